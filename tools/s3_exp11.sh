#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp11; mkdir -p $O
for C in 7B 1B; do SFFN_PREP_OVERLAP=1 timeout 300 python tools/timeline.py --config $C --out $O/timeline_$C.json > $O/timeline_$C.log 2>&1; tail -n 6 $O/timeline_$C.log; done
for C in 7B 1B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_PREP_OVERLAP --values 0,1 --reps 10 > $O/ab_$C.json 2>$O/ab_$C.err; echo "ab $C rc=$?"; cat $O/ab_$C.json; done
