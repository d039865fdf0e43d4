#!/bin/bash
# session-3 experiment 12: overlapped prep A/B (more reps, 3 configs) + timelines
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp12; mkdir -p $O
for C in 7B 1B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_PREP_OVERLAP --values 0,1 --reps 16 > $O/ab_$C.json 2>$O/ab_$C.err; echo "ab $C rc=$?"; cat $O/ab_$C.json; done
for C in 7B 1B; do for V in 0 1; do SFFN_PREP_OVERLAP=$V timeout 300 python tools/timeline.py --config $C --out $O/timeline_${C}_$V.json > $O/timeline_${C}_$V.log 2>&1; echo "== $C ov=$V"; tail -n 6 $O/timeline_${C}_$V.log; done; done
