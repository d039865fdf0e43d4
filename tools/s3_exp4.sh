#!/bin/bash
# session-3 experiment 4: GPU suite on the adaptive prep split; UP raster group 8 vs 32 at 7B / 1B / 70B
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
for C in 7B 1B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_UP_GROUP --values 8,16,32 --reps 10 > $O/ab_up_$C.json 2>$O/ab_up_$C.err; echo "ab $C rc=$?"; cat $O/ab_up_$C.json; done
