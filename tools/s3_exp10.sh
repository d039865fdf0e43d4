#!/bin/bash
# session-3 experiment 10: prep overlapped with the gate GEMM (SFFN_PREP_OVERLAP) — parity subset, A/B, timeline
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp10; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "prep_overlap or prep_split or pi_order or launch_count or forward_vs_oracle" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -n 3 $O/pytest_subset.log
for C in 7B 1B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_PREP_OVERLAP --values 0,1 --reps 10 > $O/ab_$C.json 2>$O/ab_$C.err; echo "ab $C rc=$?"; cat $O/ab_$C.json; tail -n 3 $O/ab_$C.err; done
for C in 7B 1B; do SFFN_PREP_OVERLAP=1 timeout 300 python tools/timeline.py --config $C --out $O/timeline_$C.json > $O/timeline_$C.log 2>&1; tail -n 6 $O/timeline_$C.log; done
