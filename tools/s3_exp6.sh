#!/bin/bash
# session-3 experiment 6: UP work list written by all warps (per-group offsets in SMEM) vs one warp per 32 groups
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp6; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "union or prep or pi or forward_vs or shard or fused or launch" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
for rep in 1 2; do for L in build/libsffn_head.so paper_2603_23198_b200/libsffn.so; do for C in 7B 1B; do
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"union_prep" -s 1 -c 2 --csv python tools/prof_run.py --config $C --iters 3 --fwd 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $NF}' | tr '\n' ' ' | sed "s|^|$L $C prep ns: |"; echo
done; done; done > $O/ncu_prep.txt; cat $O/ncu_prep.txt
for C in 7B 1B; do CFG=$C ROUNDS=8 timeout 600 python tools/ab_libs.py build/libsffn_head.so paper_2603_23198_b200/libsffn.so > $O/ab_$C.txt 2>&1; tail -2 $O/ab_$C.txt; done
