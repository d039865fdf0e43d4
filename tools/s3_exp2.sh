#!/bin/bash
# session-3 experiment 2: adaptive prep split (SFFN_PREP_BOOST) and UP raster group 8 vs 32
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "union or forward or prep or pi or hybrid or train or shard or fused" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
for C in 7B 1B; do for B in 0 1; do echo "== $C boost=$B"; SFFN_PREP_BOOST=$B timeout 300 python tools/prep_trace.py $C 2>&1 | grep -v Warn; done; done > $O/prep_trace.txt; cat $O/prep_trace.txt
for C in 7B 1B; do CFG=$C timeout 600 python tools/ab_env.py --var SFFN_PREP_BOOST --values 0,1 --reps 12 > $O/ab_boost_$C.json 2>/dev/null; echo "ab boost $C rc=$?"; cat $O/ab_boost_$C.json; done
timeout 600 python tools/ab_env.py --var SFFN_UP_GROUP --values 8,32 --reps 12 > $O/ab_up_group.json 2>/dev/null; cat $O/ab_up_group.json
for B in 0 1; do for C in 7B 1B; do
  SFFN_PREP_BOOST=$B timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"union_prep|union_gemm" -s 3 -c 6 --csv python tools/prof_run.py --config $C --iters 3 --fwd 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $5, $NF}' | sed "s/^/boost=$B $C /"
done; done > $O/ncu_prep.txt; cat $O/ncu_prep.txt
