#!/bin/bash
# session-3 experiment 15: UP work list ordered by fraction of each block's union (SFFN_UP_ORDER=1)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp15; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "prep_split or pi_order" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/pytest_subset.log
SFFN_UP_ORDER=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "forward_vs_oracle or 7b_full or 1b_full" > $O/pytest_order.log 2>&1; echo "pytest order rc=$?"; tail -n 2 $O/pytest_order.log
for V in 0 1; do for C in 7B 1B; do
  SFFN_UP_ORDER=$V timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm_kernel<1" -s 1 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ' | sed "s/^/order=$V $C UP: /"; echo
done; done > $O/ncu_up.txt; cat $O/ncu_up.txt
for C in 7B 1B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_UP_ORDER --values 0,1 --reps 12 > $O/ab_$C.json 2>$O/ab_$C.err; cat $O/ab_$C.json; done
