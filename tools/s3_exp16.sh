#!/bin/bash
# session-3 experiment 16: fraction-ordered UP work list — UP DRAM / time (ncu) and a second interleaved A/B
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp16; mkdir -p $O
for V in 0 1; do for C in 7B 1B 70B; do
  SFFN_UP_ORDER=$V timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm" -s 2 -c 2 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed "s/^/order=$V $C /"
done; done > $O/ncu_up.txt; cat $O/ncu_up.txt
for C in 7B 1B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_UP_ORDER --values 0,1 --reps 16 > $O/ab_$C.json 2>$O/ab_$C.err; cat $O/ab_$C.json; done
