#!/bin/bash
# session-3 experiment 17: DOWN raster group (j-major within the group) on the final build — ncu DRAM/time + A/B
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp17; mkdir -p $O
for G in 4 16 32 64; do for C in 7B 70B; do
  SFFN_DOWN_GROUP=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm" -s 3 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ' | sed "s/^/group=$G $C DOWN: /"; echo
done; done > $O/ncu_down.txt; cat $O/ncu_down.txt
for C in 7B 70B; do CFG=$C timeout 900 python tools/ab_env.py --var SFFN_DOWN_GROUP --values 4,16,32 --reps 12 > $O/ab_$C.json 2>$O/ab_$C.err; cat $O/ab_$C.json; done
