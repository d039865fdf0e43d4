#!/bin/bash
# session-3 experiment 18: UP raster group with the fraction-ordered work list — ncu UP DRAM/time
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp18; mkdir -p $O
for G in 8 16 32 64; do for C in 7B 70B 1B; do
  SFFN_UP_GROUP=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm" -s 2 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ' | sed "s/^/group=$G $C UP: /"; echo
done; done > $O/ncu_up.txt; cat $O/ncu_up.txt
