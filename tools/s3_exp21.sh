#!/bin/bash
# session-3 experiment 21: L2 prefetch-size hint on the UP gathers (none / L2::128B / L2::256B)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp21; mkdir -p $O
for rep in 1 2; do for L in paper_2603_23198_b200/libsffn.so build/libsffn_pf128.so build/libsffn_pf256.so; do for C in 7B 70B 1B; do
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm" -s 2 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ' | sed "s|^|$L $C UP: |"; echo
done; done; done > $O/ncu_up.txt; cat $O/ncu_up.txt
