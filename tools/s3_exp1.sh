#!/bin/bash
# session-3 experiment 1: raster groups of the union GEMMs (L2 locality / DRAM) and of the gate GEMM
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp1; mkdir -p $O
timeout 600 python tools/ab_env.py --var SFFN_UP_GROUP --values 8,16,32,64 --reps 8 > $O/ab_up_group.json 2> $O/ab_up.err; echo "ab up rc=$?"; cat $O/ab_up_group.json
timeout 600 python tools/ab_env.py --var SFFN_DOWN_GROUP --values 4,8,16,32 --reps 8 > $O/ab_down_group.json 2> $O/ab_down.err; echo "ab down rc=$?"; cat $O/ab_down_group.json
for UG in 8 32; do for DG in 4 16; do
  SFFN_UP_GROUP=$UG SFFN_DOWN_GROUP=$DG timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"union_gemm|union_prep" -s 3 -c 3 --csv python tools/prof_run.py --config 7B --iters 2 --fwd > $O/ncu_u${UG}_d${DG}.csv 2>/dev/null
  echo "ncu u$UG d$DG rc=$?"
done; done
ROUNDS=6 timeout 600 python tools/ab_libs.py paper_2603_23198_b200/libsffn.so build/libsffn_gm64.so build/libsffn_gm128.so > $O/ab_gemm_group.txt 2>&1; echo "ab libs rc=$?"; tail -5 $O/ab_gemm_group.txt
LIBS="paper_2603_23198_b200/libsffn.so build/libsffn_gm64.so build/libsffn_gm128.so" timeout 600 bash tools/gemm_group_ab.sh > $O/gemm_group_ncu.txt 2>&1; cat $O/gemm_group_ncu.txt
