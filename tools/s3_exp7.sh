#!/bin/bash
# session-3 experiment 7: gate GEMM ring depth 6 (default) vs 5 vs 4 stages (pack time, ncu duration)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp7; mkdir -p $O
for C in 7B 1B; do CFG=$C ROUNDS=8 timeout 600 python tools/ab_libs.py paper_2603_23198_b200/libsffn.so build/libsffn_st5.so build/libsffn_st4.so > $O/ab_$C.txt 2>&1; tail -3 $O/ab_$C.txt; done
LIBS="paper_2603_23198_b200/libsffn.so build/libsffn_st5.so build/libsffn_st4.so" timeout 600 bash tools/gemm_group_ab.sh > $O/ncu.txt 2>&1; cat $O/ncu.txt
