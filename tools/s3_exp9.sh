#!/bin/bash
# session-3 experiment 9: gate GEMM one TwELL epilogue group + 5 stages (new default) vs previous commit; GPU suite
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp9; mkdir -p $O
for C in 7B 1B 70B; do CFG=$C ROUNDS=6 timeout 900 python tools/ab_libs.py build/libsffn_prev.so paper_2603_23198_b200/libsffn.so > $O/ab_$C.txt 2>&1; tail -n 2 $O/ab_$C.txt; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/pytest_gpu.log
