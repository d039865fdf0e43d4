#!/bin/bash
# session-3 summary A/B: the session's starting build (4678fe9) vs the final build, interleaved in one process
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp23; mkdir -p $O
for C in 7B 1B 70B; do CFG=$C ROUNDS=8 timeout 1200 python tools/ab_libs.py build/libsffn_start.so paper_2603_23198_b200/libsffn.so > $O/ab_$C.txt 2>&1; tail -n 2 $O/ab_$C.txt; done
