#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp5; mkdir -p $O
for C in 7B 1B 70B; do SFFN_LIB=build/libsffn_epitrace.so timeout 300 python tools/s3_epi_trace.py $C 2>&1 | grep -v Warn; done > $O/epi_trace.txt; cat $O/epi_trace.txt
