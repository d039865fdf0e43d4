#!/bin/bash
# ncu --set full (source-level) of the union UP/DOWN GEMMs of a 7B forward; LIB= selects a probe build
cd "$(dirname "$0")/.."
O=gpurun_out/r02/ncu_union_${TAG:-real}; mkdir -p $O
SFFN_LIB=${LIB:-paper_2603_23198_b200/libsffn.so} timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"union_gemm" -s 2 -c 2 -o $O/u -f python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd \
    > $O/prof.log 2>&1; echo "rc=$?"
ncu -i $O/u.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
ncu -i $O/u.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
