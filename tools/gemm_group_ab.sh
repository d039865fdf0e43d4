#!/bin/bash
# gate GEMM raster group (M tiles per group) A/B: ncu duration + DRAM bytes per build, alternating twice
cd "$(dirname "$0")/.."
for rep in 1 2; do
for L in ${LIBS}; do
  echo "== $L"
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_tc -s 1 -c 2 --csv \
     python tools/prof_run.py --config ${CFG:-7B} --iters 3 --algo union --fwd 2>/dev/null \
     | grep -E "gpu__time|dram__bytes" | awk -F'","' '{printf "%-22s %14s\n", $(NF-2), $NF}'
done
done
