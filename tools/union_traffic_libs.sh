#!/bin/bash
# DRAM bytes + time of the union GEMMs for several library builds (ncu, one forward after warm-up)
cd "$(dirname "$0")/.."
for L in ${LIBS}; do
  SFFN_LIB=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
     -k regex:union_gemm -s 2 -c 2 --csv python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd 2>/dev/null \
     | grep -E "dram__bytes|gpu__time" | awk -F'","' -v L=$L '{split($5,k,"("); print L, k[1], $(NF-2), $NF}'
done
