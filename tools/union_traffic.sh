#!/bin/bash
# DRAM bytes + time of the two union GEMMs for raster group sizes (ncu, one forward after warm-up)
cd "$(dirname "$0")/.."
for UG in ${UPS:-4 8 16}; do for DG in ${DOWNS:-8 16 32}; do
  SFFN_UP_GROUP=$UG SFFN_DOWN_GROUP=$DG timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
     -k regex:union_gemm -s 2 -c 2 --csv python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd 2>/dev/null \
     | grep -E "dram__bytes|gpu__time" | awk -F'","' -v U=$UG -v D=$DG '{split($5,k,"("); print "up", U, "down", D, k[1], $(NF-2), $NF}'
done; done
