#!/bin/bash
# ncu --set full of one kernel (regex $K) of one forward on config $CFG: details + source (sass) under gpurun_out/ncu_one
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu_one; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-1} -c 1 \
    -o $OUT/one -f python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd > $OUT/prof.log 2>&1; echo "rc=$?"
ncu -i $OUT/one.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/one.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2>/dev/null
ls -la $OUT
