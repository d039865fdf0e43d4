#!/bin/bash
# ncu --set full (source-level) of the union prep kernel on the 7B forward
cd "$(dirname "$0")/.."
O=gpurun_out/r02/ncu_prep; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"union_prep" -s 1 -c 1 \
    -o $O/prep -f python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd > $O/prof.log 2>&1; echo "prep rc=$?"
ncu -i $O/prep.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/prep.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
ncu -i $O/prep.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ls -la $O
