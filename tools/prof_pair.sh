#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu_pair; mkdir -p $OUT
export SFFN_UNION_PAIR=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_gemm_pair -s 2 -c 2 \
    -o $OUT/pair -f python tools/prof_run.py --config 7B --iters 2 --algo union --fwd > $OUT/prof.log 2>&1; echo "full rc=$?"
ncu -i $OUT/pair.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/pair.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/pair.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2>/dev/null
ls -la $OUT
