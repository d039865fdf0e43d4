#!/bin/bash
# ncu --set full (source-level) of the CTA-pair union GEMMs (SFFN_UNION_PAIR=1) on the 7B forward
cd "$(dirname "$0")/.."
O=gpurun_out/r02/ncu_pair; mkdir -p $O
SFFN_UNION_PAIR=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"union_gemm_pair" -s 2 -c 2 \
    -o $O/pair -f python tools/prof_run.py --config 7B --iters 2 --algo union --fwd > $O/prof.log 2>&1; echo "pair rc=$?"
ncu -i $O/pair.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/pair.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
ls -la $O
