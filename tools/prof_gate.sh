#!/bin/bash
# ncu --set full (source-level) of the gate GEMM (TwELL epilogue) on a config (default 1B)
cd "$(dirname "$0")/.."
C=${CFG:-1B}; O=gpurun_out/r02/ncu_gate_$C; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel" -s 1 -c 1 \
    -o $O/gate -f python tools/prof_run.py --config $C --iters 2 --algo union --fwd > $O/prof.log 2>&1; echo "gate rc=$?"
ncu -i $O/gate.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/gate.ncu-rep --page source --csv --print-source cuda,sass > $O/mixed.csv 2>/dev/null
ncu -i $O/gate.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
ls -la $O
