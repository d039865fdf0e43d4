#!/bin/bash
# ncu --set full of every kernel of ONE sparse forward (the bench step) on the 7B config: per-kernel DRAM traffic,
# tensor-pipe and L2 metrics; plus the launch list of the same command.  Outputs under gpurun_out/ncu_step/.
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu_step; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python tools/prof_run.py --config 7B --iters 2 --algo union --fwd > $OUT/launches.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|union_|permute" -s 7 -c 7 \
    -o $OUT/step -f python tools/prof_run.py --config 7B --iters 2 --algo union --fwd > $OUT/prof.log 2>&1; echo "full rc=$?"
ncu -i $OUT/step.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/step.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT
