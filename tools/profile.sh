#!/bin/bash
# ncu evidence: launch list (cold, serialised) + one --set full capture per hot kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
CFG=${CFG:-7B}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_${CFG}.csv \
    python tools/prof_run.py --config $CFG --iters 2 --dense --algo ${ALGO:-auto} > gpurun_out/ncu/launches.log 2>&1
for K in ${KERNELS:-gemm_tc_kernel updown_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-1} -c ${COUNT:-1} \
      -o gpurun_out/ncu/prof_${K}_${CFG} -f python tools/prof_run.py --config $CFG --iters 2 --algo ${ALGO:-auto} > gpurun_out/ncu/prof_${K}.log 2>&1
  ncu -i gpurun_out/ncu/prof_${K}_${CFG}.ncu-rep --page raw --csv > gpurun_out/ncu/raw_${K}_${CFG}.csv 2>/dev/null
  ncu -i gpurun_out/ncu/prof_${K}_${CFG}.ncu-rep --page details --csv > gpurun_out/ncu/details_${K}_${CFG}.csv 2>/dev/null
done
ls -la gpurun_out/ncu
