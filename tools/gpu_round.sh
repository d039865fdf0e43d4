#!/bin/bash
# tests + bench (both up/down algorithms), each under its own timeout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_tests.sh
for A in ${ALGOS:-union gather}; do
  timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 --algo $A --no-cpu-baseline ${BENCH_ARGS} \
      > gpurun_out/bench_$A.json 2> gpurun_out/bench_$A.err
  echo "bench $A rc=$?"; tail -c 1500 gpurun_out/bench_$A.err | grep -v Warning; cat gpurun_out/bench_$A.json
done
