#!/bin/bash
# round-2 GPU validation: smoke, the whole GPU suite (no -x: every failure listed), then the default bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYT_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=20 ${PYTEST_ARGS} \
    > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/smoke.log; tail -45 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.err | grep -v Warning; cat gpurun_out/bench.json
fi
if [ -n "$TIMELINE" ]; then
  timeout 300 python tools/timeline.py --config 7B --out gpurun_out/timeline_7B.json > gpurun_out/timeline.log 2>&1
  echo "timeline rc=$?"; cat gpurun_out/timeline.log | grep -v Warning | tail -20
fi
