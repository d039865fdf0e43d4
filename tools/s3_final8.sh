#!/bin/bash
# session-3 validation of the final build (snake UP order): GPU suite, smoke(), 7B / 70B bench lines, CUPTI timeline
cd "$(dirname "$0")/.."
O=gpurun_out/r02/final_v8; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench_7B.json 2> $O/bench_7B.err; echo "bench 7B rc=$?"
timeout 900 python bench.py --config 70B --steps 10 --no-cpu-baseline --no-e2e > $O/bench_70B.json 2> $O/bench_70B.err; echo "bench 70B rc=$?"
for C in 7B 1B; do timeout 300 python tools/timeline.py --config $C --out $O/timeline_$C.json > $O/timeline_$C.log 2>&1; tail -n 6 $O/timeline_$C.log; done
