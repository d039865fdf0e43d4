#!/bin/bash
# session-3 validation of the committed build: GPU suite, smoke(), one 7B bench line
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_validate; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_7B.json 2> $O/bench_7B.err; echo "bench rc=$?"; head -c 400 $O/bench_7B.json
