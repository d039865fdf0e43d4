#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/timeline.py --config 7B --out gpurun_out/timeline_7B.json > gpurun_out/timeline.log 2>&1
echo "timeline rc=$?"; grep -v -i warn gpurun_out/timeline.log | tail -14
timeout 300 python tools/e2e_timeline.py --config 7B --out gpurun_out/e2e_timeline.json > gpurun_out/e2e_timeline.log 2>&1
echo "e2e timeline rc=$?"; grep -v -i warn gpurun_out/e2e_timeline.log | head -12
