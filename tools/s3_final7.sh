#!/bin/bash
# session-3 final evidence on the final build (+ UP group by X working set)
cd "$(dirname "$0")/.."
TAG=final_v7 bash tools/r2_final.sh
O=gpurun_out/r02/final_v7
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
