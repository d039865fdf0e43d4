#!/bin/bash
# session-3 final evidence: the round-2 final script (GPU suite, benches, sweep, reference arm, launch list, ncu step
# capture, timelines) on this build, then compute-sanitizer on the prep kernel's boosted split
cd "$(dirname "$0")/.."
TAG=${TAG:-final_v4} bash tools/r2_final.sh
O=gpurun_out/r02/${TAG:-final_v4}/sanitizer; mkdir -p $O
for tool in memcheck racecheck; do
  SFFN_PREP_BOOST=2 SFFN_PREP_SPLIT=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/sanitize_${tool}_boost2.log 2>&1
  echo "$tool boost2 rc=$?"; tail -3 $O/sanitize_${tool}_boost2.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > $O/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -3 $O/sanitize_memcheck.log
