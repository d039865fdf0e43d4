#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every entry point (small shapes), single and pair union
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitizer; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $OUT/sanitize_$tool.log
done
SFFN_UNION_PAIR=1 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_memcheck_pair.log 2>&1
echo "memcheck pair rc=$?"; tail -3 $OUT/sanitize_memcheck_pair.log
# the prep kernel with one CTA per union block (the large-M default; small shapes otherwise split blocks over CTAs)
for tool in memcheck racecheck; do
  SFFN_PREP_SPLIT=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_${tool}_split1.log 2>&1
  echo "$tool split1 rc=$?"; tail -3 $OUT/sanitize_${tool}_split1.log
done
