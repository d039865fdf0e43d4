#!/bin/bash
# per-kernel ncu durations of one forward for several library builds (deterministic kernel-level A/B)
cd "$(dirname "$0")/.."
for L in ${LIBS}; do
  echo "== $L"
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-8} --csv \
     python tools/prof_run.py --config ${CFG:-7B} --iters 2 --algo union --fwd 2>/dev/null \
     | grep gpu__time | awk -F'","' '{split($5,k,"("); printf "%-40s %10s\n", substr(k[1],1,40), $NF}'
done
