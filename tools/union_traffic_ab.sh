#!/bin/bash
# union GEMM durations + DRAM reads for several library builds (LIBS), alternating twice (ncu, deterministic A/B)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for L in ${LIBS}; do
  echo "== $L"
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:union_gemm -s 2 -c 2 --csv \
     python tools/prof_run.py --config ${CFG:-7B} --iters 3 --algo union --fwd 2>/dev/null \
     | grep -E "gpu__time|dram__bytes|lts__t" | awk -F'","' '{split($5,k,"("); printf "%-26s %-30s %s\n", substr(k[1],1,26), $(NF-2), $NF}'
done
done
