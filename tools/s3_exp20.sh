#!/bin/bash
# session-3 experiment 20: snake order of the UP groups (probe) — ncu UP time/DRAM; parity subset
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp20; mkdir -p $O
SFFN_UP_SNAKE=1 timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "prep_split or forward_vs_oracle" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/pytest.log
for rep in 1 2; do for V in 0 1; do for C in 7B 70B; do
  SFFN_UP_SNAKE=$V timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"union_gemm" -s 2 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_gemm" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ' | sed "s/^/snake=$V $C UP: /"; echo
done; done; done > $O/ncu_up.txt; cat $O/ncu_up.txt
