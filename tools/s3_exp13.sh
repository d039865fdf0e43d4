#!/bin/bash
# session-3 experiment 13: where the overlapped prep's gate-GEMM slowdown comes from (signals alone vs co-running)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp13; mkdir -p $O
for C in 7B 1B; do for V in "SFFN_PREP_OVERLAP=0" "SFFN_PREP_OVERLAP=1 SFFN_PREP_OV_NOPDL=1" "SFFN_PREP_OVERLAP=1"; do
  echo "== $C $V"; env $V timeout 300 python tools/timeline.py --config $C --out $O/tl.json 2>&1 | tail -n 5 | head -n 3
done; done > $O/timelines.txt; cat $O/timelines.txt
for C in 7B; do for V in 0 1; do
  SFFN_PREP_OVERLAP=$V timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:"gemm_tc" -s 1 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "gemm_tc" | awk -F'","' '{print $(NF-2), $NF}' | sed "s/^/ov=$V /"
done; done > $O/ncu_gate.txt; cat $O/ncu_gate.txt
