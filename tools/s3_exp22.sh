#!/bin/bash
# session-3 experiment 22: CTA-pair union GEMMs (256-row unions) vs single-CTA with the ordered work list (ncu) + forward
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp22; mkdir -p $O
for P in 0 1; do for C in 7B 70B 1B; do
  SFFN_UNION_PAIR=$P timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"union_gemm|union_prep" -s 3 -c 3 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "union_" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed "s/(.*)//" | sed "s/^/pair=$P $C /"
done; done > $O/ncu.txt; cat $O/ncu.txt
for P in 0 1; do SFFN_UNION_PAIR=$P timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-ncu --no-dense > $O/bench_$P.json 2>/dev/null; python -c "import json; d=json.load(open('$O/bench_$P.json')); print('pair=$P', d['ms_per_step'], d['clocks'])"; done
