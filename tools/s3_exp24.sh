#!/bin/bash
# session-3 experiment 24: DOWN raster group 4 vs 32 in the bench's own regime (30 steps, power cap), alternating runs
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp24; mkdir -p $O
for rep in 1 2 3; do for G in 4 32; do
  SFFN_DOWN_GROUP=$G timeout 600 python bench.py --no-cpu-baseline --no-ncu --no-dense > $O/bench_${G}_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/bench_${G}_$rep.json')); print('group=$G rep=$rep', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
