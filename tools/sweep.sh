#!/bin/bash
# sparsity sweep (BASELINE.json configs[3]) + 1B, each vs our own dense tcgen05 FFN; one JSON line per config
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
for CFG in ${CFGS:-7B-s90 7B-s95 7B-s99 7B-s995 7B-s999 7B-tail 1B}; do
  for A in ${ALGOS:-union gather}; do
    timeout 600 python bench.py --config $CFG --algo $A --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
        >> gpurun_out/sweep.jsonl 2> gpurun_out/sweep_$CFG_$A.err || echo "{\"config\": \"$CFG\", \"algo\": \"$A\", \"error\": true}" >> gpurun_out/sweep.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    d = json.loads(l)
    if "error" in d: print(d); continue
    print(f'{d["config"]["workload"]:8s} {d["algo"]:6s} sparse {d["ms_per_step"]:7.3f} ms  dense {d["dense"]["ms_per_step"]:7.3f} ms  speedup {d["dense"]["speedup_sparse_vs_dense"]:5.2f}  nnz/tok {d["nnz_per_token"]:7.1f}  overflow {d["overflow_tiles"]}')
PY
