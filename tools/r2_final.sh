#!/bin/bash
# Round-2 evidence on the final build: GPU suite, bench (7B default + 1B + 70B), sparsity sweep, reference arm,
# the bench's ncu launch list, one ncu --set full capture of every kernel of a 7B forward, CUPTI timelines.
cd "$(dirname "$0")/.."
O=gpurun_out/r02/${TAG:-final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_7B.json 2> $O/bench_7B.err; echo "bench 7B rc=$?"
for C in 1B 70B; do timeout 900 python bench.py --config $C --steps 10 --no-cpu-baseline --no-e2e > $O/bench_$C.json 2> $O/bench_$C.err; echo "bench $C rc=$?"; done
: > $O/sweep_7B.jsonl
for C in 7B-s90 7B-s95 7B-s99 7B-s995 7B-s999 7B-tail; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu >> $O/sweep_7B.jsonl 2>> $O/sweep.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_7B.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-ncu > $O/launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|union_" -s 4 -c 4 \
    -o $O/step_7B -f python tools/prof_run.py --config 7B --iters 2 --fwd > $O/prof_step.log 2>&1; echo "ncu step rc=$?"
ncu -i $O/step_7B.ncu-rep --page raw --csv > $O/step_raw_7B.csv 2>/dev/null
ncu -i $O/step_7B.ncu-rep --page details --csv > $O/step_details_7B.csv 2>/dev/null
for C in 7B 1B; do timeout 300 python tools/timeline.py --config $C --out $O/timeline_$C.json > $O/timeline_$C.log 2>&1; done
ls -la $O
