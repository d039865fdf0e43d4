cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/s3_sanity; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $O/bench_7B.json 2> $O/bench_7B.err; echo "bench rc=$?"; cat $O/bench_7B.json | head -c 600
