cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu2
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:union_gemm -s 2 -c 2 \
   -o gpurun_out/ncu2/union -f python tools/prof_run.py --config 7B --iters 2 --algo union > gpurun_out/ncu2/prof.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ncu2/union.ncu-rep --page details --csv > gpurun_out/ncu2/details.csv 2>/dev/null
ncu -i gpurun_out/ncu2/union.ncu-rep --page raw --csv > gpurun_out/ncu2/raw.csv 2>/dev/null
ncu -i gpurun_out/ncu2/union.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu2/source.csv 2>gpurun_out/ncu2/source.err
ls -la gpurun_out/ncu2
