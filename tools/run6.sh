cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu6
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_gemm -s 2 -c 2 -o gpurun_out/ncu6/ug -f python tools/prof_run.py --config 7B --iters 2 --fwd > gpurun_out/ncu6/prof.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu6/ug.ncu-rep --page raw --csv > gpurun_out/ncu6/ug_raw.csv 2>/dev/null
ls -la gpurun_out/ncu6
