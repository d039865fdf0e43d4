cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu11
for P in 0 1; do echo "== pair=$P"; SFFN_UNION_PAIR=$P timeout 300 python tools/timeline.py --config 7B --steps 2 2>&1 | grep -v -i warn | tail -8; done
SFFN_UNION_PAIR=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_gemm -s 2 -c 2 -o gpurun_out/ncu11/ugp -f python tools/prof_run.py --config 7B --iters 2 --fwd > gpurun_out/ncu11/prof.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu11/ugp.ncu-rep --page raw --csv > gpurun_out/ncu11/ugp_raw.csv 2>/dev/null
