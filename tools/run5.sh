cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu5
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "pack or gate_gemm or forward_vs or full_size or all_rows or continuous or overflow or hybrid or nongated" > gpurun_out/pyt5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pyt5.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/ncu5/gate -f python tools/prof_run.py --config 7B --iters 2 --fwd > gpurun_out/ncu5/prof.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu5/gate.ncu-rep --page raw --csv > gpurun_out/ncu5/gate_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ncu5/gate_raw.csv')))
h,u,v=rows[0],rows[1],rows[2]
for k in ["gpu__time_duration.sum","sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed","l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum","l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum","dram__bytes_read.sum","dram__bytes_write.sum","sm__cycles_elapsed.avg.per_second","smsp__inst_executed.sum"]:
    for i,n in enumerate(h):
        if n==k: print(k, v[i], u[i])
PY
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench5.json'))
print(d['ms_per_step'], d['kernels']['gate_gemm_twell']['ms'], d['kernels']['fused_up_down']['ms'], d['dense']['ms_per_step'], d['e2e']['ms_per_step'], d['clocks'], d['hbm'].get('step_dram_bytes'))"
