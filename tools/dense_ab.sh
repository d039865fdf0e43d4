cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense" 2>&1 | tail -1
for P in 0 1; do
  SFFN_GATE_PAIR=$P timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc --csv python tools/prof_run.py --config 7B --iters 1 --dense --algo union 2>/dev/null | grep gpu__time | awk -F'","' -v P=$P '{split($5,k,"("); print "pair=" P, k[1], $NF}'
done
