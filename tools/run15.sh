cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "pack or gate_gemm or all_rows or forward_vs or continuous or dynamic or dense_forward or nongated or hybrid" > gpurun_out/pyt15.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pyt15.log
for i in 1 2; do for C in 1B 7B 70B; do for L in build/libsffn_base.so paper_2603_23198_b200/libsffn.so; do
  echo "== $C $L"; SFFN_LIB=$L timeout 300 python tools/timeline.py --config $C --steps 2 2>&1 | grep -v -i warn | grep "gemm_tc\|step span" | tail -2
done; done; done
