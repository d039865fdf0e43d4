cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "union or forward_vs or full_size or up_down or nongated or fused or continuous or direct" > gpurun_out/pyt7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pyt7.log
for i in 1 2; do
for L in paper_2603_23198_b200/libsffn.so build/libsffn_bk64.so; do
  echo "== $L"; SFFN_LIB=$L timeout 300 python tools/timeline.py --config 7B 2>&1 | grep -v -i warn | tail -9
done; done
