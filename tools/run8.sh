cd $GRAFT_REPO_ROOT
for i in 1 2; do
for L in build/libsffn_base.so paper_2603_23198_b200/libsffn.so build/libsffn_PF3.so build/libsffn_PF4.so; do
  echo "== $L"; SFFN_LIB=$L timeout 300 python tools/timeline.py --config 7B --steps 2 2>&1 | grep -v -i warn | grep "union_gemm\|step span" | tail -3
done; done
