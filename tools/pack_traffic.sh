cd $GRAFT_REPO_ROOT
for L in ${LIBS:-paper_2603_23198_b200/libsffn.so}; do
  SFFN_LIB=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/prof_run.py --config 7B --iters 3 --algo union --fwd 2>/dev/null | grep -E "dram__bytes|gpu__time|hit_rate" | awk -F'","' -v L=$L '{print L, $(NF-2), $(NF-1), $NF}'
done
