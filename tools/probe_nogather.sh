#!/bin/bash
# timing probe: union GEMMs with the B gathers skipped (lib built with -DSFFN_UG_NOGATHER), single-CTA and pair mode,
# ncu tensor-pipe activity and durations next to the real build
cd "$(dirname "$0")/.."
O=gpurun_out/r02/nogather; mkdir -p $O
for P in 0 1; do for L in paper_2603_23198_b200/libsffn.so build/ab/lib_nogather.so; do
  SFFN_UNION_PAIR=$P SFFN_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"union_gemm" -s 2 -c 2 --csv python tools/prof_run.py --config 7B --iters 2 --algo union --fwd 2>/dev/null \
    | grep -E "union_gemm" | awk -F'","' -v p=$P -v l=$L '{print "pair=" p, l, substr($5,1,40), $(NF-2), $NF}'
done; done | tee $O/probe.txt
