#!/bin/bash
# session-3 experiment 8: gate GEMM with one TwELL epilogue group and 5 stages (room for a co-resident prep CTA)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp8; mkdir -p $O
for rep in 1 2; do for L in paper_2603_23198_b200/libsffn.so build/libsffn_st5g1.so; do for C in 7B 1B 70B; do
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tc" -s 1 -c 1 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $NF}' | tr '\n' ' ' | sed "s|^|$L $C gate ns: |"; echo
done; done; done > $O/ncu_gate.txt; cat $O/ncu_gate.txt
