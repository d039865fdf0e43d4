#!/bin/bash
# session-3 experiment 14: union GEMM gather warps (8 / 10 / 12) and epilogue groups (2 / 1)
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp14; mkdir -p $O
LIBS="paper_2603_23198_b200/libsffn.so build/libsffn_ngw10.so build/libsffn_ngw12.so build/libsffn_eg1.so build/libsffn_ngw12eg1.so"
for rep in 1 2; do for L in $LIBS; do for C in 7B 1B; do
  SFFN_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"union_gemm" -s 2 -c 2 --csv python tools/prof_run.py --config $C --iters 2 --fwd 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $NF}' | tr '\n' ' ' | sed "s|^|$L $C UP/DOWN ns: |"; echo
done; done; done > $O/ncu_union.txt; cat $O/ncu_union.txt
for C in 7B 1B; do CFG=$C ROUNDS=6 timeout 900 python tools/ab_libs.py $LIBS > $O/ab_$C.txt 2>&1; tail -n 5 $O/ab_$C.txt; done
