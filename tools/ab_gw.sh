#!/bin/bash
# A/B: union GEMM gather-warp count (8 vs 16) in single-CTA and CTA-pair union mode (interleaved, one process per mode)
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
for P in 0 1; do
  echo "SFFN_UNION_PAIR=$P"; SFFN_UNION_PAIR=$P ROUNDS=8 timeout 600 python tools/ab_libs.py build/ab/lib_base.so build/ab/lib_gw16.so 2>&1 | grep -v Warn
done | tee $O/ab_gw.txt
