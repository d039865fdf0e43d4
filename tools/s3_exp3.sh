#!/bin/bash
# session-3 experiment 3: prep boost levels x early X copy
cd "$(dirname "$0")/.."
O=gpurun_out/r02/s3_exp3; mkdir -p $O
for C in 7B 1B; do for B in 0 1 2; do for E in 0 1; do echo "== $C boost=$B early=$E"; SFFN_PREP_BOOST=$B SFFN_PREP_COPY_EARLY=$E timeout 300 python tools/prep_trace.py $C 2>&1 | grep -v Warn | head -3; done; done; done > $O/prep_trace.txt; cat $O/prep_trace.txt
A="SFFN_PREP_BOOST=0,SFFN_PREP_COPY_EARLY=0;SFFN_PREP_BOOST=1,SFFN_PREP_COPY_EARLY=0;SFFN_PREP_BOOST=2,SFFN_PREP_COPY_EARLY=0;SFFN_PREP_BOOST=1,SFFN_PREP_COPY_EARLY=1;SFFN_PREP_BOOST=0,SFFN_PREP_COPY_EARLY=1"
for C in 7B 1B; do CFG=$C timeout 900 python tools/ab_env.py --arms "$A" --reps 12 > $O/ab_$C.json 2>$O/ab_$C.err; echo "ab $C rc=$?"; cat $O/ab_$C.json; done
