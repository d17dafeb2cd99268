#!/bin/bash
# EM time of several builds on a cfg4-shaped species subset (tools).
#   bash tools/ab_libs.sh <cells> lib1.so lib2.so ...   ("-" = the in-tree build)
C=$1; shift
for i in 1 2; do
  for L in "$@"; do
    if [ "$L" == "-" ]; then R=$(python tools/prof_cells.py --cells $C --reps 2 2>/dev/null | head -1)
    else R=$(VDFCG_LIB=$L python tools/prof_cells.py --cells $C --reps 2 2>/dev/null | head -1); fi
    echo "$L $(echo $R | grep -o "'em_fit': [0-9.]*")"
  done
done
