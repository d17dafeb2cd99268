#!/bin/bash
# A/B the EM kernel: exp/lib_base.so (baseline build) vs the in-tree libvdfcg.so (and the
# in-tree build with VDFCG_EM_WF=0) on a cfg4-shaped species subset (65536 cells x 1907
# particles, 48^3, K=4). Tools only.   bash tools/ab_em.sh [cells] [extra prof_cells args]
C=${1:-65536}
shift
for i in 1 2; do
  echo "base: $(VDFCG_LIB=exp/lib_base.so python tools/prof_cells.py --cells $C --reps 2 "$@" 2>/dev/null | head -1)"
  echo "new:  $(python tools/prof_cells.py --cells $C --reps 2 "$@" 2>/dev/null | head -1)"

done
