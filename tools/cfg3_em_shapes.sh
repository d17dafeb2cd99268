#!/bin/bash
# cfg3 EM kernel time under forced launch shapes (warps per CTA, CTAs per cell). Tools only.
for sh in default 8,1 4,1 8,2 4,2 2,4 4,4 2,8 1,8; do
  if [ $sh == default ]; then R=$(python bench.py --config cfg3 --steps 5 --warmup 2 --no-e2e --no-cpu --no-indexed 2>/dev/null)
  else R=$(VDFCG_EM_SHAPE=$sh python bench.py --config cfg3 --steps 5 --warmup 2 --no-e2e --no-cpu --no-indexed 2>/dev/null); fi
  echo "$sh $(echo $R | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["kernel_ms"]["em_fit"],3), "ms em;", round(d["ms_per_step"],3), "ms step")')"
done
