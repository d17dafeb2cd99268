"""Profiling driver: one cfg4-shaped species batch (subset of cells) through
compress_cells on cuda:0. Used under ncu (tools only; not a bench number)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200.cells import CellBatch, CellBins, CellResults  # noqa: E402
from paper_2504_14897_b200.types import AxisRange, FitConfig, ModelMeta  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=4096)
ap.add_argument("--per-cell", type=int, default=1907)
ap.add_argument("--bins", type=int, default=48)
ap.add_argument("--K", type=int, default=4)
ap.add_argument("--range", type=float, default=6.0)
ap.add_argument("--species", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fp32", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
offs = torch.arange(a.cells + 1, dtype=torch.int64, device=dev) * a.per_cell
n = a.cells * a.per_cell
axes = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3)]
G.synth_cells(3, offs, 11, a.species, *axes)
b = CellBatch(axes, offs, a.bins, [-a.range] * 3, [a.range] * 3)
bins = CellBins.alloc(b)
res = CellResults(axes[0], b.n_cells, 3, a.K, 0)
cfg = FitConfig(initial_components=a.K, seed=11, temperature=np.full(3, (a.range / 6) ** 2),
                estep_fp32=a.fp32)
meta = ModelMeta("e", None, 0, [AxisRange(-a.range, a.range)] * 3)
ctx = G.api.context(0)
ctx.enable_timing(True)
for _ in range(a.reps):
    G.compress_cells(b, cfg, meta, bins=bins, results=res)
torch.cuda.synchronize()
print({k: round(v[0] / a.reps, 3) for k, v in ctx.kernel_times().items()})
print("exact passes per fit-iteration:", ctx.exact_passes() / (a.reps * a.cells * 100.0))
it = res.iterations.cpu().numpy()
print("iterations mean", it.mean(), "converged", res.converged.cpu().numpy().mean(),
      "nnz mean", bins.nnz.cpu().numpy().mean())
