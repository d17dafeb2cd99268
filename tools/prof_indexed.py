"""Profiling driver for the cell-index input path: one cfg4-shaped species (n particles in
a random order over n_cells cells, int32 cell id each) through bin_cells_indexed on cuda:0.
Prints per-kernel CUDA-event times (tools only; a run under ncu is never a bench number)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200.cells import ParticleBatch, bin_cells_indexed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=64 ** 3)
ap.add_argument("--particles", type=int, default=500_000_000)
ap.add_argument("--bins", type=int, default=48)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sorted", action="store_true", help="cell ids ascending (PIC sorted order)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
n, nc = a.particles, a.cells
counts = torch.full((nc,), n // nc, dtype=torch.int64, device=dev)
counts[: n % nc] += 1
offs = torch.zeros(nc + 1, dtype=torch.int64, device=dev)
offs[1:] = torch.cumsum(counts, 0)
axes = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3)]
G.synth_cells(3, offs, 11, 0, *axes)
cid = torch.repeat_interleave(torch.arange(nc, device=dev, dtype=torch.int32), counts)
if not a.sorted:
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    perm = torch.randperm(n, device=dev, generator=g)
    axes = [x[perm].contiguous() for x in axes]
    cid = cid[perm].contiguous()
    del perm
torch.cuda.empty_cache()
pb = ParticleBatch(axes, cid, nc, a.bins, [-6.0] * 3, [6.0] * 3)
ctx = G.api.context(0)
bin_cells_indexed(pb)
torch.cuda.synchronize()
ctx.enable_timing(True)
ctx.reset_timing()
for _ in range(a.reps):
    o, b = bin_cells_indexed(pb)
torch.cuda.synchronize()
kt = ctx.kernel_times()
print({k: (round(v[0] / a.reps, 3), v[1] // a.reps) for k, v in kt.items()})
tot = sum(v[0] for v in kt.values()) / a.reps
print(f"total {tot:.3f} ms  -> {n * 28 / (tot * 1e-3) / 1e9:.0f} GB/s algorithmic (28 B/particle)")
