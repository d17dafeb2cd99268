"""cfg3 histogram (256 cells x 390625, 32^3, cells_dense) kernel time (tools)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402

dev = torch.device("cuda", 0)
cells, per = 256, 390625
offs = torch.arange(cells + 1, dtype=torch.int64, device=dev) * per
axes = [torch.empty(cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
G.synth_cells(3, offs, 11, 0, *axes)
b = G.CellBatch(axes, offs, 32, [-6] * 3, [6] * 3)
ctx = api.context()
bins = G.bin_cells(b)
torch.cuda.synchronize()
ctx.enable_timing(True)
ctx.reset_timing()
for _ in range(5):
    G.bin_cells(b, bins)
torch.cuda.synchronize()
kt = ctx.kernel_times()
nnz = float(bins.nnz.sum().item())
byt = cells * per * 24 + nnz * 12 + (cells + 1) * 8
d = kt["cells_dense"][0] / 5
print(os.environ.get("VDFCG_DENSE_GQ", "default"), f"cells_dense {d:.3f} ms {byt / d / 1e6 / bench.peaks()[0]:.3f} of HBM",
      {k: round(v[0] / 5, 3) for k, v in kt.items()})
