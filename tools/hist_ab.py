"""Histogram kernel time for one species of cfg4-shaped cells at several bin counts (tools;
run under different VDFCG_HIST_* settings to compare kernel paths)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1907
dev = torch.device("cuda", 0)
offs = torch.arange(cells + 1, dtype=torch.int64, device=dev) * per
axes = [torch.empty(cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
G.synth_cells(3, offs, 1, 0, *axes)
ctx = api.context()
hbm = bench.peaks()[0]
out = []
for nb in (16, 24, 32, 48, 64):
    b = G.CellBatch(axes, offs, nb, [-6] * 3, [6] * 3)
    bins = G.bin_cells(b)
    torch.cuda.synchronize()
    ctx.enable_timing(True)
    ctx.reset_timing()
    for _ in range(3):
        G.bin_cells(b, bins)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.enable_timing(False)
    name = max((k for k in kt if k.startswith("cells_")), key=lambda k: kt[k][0])
    ms = sum(v[0] for k, v in kt.items() if k.startswith("cells_")) / 3
    nnz = float(bins.nnz.sum().item())
    byt = cells * per * 24 + nnz * 12 + (cells + 1) * 8 + cells * 20
    out.append(f"{nb}^3 {name:18s} {ms:7.3f} ms  {byt / ms / 1e6:7.0f} GB/s  {byt / ms / 1e6 / hbm:.3f} of HBM")
print(os.environ.get("VDFCG_HIST_2L", "auto"), os.environ.get("VDFCG_HIST_PATH", "auto"))
print("\n".join(out))
