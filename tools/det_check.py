"""Bitwise run-to-run determinism of compress_cells: python tools/det_check.py [n_cells] [runs]"""
import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import paper_2504_14897_b200 as G
from paper_2504_14897_b200.types import FitConfig, ModelMeta, AxisRange
dev = torch.device("cuda", 0)
NC = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
RUNS = int(sys.argv[2]) if len(sys.argv) > 2 else 30
offs = torch.arange(NC + 1, dtype=torch.int64, device=dev) * 1900
axes = [torch.empty(NC * 1900, dtype=torch.float64, device=dev) for _ in range(3)]
G.synth_cells(3, offs, 11, 0, *axes)
b = G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3)
cfg = FitConfig(initial_components=4, seed=11, temperature=np.ones(3))
meta = ModelMeta("e", None, 0, [AxisRange(-6, 6)] * 3)
bins0, r0, rec0, _ = G.compress_cells(b, cfg, meta)
k0 = bins0.keys.clone(); c0 = bins0.counts.clone(); n0 = bins0.nnz.clone()
bad = 0
for t in range(RUNS):
    bins, r, rec, _ = G.compress_cells(b, cfg, meta)
    msgs = []
    if not torch.equal(bins.nnz, n0): msgs.append("nnz")
    for f in ("weights", "means", "covariances", "final_loglik", "iterations", "status", "components"):
        a, c = getattr(r0, f), getattr(r, f)
        if a.dtype == torch.float64: a, c = a.view(torch.int64), c.view(torch.int64)
        if not torch.equal(a, c):
            diff = (a != c)
            msgs.append(f"{f}:{int(diff.sum())}")
    if not torch.equal(rec0, rec): msgs.append("records")
    if msgs:
        bad += 1
        print("run", t, msgs, "status!=0:", int((r.status != 0).sum()))
print("bad runs", bad, "failed cells", int((r0.status != 0).sum()))
