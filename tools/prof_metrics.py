"""Time the per-cell metrics pass (vdfcg_metrics_cells) on a cfg4-like species.
Usage: python tools/prof_metrics.py [--cells 262144] [--per 1907] [--bins 48] [--d 3]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402
from paper_2504_14897_b200.types import FitConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=262144)
    ap.add_argument("--per", type=int, default=1907)
    ap.add_argument("--bins", type=int, default=48)
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    offs = torch.arange(a.cells + 1, dtype=torch.int64, device=dev) * a.per
    axes = [torch.empty(a.cells * a.per, dtype=torch.float64, device=dev) for _ in range(a.d)]
    G.synth_cells(a.d, offs, 1, 0, *axes, *([None] if a.d == 2 else []))
    batch = G.CellBatch(axes, offs, a.bins, [-6] * a.d, [6] * a.d)
    bins, res, _, _ = G.compress_cells(batch, FitConfig(initial_components=4, seed=0, temperature=np.ones(a.d)))
    out = G.cell_metrics(batch, bins, res)
    ctx = api.context()
    ctx.enable_timing(True)
    ctx.reset_timing()
    for _ in range(a.reps):
        G.cell_metrics(batch, bins, res, out=out)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ms = kt["cell_metrics"][0] / a.reps
    comps = res.components.double().mean().item()
    evals = a.cells * a.bins ** a.d * comps
    print(f"cell_metrics: {ms:.2f} ms per pass over {a.cells} cells ({a.bins}^{a.d} bins, "
          f"mean M {comps:.2f}) = {evals / ms / 1e6:.3g} G component-evals/s")
    print("jsd median", out.jsd.nanmedian().item(), "kl_pq median", out.kl_pq.nanmedian().item())


if __name__ == "__main__":
    main()
