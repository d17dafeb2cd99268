"""In-situ time series on a cfg4 species: cycle 0 fits every cell from
the seeded random init; cycles 1..3 restart every cell from its own previous model
(vdfcg_compress_cells_warm) on freshly drawn particles of the same distributions.
Usage: python tools/prof_warm.py [--cells 262144] [--per 1907]"""
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
    ap.add_argument("--static", action="store_true", help="same particles every cycle")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    offs = torch.arange(a.cells + 1, dtype=torch.int64, device=dev) * a.per
    axes = [torch.empty(a.cells * a.per, dtype=torch.float64, device=dev) for _ in range(3)]
    cfg = FitConfig(initial_components=4, seed=0, temperature=np.full(3, 1.0))
    ctx = api.context()
    prev = None
    for cycle in range(4):
        # new particles of the same per-cell distributions (or the same ones with --static)
        G.synth_cells(3, offs, 100 + (0 if a.static else cycle), 0, *axes)
        b = G.CellBatch(axes, offs, a.bins, [-6] * 3, [6] * 3)
        torch.cuda.synchronize()
        ctx.enable_timing(True)
        ctx.reset_timing()
        _, res, _, _ = G.compress_cells(b, cfg, keep_bins=False, warm=prev)
        torch.cuda.synchronize()
        kt = ctx.kernel_times()
        ctx.enable_timing(False)
        em = kt["em_fit"][0]
        it = res.iterations.double().mean().item()
        print(f"cycle {cycle} ({'warm' if prev is not None else 'cold'}): em_fit {em:.1f} ms, "
              f"mean iterations {it:.2f}, converged {res.converged.double().mean().item():.3f}, "
              f"{a.cells / (em * 1e-3):.3g} fits/s (EM only)")
        prev = res


if __name__ == "__main__":
    main()
