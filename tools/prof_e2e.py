"""Break down the end-to-end (host-input) compress path of one cfg4-like species.

Prints: raw pinned H2D bandwidth, device-resident compress time, host-input compress time
(pinned and pageable outputs), so the e2e overhead over max(H2D, compute) is visible.
Usage: python tools/prof_e2e.py [--cells 262144] [--per 1907] [--reps 2]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402
from paper_2504_14897_b200.cells import CellResults  # noqa: E402
from paper_2504_14897_b200.types import AxisRange, FitConfig, ModelMeta  # noqa: E402


def timed(fn, reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=262144)
    ap.add_argument("--per", type=int, default=1907)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = a.cells * a.per
    offs = torch.arange(a.cells + 1, dtype=torch.int64, device=dev) * a.per
    axes = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 1, 0, *axes)
    cfg = FitConfig(initial_components=4, seed=0, temperature=np.ones(3))
    meta = ModelMeta("e", None, 0, [AxisRange(-6, 6)] * 3)
    dbatch = G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3)
    hax = [x.cpu().pin_memory() for x in axes]
    hoffs = offs.cpu().pin_memory()
    hbatch = G.CellBatch(hax, hoffs, 48, [-6] * 3, [6] * 3)
    dst = torch.empty(n, dtype=torch.float64, device=dev)
    h2d = timed(lambda: [dst.copy_(x, non_blocking=True) for x in hax], a.reps)
    print(f"raw pinned H2D {3 * n * 8 / 1e9:.2f} GB: {h2d:.1f} ms = {3 * n * 8 / h2d / 1e6:.1f} GB/s")
    G.compress_cells(dbatch, cfg, meta, keep_bins=False)
    dt = timed(lambda: G.compress_cells(dbatch, cfg, meta, keep_bins=False), a.reps)
    print(f"device-resident compress: {dt:.1f} ms")
    G.compress_cells(hbatch, cfg, meta, keep_bins=False)
    ht = timed(lambda: G.compress_cells(hbatch, cfg, meta, keep_bins=False), a.reps)
    print(f"host-input compress (default outputs): {ht:.1f} ms")
    hr = CellResults(torch.empty(1).pin_memory(), a.cells, 3, 4, 0)
    pt = timed(lambda: G.compress_cells(hbatch, cfg, meta, keep_bins=False, results=hr), a.reps)
    print(f"host-input compress (results buffers reused): {pt:.1f} ms")
    ctx = api.context()
    ctx.enable_timing(True)
    G.compress_cells(hbatch, cfg, meta, keep_bins=False, results=hr)
    torch.cuda.synchronize()
    for k, v in sorted(ctx.kernel_times().items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:24s} {v[0]:9.2f} ms  x{v[1]}")
    ctx.enable_timing(False)


if __name__ == "__main__":
    main()
