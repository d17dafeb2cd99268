"""Throughput of the device reference generator (vdfcg_generate, synthdata.cpp:54-86) next to
the oracle's CPU restatement (1 thread: the reference generator is one sequential stream).
Kernel times come from the context's CUDA events; the mt19937_64 stream kernel is one CTA.
Usage: python tools/prof_generate.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402


def case(name, fr, mu, cv, n, seed=11, reps=3):
    d = len(mu[0])
    out = torch.empty(n * d, dtype=torch.float64, device="cuda")
    G.generate(fr, mu, cv, n, seed, out=out)  # warm-up (arena growth)
    torch.cuda.synchronize()
    ctx = api.context()
    ctx.enable_timing(True)
    ctx.reset_timing()
    t0 = time.perf_counter()
    for _ in range(reps):
        G.generate(fr, mu, cv, n, seed, out=out)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    kt = {k: v[0] / reps for k, v in ctx.kernel_times().items()}
    ctx.enable_timing(False)
    dev_ms = sum(kt.values())
    n_cpu = min(n, 2_000_000)
    t0 = time.perf_counter()
    O.generate(fr, mu, cv, n_cpu, seed)
    cpu = (time.perf_counter() - t0) / n_cpu
    print(f"{name}: n={n} d={d}: device {dev_ms:.2f} ms ({n / dev_ms * 1e3:.3e} p/s; "
          + ", ".join(f"{k} {v:.2f} ms" for k, v in kt.items())
          + f"), call wall {wall * 1e3:.2f} ms; oracle 1 thread {cpu * n * 1e3:.1f} ms "
          f"({1 / cpu:.3e} p/s, timed on {n_cpu} particles)")


if __name__ == "__main__":
    case("cfg1", [0.8, 0.2], [[0, 0], [3, 0]], [np.eye(2), 0.25 * np.eye(2)], 1_000_000)
    cov = np.array([[1.0, 0.3, 0.3], [0.3, 1.0, 0.3], [0.3, 0.3, 1.0]])
    case("cfg2", [0.4, 0.3, 0.2, 0.1], [[0, 0, 0], [2.5, 0, 0], [-1.5, 1.5, 0], [0, -2, 1.5]],
         [cov, 0.5 * cov, 0.25 * cov, 0.3 * np.eye(3)], 10_000_000)
