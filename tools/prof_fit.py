"""Single-fit latency of the reference-facing fit() (vdfcg_fit): cfg1 (2V 64^2, K=2),
the reference pipeline's plane fit (2V 200^2, K=12) and cfg2 (3V 32^3, K=4).
Usage: python tools/prof_fit.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402
from paper_2504_14897_b200.types import AxisRange, FitConfig, Plane, WeightedPoints  # noqa: E402


def case(name, pts, cfg, reps=5):
    r = G.fit(pts, cfg)
    torch.cuda.synchronize()
    ctx = api.context()
    ctx.enable_timing(True)
    ctx.reset_timing()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = G.fit(pts, cfg)
    wall = (time.perf_counter() - t0) * 1e3 / reps
    kt = {k: round(v[0] / reps, 3) for k, v in ctx.kernel_times().items()}
    ctx.enable_timing(False)
    print(f"{name}: {pts.count()} points, M={r.model.size()}, its={r.iterations_used}: "
          f"{wall:.2f} ms per fit (host API)  kernels {kt}")


def main():
    import oracle as O
    p1 = O.generate([0.8, 0.2], [[0, 0], [3, 0]], [np.eye(2), 0.25 * np.eye(2)], 1_000_000, 11)
    h = G.bin_particles(p1, Plane.uv, 64, AxisRange(-6, 6), AxisRange(-6, 6))
    case("cfg1 2V 64^2 K=2", G.to_weighted_points(h),
         FitConfig(initial_components=2, seed=11, temperature=np.array([0.85, 0.85])))
    h2 = G.bin_particles(p1, Plane.uv, 200, AxisRange(-6, 6), AxisRange(-6, 6))
    case("plane 2V 200^2 K=12", G.to_weighted_points(h2),
         FitConfig(initial_components=12, seed=1, temperature=np.array([1.0, 1.0])))
    rng = np.random.default_rng(2)
    x = rng.normal(size=(32768, 3))
    w = rng.uniform(0.5, 3.0, 32768)
    case("cfg2-size 3V 32^3 K=4", WeightedPoints.from_(x, w),
         FitConfig(initial_components=4, seed=2, temperature=np.ones(3)))


if __name__ == "__main__":
    main()
