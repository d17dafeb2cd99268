"""Small end-to-end run of every device entry point (odd cell sizes, empty cells, host and
device buffers, streams): python tools/sanitize_smoke.py"""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200.stream import H2D, RecordStream  # noqa: E402
from paper_2504_14897_b200.types import (AxisRange, FitConfig, ModelMeta, ParticleSet,  # noqa: E402
                                         Plane)


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 900, 37)
    counts[-1] = 0
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = int(offs[-1])
    for d, nb in ((3, 24), (2, 32)):
        v = [torch.from_numpy(rng.normal(size=n) * 1.5).to(dev) for _ in range(d)]
        b = G.CellBatch(v, torch.from_numpy(offs).to(dev), nb, [-5] * d, [5] * d)
        meta = ModelMeta("e", None, 1, [AxisRange(-5, 5)] * d)
        bins, res, rec, ro = G.compress_cells(b, FitConfig(initial_components=3, seed=1, temperature=np.ones(d)), meta)
        G.cell_metrics(b, bins, res)
        hb = G.CellBatch([x.cpu().numpy() for x in v], offs, nb, [-5] * d, [5] * d)
        G.compress_cells(hb, FitConfig(initial_components=3, seed=1, temperature=np.ones(d)), meta)
        with tempfile.TemporaryDirectory() as t:
            with RecordStream(os.path.join(t, "a.gmmcs")) as s:
                s.append_records(rec, ro)
            if d == 2:
                with RecordStream(os.path.join(t, "h.h2ds"), H2D) as s:
                    s.append_h2d(b, bins)
    p = ParticleSet(rng.normal(size=(5000, 3)), None, "e", np.ones(3))
    h = G.bin_particles(p, Plane.uv, 40, AxisRange(-4, 4), AxisRange(-4, 4))
    G.all_planes(p, 40, AxisRange(-4, 4))
    pts = G.to_weighted_points(h)
    r = G.fit(pts, FitConfig(initial_components=4, seed=2, temperature=np.ones(2)))
    G.assemble_metrics(r.model, h, pts, 5000, 3)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
