"""Per-cell fit quality on the device (vdfcg_metrics_cells) vs the oracle restatement of
assemble_metrics (pipeline.cpp:106-128), 2V and 3V, host and device buffers."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200.types import FitConfig

pytestmark = pytest.mark.gpu

FIELDS = ("jsd", "kl_pq", "kl_qp", "loglik", "bic", "bic_bin_count", "mean_moment_error",
          "second_moment_error", "compression_ratio_vs_histogram", "compression_ratio_vs_raw")


def _cells(d, n_cells, per, seed, weighted=False):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(per // 2, per * 2, n_cells)
    sizes[1] = 0
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offs[-1])
    v = rng.normal(size=(n, d))
    beam = rng.uniform(size=n) < 0.25
    v[beam, 0] = 0.4 * v[beam, 0] + 2.5
    w = rng.uniform(0.2, 3.0, n) if weighted else None
    return v, offs, w


def _oracle_metrics(v, offs, nb, lo, hi, w, bins, res):
    """Oracle metrics on exactly the product's bins and results."""
    cells = O.CellsHost(v, offs, nb, lo, hi, w)
    ob = O.CellBinsHost(cells.n, cells.n_cells)
    for f in ("nnz", "keys", "counts", "out_of_range", "in_range"):
        getattr(ob, f)[:len(getattr(bins, f))] = getattr(bins, f)
    d = v.shape[1]
    orr = O.CellResultsHost(cells.n_cells, d, res.k)
    for f in ("status", "components", "weights", "means", "covariances"):
        getattr(orr, f)[:] = getattr(res, f)
    return O.cell_metrics(cells, ob, orr)


@pytest.mark.parametrize("d,weighted", [(2, False), (3, False), (3, True)])
def test_cell_metrics_vs_oracle(d, weighted):
    import paper_2504_14897_b200 as G
    v, offs, w = _cells(d, 64, 2500, 7 + d, weighted)
    nb = 40 if d == 2 else 24
    lo, hi = [-5.0] * d, [5.0] * d
    batch = G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(d)], offs, nb, lo, hi, w)
    cfg = FitConfig(initial_components=4, seed=3, temperature=np.ones(d))
    bins, res, _, _ = G.compress_cells(batch, cfg)
    got = G.cell_metrics(batch, bins, res)
    ref = _oracle_metrics(v, offs, nb, lo, hi, w, bins, res)
    ok = res.status == 0
    assert ok.sum() >= 50 and not ok[1]
    for f in FIELDS:
        a, b = getattr(got, f), getattr(ref, f)
        assert np.array_equal(np.isnan(a), np.isnan(b)), f
        assert np.array_equal(np.isinf(a), np.isinf(b)), f
        fin = np.isfinite(b)
        np.testing.assert_allclose(a[fin], b[fin], rtol=1e-9, atol=1e-13, err_msg=f)


def test_cell_metrics_device_buffers_and_determinism():
    import torch
    import paper_2504_14897_b200 as G
    dev = torch.device("cuda", 0)
    n_cells, per = 2048, 1900
    offs = torch.arange(n_cells + 1, dtype=torch.int64, device=dev) * per
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 5, 0, *axes)
    batch = G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3)
    bins, res, _, _ = G.compress_cells(batch, FitConfig(initial_components=4, seed=0, temperature=np.ones(3)))
    m1 = G.cell_metrics(batch, bins, res)
    m2 = G.cell_metrics(batch, bins, res)
    for f in FIELDS:
        assert torch.equal(getattr(m1, f).view(torch.int64), getattr(m2, f).view(torch.int64)), f
    # spot check 32 cells against the oracle
    sel = np.arange(0, n_cells, n_cells // 32)
    hb = bins.__class__(*(getattr(bins, f).cpu().numpy() for f in ("nnz", "keys", "counts", "out_of_range", "in_range")))
    hr = res.numpy()
    v = np.stack([a.cpu().numpy() for a in axes], 1)
    ref = _oracle_metrics(v, offs.cpu().numpy(), 48, [-6] * 3, [6] * 3, None, hb, hr)
    for f in FIELDS:
        a = getattr(m1, f).cpu().numpy()[sel]
        b = getattr(ref, f)[sel]
        fin = np.isfinite(b)
        assert np.array_equal(np.isinf(a), np.isinf(b)), f
        np.testing.assert_allclose(a[fin], b[fin], rtol=1e-9, atol=1e-13, err_msg=f)
    jsd = m1.jsd.cpu().numpy()
    assert np.all((jsd >= 0) & (jsd <= math.log(2)))
