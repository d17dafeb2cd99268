"""Per-particle cell-index input (vdfcg_bin_cells_indexed / vdfcg_compress_cells_indexed):
particles in any order with an int32 cell id each (BASELINE north_star: "streams particle
(u,v,w) and cell-index arrays"). The device groups them with a stable radix sort whose first
pass computes the bin keys; histograms must equal the oracle's stable group-by-cell +
per-cell binning BIT-EXACTLY (unit and fractional weights), and the fitted records must
equal the pre-grouped path's byte for byte."""
import numpy as np
import pytest

import oracle as O
from helpers import TOL_WEIGHTED_HIST
from paper_2504_14897_b200 import FitConfig, InvalidArgument, ModelMeta, AxisRange
from paper_2504_14897_b200 import cells as G

pytestmark = pytest.mark.gpu


def _case(n, n_cells, d, seed, weighted=False, sorted_ids=False, empty_every=0):
    rng = np.random.default_rng(seed)
    cell = rng.integers(0, n_cells, size=n).astype(np.int32)
    if empty_every:
        cell = np.where(cell % empty_every == 0, (cell + 1) % n_cells, cell).astype(np.int32)
    if sorted_ids:
        cell = np.sort(cell)
    drift = (cell.astype(np.float64) / max(n_cells, 1))[:, None] * 2.0 - 1.0
    v = rng.normal(size=(n, d)) * 1.3 + drift
    v[rng.random(n) < 0.01, 0] = 9.0  # some out of range
    w = rng.uniform(0.1, 4.0, size=n) if weighted else None
    return v, cell, w


def _check_bins(offs, bins, ooffs, ob, n_cells, weighted=False):
    offs = np.asarray(offs)
    assert np.array_equal(offs, ooffs)
    nnz = np.asarray(bins.nnz)
    assert np.array_equal(nnz, ob.nnz)
    assert np.array_equal(np.asarray(bins.out_of_range), ob.out_of_range)
    if weighted:  # the sum over bins (Eigen sum(), histogram.hpp:25) has no fixed order
        np.testing.assert_allclose(np.asarray(bins.in_range), ob.in_range, rtol=TOL_WEIGHTED_HIST)
    else:
        assert np.array_equal(np.asarray(bins.in_range), ob.in_range)
    keys, counts = np.asarray(bins.keys), np.asarray(bins.counts)
    for c in range(n_cells):
        b, k = ooffs[c], ob.nnz[c]
        assert np.array_equal(keys[b:b + k], ob.keys[b:b + k]), c
        assert np.array_equal(counts[b:b + k], ob.counts[b:b + k]), c


@pytest.mark.parametrize("n,n_cells,d,nb,weighted,sorted_ids", [
    (200_000, 200, 3, 32, False, False),      # one radix pass (8 bits)
    (300_000, 1000, 3, 48, False, False),     # two passes
    (300_000, 1000, 3, 48, False, True),      # pre-sorted ids (PIC order)
    (400_000, 300_000, 3, 16, False, False),  # three passes, mostly 1-2 particles per cell
    (250_000, 500, 2, 64, True, False),       # weighted: stable order -> exact sums
    (150_000, 5000, 3, 24, True, False),      # weighted 3V, two passes
    (3_000_000, 64, 3, 32, False, False),     # big cells (dense path)
])
def test_indexed_bins_bit_exact(n, n_cells, d, nb, weighted, sorted_ids):
    v, cell, w = _case(n, n_cells, d, seed=n_cells + d, weighted=weighted, sorted_ids=sorted_ids,
                       empty_every=7)
    lo, hi = [-5.0] * d, [5.0] * d
    ooffs, ob = O.bin_cells_indexed(O.ParticlesHost(v, cell, n_cells, nb, lo, hi, w))
    batch = G.ParticleBatch(v, cell, n_cells, nb, lo, hi, weights=w)
    offs, bins = G.bin_cells_indexed(batch)
    _check_bins(offs, bins, ooffs, ob, n_cells, weighted)


def test_indexed_device_tensors_match_host():
    import torch
    v, cell, _ = _case(100_000, 777, 3, seed=5)
    lo, hi = [-5.0] * 3, [5.0] * 3
    ho, hb = G.bin_cells_indexed(G.ParticleBatch(v, cell, 777, 32, lo, hi))
    tv = [torch.from_numpy(np.ascontiguousarray(v[:, a])).cuda() for a in range(3)]
    do, db = G.bin_cells_indexed(G.ParticleBatch(tv, torch.from_numpy(cell).cuda(), 777, 32, lo, hi))
    torch.cuda.synchronize()
    assert np.array_equal(do.cpu().numpy(), ho)
    keys = db.keys.cpu().numpy().view(np.uint32)
    counts = db.counts.cpu().numpy()
    assert np.array_equal(db.nnz.cpu().numpy(), hb.nnz)
    assert np.array_equal(db.out_of_range.cpu().numpy(), hb.out_of_range)
    for c in range(777):
        b, k = ho[c], hb.nnz[c]
        assert np.array_equal(keys[b:b + k], hb.keys[b:b + k])
        assert np.array_equal(counts[b:b + k], hb.counts[b:b + k])


def test_indexed_empty_and_single_cell():
    lo, hi = [-5.0] * 3, [5.0] * 3
    v = np.zeros((0, 3))
    offs, bins = G.bin_cells_indexed(G.ParticleBatch(v, np.zeros(0, np.int32), 5, 16, lo, hi))
    assert np.array_equal(offs, np.zeros(6, np.int64))
    assert np.array_equal(bins.nnz, np.zeros(5, np.int32))
    v, cell, _ = _case(10_000, 1, 3, seed=2)
    ooffs, ob = O.bin_cells_indexed(O.ParticlesHost(v, cell, 1, 16, lo, hi))
    offs, bins = G.bin_cells_indexed(G.ParticleBatch(v, cell, 1, 16, lo, hi))
    _check_bins(offs, bins, ooffs, ob, 1)


@pytest.mark.parametrize("bad", [-1, 50])
def test_indexed_rejects_out_of_range_cell(bad):
    v, cell, _ = _case(20_000, 50, 3, seed=3)
    cell[1234] = bad
    with pytest.raises(InvalidArgument, match="cell index out of range"):
        G.bin_cells_indexed(G.ParticleBatch(v, cell, 50, 16, [-5.0] * 3, [5.0] * 3))
    with pytest.raises(ValueError, match="cell index out of range"):
        O.bin_cells_indexed(O.ParticlesHost(v, cell, 50, 16, [-5.0] * 3, [5.0] * 3))


def test_indexed_rejects_nonpositive_weight():
    v, cell, w = _case(20_000, 50, 3, seed=4, weighted=True)
    w[7] = 0.0
    with pytest.raises(InvalidArgument, match="weights must all be > 0"):
        G.bin_cells_indexed(G.ParticleBatch(v, cell, 50, 16, [-5.0] * 3, [5.0] * 3, weights=w))


@pytest.mark.parametrize("weighted", [False, True])
def test_compress_indexed_equals_grouped_path(weighted):
    """Fits and .gmmc records through the cell-index entry point are byte-identical to the
    pre-grouped entry point fed the stably grouped particles."""
    n_cells, n = 600, 600 * 1500
    v, cell, w = _case(n, n_cells, 3, seed=9, weighted=weighted)
    lo, hi = [-5.0] * 3, [5.0] * 3
    order = np.argsort(cell, kind="stable")
    offs_ref = np.zeros(n_cells + 1, np.int64)
    np.cumsum(np.bincount(cell, minlength=n_cells), out=offs_ref[1:])
    cfg = FitConfig(initial_components=4, max_em_iterations=60, seed=11)
    meta = ModelMeta(species_label="e", plane=None, cycle=3, axis_ranges=[AxisRange(-5, 5)] * 3)
    gb = G.CellBatch(np.ascontiguousarray(v[order]), offs_ref, 32, lo, hi,
                     weights=None if w is None else np.ascontiguousarray(w[order]))
    _, r1, rec1, ro1 = G.compress_cells(gb, cfg, meta=meta)
    offs, _, r2, rec2, ro2 = G.compress_cells_indexed(G.ParticleBatch(v, cell, n_cells, 32, lo, hi, weights=w),
                                                      cfg, meta=meta)
    assert np.array_equal(offs, offs_ref)
    for f in ("status", "components", "iterations", "weights", "means", "covariances", "final_loglik"):
        assert np.array_equal(getattr(r1, f), getattr(r2, f)), f
    assert np.array_equal(ro1, ro2)
    assert bytes(rec1) == bytes(rec2)


def test_compress_indexed_warm_start_equals_grouped_warm():
    """Time series with unsorted particles: cycle 2 restarts every cell from its cycle-1
    model (pipeline.cpp:482-564) — identical to the grouped path's warm start."""
    n_cells, n = 300, 300 * 1200
    v, cell, _ = _case(n, n_cells, 3, seed=21)
    lo, hi = [-5.0] * 3, [5.0] * 3
    order = np.argsort(cell, kind="stable")
    offs_ref = np.zeros(n_cells + 1, np.int64)
    np.cumsum(np.bincount(cell, minlength=n_cells), out=offs_ref[1:])
    cfg = FitConfig(initial_components=3, max_em_iterations=50, seed=4)
    pb = G.ParticleBatch(v, cell, n_cells, 32, lo, hi)
    _, _, r1, _, _ = G.compress_cells_indexed(pb, cfg)
    v2 = v + 0.05
    _, _, r2, _, _ = G.compress_cells_indexed(G.ParticleBatch(v2, cell, n_cells, 32, lo, hi), cfg, warm=r1)
    gb = G.CellBatch(np.ascontiguousarray(v2[order]), offs_ref, 32, lo, hi)
    _, g2, _, _ = G.compress_cells(gb, cfg, warm=r1)
    for f in ("status", "components", "iterations", "weights", "means", "covariances", "final_loglik"):
        assert np.array_equal(getattr(r2, f), getattr(g2, f)), f
    assert np.mean(r2.iterations) < np.mean(r1.iterations) + 1  # warm restarts are no slower
