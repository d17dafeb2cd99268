"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same inputs.

Tolerances: histograms bit-exact for unit weights, 1e-12 relative for fractional
weights; FP64 EM parameters / log-likelihood trace 1e-9 relative with identical
iteration counts, component counts and pruning events.
"""
import numpy as np
import pytest

import oracle as O
import paper_2504_14897_b200 as G
from helpers import TOL_EM, TOL_WEIGHTED_HIST, model_close, rel
from paper_2504_14897_b200.types import (AffineMap, AxisRange, FitConfig, GaussianComponent,
                                         GmmModel, ModelMeta, ParticleSet, Plane, WeightedPoints)

pytestmark = pytest.mark.gpu


def cfg1_particles(n=1_000_000, seed=11):
    """BASELINE cfg1: 2V drifting beam, fractions (0.8, 0.2), means (0,0)/(3,0), var 1/0.25."""
    return O.generate([0.8, 0.2], [[0, 0], [3, 0]], [np.eye(2), 0.25 * np.eye(2)], n, seed,
                      label="e")


def assert_fit_equal(g, o, tol=TOL_EM):
    assert g.iterations_used == o.iterations_used
    assert g.converged == o.converged
    assert g.model.size() == o.model.size()
    assert [(e.iteration, e.component) for e in g.pruning_events] == \
        [(e.iteration, e.component) for e in o.pruning_events]
    assert len(g.loglik_trace) == len(o.loglik_trace)
    for a, b in zip(g.loglik_trace, o.loglik_trace):
        assert rel(a, b) <= tol, (a, b)
    assert model_close(g.model, o.model) <= tol


def test_bin_particles_cfg1_bit_exact():
    p = cfg1_particles()
    for nb in (64, 200):
        hg = G.bin_particles(p, Plane.uv, nb, AxisRange(-6, 6), AxisRange(-6, 6))
        ho = O.bin_particles(p, Plane.uv, nb, AxisRange(-6, 6), AxisRange(-6, 6))
        assert np.array_equal(hg.counts, ho.counts)
        assert hg.out_of_range_count == ho.out_of_range_count


def test_bin_particles_weighted_and_edges():
    rng = np.random.default_rng(99)
    v = rng.uniform(-3, 3, size=(5000, 2))
    w = rng.uniform(0.1, 4.0, size=5000)
    v[:4] = [[0.0, 0.0], [1.0, 1.0], [np.nan, 0.0], [np.inf, -np.inf]]
    p = ParticleSet(v, w, "x", np.ones(2))
    hg = G.bin_particles(p, Plane.uv, 50, AxisRange(-1, 1), AxisRange(-1, 1))
    ho = O.bin_particles(p, Plane.uv, 50, AxisRange(-1, 1), AxisRange(-1, 1))
    # every bin summed in particle order, like the reference's sequential `+=`: bit-exact
    assert np.array_equal(hg.counts, ho.counts)
    assert hg.out_of_range_count == ho.out_of_range_count


@pytest.mark.parametrize("n,nb", [(1_000_000, 64), (300_000, 200), (50_000, 2)])
def test_weighted_bin_particles_and_all_planes_bit_exact(n, nb):
    """Fractional weights (w ~ U(0.1, 4), test_histogram.cpp:76): bit-identical to the
    reference's sequential sums for bin_particles and all_planes, and run-to-run stable."""
    rng = np.random.default_rng(n + nb)
    v = rng.normal(size=(n, 3)) * 1.7
    w = rng.uniform(0.1, 4.0, size=n)
    p = ParticleSet(v, w, "x", np.ones(3))
    hg = G.bin_particles(p, Plane.vw, nb, AxisRange(-4, 4), AxisRange(-4, 4))
    ho = O.bin_particles(p, Plane.vw, nb, AxisRange(-4, 4), AxisRange(-4, 4))
    assert np.array_equal(hg.counts, ho.counts)
    assert hg.out_of_range_count == ho.out_of_range_count
    ag = G.all_planes(p, nb, AxisRange(-4, 4))
    ao = O.all_planes(p, nb, AxisRange(-4, 4))
    for a, b in zip(ag, ao):
        assert np.array_equal(a.counts, b.counts)
        assert a.out_of_range_count == b.out_of_range_count
    again = G.all_planes(p, nb, AxisRange(-4, 4))
    assert all(np.array_equal(a.counts, b.counts) for a, b in zip(ag, again))


def test_all_planes_bit_exact():
    p = O.preset("drifting-beam", 200_000, 5)
    hg = G.all_planes(p, 64, AxisRange(-5, 5))
    ho = O.all_planes(p, 64, AxisRange(-5, 5))
    for a, b in zip(hg, ho):
        assert np.array_equal(a.counts, b.counts)
        assert a.out_of_range_count == b.out_of_range_count


def test_to_weighted_points_bit_exact():
    p = cfg1_particles(100_000, 3)
    h = O.bin_particles(p, Plane.uv, 64, AxisRange(-6, 6), AxisRange(-6, 6))
    for drop in (True, False):
        a = G.to_weighted_points(h, drop)
        b = O.to_weighted_points(h, drop)
        assert np.array_equal(a.points, b.points)
        assert np.array_equal(a.weights, b.weights)
        assert a.total_weight == b.total_weight


def test_fit_cfg1_end_to_end_parity():
    p = cfg1_particles()
    h = O.bin_particles(p, Plane.uv, 64, AxisRange(-6, 6), AxisRange(-6, 6))
    pts = O.to_weighted_points(h)
    cfg = FitConfig(initial_components=2, seed=11, temperature=np.array([0.85, 0.85]))
    assert_fit_equal(G.fit(pts, cfg), O.fit(pts, cfg))


@pytest.mark.parametrize("seed", range(8))
def test_fit_random_weighted_clouds(seed):
    rng = np.random.default_rng(seed)
    n = 2000
    pts = np.stack([2.0 * rng.normal(size=n) + 1.0, 0.5 * rng.normal(size=n) - 3.0], 1)
    w = rng.uniform(0.2, 5.0, size=n)
    wp = WeightedPoints.from_(pts, w)
    cfg = FitConfig(initial_components=6, seed=9 + seed)
    assert_fit_equal(G.fit(wp, cfg), O.fit(wp, cfg))


def test_fit_default_config_12_components():
    p = O.preset("drifting-beam", 100_000, 7)
    h = O.bin_particles(p, Plane.uv, 100, AxisRange(-5, 5), AxisRange(-5, 5))
    pts = O.to_weighted_points(h)
    cfg = FitConfig(seed=3, temperature=np.ones(2))
    assert_fit_equal(G.fit(pts, cfg), O.fit(pts, cfg))


def test_fit_3d_points():
    p = O.preset("counter-streaming", 20000, 4)
    wp = WeightedPoints.from_(p.velocities, np.ones(p.count()))
    cfg = FitConfig(initial_components=4, seed=2, temperature=np.ones(3))
    assert_fit_equal(G.fit(wp, cfg), O.fit(wp, cfg))


def test_encode_model_hex_vector():
    m = GmmModel([GaussianComponent(1.0, np.array([0.5, -0.25]),
                                    np.array([[1, 0.125], [0.125, 2.0]]))], AffineMap.identity(2), 2)
    b = G.encode_model(m, ModelMeta("e", Plane.uv, 50, [AxisRange(-5, 5), AxisRange(-5, 5)]))
    assert len(b) == 107
    assert b[55:59].hex() == "525af6d7"  # header CRC-32, FORMATS.md:35-47
    assert b == O.encode_model(m, ModelMeta("e", Plane.uv, 50, [AxisRange(-5, 5), AxisRange(-5, 5)]))


def _cells_case(d, n_cells, per_cell, n_bins, seed=1, weighted=False):
    rng = np.random.default_rng(seed)
    counts = rng.integers(max(per_cell // 2, 1), per_cell * 3 // 2 + 1, size=n_cells)
    counts[0] = 0 if n_cells > 3 else counts[0]  # an empty cell
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = int(offs[-1])
    v = np.zeros((n, d), order="F")
    for c in range(n_cells):
        b, e = offs[c], offs[c + 1]
        k = e - b
        beam = rng.random(k) < 0.25
        v[b:e] = rng.normal(size=(k, d)) * np.where(beam[:, None], 0.5, 1.0)
        v[b:e, 0] += np.where(beam, 2.5 + 0.01 * c, 0.0)
    w = rng.uniform(0.1, 4.0, size=n) if weighted else None
    lo, hi = [-6.0] * d, [6.0] * d
    return v, offs, w, lo, hi


@pytest.mark.parametrize("d,n_cells,per_cell,n_bins,weighted", [
    (3, 16, 3000, 32, False),    # dense shared-memory path
    (3, 64, 1900, 48, False),    # sparse bitmap path, TMA-staged (cfg4 shape)
    (3, 48, 1900, 64, False),    # TMA-staged, 8192 bitmap words (16 per thread)
    (3, 32, 1900, 48, True),     # weighted: sort path, bit-exact sequential sums
    (2, 8, 50000, 64, False),    # 2V dense
    (3, 4, 20000, 64, False),    # dense global path
])
def test_bin_cells_bit_exact(d, n_cells, per_cell, n_bins, weighted):
    v, offs, w, lo, hi = _cells_case(d, n_cells, per_cell, n_bins, weighted=weighted)
    ob = O.bin_cells(O.CellsHost(v, offs, n_bins, lo, hi, w))
    gb = G.bin_cells(G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(d)], offs, n_bins,
                                 lo, hi, w))
    assert np.array_equal(gb.nnz, ob.nnz)
    for c in range(len(offs) - 1):
        b = offs[c]
        k = ob.nnz[c]
        assert np.array_equal(gb.keys[b:b + k], ob.keys[b:b + k])
        assert np.array_equal(gb.counts[b:b + k], ob.counts[b:b + k])
    assert np.array_equal(gb.out_of_range, ob.out_of_range)
    if weighted:
        np.testing.assert_allclose(gb.in_range, ob.in_range, rtol=TOL_WEIGHTED_HIST)
    else:
        assert np.array_equal(gb.in_range, ob.in_range)


@pytest.mark.parametrize("d,n_cells,per_cell,n_bins,K", [
    (3, 24, 1900, 48, 4),
    (3, 8, 20000, 32, 3),
    (2, 16, 5000, 64, 2),
])
def test_compress_cells_parity(d, n_cells, per_cell, n_bins, K):
    v, offs, w, lo, hi = _cells_case(d, n_cells, per_cell, n_bins, seed=5)
    cfg = FitConfig(initial_components=K, seed=11, temperature=np.ones(d))
    ob, orr = O.compress_cells(O.CellsHost(v, offs, n_bins, lo, hi), cfg, trace=cfg.max_em_iterations)
    batch = G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(d)], offs, n_bins, lo, hi)
    gbins, gres, _, _ = G.compress_cells(batch, cfg, trace=True)
    assert np.array_equal(gres.status, orr.status)
    assert np.array_equal(gres.iterations, orr.iterations)
    assert np.array_equal(gres.components, orr.components)
    assert np.array_equal(gres.converged, orr.converged)
    ok = orr.status == 0
    np.testing.assert_allclose(gres.final_loglik[ok], orr.final_loglik[ok], rtol=TOL_EM)
    for c in np.nonzero(ok)[0]:
        mg, mo = gres.model(c), None
        # oracle model for cell c
        k = orr.k
        from paper_2504_14897_b200.types import GaussianComponent as GC
        comps = [GC(orr.weights[c * k + i], orr.means[(c * k + i) * d:(c * k + i + 1) * d],
                    orr.covariances[(c * k + i) * d * d:(c * k + i + 1) * d * d].reshape(d, d))
                 for i in range(orr.components[c])]
        mo = GmmModel(comps, AffineMap.identity(d), d)
        assert model_close(mg, mo) <= TOL_EM, c


@pytest.mark.parametrize("misaligned", [False, True])
def test_bin_cells_staging_edges(misaligned):
    """Odd cell boundaries, empty first/last cells and an odd particle total exercise the
    16-byte widening of the TMA-staged bitmap kernel; 8-byte-misaligned device axes take
    the non-TMA bitmap kernel. Both must equal the oracle bit for bit."""
    import torch
    rng = np.random.default_rng(21)
    counts = rng.integers(1, 2400, size=97)
    counts[[0, 5, 96]] = 0
    counts[1] = 1
    if counts.sum() % 2 == 0:
        counts[2] += 1
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = int(offs[-1])
    v = np.asfortranarray(rng.normal(size=(n, 3)) * 1.7)
    ob = O.bin_cells(O.CellsHost(v, offs, 48, [-6] * 3, [6] * 3))
    dev = torch.device("cuda", 0)
    if misaligned:
        axes = [torch.from_numpy(np.concatenate([[0.0], v[:, a]])).to(dev)[1:] for a in range(3)]
        assert axes[0].data_ptr() % 16 == 8
    else:
        axes = [torch.from_numpy(np.ascontiguousarray(v[:, a])).to(dev) for a in range(3)]
    gb = G.bin_cells(G.CellBatch(axes, torch.from_numpy(offs).to(dev), 48, [-6] * 3, [6] * 3))
    nnz = gb.nnz.cpu().numpy()
    keys, cnts = gb.keys.cpu().numpy(), gb.counts.cpu().numpy()
    assert np.array_equal(nnz, ob.nnz)
    for c in range(len(counts)):
        b, k = offs[c], ob.nnz[c]
        assert np.array_equal(keys[b:b + k], ob.keys[b:b + k])
        assert np.array_equal(cnts[b:b + k], ob.counts[b:b + k])
    assert np.array_equal(gb.out_of_range.cpu().numpy(), ob.out_of_range)


def test_weighted_dense_cells_bit_exact():
    """Weighted cells larger than the per-cell sort (> 8192 particles: cfg3-like dense cells)
    take the ordered composite-id path: every (cell, bin) summed in particle order — equal
    to the oracle's sequential sums bit for bit; in_range (Eigen sum()) within 1e-12."""
    v, offs, w, lo, hi = _cells_case(3, 6, 40_000, 32, seed=4, weighted=True)
    from paper_2504_14897_b200 import cells as GC
    gb = GC.bin_cells(GC.CellBatch(v, offs, 32, lo, hi, weights=w))
    ob = O.bin_cells(O.CellsHost(v, offs, 32, lo, hi, w))
    assert np.array_equal(gb.nnz, ob.nnz)
    assert np.array_equal(gb.out_of_range, ob.out_of_range)
    np.testing.assert_allclose(gb.in_range, ob.in_range, rtol=TOL_WEIGHTED_HIST)
    for c in range(len(offs) - 1):
        b, k = offs[c], ob.nnz[c]
        assert np.array_equal(gb.keys[b:b + k], ob.keys[b:b + k]), c
        assert np.array_equal(gb.counts[b:b + k], ob.counts[b:b + k]), c
