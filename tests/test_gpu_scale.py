"""GPU: golden vectors produced by the reference's own refem::fit, full-size BASELINE
configs against the oracle, bitwise determinism, and size-independent properties at
full cfg4 scale (mass conservation, unit weight sums, record integrity)."""
import glob
import os
import struct
import zlib

import numpy as np
import pytest

import oracle as O
import paper_2504_14897_b200 as G
from helpers import TOL_EM, model_close
from paper_2504_14897_b200.types import (AffineMap, AxisRange, FitConfig, GaussianComponent,
                                         GmmModel, ModelMeta, WeightedPoints)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "refem_*.npz"))))
def test_gpu_fit_matches_reference_refem(path):
    """Acceptance criterion 5 against the reference's own EM (golden outputs)."""
    g = np.load(path)
    wp = WeightedPoints.from_(np.stack([g["xs"], g["ys"]], 1), np.ones(len(g["xs"])))
    r = G.fit(wp, FitConfig(initial_components=int(g["m"]), seed=int(g["seed"]), temperature=np.ones(2)))
    assert r.iterations_used == int(g["iterations"]) and r.model.size() == len(g["alpha"])
    for i, c in enumerate(r.model.components):
        assert _rel(c.weight, g["alpha"][i]) <= TOL_EM
        assert _rel(c.mean, g["means"][i]) <= TOL_EM
        assert _rel(c.covariance, g["covs"][i]) <= TOL_EM
    assert _rel(r.loglik_trace, g["trace"]) <= TOL_EM


def _batch(v, offs, nb, r, w=None):
    d = v.shape[1]
    return G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(d)], offs, nb, [-r] * d, [r] * d, w)


def _oracle_model(res, c, d):
    k = res.k
    comps = [GaussianComponent(res.weights[c * k + i], res.means[(c * k + i) * d:(c * k + i + 1) * d],
                               res.covariances[(c * k + i) * d * d:(c * k + i + 1) * d * d].reshape(d, d))
             for i in range(res.components[c])]
    return GmmModel(comps, AffineMap.identity(d), d)


def test_cfg2_full_size_parity():
    """BASELINE cfg2: one cell, 1e7 particles, 3V 32^3 bins, K=4 full covariances."""
    covs = []
    rng = np.random.default_rng(7)
    for k in range(4):
        a = np.eye(3) + 0.3 * (np.ones((3, 3)) - np.eye(3))
        covs.append(a * rng.uniform(0.3, 1.0))
    p = O.generate([0.4, 0.3, 0.2, 0.1], [[0, 0, 0], [2.5, 0, 0], [-1.5, 1.5, 0], [0, -2, 1.5]],
                   covs, 10_000_000, 17)
    offs = np.array([0, p.count()], dtype=np.int64)
    cfg = FitConfig(initial_components=4, seed=17, temperature=p.nominal_temperature)
    ob, orr = O.compress_cells(O.CellsHost(p.velocities, offs, 32, [-6] * 3, [6] * 3), cfg,
                               trace=cfg.max_em_iterations)
    gb, gr, _, _ = G.compress_cells(_batch(p.velocities, offs, 32, 6.0), cfg, trace=True)
    assert np.array_equal(gb.nnz, ob.nnz)
    k = int(ob.nnz[0])
    assert np.array_equal(gb.keys[:k], ob.keys[:k]) and np.array_equal(gb.counts[:k], ob.counts[:k])
    assert gr.status[0] == 0 and gr.iterations[0] == orr.iterations[0]
    assert gr.components[0] == orr.components[0]
    n_it = int(orr.iterations[0])
    assert _rel(gr.loglik_trace[:n_it], orr.loglik_trace[:n_it]) <= TOL_EM
    assert model_close(gr.model(0), _oracle_model(orr, 0, 3)) <= TOL_EM


def test_cfg1_full_size_all_planes_and_fit():
    p = O.preset("drifting-beam", 1_000_000, 11)
    hg = G.all_planes(p, 64, AxisRange(-6, 6))
    ho = O.all_planes(p, 64, AxisRange(-6, 6))
    cfg = FitConfig(initial_components=2, seed=11, temperature=np.ones(2))
    for a, b in zip(hg, ho):
        assert np.array_equal(a.counts, b.counts)
        rg, ro = G.fit(G.to_weighted_points(a), cfg), O.fit(O.to_weighted_points(b), cfg)
        assert rg.iterations_used == ro.iterations_used and model_close(rg.model, ro.model) <= TOL_EM


def test_weighted_cells_parity():
    rng = np.random.default_rng(4)
    offs = np.arange(33, dtype=np.int64) * 1500
    v = rng.normal(size=(int(offs[-1]), 3))
    w = rng.uniform(0.1, 4.0, size=int(offs[-1]))
    cfg = FitConfig(initial_components=3, seed=5, temperature=np.ones(3))
    ob, orr = O.compress_cells(O.CellsHost(v, offs, 48, [-5] * 3, [5] * 3, w), cfg)
    gb, gr, _, _ = G.compress_cells(_batch(v, offs, 48, 5.0, w), cfg)
    for c in range(32):
        b, k = offs[c], ob.nnz[c]
        assert np.array_equal(gb.counts[b:b + k], ob.counts[b:b + k])  # sequential sums: bit-exact
    assert np.array_equal(gr.iterations, orr.iterations)
    for c in range(32):
        assert model_close(gr.model(c), _oracle_model(orr, c, 3)) <= TOL_EM


def test_determinism_bitwise():
    import torch
    dev = torch.device("cuda", 0)
    offs = torch.arange(2049, dtype=torch.int64, device=dev) * 1900
    axes = [torch.empty(2048 * 1900, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 11, 0, *axes)
    b = G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3)
    cfg = FitConfig(initial_components=4, seed=11, temperature=np.ones(3))
    meta = ModelMeta("e", None, 0, [AxisRange(-6, 6)] * 3)
    _, r1, rec1, _ = G.compress_cells(b, cfg, meta)
    _, r2, rec2, _ = G.compress_cells(b, cfg, meta)
    assert torch.equal(rec1, rec2)
    for f in ("weights", "means", "covariances", "final_loglik", "iterations", "status"):
        a, b2 = getattr(r1, f), getattr(r2, f)
        if a.dtype == torch.float64:  # bit patterns (NaN-safe)
            a, b2 = a.view(torch.int64), b2.view(torch.int64)
        assert torch.equal(a, b2), f


def test_cfg4_scale_properties():
    """One cfg4 species at full scale on one GPU (262144 cells, 5e8 particles): exact mass
    conservation per cell, every fit valid (status 0, weights sum to 1 within 1e-12,
    SPD covariances), every .gmmc record well formed (magic, CRC, size)."""
    import torch
    dev = torch.device("cuda", 0)
    n_cells, total = 64 ** 3, 500_000_000
    base, extra = divmod(total, n_cells)
    counts = np.full(n_cells, base, dtype=np.int64)
    counts[:extra] += 1
    offs_h = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    offs = torch.from_numpy(offs_h).to(dev)
    axes = [torch.empty(total, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 11, 0, *axes)
    b = G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3)
    cfg = FitConfig(initial_components=4, seed=11, temperature=np.ones(3))
    bins, res, rec, roffs = G.compress_cells(b, cfg, ModelMeta("e", None, 0, [AxisRange(-6, 6)] * 3))
    tot = (bins.in_range + bins.out_of_range).cpu().numpy()
    assert np.array_equal(tot, counts.astype(np.float64))
    st = res.status.cpu().numpy()
    assert (st == 0).all()
    K = res.k
    m = res.components.cpu().numpy()
    w = res.weights.cpu().numpy().reshape(n_cells, K)
    mask = np.arange(K)[None, :] < m[:, None]
    assert np.abs((w * mask).sum(1) - 1.0).max() <= 1e-12
    cov = res.covariances.cpu().numpy().reshape(n_cells, K, 3, 3)
    ev = np.linalg.eigvalsh(cov[mask])
    assert (ev > 0).all()
    rec_h = rec.cpu().numpy().tobytes()
    ro = roffs.cpu().numpy()
    for c in np.random.default_rng(0).choice(n_cells, 2000, replace=False):
        r = rec_h[ro[c]:ro[c + 1]]
        assert r[:4] == b"GMMC" and r[5] == 3
        hb = 26 + 16 * 3 + 1
        assert struct.unpack("<I", r[hb - 4:hb])[0] == zlib.crc32(r[:hb - 4])
        assert len(r) == hb + m[c] * 80
        assert struct.unpack("<I", r[8:12])[0] == m[c]


def _cell_points(bins, offs, c, nb, r, d):
    """Data-space bin centres of cell c (the oracle's WeightedPoints for that cell)."""
    k = int(bins.nnz[c])
    keys = np.asarray(bins.keys[offs[c]:offs[c] + k]).astype(np.int64)
    idx = []
    for _ in range(d):
        idx.append(keys % nb)
        keys //= nb
    idx = idx[::-1]
    pts = np.stack([-r + (i + 0.5) * ((2 * r) / nb) for i in idx], 1)
    return WeightedPoints(pts, np.asarray(bins.counts[offs[c]:offs[c] + k]).copy(), float(bins.in_range[c]))


def test_time_series_warm_start_per_cell():
    """Per-cell warm start (pipeline.cpp:482-564): cycle 1 fits each cell from its own
    cycle-0 model; matches the oracle's fit with FitConfig.warm_start = that model
    (wgmm.cpp:142-161), and static data converges in <= 2 iterations (test_wgmm.cpp:444-479)."""
    rng = np.random.default_rng(12)
    n_cells, per = 48, 20000
    offs = np.arange(n_cells + 1, dtype=np.int64) * per
    v = rng.normal(size=(n_cells * per, 3))
    left = rng.random(n_cells * per) < 0.5
    v[:, 0] += np.where(left, -3.0, 3.0)
    cfg = FitConfig(initial_components=2, seed=13, temperature=np.ones(3))
    batch = _batch(v, offs, 24, 6.0)
    bins0, res0, _, _ = G.compress_cells(batch, cfg)
    conv = res0.converged.astype(bool)
    assert conv.sum() >= n_cells // 2
    # cycle 1, same data: every cell restarts from its own model; converged cells stay put
    bins1, res1, _, _ = G.compress_cells(batch, cfg, warm=res0)
    assert (res1.status == 0).all()
    assert (res1.iterations[conv] <= 2).all(), res1.iterations[conv]
    # cycle 1 on fresh (drifted) particles: compare against the oracle per cell
    v2 = v + 0.05 * rng.normal(size=v.shape)
    b2 = _batch(v2, offs, 24, 6.0)
    gb, gr, _, _ = G.compress_cells(b2, cfg, warm=res0)
    assert gr.iterations.mean() < res0.iterations.mean()
    for c in range(0, n_cells, 6):
        wp = _cell_points(gb, offs, c, 24, 6.0, 3)
        fc = FitConfig(initial_components=2, seed=13, temperature=np.ones(3), warm_start=res0.model(c))
        ro = O.fit(wp, fc)
        assert gr.iterations[c] == ro.iterations_used
        assert model_close(gr.model(c), ro.model) <= TOL_EM


@pytest.mark.parametrize("K,nb", [(4, 48), (3, 32)])
def test_fp32_estep_mode_within_1e4(K, nb):
    """FP32 E-step option (north star: 1e-4 FP32 / 1e-9 FP64), compared with the FP64
    oracle in fixed-iteration mode (no pruning, convergence disabled) so both run the
    same number of EM steps."""
    rng = np.random.default_rng(21)
    n_cells, per = 64, 4000
    offs = np.arange(n_cells + 1, dtype=np.int64) * per
    v = rng.normal(size=(n_cells * per, 3))
    v[rng.random(n_cells * per) < 0.3, 0] += 2.5
    base = dict(initial_components=K, seed=5, temperature=np.ones(3), max_em_iterations=30,
                loglik_rel_tolerance=1e-300, prune_threshold=1e-300)
    ob, orr = O.compress_cells(O.CellsHost(v, offs, nb, [-6] * 3, [6] * 3), FitConfig(**base))
    gb, gr, _, _ = G.compress_cells(_batch(v, offs, nb, 6.0), FitConfig(**base, estep_fp32=True))
    assert (gr.iterations == 30).all() and np.array_equal(gr.components, orr.components)
    worst = max(model_close(gr.model(c), _oracle_model(orr, c, 3), tol=1e-4) for c in range(n_cells))
    assert worst <= 1e-4, worst
    np.testing.assert_allclose(gr.final_loglik, orr.final_loglik, rtol=1e-6)


def test_pipelined_host_path_bitwise_equals_device_path():
    """Host-resident inputs take the chunked H2D/compute-overlap path; results and .gmmc
    records must be bitwise identical to the device-resident path."""
    import torch
    dev = torch.device("cuda", 0)
    n_cells, per = 4096, 1500
    offs = torch.arange(n_cells + 1, dtype=torch.int64, device=dev) * per
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 7, 0, *axes)
    cfg = FitConfig(initial_components=4, seed=11, temperature=np.ones(3))
    meta = ModelMeta("e", None, 3, [AxisRange(-6, 6)] * 3)
    _, rd, recd, offd = G.compress_cells(G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3), cfg, meta)
    host_axes = [a.cpu().pin_memory() for a in axes]
    hb = G.CellBatch(host_axes, offs.cpu(), 48, [-6] * 3, [6] * 3)
    _, rh, rech, offh = G.compress_cells(hb, cfg, meta)
    assert torch.equal(recd.cpu(), rech) and torch.equal(offd.cpu(), offh)
    for f in ("status", "components", "iterations", "weights", "means", "covariances", "final_loglik"):
        a, b = getattr(rd, f).cpu(), getattr(rh, f)
        if a.dtype == torch.float64:  # compare bit patterns
            a, b = a.view(torch.int64), b.view(torch.int64)
        if f in ("weights", "means", "covariances"):  # slots past `components` are unspecified
            a, b = a.view(n_cells, 4, -1), b.view(n_cells, 4, -1)
            used = torch.arange(4)[None, :] < rh.components[:, None].long()
            a, b = a[used], b[used]
        assert torch.equal(a, b), f


def test_pipelined_host_path_weighted_bitwise():
    """Weighted particles through the chunked host-input path == device-resident path."""
    import torch
    dev = torch.device("cuda", 0)
    n_cells, per = 2500, 1800
    offs = torch.arange(n_cells + 1, dtype=torch.int64, device=dev) * per
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 17, 1, *axes)
    w = torch.rand(n_cells * per, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(3)) * 3.0 + 0.1
    cfg = FitConfig(initial_components=3, seed=5, temperature=np.ones(3))
    meta = ModelMeta("i", None, 2, [AxisRange(-6, 6)] * 3)
    _, rd, recd, _ = G.compress_cells(G.CellBatch(axes, offs, 40, [-6] * 3, [6] * 3, w), cfg, meta)
    hb = G.CellBatch([a.cpu().pin_memory() for a in axes], offs.cpu(), 40, [-6] * 3, [6] * 3,
                     w.cpu().pin_memory())
    assert hb.n >= (1 << 22)  # large enough for the pipelined path
    _, rh, rech, _ = G.compress_cells(hb, cfg, meta)
    assert torch.equal(recd.cpu(), rech)
    for f in ("status", "components", "iterations"):
        assert torch.equal(getattr(rd, f).cpu(), getattr(rh, f)), f
    assert torch.equal(rd.weights.cpu().view(torch.int64), rh.weights.view(torch.int64))


@pytest.mark.parametrize("weighted", [False, True])
def test_pageable_host_path_bitwise_equals_device_path(weighted):
    """Pageable host inputs (plain numpy, as a reference caller's Eigen storage) go through
    the pinned staging ring (host copy threads + async H2D) and must give the device path's
    results bit for bit; small 64 MB staging slots mean many pieces per chunk."""
    import torch
    dev = torch.device("cuda", 0)
    n_cells, per = 3000, 1700
    offs = torch.arange(n_cells + 1, dtype=torch.int64, device=dev) * per
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 23, 0, *axes)
    w = None
    if weighted:
        w = torch.rand(n_cells * per, dtype=torch.float64, device=dev,
                       generator=torch.Generator(dev).manual_seed(5)) * 3.0 + 0.1
    cfg = FitConfig(initial_components=4, seed=7, temperature=np.ones(3))
    meta = ModelMeta("e", None, 4, [AxisRange(-6, 6)] * 3)
    _, rd, recd, offd = G.compress_cells(G.CellBatch(axes, offs, 48, [-6] * 3, [6] * 3, w), cfg, meta)
    hv = [np.ascontiguousarray(a.cpu().numpy()) for a in axes]  # pageable
    hw = None if w is None else np.ascontiguousarray(w.cpu().numpy())
    hb = G.CellBatch(hv, offs.cpu().numpy(), 48, [-6] * 3, [6] * 3, hw)
    assert hb.n >= (1 << 22)
    _, rh, rech, offh = G.compress_cells(hb, cfg, meta)
    assert bytes(recd.cpu().numpy()) == bytes(rech) and np.array_equal(offd.cpu().numpy(), offh)
    for f in ("status", "components", "iterations", "final_loglik"):
        assert np.array_equal(getattr(rd, f).cpu().numpy(), getattr(rh, f)), f


def test_cfg3_full_size_parity():
    """BASELINE cfg3 at full size: 16x16 cells x 390625 particles (1e8), 3V 32^3 bins, K=3
    (the reference's per-part fit_one_plane, pipeline.cpp:130-160, on every cell). Every
    cell's compacted histogram bit-exact vs the oracle; identical iterations and M-hat;
    parameters and final log-likelihood within 1e-9 on every cell."""
    import torch
    dev = torch.device("cuda", 0)
    n_cells, per = 256, 390_625
    offs = torch.arange(n_cells + 1, dtype=torch.int64, device=dev) * per
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 11, 0, *axes)
    cfg = FitConfig(initial_components=3, seed=11, temperature=np.ones(3))
    gb, gr, _, _ = G.compress_cells(G.CellBatch(axes, offs, 32, [-6] * 3, [6] * 3), cfg)
    offs_h = offs.cpu().numpy()
    v = np.empty((n_cells * per, 3), order="F")
    for a in range(3):
        v[:, a] = axes[a].cpu().numpy()
    del axes
    ob, orr = O.compress_cells(O.CellsHost(v, offs_h, 32, [-6] * 3, [6] * 3), cfg,
                               threads=os.cpu_count() or 1)
    nnz = gb.nnz.cpu().numpy()
    assert np.array_equal(nnz, ob.nnz)
    keys, counts = gb.keys.cpu().numpy(), gb.counts.cpu().numpy()
    for c in range(n_cells):
        b, k = offs_h[c], nnz[c]
        assert np.array_equal(keys[b:b + k], ob.keys[b:b + k]), c
        assert np.array_equal(counts[b:b + k], ob.counts[b:b + k]), c
    assert np.array_equal(gb.out_of_range.cpu().numpy(), ob.out_of_range)
    assert (gr.status.cpu().numpy() == 0).all()
    assert np.array_equal(gr.iterations.cpu().numpy(), orr.iterations)
    assert np.array_equal(gr.components.cpu().numpy(), orr.components)
    gres = gr.numpy()
    worst = 0.0
    for c in range(n_cells):
        worst = max(worst, model_close(gres.model(c), _oracle_model(orr, c, 3)))
    assert worst <= TOL_EM, worst
    fl = gr.final_loglik.cpu().numpy()
    assert _rel(fl, orr.final_loglik) <= TOL_EM
