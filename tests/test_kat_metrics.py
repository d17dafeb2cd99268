"""Fit-quality KATs against the CPU oracle and the CUDA product:
proj/tests/unit/test_metrics.cpp (kl / jsd / bic / moment errors / compression ratio /
report round trips) and test_wgmm.cpp:528-556 (evaluate_pdf)."""
import json
import math

import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200 import _metrics as Mx
from paper_2504_14897_b200.types import (AffineMap, AxisRange, GaussianComponent, GmmModel,
                                         GridSpec, InvalidArgument, WeightedPoints)

LN2 = 0.6931471805599453


@pytest.fixture(params=["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def impl(request):
    if request.param == "oracle":
        return O
    import paper_2504_14897_b200 as G
    return G


def grid_from(vals, n, x=(0, 1), y=(0, 1)):  # test_metrics.cpp:18-24 (row k/n, col k%n)
    m = np.zeros((n, n))
    for k, v in enumerate(vals):
        m[k // n, k % n] = v
    return Mx.PdfGrid.normalized(GridSpec(n, AxisRange(*x), AxisRange(*y)), m)


def random_grid(n, seed, with_zeros=False):  # :26-37 (any positive values)
    m = np.random.default_rng(seed).uniform(0.05, 2.0, size=(n, n))
    if with_zeros:
        m[0, 0] = 0.0
        m[n - 1, n // 2] = 0.0
    return Mx.PdfGrid.normalized(GridSpec(n, AxisRange(0, 1), AxisRange(0, 1)), m)


def unit_model(mean, cov):
    d = len(mean)
    return GmmModel([GaussianComponent(1.0, np.array(mean, float), np.array(cov, float))],
                    AffineMap.identity(d), d)


def model_from(ws, mus, covs):
    return GmmModel([GaussianComponent(w, np.array(m, float), np.array(c, float))
                     for w, m, c in zip(ws, mus, covs)], AffineMap.identity(2), 2)


def test_kl_self_is_zero(impl):  # test_metrics.cpp:53-56
    p = random_grid(8, 1)
    assert impl.kl_divergence(p, p) == 0.0


def test_kl_hand_example(impl):  # :58-66
    p = grid_from([0.5, 0.5, 0.0, 0.0], 2)
    q = grid_from([0.9, 0.1, 0.0, 0.0], 2)
    expected = 0.5 * math.log(0.5 / 0.9) + 0.5 * math.log(0.5 / 0.1)
    assert impl.kl_divergence(p, q) == pytest.approx(expected, rel=1e-12)
    assert expected == pytest.approx(0.5108, rel=1e-3)


def test_kl_divergent_marker(impl):  # :68-73
    p = grid_from([0.5, 0.5, 0.0, 0.0], 2)
    q = grid_from([0.0, 0.5, 0.5, 0.0], 2)
    v = impl.kl_divergence(p, q)
    assert math.isinf(v) and v > 0


def test_kl_misaligned(impl):  # :75-79
    with pytest.raises(InvalidArgument):
        impl.kl_divergence(random_grid(4, 2), grid_from([1, 1, 1, 1], 2))


def test_kl_nonnegative(impl):  # :81-87
    for seed in range(10):
        assert impl.kl_divergence(random_grid(6, 100 + seed), random_grid(6, 200 + seed)) >= 0.0


def test_jsd_identity_symmetry_bounds(impl):  # :89-96
    p, q = random_grid(8, 3, True), random_grid(8, 4, True)
    assert impl.jsd(p, p) == 0.0
    assert impl.jsd(p, q) == pytest.approx(impl.jsd(q, p), rel=1e-12)
    assert 0.0 <= impl.jsd(p, q) <= LN2


def test_jsd_disjoint_is_ln2(impl):  # :98-102
    p = grid_from([1.0, 1.0, 0.0, 0.0], 2)
    q = grid_from([0.0, 0.0, 1.0, 1.0], 2)
    assert impl.jsd(p, q) == pytest.approx(LN2, rel=1e-12)


def test_jsd_direct_sum(impl):  # :104-122
    for seed in range(20):
        p = random_grid(5, 300 + seed, seed % 2 == 0)
        q = random_grid(5, 400 + seed, seed % 3 == 0)
        area = p.bin_area()
        direct = 0.0
        for i in range(5):
            for j in range(5):
                pn, qn = p.values[i, j] * area, q.values[i, j] * area
                mn = 0.5 * (pn + qn)
                if pn > 0:
                    direct += 0.5 * pn * math.log(pn / mn)
                if qn > 0:
                    direct += 0.5 * qn * math.log(qn / mn)
        assert impl.jsd(p, q) == pytest.approx(direct, rel=1e-12)


def test_bic_arithmetic():  # :124-134
    assert Mx.bic_parameter_count(8, 2) == 48
    assert Mx.bic_parameter_count(12, 3) == 120
    assert Mx.bic_parameter_count(1, 2) == 6
    m = unit_model([0, 0], np.eye(2))
    assert Mx.bic(0.0, m, math.e) == pytest.approx(6.0, rel=1e-12)
    ll = -123.456
    assert Mx.bic(ll, m, 50.0) == pytest.approx(-2 * ll + 6 * math.log(50.0), rel=1e-12)
    with pytest.raises(InvalidArgument):
        Mx.bic(0.0, m, 0.0)


def test_bic_increases_with_k():  # :136-145
    m1 = unit_model([0, 0], np.eye(2))
    m2 = model_from([0.5, 0.5], [[0, 0], [0, 0]], [np.eye(2), np.eye(2)])
    assert Mx.bic(-10.0, m2, 100.0) > Mx.bic(-10.0, m1, 100.0)


def test_moment_errors():  # :147-173
    mu = np.array([1.0, -2.0])
    cov = np.array([[1.5, 0.2], [0.2, 0.5]])
    m = unit_model(mu, cov)
    L = np.linalg.cholesky(cov)
    pts = np.stack([mu + math.sqrt(2) * L[:, 0], mu - math.sqrt(2) * L[:, 0],
                    mu + math.sqrt(2) * L[:, 1], mu - math.sqrt(2) * L[:, 1]])
    wp = WeightedPoints.from_(pts, np.ones(4))
    e1, e2 = Mx.moment_errors(m, wp)
    assert e1 < 1e-12 and e2 < 1e-12
    shifted = unit_model(mu + [0.1, 0.0], cov)
    s1, s2 = Mx.moment_errors(shifted, wp)
    _, dm2 = Mx.weighted_data_moments(wp)
    assert s1 == pytest.approx(0.1 / math.sqrt(np.trace(dm2)), rel=1e-6)
    assert s2 > 0.0


def test_compression_ratio():  # :175-180
    assert Mx.compression_ratio(40000, 400) == 100.0
    assert Mx.compression_ratio(10000 * 2 * 8, 12 * 8) == pytest.approx(10000 * 2 / 12, rel=1e-12)
    with pytest.raises(InvalidArgument):
        Mx.compression_ratio(100, 0)


def test_report_round_trips():  # :182-211
    r = Mx.MetricsReport(0.0123, 0.05, math.inf, -1234.5, -1200.25, 1e-12, 2e-11, 833.33, 41666.0)
    j = json.loads(json.dumps(r.to_json()))
    assert j["jsd"] == r.jsd and j["kl_qp"] is None
    back = Mx.MetricsReport.from_json(j)
    assert back.jsd == r.jsd and back.bic == r.bic and math.isinf(back.kl_qp)
    assert "inf" in r.csv_row()
    assert Mx.MetricsReport.csv_header().startswith("jsd")


def test_evaluate_pdf_peak(impl):  # test_wgmm.cpp:528-533
    m = unit_model([0, 0], np.eye(2))
    v = impl.evaluate_pdf(m, GridSpec(3, AxisRange(-0.05, 0.05), AxisRange(-0.05, 0.05)))
    assert v[1, 1] == pytest.approx(1 / (2 * math.pi), rel=1e-6)


def test_evaluate_pdf_integrates_to_one(impl):  # :535-541
    m = model_from([0.6, 0.4], [[-1.0, 0.5], [2.0, -0.5]], [np.eye(2), [[0.5, 0.1], [0.1, 0.7]]])
    g = GridSpec(400, AxisRange(-10, 12), AxisRange(-9, 9))
    v = impl.evaluate_pdf(m, g)
    assert v.sum() * g.bin_area() == pytest.approx(1.0, rel=1e-4)


def test_evaluate_pdf_rejects(impl):  # wgmm.cpp:425-435
    with pytest.raises(InvalidArgument, match="2-dimensional"):
        impl.evaluate_pdf(unit_model([0, 0, 0], np.eye(3)), GridSpec(4, AxisRange(-1, 1), AxisRange(-1, 1)))
    with pytest.raises(InvalidArgument, match="grid"):
        impl.evaluate_pdf(unit_model([0, 0], np.eye(2)), GridSpec(4, AxisRange(1, -1), AxisRange(-1, 1)))
    bad = unit_model([0, 0], [[1.0, 2.0], [2.0, 1.0]])  # symmetric, not SPD
    with pytest.raises(RuntimeError, match="SPD"):
        impl.evaluate_pdf(bad, GridSpec(4, AxisRange(-1, 1), AxisRange(-1, 1)))


def test_evaluate_pdf_matches_oracle_with_map(impl):
    m = model_from([0.3, 0.7], [[-0.2, 0.1], [0.4, -0.3]], [[[0.05, 0.01], [0.01, 0.08]], 0.1 * np.eye(2)])
    m.normalization = AffineMap(np.array([3.0, 2.0]), np.array([0.5, -1.0]))
    g = GridSpec(64, AxisRange(-4, 5), AxisRange(-5, 3))
    np.testing.assert_allclose(impl.evaluate_pdf(m, g), O.evaluate_pdf(m, g), rtol=1e-12, atol=0)


def test_weighted_loglik_matches_oracle(impl):
    rng = np.random.default_rng(5)
    x = rng.normal(size=(3000, 3))
    w = rng.uniform(0.1, 4.0, 3000)
    wp = WeightedPoints.from_(x, w)
    m = GmmModel([GaussianComponent(0.4, np.array([0.1, 0.0, -0.2]), np.diag([1.0, 0.5, 2.0])),
                  GaussianComponent(0.6, np.array([-0.5, 0.3, 0.1]),
                                    np.array([[1.0, 0.2, 0.0], [0.2, 1.0, 0.1], [0.0, 0.1, 1.5]]))],
                 AffineMap.identity(3), 3)
    assert impl.weighted_loglik(m, wp) == pytest.approx(O.weighted_loglik(m, wp), rel=1e-12)
    # weighted_loglik == the E-step log-likelihood of the same model (wgmm.cpp:233-267)
    es = O.e_step(m, wp)
    assert O.weighted_loglik(m, wp) == pytest.approx(es.loglik, rel=1e-13)


def test_assemble_metrics_pipeline_case(impl):
    """pipeline.cpp:106-128 on a fitted cfg1-style plane: product vs oracle."""
    from paper_2504_14897_b200.types import FitConfig, ParticleSet, Plane
    rng = np.random.default_rng(11)
    vel = np.concatenate([rng.normal(size=(16000, 2)), 0.5 * rng.normal(size=(4000, 2)) + [3, 0]])
    ps = ParticleSet(vel, None, "e", np.array([0.85, 0.85]))
    rx = AxisRange(-6, 6)
    h = O.bin_particles(ps, Plane.uv, 64, rx, rx)
    pts = O.to_weighted_points(h)
    fit = O.fit(pts, FitConfig(initial_components=2, seed=11, temperature=np.array([0.85, 0.85])))
    ref = O.assemble_metrics(fit.model, h, pts, 20000, 2)
    got = impl.assemble_metrics(fit.model, h, pts, 20000, 2)
    for f in Mx.MetricsReport.FIELDS:
        a, b = getattr(got, f), getattr(ref, f)
        assert a == pytest.approx(b, rel=1e-9, abs=1e-12) or (math.isinf(a) and math.isinf(b)), f


def _cells(d, n_cells, per, seed, weighted=False):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(per // 2, per * 2, n_cells)
    sizes[1] = 0  # an empty cell -> NaN report
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offs[-1])
    v = rng.normal(size=(n, d))
    beam = rng.uniform(size=n) < 0.25
    v[beam, 0] = 0.4 * v[beam, 0] + 2.5
    w = rng.uniform(0.2, 3.0, n) if weighted else None
    return O.CellsHost(v, offs, 24 if d == 3 else 40, [-5] * d, [5] * d, w)


def test_cell_metrics_oracle_equals_assemble_metrics_2v():
    """The per-cell restatement on 2V cells is assemble_metrics (pipeline.cpp:106-128) of
    each cell's own plane histogram."""
    from paper_2504_14897_b200.types import FitConfig, ParticleSet, Plane
    cells = _cells(2, 6, 3000, 3)
    bins, res = O.compress_cells(cells, FitConfig(initial_components=3, seed=2, temperature=np.ones(2)))
    met = O.cell_metrics(cells, bins, res)
    assert all(np.isnan(getattr(met, f)[1]) for f in Mx.MetricsReport.FIELDS)
    from paper_2504_14897_b200.cells import CellResults
    for c in (0, 2, 3, 5):
        if res.status[c] != 0:
            continue
        sl = slice(cells.offsets[c], cells.offsets[c + 1])
        ps = ParticleSet(cells.velocity[sl], None, "e", np.ones(2))
        rx = AxisRange(-5, 5)
        h = O.bin_particles(ps, Plane.uv, 40, rx, rx)
        pts = O.to_weighted_points(h)
        k = res.k
        comps = [GaussianComponent(res.weights[c * k + i], res.means[(c * k + i) * 2:(c * k + i + 1) * 2],
                                   res.covariances[(c * k + i) * 4:(c * k + i + 1) * 4].reshape(2, 2))
                 for i in range(res.components[c])]
        model = GmmModel(comps, AffineMap.identity(2), 2)
        ref = O.assemble_metrics(model, h, pts, sl.stop - sl.start, 2)
        for f in Mx.MetricsReport.FIELDS:
            a, b = getattr(met, f)[c], getattr(ref, f)
            assert a == pytest.approx(b, rel=1e-12, abs=1e-15) or (math.isinf(a) and math.isinf(b)), (c, f)
