"""Reference KATs (run against the CPU oracle and the CUDA product) for wgmm.cpp pinned by the reference's KATs
(proj/tests/unit/test_wgmm.cpp, acceptance criteria 1, 2, 4, 10, 11)."""
import copy

import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200.types import (AffineMap, AxisRange, CovarianceRepairError, FitConfig,
                                         GaussianComponent, GmmModel, InvalidArgument, Plane,
                                         WeightedPoints)

@pytest.fixture(params=["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def impl(request):
    """The same reference KAT against the CPU oracle and against the CUDA product."""
    if request.param == "oracle":
        return O
    import paper_2504_14897_b200 as G
    return G



def pts(rows):
    return WeightedPoints.from_(np.array([r[0] for r in rows], float), np.array([r[1] for r in rows], float))


def cloud(n, seed, unit=False):
    rng = np.random.default_rng(seed)
    x = np.stack([2.0 * rng.normal(size=n) + 1.0, 0.5 * rng.normal(size=n) - 3.0], 1)
    w = np.ones(n) if unit else rng.uniform(0.2, 5.0, size=n)
    return WeightedPoints.from_(x, w)


def model(ws, mus, covs):
    d = len(mus[0])
    return GmmModel([GaussianComponent(w, np.array(m, float), np.array(c, float))
                     for w, m, c in zip(ws, mus, covs)], AffineMap.identity(d), d)


def test_normalize_bbox(impl):  # test_wgmm.cpp:73-85
    p = pts([([0.0, -2.0], 1.0), ([10.0, 2.0], 2.0), ([5.0, 0.0], 3.0)])
    n, m = impl.normalize(p)
    assert list(m.offset) == [5.0, 0.0] and list(m.scale) == [5.0, 2.0]
    assert n.points[:, 0].min() == -1.0 and n.points[:, 0].max() == 1.0


def test_normalize_identity_and_zero_spread(impl):  # :87-97
    n, m = impl.normalize(pts([([-1.0, -1.0], 1.0), ([1.0, 1.0], 1.0)]))
    assert m.is_identity()
    with pytest.raises(InvalidArgument, match="axis 0"):
        impl.normalize(pts([([3.0, -1.0], 1.0), ([3.0, 1.0], 1.0)]))


def test_denormalize(impl):  # :99-124
    m = model([1.0], [[0.0, 0.0]], [np.eye(2)])
    m.normalization = AffineMap(np.array([5.0, 2.0]), np.array([1.0, -1.0]))
    d = impl.denormalize_model(m)
    c = d.components[0]
    assert c.covariance[0, 0] == 25.0 and c.covariance[1, 1] == 4.0 and c.covariance[0, 1] == 0.0
    assert list(c.mean) == [1.0, -1.0]


def test_init_uniform_weights_seeded(impl):  # :126-148
    n, m = impl.normalize(cloud(500, 4))
    cfg = FitConfig(initial_components=12, seed=77)
    a = impl.init_model(n, cfg, np.ones(2), m)
    assert a.size() == 12 and all(abs(c.weight - 1 / 12) <= 1e-15 for c in a.components)
    b = impl.init_model(n, cfg, np.ones(2), m)
    assert all(np.array_equal(x.mean, y.mean) for x, y in zip(a.components, b.components))
    c = impl.init_model(n, FitConfig(initial_components=12, seed=78), np.ones(2), m)
    assert not np.array_equal(a.components[0].mean, c.components[0].mean)
    assert abs(a.components[0].covariance[0, 0] - 1 / m.scale[0] ** 2) <= 1e-14 / m.scale[0] ** 2


def test_init_uniforms_are_mt19937_64():
    """rng.hpp:22: uniforms = top 53 bits of std::mt19937_64 (C++ standard algorithm);
    10000th raw output of mt19937_64(5489) is 9981545732273789042 (the standard's check)."""
    u = O.uniforms(5489, 10000)
    assert u[-1] == (9981545732273789042 >> 11) * 2.0 ** -53


def test_warm_start_pass_through(impl):  # :150-165
    n, m = impl.normalize(cloud(500, 4))
    warm = model([1.0], [[1.0, -3.0]], [[[4.0, 0.5], [0.5, 0.25]]])
    init = impl.init_model(n, FitConfig(warm_start=warm), np.ones(2), m)
    back = impl.denormalize_model(init)
    assert np.allclose(back.components[0].mean, [1.0, -3.0], rtol=1e-12)
    assert np.allclose(back.components[0].covariance, [[4.0, 0.5], [0.5, 0.25]], rtol=1e-12)


def test_init_shrinks_to_distinct(impl):  # :167-177
    x = np.array([[0, 0], [1, 0], [0, 1], [0, 0], [1, 0], [0, 1]], float)
    n, m = impl.normalize(WeightedPoints.from_(x, np.ones(6)))
    mm = impl.init_model(n, FitConfig(initial_components=5, prune_threshold=0.01), np.ones(2), m)
    assert mm.size() == 3


def test_e_step_kats(impl):  # :188-231
    m = model([1.0], [[0.0, 0.0]], [np.eye(2)])
    es = impl.e_step(m, pts([([0.5, 0.5], 2.0), ([-4.0, 1.0], 1.0)]))
    assert np.array_equal(es.responsibilities, np.ones((1, 2)))
    m2 = model([0.5, 0.5], [[0, 0], [0, 0]], [np.eye(2), np.eye(2)])
    es = impl.e_step(m2, pts([([1.0, 2.0], 1.0), ([-3.0, 0.5], 4.0)]))
    assert np.allclose(es.responsibilities, 0.5, rtol=1e-14)
    m3 = model([0.6, 0.4], [[-1, 0], [1, 0]], [0.01 * np.eye(2), 0.01 * np.eye(2)])
    far = 4.0
    es = impl.e_step(m3, pts([([1.0 + far, 0.0], 1.0), ([-1.0, 0.0], 1.0)]))
    assert np.all(np.isfinite(es.responsibilities)) and np.isfinite(es.loglik)
    import mpmath as mp  # high-precision oracle for the far point (long double in the reference)
    d0 = mp.e ** (-0.5 * (1 + far + 1) ** 2 / 0.01) * 0.6
    d1 = mp.e ** (-0.5 * (far) ** 2 / 0.01) * 0.4
    assert abs(es.responsibilities[1, 0] - float(d1 / (d0 + d1))) <= 1e-9


def test_m_step_single_component_closed_form(impl):  # :233-244
    p = cloud(400, 21)
    nxt = impl.m_step(p, np.ones((1, 400)), model([1.0], [[0, 0]], [np.eye(2)]))
    mean, m2 = O.weighted_data_moments(p)
    c = nxt.components[0]
    assert abs(c.weight - 1.0) <= 1e-14
    assert np.allclose(c.mean, mean, rtol=1e-12)
    assert np.allclose(c.covariance, m2 - np.outer(mean, mean), rtol=1e-9)


def test_m_step_constant_weights_and_duplicates(impl):  # :246-293
    p = cloud(300, 22, unit=True)
    sc = WeightedPoints(p.points, p.weights * 3.7, p.total_weight * 3.7)
    prev = model([0.5, 0.5], [[0, -3], [2, -3]], [np.eye(2), np.eye(2)])
    m1, m2 = copy.deepcopy(prev), copy.deepcopy(prev)
    e1, e2 = impl.e_step(m1, p), impl.e_step(m2, sc)
    assert np.allclose(e1.responsibilities, e2.responsibilities, rtol=1e-13)
    u1, u2 = impl.m_step(p, e1.responsibilities, m1), impl.m_step(sc, e2.responsibilities, m2)
    for a, b in zip(u1.components, u2.components):
        assert abs(a.weight - b.weight) <= 1e-12 and np.allclose(a.mean, b.mean, rtol=1e-12)


def test_prune_kats(impl):  # :295-336
    m = model([0.5, 0.497, 0.003], [[0, 0], [1, 1], [2, 2]], [np.eye(2)] * 3)
    pr = impl.prune(m, 0.005)
    assert pr.size() == 2 and abs(pr.components[0].weight - 0.5 / 0.997) <= 1e-15
    m = model([0.002, 0.003, 0.995], [[0, 0], [1, 1], [2, 2]], [np.eye(2)] * 3)
    once = impl.prune(m, 0.005)
    assert once.size() == 2 and abs(once.components[0].weight - 0.003 / 0.998) <= 1e-15
    single = model([1.0], [[0, 0]], [np.eye(2)])
    assert impl.prune(single, 0.5).size() == 1
    m = model([0.001, 0.001, 0.998], [[0, 0], [1, 1], [2, 2]], [np.eye(2)] * 3)
    ev = impl.prune_one(m, 0.005, 30)
    assert ev.component == 0 and ev.iteration == 30 and ev.weight == 0.001


def llt_ok(a):
    """Eigen LLT<Lower> unblocked order (the acceptance test's success criterion)."""
    d = a.shape[0]
    L = np.zeros_like(a)
    for k in range(d):
        x = a[k, k] - sum(L[k, j] * L[k, j] for j in range(k))
        if not x > 0:
            return False
        L[k, k] = np.sqrt(x)
        for i in range(k + 1, d):
            L[i, k] = (a[i, k] - sum(L[i, j] * L[k, j] for j in range(k))) / L[k, k]
    return True


def test_repair_kats(impl):  # :338-371, acceptance criterion 11
    spd = np.array([[2.0, 0.3], [0.3, 1.0]])
    assert np.array_equal(impl.repair_covariance(spd), spd)
    r = impl.repair_covariance(np.ones((2, 2)))
    assert r[0, 1] == 1.0 and np.linalg.eigvalsh(r).min() > 0 and abs(r[0, 0] - 1.0) <= 1e-7
    with pytest.raises(CovarianceRepairError):
        impl.repair_covariance(np.zeros((2, 2)))
    rng = np.random.default_rng(321)
    for rnd in range(100):
        d = 2 if rnd % 2 else 3
        if rnd % 3 == 0:
            v = rng.normal(size=d)
            s = np.outer(v, v)
        else:
            a = rng.normal(size=(d, d))
            spd = a @ a.T + 0.1 * np.eye(d)
            ev, evec = np.linalg.eigh(spd)
            ev[0] = 0.0 if rnd % 3 == 1 else -1e-14
            s = evec @ np.diag(ev) @ evec.T
            s = 0.5 * (s + s.T)
        rep = impl.repair_covariance(s)
        assert llt_ok(rep)
        sym = 0.5 * (s + s.T)
        off = ~np.eye(d, dtype=bool)
        assert np.array_equal(rep[off], sym[off])


def test_fit_moments_conserved_1e9(impl):  # :373-407
    p = O.generate([1.0], [[0.5, -0.25]], [[[1.0, 0.2], [0.2, 0.8]]], 20000, 5)
    h = impl.bin_particles(p, Plane.uv, 100, AxisRange(-5, 5), AxisRange(-5, 5))
    wp = impl.to_weighted_points(h)
    r = impl.fit(wp, FitConfig(initial_components=12, seed=3, temperature=np.ones(2)))
    mm, m2 = O.mixture_moments(r.model)
    dm, d2 = O.weighted_data_moments(wp)
    assert np.linalg.norm(mm - dm) <= 1e-9 * np.sqrt(np.trace(d2))
    assert np.linalg.norm(m2 - d2) <= 1e-9 * np.linalg.norm(d2)


def test_fit_monotone_deterministic(impl):  # :409-442
    p = cloud(2000, 31)
    r = impl.fit(p, FitConfig(initial_components=6, seed=9))
    prunes = {e.iteration for e in r.pruning_events}
    for t in range(1, len(r.loglik_trace)):
        if t not in prunes:
            assert r.loglik_trace[t] >= r.loglik_trace[t - 1] - 1e-8
    a = impl.fit(cloud(1500, 41), FitConfig(initial_components=5, seed=17))
    b = impl.fit(cloud(1500, 41), FitConfig(initial_components=5, seed=17))
    assert a.loglik_trace == b.loglik_trace and a.iterations_used == b.iterations_used


def test_warm_start_converges_immediately(impl):  # :444-479
    p = O.generate([0.5, 0.5], [[-3, 0], [3, 0]], [np.eye(2), np.eye(2)], 20000, 51)
    wp = impl.to_weighted_points(impl.bin_particles(p, Plane.uv, 100, AxisRange(-6, 6), AxisRange(-6, 6)))
    cold = impl.fit(wp, FitConfig(initial_components=2, seed=13, temperature=np.ones(2)))
    assert cold.converged and cold.model.size() == 2
    left = min(cold.model.components, key=lambda c: c.mean[0]).mean
    assert np.linalg.norm(left - [-3, 0]) < 0.05
    warm = impl.fit(wp, FitConfig(initial_components=2, seed=13, temperature=np.ones(2),
                               warm_start=cold.model))
    assert warm.converged and warm.iterations_used <= 2


def test_fit_degenerate_context(impl):  # :481-488
    x = np.array([[1.0, 0.0], [1.0, 1.0], [1.0, 2.0]])
    with pytest.raises(InvalidArgument, match="fit:"):
        impl.fit(WeightedPoints.from_(x, np.ones(3)), FitConfig(initial_components=2))


def test_pruning_protocol_through_fit(impl):  # acceptance criterion 4
    p = O.generate([0.997, 0.003], [[0, 0], [6, 0]], [np.eye(2), 0.25 * np.eye(2)], 50000, 13)
    wp = impl.to_weighted_points(impl.bin_particles(p, Plane.uv, 100, AxisRange(-8, 8), AxisRange(-8, 8)))
    r = impl.fit(wp, FitConfig(initial_components=2, prune_threshold=0.005, seed=2, temperature=np.ones(2)))
    assert len(r.pruning_events) == 1 and r.pruning_events[0].iteration % 10 == 0
    assert r.pruning_events[0].weight < 0.005 and r.model.size() == 1


def test_prune_disabled_keeps_all(impl):  # acceptance criterion 10 (small N)
    p = O.generate([0.5, 0.5], [[-2, 0], [2, 0]], [np.eye(2), np.eye(2)], 10000, 97)
    wp = impl.to_weighted_points(impl.bin_particles(p, Plane.uv, 200, AxisRange(-5, 5), AxisRange(-5, 5)))
    r = impl.fit(wp, FitConfig(initial_components=8, prune_threshold=1e-300, seed=9, temperature=np.ones(2)))
    assert r.model.size() == 8


def test_config_validation(impl):  # wgmm.cpp:65-76
    with pytest.raises(InvalidArgument, match="prune_threshold must be < 1/initial_components"):
        impl.validate_fit_config(FitConfig(initial_components=12, prune_threshold=0.1), 2)
    with pytest.raises(InvalidArgument, match="max_em_iterations"):
        impl.validate_fit_config(FitConfig(max_em_iterations=0), 2)
