"""Reference acceptance criteria 3 and 9 (proj/tests/acceptance/acceptance_main.cpp:197-243,
449-504) against the CPU oracle and the CUDA product. Criteria 1, 2, 4, 5, 6, 10, 11 are in
test_kat_wgmm.py / test_oracle_refem.py; 7 and 8 in test_kat_metrics.py."""
import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200 import codec
from paper_2504_14897_b200.types import (AffineMap, AxisRange, FitConfig, GaussianComponent,
                                         GmmModel, ModelMeta, Plane)


@pytest.fixture(params=["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def impl(request):
    if request.param == "oracle":
        return O
    import paper_2504_14897_b200 as G
    return G


def test_criterion_3_two_gaussian_recovery(impl):
    """The reference documents the M-hat / mean / JSD < 0.02 targets as unreachable at
    N=1e5 (expected FAIL, acceptance_main.cpp:192-196) and requires moment conservation and a
    valid fit; here the JSD and the fit are also checked against the oracle."""
    p = O.generate([0.5, 0.5], [[-2.0, 0.0], [2.0, 0.0]], [np.eye(2), np.eye(2)], 100000, 31)
    h = impl.bin_particles(p, Plane.uv, 200, AxisRange(-5, 5), AxisRange(-5, 5))
    pts = impl.to_weighted_points(h)
    cfg = FitConfig(initial_components=12, prune_threshold=0.005, seed=31, temperature=np.ones(2))
    r = impl.fit(pts, cfg)
    ro = O.fit(O.to_weighted_points(O.bin_particles(p, Plane.uv, 200, AxisRange(-5, 5), AxisRange(-5, 5))), cfg)
    assert r.iterations_used == ro.iterations_used and r.model.size() == ro.model.size()
    mm, m2 = O.mixture_moments(r.model)
    dm, d2 = O.weighted_data_moments(pts)
    assert np.linalg.norm(mm - dm) <= 1e-9 * np.sqrt(np.trace(d2))
    assert np.linalg.norm(m2 - d2) <= 1e-9 * np.linalg.norm(d2)
    j = impl.jsd(impl.to_pdf(h), impl.PdfGrid.normalized(h.grid(), impl.evaluate_pdf(r.model, h.grid())))
    jo = O.jsd(O.to_pdf(h), O.PdfGrid.normalized(h.grid(), O.evaluate_pdf(ro.model, h.grid())))
    assert 0.0 <= j < 0.1 and j == pytest.approx(jo, rel=1e-8)


def test_criterion_9_codec_round_trip(impl):
    """1000 random models (d in {2,3}, 1..12 components): encode on the device (or oracle),
    decode with the FORMATS.md reader -> bit-identical parameters, exact size formula."""
    rng = np.random.default_rng(123)
    for rnd in range(1000 if impl is O else 300):
        d = 2 if rng.integers(2) else 3
        m = 1 + int(rng.integers(12))
        w = rng.uniform(0.05, 1.0, m)
        w /= w.sum()
        w[-1] = 1.0 - w[:-1].sum()
        comps = []
        for i in range(m):
            a = rng.normal(size=(d, d))
            c = a @ a.T + 0.05 * np.eye(d)
            c = np.triu(c) + np.triu(c, 1).T  # exactly symmetric (set_covariance)
            comps.append(GaussianComponent(float(w[i]), 4.0 * rng.normal(size=d), c))
        model = GmmModel(comps, AffineMap.identity(d), d)
        if not all(c.weight > 0 for c in comps) or abs(sum(c.weight for c in comps) - 1.0) > 1e-12:
            continue
        meta = ModelMeta("acceptance", Plane.uv if d == 2 else None, rnd, [AxisRange(-5, 5)] * d)
        b = impl.encode_model(model, meta)
        assert len(b) == 4 + 4 + 4 + 8 + 16 * d + 2 + len("acceptance") + 4 + impl.model_payload_bytes(m, d)
        back = codec.decode_model(b)
        assert back.model.size() == m and back.meta.cycle == rnd
        for x, y in zip(back.model.components, comps):
            assert x.weight == y.weight and np.array_equal(x.mean, y.mean)
            assert np.array_equal(np.triu(x.covariance), np.triu(y.covariance))
