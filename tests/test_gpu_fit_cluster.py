"""The single-fit path (vdfcg_fit) runs one fit on a thread-block cluster of up to 16 CTAs
that combine partial sufficient statistics through distributed shared memory. Parity with
the oracle at the reference's tolerance, and bitwise determinism."""
import numpy as np
import pytest

import oracle as O
from helpers import TOL_EM, model_close
from paper_2504_14897_b200.types import AxisRange, FitConfig, Plane, WeightedPoints

pytestmark = pytest.mark.gpu


def _plane_points():
    p = O.generate([0.5, 0.3, 0.2], [[0, 0], [2.5, 0.5], [-1.5, 1.0]],
                   [np.eye(2), 0.4 * np.eye(2), [[0.5, 0.2], [0.2, 0.3]]], 1_000_000, 5)
    h = O.bin_particles(p, Plane.uv, 200, AxisRange(-6, 6), AxisRange(-6, 6))
    return O.to_weighted_points(h)


@pytest.mark.parametrize("case", ["plane200_K12", "3v_32k_K4"])
def test_cluster_fit_matches_oracle(case):
    import paper_2504_14897_b200 as G
    if case == "plane200_K12":
        pts = _plane_points()
        cfg = FitConfig(initial_components=12, seed=3, temperature=np.ones(2))
    else:
        rng = np.random.default_rng(9)
        x = np.concatenate([rng.normal(size=(20000, 3)), 0.5 * rng.normal(size=(12768, 3)) + [2.0, 0.0, 1.0]])
        pts = WeightedPoints.from_(x, rng.uniform(0.5, 3.0, len(x)))
        cfg = FitConfig(initial_components=4, seed=2, temperature=np.ones(3))
    assert pts.count() > 4 * 1024  # more than one CTA's worth of points
    g, o = G.fit(pts, cfg), O.fit(pts, cfg)
    assert g.iterations_used == o.iterations_used and g.model.size() == o.model.size()
    assert [(e.iteration, e.component) for e in g.pruning_events] == \
           [(e.iteration, e.component) for e in o.pruning_events]
    assert model_close(g.model, o.model) <= TOL_EM
    np.testing.assert_allclose(g.loglik_trace, o.loglik_trace, rtol=TOL_EM)


def test_cluster_fit_bitwise_deterministic():
    import paper_2504_14897_b200 as G
    pts = _plane_points()
    cfg = FitConfig(initial_components=12, seed=3, temperature=np.ones(2))
    a, b = G.fit(pts, cfg), G.fit(pts, cfg)
    assert a.loglik_trace == b.loglik_trace
    for x, y in zip(a.model.components, b.model.components):
        assert x.weight == y.weight and np.array_equal(x.mean, y.mean) and np.array_equal(x.covariance, y.covariance)


def test_cluster_fit_error_path():
    """A large point set (cluster launch) with zero spread on one axis raises the
    reference's message, like the single-CTA path."""
    import paper_2504_14897_b200 as G
    from paper_2504_14897_b200.types import InvalidArgument
    rng = np.random.default_rng(1)
    x = rng.normal(size=(20000, 3))
    x[:, 1] = 0.25
    wp = WeightedPoints.from_(x, np.ones(len(x)))
    cfg = FitConfig(initial_components=4, seed=1, temperature=np.ones(3))
    with pytest.raises(InvalidArgument, match="axis 1 has zero spread"):
        G.fit(wp, cfg)
    with pytest.raises(InvalidArgument, match="axis 1 has zero spread"):
        O.fit(wp, cfg)
