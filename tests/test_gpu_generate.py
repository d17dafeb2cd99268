"""Device copy of the reference generator: vdfcg_generate against the
oracle's restatement of synthdata.cpp:54-86 on the same mt19937_64(seed) stream.

The stream positions and component choices are exact (one uniform per particle, then
Box-Muller pairs whose spare crosses particle boundaries when d is odd), so every value
agrees to a few ulp; only CUDA's log/sin/cos rounding differs from the host libm.
Tolerance: |gpu - oracle| <= 1e-13 * (1 + |oracle|).
"""
import numpy as np
import pytest

import oracle as O
import paper_2504_14897_b200 as G
from paper_2504_14897_b200.types import InvalidArgument

pytestmark = pytest.mark.gpu

TOL = 1e-13


def _check(fr, mu, cv, n, seed):
    g = G.generate(fr, mu, cv, n, seed)
    o = O.generate(fr, mu, cv, n, seed)
    assert g.velocities.shape == o.velocities.shape
    err = np.abs(g.velocities - o.velocities) / (1.0 + np.abs(o.velocities))
    assert err.max() <= TOL, err.max()
    np.testing.assert_array_equal(g.nominal_temperature, o.nominal_temperature)
    # most values are bit-identical; a wrong stream offset would make none of them so
    assert np.mean(g.velocities == o.velocities) > 0.25
    return g


def test_generate_jump_ahead_chunk_boundaries():
    """Streams of >= 2^20 raw words run one CTA per 2^18-word chunk from GF(2) jump-ahead
    windows (mtjump.cu): particles whose uniforms straddle chunk boundaries must still match
    the sequential stream (2V: 3 raw words per particle, boundaries at 1 + c 2^18)."""
    g = _check([0.5, 0.5], [[0, 0], [1, -1]], [np.eye(2), np.array([[0.5, 0.2], [0.2, 0.3]])],
               600_000, 123)
    assert g.velocities.shape == (600_000, 2)


def test_generate_cfg1_2v():
    _check([0.8, 0.2], [[0, 0], [3, 0]], [np.eye(2), 0.25 * np.eye(2)], 1_000_000, 11)


@pytest.mark.parametrize("n", [1, 2, 3, 311, 312, 313, 100_001, 3_000_001])
def test_generate_3v_full_covariance_odd_spares(n):
    # d = 3: the third normal of an even particle opens a pair whose spare is the first
    # normal of the next particle; n around the 312-word twist block and odd n.
    cov = np.array([[1.0, 0.3, 0.1], [0.3, 0.8, -0.2], [0.1, -0.2, 0.5]])
    _check([0.4, 0.3, 0.2, 0.1], [[0, 0, 0], [2.5, 0, 0], [-1.5, 1.5, 0], [0, -2, 1.5]],
           [cov, 0.5 * np.eye(3), 0.25 * cov, np.eye(3)], n, 7)


def test_generate_device_output_and_single_component():
    import torch
    n = 4096
    out = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    G.generate([1.0], [[0.5, -0.25]], [[[1.0, 0.2], [0.2, 0.8]]], n, 5, out=out)
    o = O.generate([1.0], [[0.5, -0.25]], [[[1.0, 0.2], [0.2, 0.8]]], n, 5)
    got = out.cpu().numpy().reshape(2, n).T
    assert (np.abs(got - o.velocities) / (1.0 + np.abs(o.velocities))).max() <= TOL
    # an (n, d) column-major view is accepted; the returned set is a usable n x d ParticleSet
    col = torch.empty(2, n, dtype=torch.float64, device="cuda").t()
    ps = G.generate([1.0], [[0.5, -0.25]], [[[1.0, 0.2], [0.2, 0.8]]], n, 5, out=col)
    assert ps.count() == n and ps.dimension() == 2
    assert torch.equal(col.cpu(), torch.from_numpy(got.copy()))
    # row-major (n, d) would be scrambled by the column-major kernel: rejected
    with pytest.raises(InvalidArgument, match="column-major"):
        G.generate([1.0], [[0.5, -0.25]], [[[1.0, 0.2], [0.2, 0.8]]], n, 5,
                   out=torch.empty(n, 2, dtype=torch.float64, device="cuda"))


def test_generate_validation_messages():  # synthdata.cpp:32-52
    with pytest.raises(InvalidArgument, match="fractions must sum to 1"):
        G.generate([0.5, 0.4], [[0, 0], [1, 1]], [np.eye(2), np.eye(2)], 10, 1)
    with pytest.raises(InvalidArgument, match="component 1: covariance is not symmetric positive"):
        G.generate([0.5, 0.5], [[0, 0], [1, 1]], [np.eye(2), -np.eye(2)], 10, 1)
    with pytest.raises(InvalidArgument, match="component 0: covariance is not symmetric"):
        G.generate([1.0], [[0, 0]], [[[1.0, 0.5], [0.0, 1.0]]], 10, 1)
    with pytest.raises(InvalidArgument, match="component 0: fraction must be >= 0"):
        G.generate([-0.5, 1.5], [[0, 0], [1, 1]], [np.eye(2), np.eye(2)], 10, 1)
    with pytest.raises(InvalidArgument, match="particle_count must be >= 1"):
        G.generate([1.0], [[0, 0]], [np.eye(2)], 0, 1)
