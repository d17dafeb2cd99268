"""Reference KATs (run against the CPU oracle and the CUDA product) for histogram.cpp pinned by the reference's own KATs
(proj/tests/unit/test_histogram.cpp:39-174, test_codec.cpp:186-200)."""
import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200.types import (AxisRange, Histogram2D, InvalidArgument, ParticleSet,
                                         Plane)

@pytest.fixture(params=["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def impl(request):
    """The same reference KAT against the CPU oracle and against the CUDA product."""
    if request.param == "oracle":
        return O
    import paper_2504_14897_b200 as G
    return G



def p2(v, w=None):
    return ParticleSet(np.asarray(v, dtype=float), None if w is None else np.asarray(w, dtype=float),
                       "", np.ones(2))


def test_one_particle_per_bin_2x2(impl):  # test_histogram.cpp:39-45
    v = [[-0.5, -0.5], [-0.5, 0.5], [0.5, -0.5], [0.5, 0.5]]
    h = impl.bin_particles(p2(v), Plane.uv, 2, AxisRange(-1, 1), AxisRange(-1, 1))
    assert np.array_equal(h.counts, np.ones((2, 2)))
    assert h.out_of_range_count == 0.0


def test_tail_mass_small(impl):  # :47-52
    p = O.gaussian_2d(10000, 11)
    h = impl.bin_particles(p, Plane.uv, 200, AxisRange(-5, 5), AxisRange(-5, 5))
    assert h.out_of_range_count / 10000 < 1e-3
    assert abs(h.in_range_count() + h.out_of_range_count - 10000) <= 1e-9 * 10000


def test_interior_edge_higher_bin_top_edge_closed(impl):  # :54-66
    h = impl.bin_particles(p2([[0.0, 0.0]]), Plane.uv, 2, AxisRange(-1, 1), AxisRange(-1, 1))
    assert h.counts[1, 1] == 1.0 and h.in_range_count() == 1.0
    h2 = impl.bin_particles(p2([[1.0, 1.0]]), Plane.uv, 2, AxisRange(-1, 1), AxisRange(-1, 1))
    assert h2.counts[1, 1] == 1.0 and h2.out_of_range_count == 0.0


def test_w_plane_rejected_for_2d(impl):  # :68-72
    p = O.gaussian_2d(10, 1)
    for pl in (Plane.vw, Plane.uw):
        with pytest.raises(InvalidArgument):
            impl.bin_particles(p, pl, 4, AxisRange(-1, 1), AxisRange(-1, 1))


def test_weighted_mass_conservation_and_permutation(impl):  # :74-104
    rng = np.random.default_rng(99)
    v = rng.uniform(-3, 3, size=(5000, 2))
    w = rng.uniform(0.1, 4.0, size=5000)
    h = impl.bin_particles(p2(v, w), Plane.uv, 50, AxisRange(-1, 1), AxisRange(-1, 1))
    assert abs(h.in_range_count() + h.out_of_range_count - w.sum()) <= 1e-9 * w.sum()
    assert h.out_of_range_count > 0
    perm = rng.permutation(5000)
    h2 = impl.bin_particles(p2(v[perm], w[perm]), Plane.uv, 50, AxisRange(-1, 1), AxisRange(-1, 1))
    assert np.linalg.norm(h.counts - h2.counts) <= 1e-12 * np.linalg.norm(h.counts)


def test_all_planes_d2_rejected_and_empty_degenerate(impl):  # :119-134
    with pytest.raises(InvalidArgument, match="bin_particles"):
        impl.all_planes(O.gaussian_2d(10, 1), 4, AxisRange(-1, 1))
    p = ParticleSet(np.zeros((0, 3)), None, "", np.ones(3))
    for h in impl.all_planes(p, 4, AxisRange(-1, 1)):
        assert h.degenerate() and not h.counts.any()


def test_all_planes_maxwellian_marginals_mass(impl):  # :106-117
    p = O.preset("maxwellian", 1000000, 5)
    hs = impl.all_planes(p, 200, AxisRange(-5, 5))
    for h in hs:
        assert abs(h.in_range_count() + h.out_of_range_count - 1e6) <= 1e-9 * 1e6
    a, b, c = (impl.to_pdf(h) for h in hs)
    assert impl.jsd(a, b) < 0.01 and impl.jsd(b, c) < 0.01 and impl.jsd(a, c) < 0.01


def test_to_weighted_points_order_centres_total(impl):  # :136-156
    h = Histogram2D(np.zeros((2, 2), order="F"), AxisRange(0, 2), AxisRange(0, 2), Plane.uv, 2)
    h.counts[0, 0] = 3
    h.counts[1, 1] = 1
    wp = impl.to_weighted_points(h, True)
    assert wp.count() == 2 and list(wp.weights) == [3.0, 1.0]
    assert list(wp.points[0]) == [0.5, 0.5] and wp.total_weight == 4.0
    assert impl.to_weighted_points(h, False).count() == 4


def test_to_weighted_points_200_grid(impl):  # :158-164
    h = impl.bin_particles(O.gaussian_2d(100000, 2), Plane.uv, 200, AxisRange(-5, 5), AxisRange(-5, 5))
    assert impl.to_weighted_points(h, True).count() <= 40000
    assert impl.to_weighted_points(h, False).count() == 40000


def test_zero_histogram_rejected(impl):  # :166-174
    h = Histogram2D(np.zeros((2, 2)), AxisRange(0, 1), AxisRange(0, 1), Plane.uv, 2)
    with pytest.raises(InvalidArgument, match="degenerate histogram"):
        impl.to_weighted_points(h, True)


def test_cells_reduce_to_bin_particles(impl):
    """App. A: a 2V cell batch equals bin_particles + to_weighted_points per cell."""
    rng = np.random.default_rng(3)
    v = rng.normal(size=(3000, 2))
    offs = np.array([0, 1000, 1000, 3000], dtype=np.int64)
    b = O.bin_cells(O.CellsHost(v, offs, 16, [-3, -3], [3, 3]))
    for c in range(3):
        seg = v[offs[c]:offs[c + 1]]
        h = impl.bin_particles(p2(seg), Plane.uv, 16, AxisRange(-3, 3), AxisRange(-3, 3))
        k = b.nnz[c]
        if h.degenerate():
            assert k == 0
            continue
        wp = impl.to_weighted_points(h)
        assert k == wp.count()
        keys = b.keys[offs[c]:offs[c] + k]
        i, j = keys // 16, keys % 16
        assert np.array_equal(np.stack([-3 + (i + 0.5) * 6 / 16, -3 + (j + 0.5) * 6 / 16], 1), wp.points)
        assert np.array_equal(b.counts[offs[c]:offs[c] + k], wp.weights)
        assert b.out_of_range[c] == h.out_of_range_count


def test_histogram_payload_size(impl):  # test_codec.cpp:186-200: 200^2 f64 = 320000 B
    h = impl.bin_particles(O.preset("maxwellian", 20000, 3), Plane.uv, 200, AxisRange(-5, 5),
                        AxisRange(-5, 5))
    assert h.counts.astype(np.float64).nbytes == 320000
