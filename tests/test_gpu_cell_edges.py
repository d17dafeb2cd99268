"""Edge cells through the batched path vs the oracle: empty cells, a single particle,
everything out of range, all particles in one bin (zero spread), fewer distinct bins than
components, and cells straddling the range edges. Statuses, component counts, iteration
counts and parameters must match (the reference's error cases)."""
import numpy as np
import pytest

import oracle as O
from helpers import TOL_EM, model_close
from paper_2504_14897_b200.types import AffineMap, FitConfig, GaussianComponent, GmmModel

pytestmark = pytest.mark.gpu


def _cells():
    rng = np.random.default_rng(8)
    parts = []
    parts.append(np.zeros((0, 3)))                                  # empty
    parts.append(np.array([[0.1, 0.2, 0.3]]))                       # one particle
    parts.append(rng.normal(size=(50, 3)) + 40.0)                   # all out of range
    parts.append(np.tile([[0.5, 0.5, 0.5]], (30, 1)))               # one bin: zero spread
    parts.append(np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [0.0, 2.0, 1.0]] * 5))  # 3 bins < K
    x = rng.normal(size=(3000, 3)) * 2.5                             # straddles the +-6 edges
    x[:20] = 6.0
    x[20:40] = -6.0
    parts.append(x)
    parts.append(rng.normal(size=(2500, 3)))                         # ordinary cell
    offs = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
    return np.concatenate(parts), offs


def test_edge_cells_match_oracle():
    import paper_2504_14897_b200 as G
    v, offs = _cells()
    cfg = FitConfig(initial_components=4, seed=6, temperature=np.ones(3))
    ob, orr = O.compress_cells(O.CellsHost(v, offs, 24, [-6] * 3, [6] * 3), cfg)
    batch = G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(3)], offs, 24, [-6] * 3, [6] * 3)
    gb, gr, _, _ = G.compress_cells(batch, cfg)
    assert np.array_equal(gb.nnz, ob.nnz) and np.array_equal(gb.out_of_range, ob.out_of_range)
    assert np.array_equal(gr.status, orr.status), (gr.status, orr.status)
    assert np.array_equal(gr.components, orr.components)
    assert np.array_equal(gr.iterations, orr.iterations)
    assert (orr.status[[0, 1, 2, 3]] != 0).all()          # the reference rejects these
    k = orr.k
    for c in np.nonzero(orr.status == 0)[0]:
        m = int(orr.components[c])
        om = GmmModel([GaussianComponent(orr.weights[c * k + i], orr.means[(c * k + i) * 3:(c * k + i + 1) * 3],
                                         orr.covariances[(c * k + i) * 9:(c * k + i + 1) * 9].reshape(3, 3))
                       for i in range(m)], AffineMap.identity(3), 3)
        assert model_close(gr.model(c), om) <= TOL_EM, c
