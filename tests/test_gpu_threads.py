"""The reference API is reentrant: host threads calling the library
concurrently (one context per thread) get the same results as sequential calls."""
import threading

import numpy as np
import pytest

from paper_2504_14897_b200.types import FitConfig, WeightedPoints

pytestmark = pytest.mark.gpu


def _work(seed):
    import paper_2504_14897_b200 as G
    rng = np.random.default_rng(seed)
    x = np.concatenate([rng.normal(size=(3000, 2)), 0.4 * rng.normal(size=(1500, 2)) + [2.5, 0.0]])
    r = G.fit(WeightedPoints.from_(x, np.ones(len(x))), FitConfig(initial_components=3, seed=seed,
                                                                  temperature=np.ones(2)))
    offs = np.arange(65, dtype=np.int64) * 900
    v = rng.normal(size=(int(offs[-1]), 3))
    b = G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(3)], offs, 24, [-5] * 3, [5] * 3)
    _, res, _, _ = G.compress_cells(b, FitConfig(initial_components=2, seed=seed, temperature=np.ones(3)))
    return r.loglik_trace, res.weights.copy(), res.iterations.copy()


def test_concurrent_host_threads_match_sequential():
    seeds = list(range(6))
    seq = [_work(s) for s in seeds]
    out = [None] * len(seeds)
    errs = []

    def run(i):
        try:
            out[i] = _work(seeds[i])
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(seeds))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(seq, out):
        assert a[0] == b[0]
        assert np.array_equal(a[1].view(np.int64), b[1].view(np.int64)) and np.array_equal(a[2], b[2])
