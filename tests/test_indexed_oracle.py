"""CPU checks of the cell-index oracle (test infrastructure for tests/test_gpu_indexed.py):
its stable group-by-cell equals numpy's stable argsort, and a cell's fractional-weight bins
equal the reference's sequential `counts += w` in input order (histogram.cpp:66-74)."""
import numpy as np
import pytest

import oracle as O


def test_indexed_oracle_equals_stable_grouping():
    rng = np.random.default_rng(1)
    n, nc, nb = 50_000, 37, 16
    cell = rng.integers(0, nc, size=n).astype(np.int32)
    v = rng.normal(size=(n, 3)) * 1.5
    w = rng.uniform(0.1, 4.0, size=n)
    lo, hi = [-5.0] * 3, [5.0] * 3
    offs, ib = O.bin_cells_indexed(O.ParticlesHost(v, cell, nc, nb, lo, hi, w))
    order = np.argsort(cell, kind="stable")
    ref_offs = np.zeros(nc + 1, np.int64)
    np.cumsum(np.bincount(cell, minlength=nc), out=ref_offs[1:])
    assert np.array_equal(offs, ref_offs)
    gb = O.bin_cells(O.CellsHost(v[order], ref_offs, nb, lo, hi, w[order]))
    for f in ("nnz", "keys", "counts", "out_of_range", "in_range"):
        assert np.array_equal(getattr(ib, f), getattr(gb, f)), f
    # cell 5, sequential sums in input order
    c = 5
    sel = np.nonzero(cell == c)[0]
    idx = np.floor((v[sel] + 5.0) * (nb / 10.0)).astype(int)
    inr = np.all((v[sel] >= -5.0) & (v[sel] <= 5.0), axis=1)
    idx = np.minimum(idx, nb - 1)
    sums = {}
    for p, ok, (i, j, k) in zip(sel, inr, idx):
        if ok:
            key = (i * nb + j) * nb + k
            sums[key] = sums.get(key, 0.0) + w[p]
    keys = sorted(sums)
    b = offs[c]
    assert list(ib.keys[b:b + ib.nnz[c]]) == keys
    assert np.array_equal(ib.counts[b:b + ib.nnz[c]], np.array([sums[k] for k in keys]))


def test_indexed_oracle_rejects_bad_cell():
    v = np.zeros((4, 3))
    with pytest.raises(ValueError, match="cell index out of range"):
        O.bin_cells_indexed(O.ParticlesHost(v, np.array([0, 1, 2, 3], np.int32), 3, 8, [-1] * 3, [1] * 3))
