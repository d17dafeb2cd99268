"""Bin a fixed cell batch with the histogram path forced by VDFCG_HIST_PATH and save the
compacted result (run by tests/test_gpu_hist_paths.py in a subprocess per path)."""
import sys

import numpy as np

sys.path.insert(0, sys.argv[2])
import paper_2504_14897_b200 as G  # noqa: E402


def case():
    rng = np.random.default_rng(31)
    counts = rng.integers(200, 3000, size=40)
    counts[[0, 17]] = 0
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    v = rng.normal(size=(int(offs[-1]), 3)) * 1.6
    return v, offs


if __name__ == "__main__":
    v, offs = case()
    out = {}
    for nb in (16, 32, 48):
        b = G.CellBatch([np.ascontiguousarray(v[:, a]) for a in range(3)], offs, nb, [-5] * 3, [5] * 3)
        bins = G.bin_cells(b)
        out[f"nnz{nb}"] = bins.nnz
        out[f"keys{nb}"] = bins.keys
        out[f"counts{nb}"] = bins.counts
        out[f"oor{nb}"] = bins.out_of_range
    np.savez(sys.argv[1], **out)
