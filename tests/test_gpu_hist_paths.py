"""Every histogram kernel (TMA bitmap, bitmap, radix sort, dense), forced through
VDFCG_HIST_PATH in a subprocess, is bit-exact against the oracle on the same cells — the
automatic path choice is a performance decision only."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "scripts"))


@pytest.mark.parametrize("path", ["auto", "tma", "bitmap", "sort", "dense"])
def test_forced_histogram_path_bit_exact(path, tmp_path):
    from hist_path_case import case
    out = str(tmp_path / f"{path}.npz")
    env = dict(os.environ)
    if path != "auto":
        env["VDFCG_HIST_PATH"] = path
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "scripts", "hist_path_case.py"), out, ROOT],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    g = np.load(out)
    v, offs = case()
    for nb in (16, 32, 48):
        ob = O.bin_cells(O.CellsHost(v, offs, nb, [-5] * 3, [5] * 3))
        assert np.array_equal(g[f"nnz{nb}"], ob.nnz), nb
        assert np.array_equal(g[f"oor{nb}"], ob.out_of_range), nb
        for c in range(len(offs) - 1):
            b, k = offs[c], ob.nnz[c]
            assert np.array_equal(g[f"keys{nb}"][b:b + k], ob.keys[b:b + k]), (nb, c)
            assert np.array_equal(g[f"counts{nb}"][b:b + k], ob.counts[b:b + k]), (nb, c)
