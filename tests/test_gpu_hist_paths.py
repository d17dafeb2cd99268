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


@pytest.mark.parametrize("n_per_cell,nb,eigen", [(1907, 48, True), (1906, 48, True), (1907, 32, True),
                                                (1907, 32, False), (1200, 32, False),
                                                (1907, 64, True), (1907, 64, False),
                                                (1907, 63, True), (1907, 63, False)])
def test_tma_path_accepts_eigen_column_bases(n_per_cell, nb, eigen):
    """An Eigen N x 3 column-major matrix with odd N has its v and w columns 8 bytes off a
    16-byte boundary (ParticleSet::velocities, synthdata.hpp:13-28). The TMA kernel carries
    the per-axis skew, so such device columns bin bit-exactly (forced TMA path). 32^3 with
    ~1.9K particles per cell runs the packed-u16-count form (three CTAs per SM), 64^3 the
    4-word prefix groups (two CTAs per SM), aligned and skewed; 63^3 (7814 bitmap words) the
    same with the swizzled bitmap padded to a multiple of 16 words."""
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from paper_2504_14897_b200 import cells as G
rng = np.random.default_rng(3)
nc = 300
n = nc * {n_per_cell} + 1            # odd N: columns 1 and 2 start 8 bytes off
v = rng.normal(size=(n, 3)) * 1.5
offs = np.arange(nc + 1, dtype=np.int64) * {n_per_cell}
flat = torch.from_numpy(np.asfortranarray(v).reshape(-1, order="F").copy()).cuda()
cols = [flat[a * n:(a + 1) * n] for a in range(3)]
if {eigen}:
    assert cols[1].data_ptr() % 16 == 8
else:
    cols = [c.clone() for c in cols]
    assert all(c.data_ptr() % 16 == 0 for c in cols)
b = G.bin_cells(G.CellBatch(cols, torch.from_numpy(offs).cuda(), {nb}, [-5] * 3, [5] * 3))
torch.cuda.synchronize()
np.savez(sys.argv[1], nnz=b.nnz.cpu().numpy(), keys=b.keys.cpu().numpy().view(np.uint32),
         counts=b.counts.cpu().numpy(), v=v, offs=offs)
"""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "o.npz")
        env = dict(os.environ, VDFCG_HIST_PATH="tma")
        r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        g = np.load(out)
        ob = O.bin_cells(O.CellsHost(g["v"], g["offs"], nb, [-5] * 3, [5] * 3))
        assert np.array_equal(g["nnz"], ob.nnz)
        offs = g["offs"]
        for c in range(len(offs) - 1):
            b, k = offs[c], ob.nnz[c]
            assert np.array_equal(g["keys"][b:b + k], ob.keys[b:b + k]), c
            assert np.array_equal(g["counts"][b:b + k], ob.counts[b:b + k]), c
