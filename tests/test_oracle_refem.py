"""Pin the oracle restatement against the reference's OWN code: refem::fit
(proj/tests/support/reference_em.cpp) compiled from /root/reference into oracle/_ref by
oracle/Makefile, and the committed golden fixtures it produced (tests/golden/). Mirrors
acceptance criterion 5 (acceptance_main.cpp:306-361): unit-weight fits agree to 1e-10
relative with identical iteration counts."""
import glob
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200.types import (AffineMap, AxisRange, FitConfig, GaussianComponent,
                                         GmmModel, ModelMeta, Plane, WeightedPoints)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0))


def check_against(res, alpha, means, covs, trace, iterations, tol=1e-10):
    assert res.iterations_used == int(iterations)
    assert res.model.size() == len(alpha)
    for i, c in enumerate(res.model.components):
        assert _rel(c.weight, alpha[i]) <= tol
        assert _rel(c.mean, means[i]) <= tol
        assert _rel(c.covariance, covs[i]) <= tol
    assert _rel(res.loglik_trace, trace) <= tol


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "refem_*.npz"))))
def test_oracle_matches_refem_golden(path):
    g = np.load(path)
    wp = WeightedPoints.from_(np.stack([g["xs"], g["ys"]], 1), np.ones(len(g["xs"])))
    r = O.fit(wp, FitConfig(initial_components=int(g["m"]), seed=int(g["seed"]), temperature=np.ones(2)))
    check_against(r, g["alpha"], g["means"], g["covs"], g["trace"], g["iterations"])


@pytest.mark.skipif(not O.refem_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(20))
def test_oracle_matches_refem_live(seed):
    rng = np.random.default_rng(5000 + seed)
    n = 1500
    left = rng.integers(0, 2, n) == 0
    xs = rng.normal(size=n) * 0.8 + np.where(left, -2.5, 2.5)
    ys = rng.normal(size=n) * 1.1
    ref = O.refem_fit(xs, ys, m=3, seed=50 + seed)
    r = O.fit(WeightedPoints.from_(np.stack([xs, ys], 1), np.ones(n)),
              FitConfig(initial_components=3, seed=50 + seed, temperature=np.ones(2)))
    check_against(r, ref["alpha"], ref["means"], ref["covs"], ref["trace"], ref["iterations"])


def test_formats_hex_vector():  # FORMATS.md:35-47
    g = json.load(open(os.path.join(GOLD, "formats_hex.json")))
    m = GmmModel([GaussianComponent(1.0, np.array(g["model"]["mean"]), np.array(g["model"]["cov"]))],
                 AffineMap.identity(2), 2)
    b = O.encode_model(m, ModelMeta("e", Plane.uv, 50, [AxisRange(-5, 5)] * 2))
    assert b.hex() == g["hex"] and len(b) == 107
    assert b[55:59].hex() == "525af6d7"  # header CRC-32 d7f65a52, little-endian


def test_payload_and_header_sizes():  # test_codec.cpp:62-78, acceptance criterion 9
    assert O.model_payload_bytes(2, 2) == 96 and O.model_payload_bytes(8, 3) == 640
    rng = np.random.default_rng(0)
    for d, m, label in [(2, 2, "electrons"), (3, 8, "electrons"), (3, 1, "")]:
        comps = []
        w = rng.uniform(0.1, 1.0, m)
        w /= w.sum()
        w[-1] = 1.0 - w[:-1].sum()
        for i in range(m):
            a = rng.normal(size=(d, d))
            comps.append(GaussianComponent(w[i], rng.normal(size=d), a @ a.T + 0.1 * np.eye(d)))
        b = O.encode_model(GmmModel(comps, AffineMap.identity(d), d),
                           ModelMeta(label, Plane.uv if d == 2 else None, 0, [AxisRange(-5, 5)] * d))
        assert len(b) == 4 + 4 + 4 + 8 + 16 * d + 2 + len(label) + 4 + O.model_payload_bytes(m, d)
