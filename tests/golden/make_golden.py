"""Generate the golden fixtures from the REFERENCE's own code (run in the container
where /root/reference exists; the GPU box only reads the committed files):

* refem_*.npz — inputs and outputs of refem::fit (proj/tests/support/reference_em.cpp,
  compiled from /root/reference into oracle/_ref/librefem.so by oracle/Makefile), the
  reference's independent unit-weight d=2 EM, on the acceptance-criterion-5 protocol
  (acceptance_main.cpp:306-361): two blobs at +-2.5, 1500 points, M=3, seed 50+s,
  temperature (1,1).
* formats_hex.json — the FORMATS.md:35-47 .gmmc example (107 bytes, CRC d7f65a52).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def main():
    assert O.refem_available(), "build oracle/_ref first (make -C oracle)"
    for s in range(6):
        rng = np.random.default_rng(900 + s)
        n = 1500
        left = rng.integers(0, 2, n) == 0
        xs = rng.normal(size=n) * 0.8 + np.where(left, -2.5, 2.5)
        ys = rng.normal(size=n) * 1.1
        r = O.refem_fit(xs, ys, m=3, seed=50 + s)
        np.savez(os.path.join(HERE, f"refem_{s}.npz"), xs=xs, ys=ys, seed=50 + s, m=3,
                 alpha=r["alpha"], means=r["means"], covs=r["covs"], trace=r["trace"],
                 iterations=r["iterations"], converged=r["converged"])
    hexv = ("474d4d430102000001000000320000000000000000000000000014c0000000000000144000000000000014c0"
            "0000000000001440010065525af6d7000000000000f03f000000000000e03f000000000000d0bf00000000"
            "0000f03f000000000000c03f0000000000000040")
    with open(os.path.join(HERE, "formats_hex.json"), "w") as f:
        json.dump({"source": "proj/FORMATS.md:35-47", "hex": hexv, "bytes": 107,
                   "crc": "d7f65a52", "model": {"weight": 1.0, "mean": [0.5, -0.25],
                                               "cov": [[1.0, 0.125], [0.125, 2.0]]},
                   "meta": {"label": "e", "plane": 0, "cycle": 50, "range": [-5.0, 5.0]}}, f,
                  indent=1)


if __name__ == "__main__":
    main()
