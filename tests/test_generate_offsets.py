"""Host check of the closed-form stream offsets the device generator uses (synth.cu
generate_kernel) against a replay of the reference's sequential call pattern
(synthdata.cpp:77-82: one uniform(), then d normal() per particle; rng.hpp:27-37: a normal()
without a spare draws two uniforms and keeps r·sin for the next call)."""
import pytest


def replay(n, d):
    pos, spare = 0, None
    sel, normals = [], []
    for _ in range(n):
        sel.append(pos)
        pos += 1
        for _ in range(d):
            if spare is not None:
                normals.append(("sin", spare))
                spare = None
            else:
                normals.append(("cos", pos))
                spare = pos
                pos += 2
    return sel, normals, pos


def closed_form(n, d):
    sel = [r + 2 * ((r * d + 1) >> 1) for r in range(n)]
    normals = []
    for j in range(n * d):
        q = j >> 1
        normals.append(("sin" if j & 1 else "cos", (2 * q) // d + 1 + 2 * q))
    return sel, normals, n + 2 * ((n * d + 1) // 2)


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 311, 312, 313, 1000])
def test_stream_offsets_match_sequential_replay(n, d):
    assert closed_form(n, d) == replay(n, d)
