"""Host check of the closed-form stream offsets the device generator uses (synth.cu
generate_kernel) against a replay of the reference's sequential call pattern
(synthdata.cpp:77-82: one uniform(), then d normal() per particle; rng.hpp:27-37: a normal()
without a spare draws two uniforms and keeps r·sin for the next call), and of the
register-pair decomposition of the mt19937_64 twist that mt_stream_kernel runs."""
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


def _twist(upper, lower):
    xx = (upper & 0xFFFFFFFF80000000) | (lower & 0x7FFFFFFF)
    return (xx >> 1) ^ (0xB5026F5AA96619E9 if xx & 1 else 0)


def _temper(y):
    M = 0xFFFFFFFFFFFFFFFF
    y ^= (y >> 29) & 0x5555555555555555
    y ^= (y << 17) & 0x71D67FFFEDA60000 & M
    y ^= (y << 37) & 0xFFF7EEE000000000 & M
    y ^= y >> 43
    return (y >> 11) * 2.0 ** -53


def test_register_pair_twist_matches_mt19937_64():
    """synth.cu mt_stream_kernel: thread t keeps (mt[t], mt[t+156]) and needs only thread
    t+1's old pair (thread 155: mt[156] and the new mt[0]); replayed here for 3 blocks
    against std::mt19937_64 in the oracle (rng.hpp:22)."""
    import numpy as np
    import oracle as O
    seed, M = 11, 0xFFFFFFFFFFFFFFFF
    mt = [seed]
    for i in range(1, 312):
        mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & M)
    A, B = mt[:156], mt[156:]
    out = []
    for _ in range(3):
        nA, nB = [0] * 156, [0] * 156
        for t in range(156):
            if t + 1 < 156:
                A1, B1 = A[t + 1], B[t + 1]
            else:
                A1, B1 = B[0], B[0] ^ _twist(A[0], A[1])
            nA[t] = B[t] ^ _twist(A[t], A1)
            nB[t] = nA[t] ^ _twist(B[t], B1)
        A, B = nA, nB
        out += [_temper(x) for x in A + B]
    np.testing.assert_array_equal(np.array(out), O.uniforms(seed, 3 * 312))


@pytest.mark.parametrize("offset", [1, 2, 311, 312, 313, 19937, 262145, 1_000_003, 12_000_000])
def test_mt19937_64_jump_window_matches_sequential_stream(offset):
    """mtjump.cu: the 312 raw words at stream offset J >= 1 as a GF(2) correlation of the first
    19937 + 312 words with x^(J-1) mod phi (phi from Berlekamp-Massey) equal the sequential
    mt19937_64 stream — checked through the tempered top-53-bit uniforms the reference draws
    (rng.hpp:22) against the oracle's std::mt19937_64. Host-only (no device)."""
    import ctypes as C

    import numpy as np

    import oracle as O
    from paper_2504_14897_b200 import api
    lib = api.lib()
    fn = lib.vdfcg_debug_mt_window
    fn.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
    seed = 0x1234567 + offset
    raw = np.zeros(312, np.uint64)
    assert fn(seed, offset, raw.ctypes.data) == 0
    y = raw.copy()
    y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
    y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
    y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
    y ^= y >> np.uint64(43)
    got = (y >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    ref = O.uniforms(seed, offset + 312)[offset:]
    assert np.array_equal(got, ref)
