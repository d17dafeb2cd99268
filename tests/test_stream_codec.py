"""FORMATS.md readers (codec.cpp:136-190, 260-300) and the record-stream host logic
(SURVEY.md 8(f) row 3). Device appends are covered in tests/test_gpu_stream.py."""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200 import codec
from paper_2504_14897_b200.types import (AffineMap, AxisRange, CodecError, GaussianComponent,
                                         GmmModel, Histogram2D, ModelMeta, Plane)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "formats_hex.json")))


def test_decode_formats_md_vector():  # FORMATS.md:35-47
    dm = codec.decode_model(bytes.fromhex(GOLD["hex"]))
    c = dm.model.components[0]
    assert dm.model.size() == 1 and c.weight == 1.0 and list(c.mean) == [0.5, -0.25]
    assert c.covariance.tolist() == [[1.0, 0.125], [0.125, 2.0]]
    assert dm.meta.species_label == "e" and dm.meta.plane == Plane.uv and dm.meta.cycle == 50
    assert [(r.lo, r.hi) for r in dm.meta.axis_ranges] == [(-5.0, 5.0)] * 2


def test_decode_errors():  # test_codec.cpp corruption cases
    b = bytearray.fromhex(GOLD["hex"])
    with pytest.raises(CodecError, match="bad magic"):
        codec.decode_model(b"XMMC" + bytes(b[4:]))
    bad = bytearray(b)
    bad[12] ^= 1
    with pytest.raises(CodecError, match="CRC"):
        codec.decode_model(bytes(bad))
    with pytest.raises(CodecError, match="truncated"):
        codec.decode_model(bytes(b[:-8]))
    with pytest.raises(CodecError, match="size mismatch"):
        codec.decode_model(bytes(b) + b"\0" * 8)
    v = bytearray(b)
    v[4] = 2
    with pytest.raises(CodecError, match="unsupported version"):
        codec.decode_model(bytes(v))
    nspd = bytearray(b)
    nspd[-24:-16] = np.array([-1.0]).tobytes()  # Sigma00 < 0
    with pytest.raises(CodecError, match="positive definite"):
        codec.decode_model(bytes(nspd))


def test_decode_roundtrip_3v():
    rng = np.random.default_rng(4)
    comps = []
    for w in (0.2, 0.5, 0.3):
        a = rng.normal(size=(3, 3))
        comps.append(GaussianComponent(w, rng.normal(size=3), a @ a.T + np.eye(3)))
    m = GmmModel(comps, AffineMap.identity(3), 3)
    meta = ModelMeta("ions", None, -7, [AxisRange(-1, 2)] * 3)
    dm = codec.decode_model(O.encode_model(m, meta))
    for a, b in zip(dm.model.components, m.components):
        assert a.weight == b.weight and np.array_equal(a.mean, b.mean)
        assert np.array_equal(np.triu(a.covariance), np.triu(b.covariance))
    assert dm.meta.plane is None and dm.meta.cycle == -7 and dm.meta.species_label == "ions"


def test_h2d_roundtrip_and_size():  # test_codec.cpp:186-200
    rng = np.random.default_rng(1)
    counts = rng.integers(0, 9, size=(200, 200)).astype(float)
    h = Histogram2D(np.asfortranarray(counts), AxisRange(-5, 5), AxisRange(-4, 4), Plane.vw, 200, 3.0, "e")
    payload = codec.encode_histogram(h)
    assert len(payload) == 320000
    assert np.frombuffer(payload, "<f8")[1 * 200 + 2] == counts[1, 2]  # x bin = row
    side = codec.histogram_sidecar(h)
    back = codec.decode_histogram(payload, json.dumps(side))
    assert np.array_equal(back.counts, counts) and back.plane == Plane.vw
    assert back.out_of_range_count == 3.0 and back.range_y.hi == 4
    with pytest.raises(CodecError, match="header implies"):
        codec.decode_histogram(payload[:-8], side)
    with pytest.raises(CodecError, match="not an h2d"):
        codec.decode_histogram(payload, dict(side, format="x"))


def test_empty_stream_writes_index(tmp_path):
    """Stream open/close is host-only (no device work without appends)."""
    from paper_2504_14897_b200.stream import GMMC, RecordStream, read_index, stream_kind
    p = str(tmp_path / "empty.gmmcs")
    s = RecordStream(p, GMMC)
    assert s.close() == (0, 0)
    assert os.path.getsize(p) == 0 and len(read_index(p)) == 0 and stream_kind(p) == GMMC
    from paper_2504_14897_b200.types import InvalidArgument
    with pytest.raises(InvalidArgument):
        RecordStream(str(tmp_path / "x"), 7)


def test_model_json_round_trip():  # FORMATS.md:52-70, codec.cpp:192-255
    rng = np.random.default_rng(8)
    a = rng.normal(size=(3, 3))
    cov = a @ a.T + np.eye(3)
    cov = np.triu(cov) + np.triu(cov, 1).T
    m = GmmModel([GaussianComponent(0.3, rng.normal(size=3), cov),
                  GaussianComponent(0.7, rng.normal(size=3), np.eye(3) * 0.1)], AffineMap.identity(3), 3)
    meta = ModelMeta("ions", None, 9, [AxisRange(-1.5, 2.0)] * 3)
    j = json.loads(json.dumps(codec.model_to_json(m, meta)))
    assert j["format"] == "gmm-model" and j["plane"] is None and len(j["components"][0]["covariance_upper"]) == 6
    back = codec.model_from_json(j)
    for x, y in zip(back.model.components, m.components):
        assert x.weight == y.weight and np.array_equal(x.mean, y.mean) and np.array_equal(x.covariance, y.covariance)
    # the JSON and the binary record carry the same information
    dm = codec.decode_model(O.encode_model(m, meta))
    assert [c.weight for c in dm.model.components] == [c.weight for c in back.model.components]
    with pytest.raises(CodecError, match="gmm-model"):
        codec.model_from_json(dict(j, format="x"))
