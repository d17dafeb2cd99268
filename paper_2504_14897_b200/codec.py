"""Readers for the FORMATS.md payloads the device path writes (codec.hpp:50-64).

``decode_model`` (codec.cpp:136-190), the ``.gmm.json`` rendering (codec.cpp:192-255) and
the ``.h2d`` helpers (codec.cpp:260-300) are
byte-format parsing on the host — the reference does the same on the host — used to
read back ``.gmmc`` records and record streams. Errors raise ``CodecError`` with the
reference's messages.
"""
from __future__ import annotations

import json
import struct
import zlib
from dataclasses import dataclass

import numpy as np

from .types import (AffineMap, AxisRange, CodecError, GaussianComponent, GmmModel, Histogram2D,
                    InvalidArgument, ModelMeta, Plane)

_PLANES = {0: Plane.uv, 1: Plane.vw, 2: Plane.uw}
_PLANE_NAMES = {Plane.uv: "uv", Plane.vw: "vw", Plane.uw: "uw"}


@dataclass
class DecodedModel:
    """codec.hpp:27-30."""
    model: GmmModel
    meta: ModelMeta


def _llt_ok(c: np.ndarray) -> bool:
    """Eigen LLT success + llt_ok (gaussian.hpp:15-19), restated for d <= 8."""
    d = c.shape[0]
    L = np.zeros_like(c)
    for k in range(d):
        x = c[k, k] - float(np.dot(L[k, :k], L[k, :k]))
        if not (x > 0.0) or not np.isfinite(np.sqrt(x)):
            return False
        L[k, k] = np.sqrt(x)
        for i in range(k + 1, d):
            L[i, k] = (c[i, k] - float(np.dot(L[i, :k], L[k, :k]))) / L[k, k]
    return True


def decode_model(data: bytes) -> DecodedModel:
    """codec.cpp:136-190."""
    data = bytes(data)
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(data):
            raise CodecError("truncated")
        out = data[pos:pos + n]
        pos += n
        return out

    if take(4) != b"GMMC":
        raise CodecError("bad magic: not a gmmc model")
    version = take(1)[0]
    if version != 1:
        raise CodecError(f"unsupported version {version}")
    d = take(1)[0]
    if d < 1 or d > 8:
        raise CodecError("implausible dimension")
    plane_id = take(1)[0]
    take(1)
    m = struct.unpack("<I", take(4))[0]
    cycle = struct.unpack("<q", take(8))[0]
    ranges = []
    for _ in range(d):
        lo, hi = struct.unpack("<dd", take(16))
        ranges.append(AxisRange(lo, hi))
    ll = struct.unpack("<H", take(2))[0]
    label = take(ll).decode("utf-8", errors="replace")
    header_len = pos
    crc = struct.unpack("<I", take(4))[0]
    if crc != zlib.crc32(data[:header_len]) & 0xFFFFFFFF:
        raise CodecError("header CRC mismatch")
    plane = None
    if plane_id != 255:
        if plane_id > 2:
            raise CodecError("invalid plane id")
        plane = _PLANES[plane_id]
    expected = m * (1 + d + d * (d + 1) // 2) * 8
    rem = len(data) - pos
    if rem < expected:
        raise CodecError("truncated payload")
    if rem > expected:
        raise CodecError("payload size mismatch vs header")
    vals = np.frombuffer(data, dtype="<f8", count=expected // 8, offset=pos)
    comps = []
    k = 0
    iu = np.triu_indices(d)
    for _ in range(m):
        w = float(vals[k])
        mean = np.array(vals[k + 1:k + 1 + d])
        k += 1 + d
        cov = np.zeros((d, d))
        cov[iu] = vals[k:k + d * (d + 1) // 2]
        k += d * (d + 1) // 2
        cov[(iu[1], iu[0])] = cov[iu]  # set_covariance mirrors the upper triangle
        if not _llt_ok(cov):
            raise CodecError("decoded covariance is not symmetric positive definite")
        comps.append(GaussianComponent(w, mean, cov))
    return DecodedModel(GmmModel(comps, AffineMap.identity(d), d),
                        ModelMeta(label, plane, cycle, ranges))


def model_to_json(model: GmmModel, meta: ModelMeta) -> dict:
    """codec.cpp:192-220 (`.gmm.json`): same information as `.gmmc`; json.dumps prints
    doubles in their shortest round-trip form, so parsing reproduces the exact bits.
    Expects a canonical (data-space) model, as the writers produce."""
    model.validate()
    if not model.normalization.is_identity():
        raise InvalidArgument("model_to_json: denormalize the model first (denormalize_model)")
    d = model.dimension
    if len(meta.axis_ranges) != d:
        raise InvalidArgument("model meta must carry one axis range per dimension")
    comps = []
    for c in model.components:
        cov = np.asarray(c.covariance, float)
        comps.append({"weight": float(c.weight), "mean": [float(x) for x in c.mean],
                      "covariance_upper": [float(cov[i, j]) for i in range(d) for j in range(i, d)]})
    return {"format": "gmm-model", "version": 1, "dimension": d, "components": comps,
            "plane": _PLANE_NAMES[Plane(meta.plane)] if meta.plane is not None else None,
            "species": meta.species_label, "cycle": int(meta.cycle),
            "axis_ranges": [[r.lo, r.hi] for r in meta.axis_ranges]}


def model_from_json(j) -> DecodedModel:
    """codec.cpp:222-255."""
    if isinstance(j, (str, bytes)):
        j = json.loads(j)
    if j.get("format", "") != "gmm-model":
        raise CodecError("not a gmm-model JSON document")
    if j["version"] != 1:
        raise CodecError("unsupported gmm-model JSON version")
    d = int(j["dimension"])
    iu = np.triu_indices(d)
    comps = []
    for jc in j["components"]:
        mean, upper = jc["mean"], jc["covariance_upper"]
        if len(mean) != d or len(upper) != d * (d + 1) // 2:
            raise CodecError("component shape mismatch")
        cov = np.zeros((d, d))
        cov[iu] = upper
        cov[(iu[1], iu[0])] = cov[iu]
        if not _llt_ok(cov):
            raise CodecError("decoded covariance is not symmetric positive definite")
        comps.append(GaussianComponent(float(jc["weight"]), np.array(mean, float), cov))
    names = {v: k for k, v in _PLANE_NAMES.items()}
    plane = None if j["plane"] is None else names[j["plane"]]
    meta = ModelMeta(j["species"], plane, int(j["cycle"]), [AxisRange(*r) for r in j["axis_ranges"]])
    return DecodedModel(GmmModel(comps, AffineMap.identity(d), d), meta)


def encode_histogram(hist: Histogram2D) -> bytes:
    """codec.cpp:260-267: n^2 little-endian f64, row-major with the x bin as the row."""
    return np.ascontiguousarray(hist.counts, dtype="<f8").tobytes(order="C")


def histogram_sidecar(hist: Histogram2D) -> dict:
    """codec.cpp:269-278."""
    return {"format": "h2d", "version": 1, "n_bins": hist.n_bins,
            "plane": _PLANE_NAMES[Plane(hist.plane)],
            "range_x": [hist.range_x.lo, hist.range_x.hi],
            "range_y": [hist.range_y.lo, hist.range_y.hi],
            "out_of_range_count": hist.out_of_range_count, "species": hist.species_label}


def decode_histogram(payload: bytes, sidecar) -> Histogram2D:
    """codec.cpp:280-300."""
    if isinstance(sidecar, (str, bytes)):
        sidecar = json.loads(sidecar)
    if sidecar.get("format", "") != "h2d":
        raise CodecError("not an h2d sidecar")
    if sidecar["version"] != 1:
        raise CodecError("unsupported h2d version")
    n = int(sidecar["n_bins"])
    if n < 1:
        raise CodecError("invalid n_bins")
    expected = n * n * 8
    if len(payload) != expected:
        raise CodecError(f"histogram payload is {len(payload)} bytes, header implies {expected}")
    names = {v: k for k, v in _PLANE_NAMES.items()}
    if sidecar["plane"] not in names:
        raise CodecError(f"unknown plane {sidecar['plane']}")
    counts = np.frombuffer(bytes(payload), dtype="<f8").reshape(n, n).astype(np.float64)
    return Histogram2D(counts=np.asfortranarray(counts), range_x=AxisRange(*sidecar["range_x"]),
                       range_y=AxisRange(*sidecar["range_y"]), plane=names[sidecar["plane"]],
                       n_bins=n, out_of_range_count=float(sidecar["out_of_range_count"]),
                       species_label=sidecar.get("species", ""))
