"""Record streams (vdfcg_stream_*): batches of per-cell .gmmc
records or .h2d histogram payloads appended to one file plus a binary index, written by
the library's IO thread while the device works on the next batch.

    with RecordStream("run.gmmcs") as s:
        for batch in batches:
            _, res, rec, offs = compress_cells(batch, cfg, meta)
            s.append_records(rec, offs, cell_base=batch_first_cell)
    idx = read_index("run.gmmcs")            # numpy structured array
    m = decode_model(read_record("run.gmmcs", idx[0]))
"""
from __future__ import annotations

import ctypes as C
import zlib

import numpy as np

INDEX_DTYPE = np.dtype([("cell", "<i8"), ("offset", "<u8"), ("length", "<u4"), ("crc", "<u4"),
                        ("aux", "<f8")])
GMMC, H2D = 0, 1


def _api():
    from . import api
    return api


def _bind():
    lib = _api().lib()
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    for name, args in {"vdfcg_stream_open": [C.c_char_p, i32, C.POINTER(vp)],
                       "vdfcg_stream_append_records": [vp, vp, vp, vp, i32, i64],
                       "vdfcg_stream_append_h2d": [vp, vp, vp, vp, i64],
                       "vdfcg_stream_close": [vp, vp, vp]}.items():
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = args
    return lib


def _check(rc):
    from ._marshal import check
    check(rc, _api().last_error)


def _ptr(x):
    if x is None:
        return None
    return x.data_ptr() if type(x).__module__.startswith("torch") else x.ctypes.data


class RecordStream:
    """An open stream file of kind GMMC (records) or H2D (2V cell histograms)."""

    def __init__(self, path: str, kind: int = GMMC):
        self.path, self.kind = path, kind
        self._lib = _bind()
        self._h = C.c_void_p()
        _check(self._lib.vdfcg_stream_open(path.encode(), kind, C.byref(self._h)))

    def append_records(self, records, offsets, cell_base: int = 0) -> None:
        """records / offsets from compress_cells or pack_cells (host or device)."""
        n = int(offsets.shape[0]) - 1
        from .cells import _ctx
        _check(self._lib.vdfcg_stream_append_records(self._h, _ctx(records, offsets).handle,
                                                     _ptr(records), _ptr(offsets), n, int(cell_base)))

    def append_h2d(self, batch, bins, cell_base: int = 0) -> None:
        """One .h2d payload per cell of a 2V CellBatch from its CellBins."""
        bs = bins.struct()
        from .cells import _ctx
        _check(self._lib.vdfcg_stream_append_h2d(self._h, _ctx(batch.axes[0]).handle,
                                                 C.byref(batch.struct), C.byref(bs), int(cell_base)))

    def close(self) -> tuple[int, int]:
        """Flush, write the index; returns (records, payload bytes)."""
        if not self._h:
            return 0, 0
        n, b = C.c_int64(), C.c_int64()
        h, self._h = self._h, C.c_void_p()
        _check(self._lib.vdfcg_stream_close(h, C.byref(n), C.byref(b)))
        return n.value, b.value

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_index(path: str, verify: bool = False) -> np.ndarray:
    """The `<path>.idx` entries; verify=True also checks each record's CRC-32."""
    raw = open(path + ".idx", "rb").read()
    if raw[:4] != b"GMIX" or raw[4] != 1:
        raise ValueError("not a vdfcg stream index")
    n = int(np.frombuffer(raw, "<u8", 1, 8)[0])
    idx = np.frombuffer(raw, INDEX_DTYPE, n, 16)
    if verify:
        with open(path, "rb") as f:
            for e in idx:
                f.seek(int(e["offset"]))
                if zlib.crc32(f.read(int(e["length"]))) & 0xFFFFFFFF != int(e["crc"]):
                    raise ValueError(f"CRC mismatch for cell {int(e['cell'])}")
    return idx


def stream_kind(path: str) -> int:
    return open(path + ".idx", "rb").read(6)[5]


def read_record(path: str, entry) -> bytes:
    with open(path, "rb") as f:
        f.seek(int(entry["offset"]))
        return f.read(int(entry["length"]))


__all__ = ["RecordStream", "read_index", "read_record", "stream_kind", "INDEX_DTYPE", "GMMC", "H2D"]
