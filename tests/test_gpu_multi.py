"""Several devices from one host process (vdfcg_multi_compress_cells): cells split
by particle count, one context + host thread per device, records gathered in cell order.
The results must equal a one-device compress_cells byte for byte. With one GPU the same
device is used twice (two contexts, two threads, two partitions) — the partition and the
gather are exercised for real; with >= 2 GPUs every device is used."""
import numpy as np
import pytest
import torch

from paper_2504_14897_b200 import AxisRange, FitConfig, ModelMeta
from paper_2504_14897_b200 import cells as G

pytestmark = pytest.mark.gpu


def _batch(n_cells=4096, seed=5):
    rng = np.random.default_rng(seed)
    counts = rng.integers(150, 450, size=n_cells)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = int(offs[-1])
    cid = np.repeat(np.arange(n_cells), counts)
    v = rng.normal(size=(n, 3)) * (1.0 + 0.3 * np.sin(cid))[:, None] + 0.5 * np.cos(cid)[:, None]
    return G.CellBatch(np.asfortranarray(v), offs, 24, [-6.0] * 3, [6.0] * 3), offs


def _check_same(ref, got):
    _, r1, rec1, ro1 = ref
    _, r2, rec2, ro2, cb = got
    for f in ("status", "components", "iterations", "converged", "weights", "means", "covariances",
              "final_loglik", "n_events"):
        assert np.array_equal(getattr(r1, f), getattr(r2, f)), f
    k = r1.k  # event slots past n_events are unspecified
    for f in ("event_iteration", "event_component", "event_weight"):
        a, b = getattr(r1, f).reshape(-1, k), getattr(r2, f).reshape(-1, k)
        used = np.arange(k)[None, :] < r1.n_events[:, None]
        assert np.array_equal(a[used], b[used]), f
    assert np.array_equal(ro1, ro2)
    assert bytes(rec1) == bytes(rec2)
    return cb


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_on_one_gpu_equals_single_call(devices):
    b, offs = _batch()
    cfg = FitConfig(initial_components=4, max_em_iterations=40, seed=3, temperature=np.ones(3))
    meta = ModelMeta("e", None, 7, [AxisRange(-6, 6)] * 3)
    ref = G.compress_cells(b, cfg, meta, keep_bins=False)
    md = G.MultiDevice(devices)
    cb = _check_same(ref, md.compress_cells(b, cfg, meta))
    assert np.array_equal(cb, G.partition_cells(offs, len(devices)))
    md.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="one GPU: covered by the [0, 0] case")
def test_multi_all_devices_equals_single_call():
    b, offs = _batch(n_cells=8192, seed=9)
    cfg = FitConfig(initial_components=4, max_em_iterations=40, seed=3, temperature=np.ones(3))
    meta = ModelMeta("e", None, 7, [AxisRange(-6, 6)] * 3)
    ref = G.compress_cells(b, cfg, meta, keep_bins=False)
    md = G.MultiDevice(list(range(torch.cuda.device_count())))
    _check_same(ref, md.compress_cells(b, cfg, meta))
    md.close()


def test_multi_keeps_bins_and_reports_errors():
    b, offs = _batch(n_cells=2048, seed=4)
    cfg = FitConfig(initial_components=3, max_em_iterations=20, seed=1, temperature=np.ones(3))
    md = G.MultiDevice([0, 0])
    bins, res, rec, ro, cb = md.compress_cells(b, cfg, None, keep_bins=True)
    ref_bins = G.bin_cells(b)
    for f in ("nnz", "out_of_range", "in_range"):
        assert np.array_equal(getattr(bins, f), getattr(ref_bins, f)), f
    for c in range(0, 2048, 97):
        s, k = offs[c], ref_bins.nnz[c]
        assert np.array_equal(bins.keys[s:s + k], ref_bins.keys[s:s + k])
        assert np.array_equal(bins.counts[s:s + k], ref_bins.counts[s:s + k])
    bad = FitConfig(initial_components=3, prune_threshold=0.9)
    with pytest.raises(ValueError, match="prune_threshold"):
        md.compress_cells(b, bad, None)
    md.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_device_pointer_of_another_gpu_is_rejected():
    """A context's kernels cannot read another GPU's memory (no peer mapping): the call
    fails with invalid_argument naming both devices instead of faulting."""
    import ctypes as C
    from paper_2504_14897_b200 import api
    from paper_2504_14897_b200.types import InvalidArgument
    v = [torch.randn(1000, dtype=torch.float64, device="cuda:1") for _ in range(3)]
    offs = torch.tensor([0, 1000], dtype=torch.int64, device="cuda:1")
    b = G.CellBatch(v, offs, 16, [-5.0] * 3, [5.0] * 3)
    bins = G.CellBins.alloc(b)
    bs = bins.struct()
    rc = api.lib().vdfcg_bin_cells(api.context(0).handle, C.byref(b.struct), C.byref(bs))
    assert rc == 1
    assert "passed to a context on cuda:0" in api.lib().vdfcg_last_error().decode()
    with pytest.raises(InvalidArgument):
        G._check(rc)
