"""Record streams on the device path: batched .gmmc records and
.h2d payloads written by the IO thread, read back through the FORMATS.md decoders."""
import numpy as np
import pytest

import oracle as O
from paper_2504_14897_b200.types import AxisRange, FitConfig, ModelMeta

pytestmark = pytest.mark.gpu


def _batch(G, torch, n_cells, per, d, seed, base):
    dev = torch.device("cuda", 0)
    offs = (torch.arange(n_cells + 1, dtype=torch.int64, device=dev) + base) * per  # global
    axes = [torch.empty(n_cells * per, dtype=torch.float64, device=dev) for _ in range(d)]
    G.synth_cells(d, offs, seed, 0, *axes, *([None] if d == 2 else []), cell_base=base)
    return G.CellBatch(axes, offs - offs[0], 32 if d == 3 else 40, [-6] * d, [6] * d)


def test_gmmc_stream_roundtrip(tmp_path):
    import torch
    import paper_2504_14897_b200 as G
    from paper_2504_14897_b200.codec import decode_model
    from paper_2504_14897_b200.stream import RecordStream, read_index, read_record
    cfg = FitConfig(initial_components=4, seed=1, temperature=np.ones(3))
    meta = ModelMeta("e", None, 12, [AxisRange(-6, 6)] * 3)
    path = str(tmp_path / "run.gmmcs")
    kept = []
    with RecordStream(path) as s:
        for j, (nc, base) in enumerate([(300, 0), (500, 300), (7, 800)]):
            b = _batch(G, torch, nc, 1200, 3, 9, base)
            _, res, rec, offs = G.compress_cells(b, cfg, meta)
            s.append_records(rec, offs, cell_base=base)
            kept.append((base, res.numpy(), rec.cpu().numpy().tobytes(), offs.cpu().numpy()))
    idx = read_index(path, verify=True)
    assert len(idx) == 807 and list(idx["cell"]) == list(range(807))
    assert np.all(np.diff(idx["offset"].astype(np.int64)) == idx["length"][:-1].astype(np.int64))
    for base, res, recb, offs in kept:
        for c in range(0, len(offs) - 1, 37):
            e = idx[base + c]
            raw = read_record(path, e)
            assert raw == recb[offs[c]:offs[c + 1]]
            if res.status[c] != 0:
                assert e["length"] == 0
                continue
            dm = decode_model(raw)
            k = res.k
            assert dm.model.size() == res.components[c] and dm.meta.cycle == 12
            for i, comp in enumerate(dm.model.components):
                assert comp.weight == res.weights[c * k + i]
                assert np.array_equal(comp.mean, res.means[(c * k + i) * 3:(c * k + i + 1) * 3])


def test_h2d_stream_matches_oracle_histograms(tmp_path):
    import torch
    import paper_2504_14897_b200 as G
    from paper_2504_14897_b200.codec import decode_histogram
    from paper_2504_14897_b200.stream import H2D, RecordStream, read_index, read_record
    b = _batch(G, torch, 64, 3000, 2, 4, 0)
    bins = G.bin_cells(b)
    path = str(tmp_path / "h.h2ds")
    with RecordStream(path, H2D) as s:
        s.append_h2d(b, bins, cell_base=100)
    idx = read_index(path, verify=True)
    assert len(idx) == 64 and idx["cell"][0] == 100 and np.all(idx["length"] == 40 * 40 * 8)
    v = np.stack([a.cpu().numpy() for a in b.axes], 1)
    oc = O.CellsHost(v, b.offsets.cpu().numpy(), 40, [-6] * 2, [6] * 2)
    ob = O.bin_cells(oc)
    for c in (0, 17, 63):
        side = {"format": "h2d", "version": 1, "n_bins": 40, "plane": "uv", "range_x": [-6, 6],
                "range_y": [-6, 6], "out_of_range_count": float(idx["aux"][c]), "species": "e"}
        h = decode_histogram(read_record(path, idx[c]), side)
        dense = np.zeros(40 * 40)
        o = oc.offsets[c]
        dense[ob.keys[o:o + ob.nnz[c]]] = ob.counts[o:o + ob.nnz[c]]
        assert np.array_equal(h.counts, dense.reshape(40, 40))
        assert h.out_of_range_count == ob.out_of_range[c]
