"""Multi-GPU sharding logic on CPU: world_size=2 gloo processes each own a contiguous
half of the cells (bench.py my_cells), compress them (the CPU oracle stands in for the
device here), and the gathered records equal the single-process run byte for byte —
cells are independent, so no collective is needed on the data path."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _cfg():
    # skewed cells: the split must balance particles, not cells
    counts = [300 + (c * 997) % 1400 for c in range(24)]
    return dict(workload="t", d=3, species=[("e", 6.0)], cells=24, particles=sum(counts), n_bins=24,
                K=3, scaling="strong", counts=counts)


def _compress(c0, c1):
    import bench
    import oracle as O
    from paper_2504_14897_b200.types import AxisRange, FitConfig, ModelMeta
    cfg = _cfg()
    counts = bench.cell_counts(cfg)
    offs_all = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    v = bench.synth_numpy(3, offs_all[c0:c1 + 1], c0, 11, 0)
    offs = offs_all[c0:c1 + 1] - offs_all[c0]
    _, res = O.compress_cells(O.CellsHost(v, offs, 24, [-6] * 3, [6] * 3),
                              FitConfig(initial_components=3, seed=11, temperature=np.ones(3)))
    rec, ro = O.pack_cells(res, c1 - c0, ModelMeta("e", None, 0, [AxisRange(-6, 6)] * 3))
    return rec


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    c0, c1 = bench.my_cells(_cfg(), rank, world)
    rec = _compress(c0, c1)
    gathered = [None] * world
    dist.all_gather_object(gathered, (c0, c1, rec))
    if rank == 0:
        out.put(gathered)
    dist.destroy_process_group()


def test_partition_balances_particles():
    """vdfcg_partition_cells (host-only): contiguous ranges covering every cell, each part's
    particle count within one cell of total/n, identical to a numpy restatement."""
    from paper_2504_14897_b200.cells import partition_cells
    rng = np.random.default_rng(2)
    for n_cells, parts in ((1000, 8), (37, 4), (5, 8), (262144, 8), (0, 3)):
        counts = rng.integers(0, 4000, size=n_cells)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        b = partition_cells(offs, parts)
        assert b[0] == 0 and b[-1] == n_cells and np.all(np.diff(b) >= 0)
        total = offs[-1]
        for r in range(1, parts):
            t = total * r // parts
            c = np.searchsorted(offs, t, side="left")
            if c > 0 and (c > n_cells or t - offs[c - 1] <= offs[c] - t):
                c -= 1
            assert b[r] == max(c, b[r - 1]), (n_cells, parts, r)
        if n_cells:
            per = offs[b[1:]] - offs[b[:-1]]
            assert per.max() - total / parts <= counts.max() + 1


def test_two_rank_shards_cover_cells_and_match_single_process():
    import bench
    cfg = _cfg()
    spans = [bench.my_cells(cfg, r, 2) for r in range(2)]
    assert spans[0][0] == 0 and spans[0][1] == spans[1][0] and spans[1][1] == cfg["cells"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    gathered = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    single = _compress(0, cfg["cells"])
    assert b"".join(g[2] for g in sorted(gathered)) == single
