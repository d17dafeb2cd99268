"""K sweep x bin sweep on one B200 (BASELINE.json configs[4], single-GPU part): for each
(K, n_bins) one species of `--cells` 3V cells x `--per` particles is binned and fitted on
the device; prints histogram GB/s and EM algorithmic TFLOP/s with their roofline
fractions, particles/s and fits/s, as a markdown table.
Usage: python tools/sweep.py [--cells 65536] [--per 1907]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2504_14897_b200 as G  # noqa: E402
from paper_2504_14897_b200 import api  # noqa: E402
from paper_2504_14897_b200.types import FitConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=65536)
    ap.add_argument("--per", type=int, default=1907)
    ap.add_argument("--json", default=None)
    ap.add_argument("--cpu-cells", type=int, default=64, help="CPU-oracle sample cells per config (0: skip)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    hbm = bench.peaks()[0] if hasattr(bench, "peaks") else 6540.8
    fp64_peak, _ = api.probe_peaks()
    offs = torch.arange(a.cells + 1, dtype=torch.int64, device=dev) * a.per
    axes = [torch.empty(a.cells * a.per, dtype=torch.float64, device=dev) for _ in range(3)]
    G.synth_cells(3, offs, 1, 0, *axes)
    ctx = api.context()
    rows = []
    threads = os.cpu_count() or 1
    if a.cpu_cells:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        stride = max(1, a.cells // a.cpu_cells)
        sel = np.arange(0, a.cells, stride)[:a.cpu_cells]
        idx = np.concatenate([np.arange(c * a.per, (c + 1) * a.per) for c in sel])
        hv = np.asfortranarray(np.stack([ax.cpu().numpy()[idx] for ax in axes], axis=1))
        hoffs = np.arange(len(sel) + 1, dtype=np.int64) * a.per
    for nb in (16, 24, 32, 48, 64):
        b = G.CellBatch(axes, offs, nb, [-6] * 3, [6] * 3)
        for K in (1, 2, 4, 8):
            cfg = FitConfig(initial_components=K, seed=0, temperature=np.ones(3))
            bins, res, _, _ = G.compress_cells(b, cfg, keep_bins=True)  # warm-up
            torch.cuda.synchronize()
            ctx.enable_timing(True)
            ctx.reset_timing()
            bins, res, _, _ = G.compress_cells(b, cfg, keep_bins=True)
            torch.cuda.synchronize()
            kt = ctx.kernel_times()
            ctx.enable_timing(False)
            hist_name = max((k for k in kt if k.startswith("cells_")), key=lambda k: kt[k][0])
            h_ms, em_ms = kt[hist_name][0], kt["em_fit"][0]
            total_ms = sum(v[0] for v in kt.values())
            nnz = bins.nnz.cpu().numpy().astype(np.float64)
            r = res.numpy()
            flops = bench.em_flops({"status": r.status, "iterations": r.iterations,
                                    "n_events": r.n_events, "event_iteration": r.event_iteration},
                                   nnz, K, 3)
            hbytes = a.cells * a.per * 24 + nnz.sum() * 12 + (a.cells + 1) * 8
            row = {"n_bins": nb, "K": K, "hist_kernel": hist_name, "hist_ms": h_ms,
                   "hist_GBps": hbytes / h_ms / 1e6, "hist_frac": hbytes / h_ms / 1e6 / hbm,
                   "em_ms": em_ms, "em_TFLOPs": flops / em_ms / 1e9,
                   "em_frac": flops / em_ms / 1e9 / fp64_peak, "mean_iterations": float(r.iterations.mean()),
                   "mean_nnz": float(nnz.mean()), "particles_per_s": a.cells * a.per / (total_ms * 1e-3),
                   "fits_per_s": a.cells / (total_ms * 1e-3)}
            if a.cpu_cells:  # the CPU oracle (reference algorithm, oracle/) on a cell sample
                import time
                t0 = time.perf_counter()
                O.compress_cells(O.CellsHost(hv, hoffs, nb, [-6] * 3, [6] * 3), cfg, threads=threads)
                dt = time.perf_counter() - t0
                row["cpu_particles_per_s"] = len(sel) * a.per / dt
                row["cpu_fits_per_s"] = len(sel) / dt
                row["gpu_over_cpu"] = row["particles_per_s"] / row["cpu_particles_per_s"]
            rows.append(row)
    print(f"one B200, {a.cells} cells x {a.per} particles (3V), FP64 peak {fp64_peak:.1f} TFLOP/s, "
          f"HBM {hbm:.0f} GB/s; CPU = oracle/ (reference algorithm restated) on {a.cpu_cells} sampled cells, "
          f"{threads} host threads\n")
    print("| bins | K | hist kernel | hist ms | hist % HBM | EM ms | EM TFLOP/s | EM % FP64 | mean its | particles/s | fits/s | CPU particles/s | GPU/CPU |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        cpu = f"{r['cpu_particles_per_s']:.3g} | {r['gpu_over_cpu']:.0f}" if "cpu_particles_per_s" in r else "- | -"
        print(f"| {r['n_bins']}³ | {r['K']} | {r['hist_kernel']} | {r['hist_ms']:.2f} | {100 * r['hist_frac']:.1f} | "
              f"{r['em_ms']:.1f} | {r['em_TFLOPs']:.2f} | {100 * r['em_frac']:.1f} | {r['mean_iterations']:.1f} | "
              f"{r['particles_per_s']:.3g} | {r['fits_per_s']:.3g} | {cpu} |")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
