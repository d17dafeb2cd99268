"""Per-launch DRAM traffic of the bench's kernels from an `ncu --set full` capture, keyed by
the labels the library's timing uses (what bench.py reports as roofline.traffic).
Usage: python tools/ncu_traffic.py rep.ncu-rep profiles/ncu_traffic_cfg4.json"""
import csv
import io
import json
import subprocess
import sys

LABELS = [("cells_bitmap_tma_kernel", "cells_bitmap_tma"), ("cells_bitmap_kernel", "cells_bitmap"),
          ("cells_sort_kernel", "cells_sort"), ("cells_dense_kernel", "cells_dense"),
          ("em_kernel", "em_fit"), ("cell_metrics_kernel", "cell_metrics")]
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {"source": f"ncu --set full capture {rep} (tools/round_run.sh)", "kernels": {}}
    for r in data:
        name = r[hdr.index("Kernel Name")]
        label = next((lab for key, lab in LABELS if key in name), None)
        if label is None or label in res["kernels"]:
            continue

        def val(m):
            i = hdr.index(m)
            return float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        res["kernels"][label] = {
            "kernel": name[:120],
            "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "duration_ms_under_ncu": val("gpu__time_duration.sum"),
            "fp64_pipe_pct": val(METRICS[3]), "issue_active_pct": val(METRICS[4]),
            "warps_active_pct": val(METRICS[5])}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
