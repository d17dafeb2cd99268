"""Summarise an .ncu-rep: per kernel SOL, DRAM traffic, occupancy, pipes, stall reasons,
and the hottest SASS (samples by opcode). Usage: python tools/ncu_summary.py rep [--json out]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
json_out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum"]

rows = page("raw")
h, units = rows[0], rows[1]
summary = []
for vals in rows[2:]:
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    name = d.get("Kernel Name", "?")
    print(f"=== {name[:110]}")
    rec = {"kernel": name}
    for k in KEYS:
        print(f"  {k:66s} {d.get(k)} {u.get(k, '')}")
        rec[k] = d.get(k)
        rec[k + ".unit"] = u.get(k, "")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    stalls = [(k, round(100 * v / tot, 1)) for v, k in sorted(st, reverse=True)[:10]]
    print("  stalls:", ", ".join(f"{k} {p}%" for k, p in stalls))
    rec["stalls_pct"] = stalls
    summary.append(rec)

# SASS hot spots per kernel section of the source page
src = page("source", ["--print-source=sass"])
sections, cur = [], None
for row in src:
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1] if len(row) > 1 else "?", "rows": []}
        sections.append(cur)
    elif row and row[0] == "Address":
        cur["hdr"] = row
    elif cur is not None and "hdr" in cur and row:
        cur["rows"].append(dict(zip(cur["hdr"], row)))
for sec in sections:
    ins = sec["rows"]
    col = "Warp Stall Sampling (All Samples)"

    def val(x):
        try:
            return int(x.get(col) or 0)
        except ValueError:
            return 0
    tot = sum(val(x) for x in ins) or 1
    by = collections.Counter()
    for x in ins:
        t = x.get("Source", "").split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        by[op.split(".")[0]] += val(x)
    print(f"--- SASS samples by opcode: {sec['name'][:80]}")
    print("  ", [(k, round(100 * v / tot, 1)) for k, v in by.most_common(14)])
if json_out:
    json.dump(summary, open(json_out, "w"), indent=1)
