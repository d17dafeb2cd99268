"""Summarise an .ncu-rep: SOL, occupancy, pipes, stall reasons, hottest SASS."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("raw")
h, vals = rows[0], rows[2]
d = dict(zip(h, vals))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1
print("stalls:", ", ".join(f"{k} {100 * v / tot:.1f}%" for v, k in sorted(st, reverse=True)[:10]))
src = page("source", ["--print-source=sass"])
hh = src[1]
ins = [dict(zip(hh, x)) for x in src[2:]]
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in ins) or 1
by = collections.Counter()
for x in ins:
    t = x["Source"].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    by[op.split(".")[0]] += int(x["Warp Stall Sampling (All Samples)"] or 0)
print("samples by opcode:", [(k, round(100 * v / tot, 1)) for k, v in by.most_common(16)])
for x in sorted(ins, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:12]:
    print(f"  {100 * int(x['Warp Stall Sampling (All Samples)']) / tot:5.1f}%  exec={x['Instructions Executed']:>12s}  {x['Source'][:80]}")
