"""Summarise an .ncu-rep: key throughput metrics + top stall reasons + instruction mix."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def page(p, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout

keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Block Size", "Grid Size", "Warp Cycles Per Issued Instruction"]
rows = list(csv.reader(io.StringIO(page("details"))))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:38s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(page("raw"))))
if len(raw) > 2:
    hh = raw[0]; vals = raw[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if k in hh:
            i = hh.index(k); print(f"{k:60s} {vals[i]} {raw[1][i]}")
src = list(csv.reader(io.StringIO(page("source", ("--print-source", "sass")))))
if len(src) > 2:
    h = src[1]
    data = [dict(zip(h, r)) for r in src[2:] if len(r) == len(h) and r[0] != "Address"]
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    S = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
    tot = collections.Counter()
    for d in data:
        for c in stalls:
            tot[c] += int(d[c] or 0)
    print("stall samples", S)
    for c, v in tot.most_common(8):
        print(f"  {c:25s} {100 * v / S:5.1f}%")
    mix = collections.Counter()
    for d in data:
        toks = d["Source"].split()
        if not toks: continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        mix[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
    tot_i = sum(mix.values())
    print("warp instructions", tot_i, "top:", ", ".join(f"{k} {100*v/tot_i:.1f}%" for k, v in mix.most_common(12)))
