"""Per-CUDA-source-line warp-stall samples of an .ncu-rep (needs -lineinfo).

  python tools/ncu_lines.py rep.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, header, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(header[4:], r[4:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
              and v.isdigit() and int(v) > 0}
    ie = d.get("Instructions Executed", "0")
    rows.append((s, f"{fname}:{r[0]}", r[1][:70], stalls, int(ie) if ie.isdigit() else 0))
tot = sum(r[0] for r in rows) or 1
rows.sort(key=lambda r: -r[0])
print(f"total stall samples {tot}")
for s, loc, src, st, ie in rows[:top]:
    big = ", ".join(f"{k[6:]} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * s / tot:5.1f}% {loc:24s} inst {ie:>10d}  {src:70s} [{big}]")
