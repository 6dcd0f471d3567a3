"""Per-CUDA-line executed warp instructions (and top opcodes) of an .ncu-rep."""
import collections, csv, io, subprocess, sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = header = cur = None
per, ops = collections.Counter(), collections.defaultdict(collections.Counter)
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = f"{fname}:{r[0]} {r[1][:58]}"
        continue
    d = dict(zip(header[2:], r[2:]))
    src = d.get("Source", "").split()
    if not src:
        continue
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    try:
        ie = int(d.get("Instructions Executed", "0"))
    except ValueError:
        continue
    per[cur] += ie
    ops[cur][op] += ie
tot = sum(per.values()) or 1
print("total warp instructions", tot)
for k, v in per.most_common(top):
    print(f"{100 * v / tot:5.1f}% {k:76s} {dict(ops[k].most_common(3))}")
