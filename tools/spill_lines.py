"""Local-memory (LDL/STL) instructions per source line of one kernel in a cubin.
usage: python tools/spill_lines.py <obj.o|.cubin> <kernel-substring>"""
import collections, os, re, subprocess, sys, tempfile

obj, pat = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
if obj.endswith(".o") or obj.endswith(".so"):
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cubins = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")]
else:
    cubins = [obj]
for cb in cubins:
    dis = subprocess.run(["nvdisasm", "-gi", cb], capture_output=True, text=True).stdout.split("\n")
    start = None
    for i, l in enumerate(dis):
        if ".section" in l and ".text." in l and pat in l:
            start = i
            break
    if start is None:
        continue
    cur, cnt, tot = None, collections.Counter(), 0
    for l in dis[start + 1:]:
        if ".section" in l and ".text." in l:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        if re.search(r"\b(LDL|STL)(\.\w+)*\b", l):
            cnt[cur] += 1
            tot += 1
    print(os.path.basename(cb), "total", tot)
    for k, v in cnt.most_common(40):
        print(f"{v:4d} {k[0]}:{k[1]}")
