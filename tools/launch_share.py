"""Per-kernel count / total / share of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, io, sys

txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if len(r) < len(h) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    try:
        v = float(r[vi])
    except ValueError:
        continue
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T / 1e3:.1f} us total (ncu: cold cache, serialised)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} n={cnt[k]:5d} total {v / 1e3:12.1f} us  share {100 * v / T:5.1f}%")
