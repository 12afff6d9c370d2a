"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel totals/shares.
python tools/launch_summary.py launches.csv [--ours] [name-filter]; --ours drops the harness's
torch / cuBLAS kernels (parity checks of bench.py) so the shares are those of the library's step."""
import collections
import csv
import sys

ours = "--ours" in sys.argv
argv = [a for a in sys.argv if a != "--ours"]
rows = list(csv.reader(open(argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size")
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("tcqr::", "")
    if ours and (name.startswith("at::") or name.startswith("cutlass::") or "cublas" in name):
        continue
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
    agg[name][0] += 1
    agg[name][1] += v
    seq.append((name, v, r[gi]))
tot = sum(a[1] for a in agg.values())
print(f"total {tot/1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches (cold-cache, serialized)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:40s} n={n:5d} total={t/1e3:9.3f} ms avg={t/n:9.2f} us share={t/tot:.3f}")
if len(argv) > 2:
    for name, v, g in seq:
        if argv[2] in name:
            print(f"    {name:40s} {v:9.2f} us grid {g}")
