"""Per-recursion-level kernel times of one config-3 factorization from an ncu launch list.

Usage: python tools/level_breakdown.py launches.csv [factorization index]
Nodes are visited in order (in-order index i -> width w = 256 * 2^tz(i)); kernels between two
leaf launches belong to the node that follows the earlier leaf.
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr, out = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append((d['Kernel Name'].split('(')[0].replace('void ', '').replace('tcqr::', ''),
                    float(d['Metric Value']) / 1000))
ends = [i for i, o in enumerate(out) if 'zero_lower' in o[0]]
start = ends[which - 1] + 1 if which > 0 else 0
seq = out[start:ends[which] + 1]


def tz(i):
    c = 0
    while i % 2 == 0:
        i //= 2
        c += 1
    return c


nodes, cur, pre, leaf = [], [], [], 0.0
for n, t in seq:
    if 'leaf' in n:
        leaf += t
        if nodes or cur:
            nodes.append(cur)
        cur = []
        if len(nodes) == 0 and not cur:
            nodes.append([])  # marker: first leaf seen
    else:
        cur.append((n, t))
nodes = [x for x in nodes if x is not None][1:]
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for i, nd in enumerate(nodes[:127], 1):
    for n, t in nd:
        agg[256 * 2 ** tz(i)][n] += t
tot = 0.0
print(f"leaves: {leaf/1000:.2f} ms")
for w in sorted(agg):
    s = sum(agg[w].values())
    tot += s
    print(w, f"{s/1000:.2f} ms", {k: round(v / 1000, 3) for k, v in agg[w].items()})
print(f"non-leaf total {tot/1000:.2f} ms")
