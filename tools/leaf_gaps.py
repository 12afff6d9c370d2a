"""Critical-path gaps of one config-3 factorization (32768 x 16384, cutoff 128): CTA 0's start /
end of every leaf launch (debug hook tcqr_debug_leaf_trace), the leaf durations and the gaps
between consecutive leaves grouped by the node whose products run in the gap (leaf i -> i + 1:
the node of width 256 * 2^tz(i + 1)).  Graph replay as in the bench (the hook is set before the
first call, so the captured launches carry it)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import collections
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_leaf_trace.argtypes = [ctypes.c_void_p]
m, n = int(os.environ.get("M", 32768)), int(os.environ.get("N", 16384))
A = W.gaussian_cuda(m, n, 3)
Q = torch.empty_like(A)
R = torch.empty(n, n, device="cuda").t()
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
L.tcqr_debug_leaf_trace(ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    tq.factor(A, Q, R)
torch.cuda.synchronize()
res = []
for rep in range(3):
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tq.factor(A, Q, R)
    e1.record()
    torch.cuda.synchronize()
    d = tr.cpu().numpy().astype(np.int64)
    k = int(d[0])
    se = d[1:1 + 2 * k].reshape(k, 2)
    dur = (se[:, 1] - se[:, 0]) / 1000.0
    gaps = (se[1:, 0] - se[:-1, 1]) / 1000.0
    by = collections.defaultdict(list)
    for i, g in enumerate(gaps):
        j, z = i + 1, 0
        while j % 2 == 0:
            j //= 2
            z += 1
        by[256 << z].append(g)
    res.append((e0.elapsed_time(e1), k, dur, gaps, by, (se[-1, 1] - se[0, 0]) / 1e3))
L.tcqr_debug_leaf_trace(None)
for ms, k, dur, gaps, by, span in res:
    print(f"factor {ms:.2f} ms, {k} leaves, first leaf start -> last leaf end {span / 1e3:.2f} ms; "
          f"leaves {dur.sum() / 1e3:.2f} ms (mean {dur.mean():.1f} us, min {dur.min():.1f}, max "
          f"{dur.max():.1f}), gaps {gaps.sum() / 1e3:.2f} ms")
    for w in sorted(by):
        g = np.array(by[w])
        print(f"  gaps before the right half of w={w:6d} nodes: {len(g):4d} x mean {g.mean():8.1f} us "
              f"(min {g.min():8.1f}, median {np.median(g):8.1f}, max {g.max():8.1f}) = {g.sum() / 1e3:6.2f} ms")
if os.environ.get("DUMP"):
    ms, k, dur, gaps, by, span = res[-1]
    print("leaf durations (us):", " ".join(f"{v:.0f}" for v in dur))
    print("gaps (us):", " ".join(f"{v:.0f}" for v in gaps))
