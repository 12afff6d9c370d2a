"""Leaf phases inside the config-3 factorization (32768 x 16384): CTA 0's phase timestamps of every
leaf launch (debug hook tcqr_debug_leaf_timestamps_multi), the median phase times of the left
(even) and right (odd) leaves, and of an isolated 32768 x 128 factorization for comparison."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_leaf_timestamps_multi.argtypes = [ctypes.c_void_p]
names = ["load"]
for op in ["P0", "J01", "P1", "J0123", "P2", "J23", "P3"]:
    if op[0] == "P":
        names += [op + s for s in (":mgs", ":publish", ":ownersum", ":gather", ":chol+S", ":apply+st")]
    else:
        names += [op + s for s in (":partial+pub", ":ownersum", ":gather", ":update")]
names += ["write"]
K = len(names) + 1
m, n = int(os.environ.get("M", 32768)), int(os.environ.get("N", 16384))
tq.set_config(use_graphs=int(os.environ.get("GRAPHS", 0)))


BIG = torch.empty(64 << 20, device="cuda")  # 256 MB: evicts L2 (126 MB)
SA, SB = torch.randn(256, 256, device="cuda"), torch.randn(256, 256, device="cuda")


def pollute(kind):
    if kind in ("data", "both"):
        BIG.zero_()
    if kind in ("ef", "ef+code"):  # the same bytes with evict_first stores
        L.tcqr_debug_pollute(ctypes.c_void_p(BIG.data_ptr()), ctypes.c_int64(BIG.numel()), 1)
    if kind in ("nf", "nf+code"):  # the same kernel with plain stores
        L.tcqr_debug_pollute(ctypes.c_void_p(BIG.data_ptr()), ctypes.c_int64(BIG.numel()), 0)
    if kind in ("code", "both", "ef+code", "nf+code"):
        for _ in range(4):  # other kernels' code through every SM (little data)
            torch.matmul(SA, SB)
            torch.nn.functional.softmax(SA, dim=0)
            torch.cumsum(SA, 0)


def run(A, Q, R, reps=3, kind=None):
    out = []
    for _ in range(reps):
        dbg = torch.zeros(128 * 128, dtype=torch.int64, device="cuda")
        if kind:
            pollute(kind)
        L.tcqr_debug_leaf_timestamps_multi(ctypes.c_void_p(dbg.data_ptr()))
        tq.factor(A, Q, R)
        torch.cuda.synchronize()
        L.tcqr_debug_leaf_timestamps_multi(None)
        d = dbg.cpu().numpy().astype(np.int64).reshape(128, 128)
        out.append(d)
    return out


A = W.gaussian_cuda(m, n, 3)
Q = torch.empty_like(A)
R = torch.empty(n, n, device="cuda").t()
for _ in range(2):
    tq.factor(A, Q, R)
ds = run(A, Q, R)
nl = n // 128
ph = np.array([np.diff(d[i, :K]) / 1000.0 for d in ds for i in range(nl)])  # (reps * nl, K - 1)
idx = np.array([i for _ in ds for i in range(nl)])
even, odd = ph[idx % 2 == 0], ph[idx % 2 == 1]
A1 = W.gaussian_cuda(m, 128, 3)
Q1 = torch.empty_like(A1)
R1 = torch.empty(128, 128, device="cuda").t()
for _ in range(3):
    tq.factor(A1, Q1, R1)
iso = np.array([np.diff(d[0, :K]) / 1000.0 for d in run(A1, Q1, R1, 5)])
for kind in ("data", "code", "both", "ef+code", "nf+code"):
    pk = np.median(np.array([np.diff(d[0, :K]) / 1000.0 for d in run(A1, Q1, R1, 7, kind)]), 0)
    print(f"isolated after {kind} pollution: total {pk.sum():.1f} us; " +
          ", ".join(f"{names[j]} {pk[j]:.2f}" for j in (1, 5, 6, 7, 8, 12, 16, 17)))
me, mo, mi = np.median(even, 0), np.median(odd, 0), np.median(iso, 0)
print(f"total (us): left leaves {me.sum():.1f}, right leaves {mo.sum():.1f}, isolated {mi.sum():.1f}")
print(f"  {'phase':16s} {'left':>8s} {'right':>8s} {'isolated':>8s}")
for j, nm in enumerate(names):
    print(f"  {nm:16s} {me[j]:8.2f} {mo[j]:8.2f} {mi[j]:8.2f}")
