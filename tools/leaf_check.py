"""GPU check of the whole-leaf kernel (k_leaf.cu) against the per-panel path and the oracle gates,
plus a timing comparison of the two paths (tools/, not a test)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1912_05508_b200 as tq
import workloads as W
from oracle.metrics import backward_error_f, orthogonality_f, r_rel_error
from oracle.qr import rgs

tq.init(0)
for (m, n, cut) in [(1024, 128, 128), (1000, 100, 128), (777, 96, 64), (4100, 300, 64), (2048, 512, 128),
                    (1024, 128, 32), (300, 300, 128), (16384, 1024, 128)]:
    a = W.gaussian(m, n, seed=m + n)
    out = {}
    for lk in (0, 1):
        tq.set_config(cutoff=cut, leaf_kernel=lk)
        A = tq.to_device_colmajor(a)
        Q, R = tq.factor(A)
        torch.cuda.synchronize()
        out[lk] = (Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64))
    _, r_o = rgs(a.astype(np.float64)) if m * n <= 4100 * 1024 else (None, None)
    for lk in (0, 1):
        q, r = out[lk]
        msg = f"m={m} n={n} c={cut} leaf={lk}: be {backward_error_f(a, q, r):.2e} orth {orthogonality_f(q):.2e}"
        if r_o is not None:
            msg += f" Rerr {r_rel_error(r, r_o):.2e}"
        msg += f" triu {np.array_equal(r, np.triu(r))} diag>0 {bool(np.all(np.diag(r) > 0))}"
        print(msg, flush=True)
# planted
for (m, n, cut) in [(1024, 128, 32), (1024, 128, 128), (4096, 512, 128), (1024, 256, 64)]:
    a, qt, r0 = W.planted_hadamard(m, n, seed=201)
    tq.set_config(cutoff=cut, leaf_kernel=1)
    Q, R = tq.factor(tq.to_device_colmajor(a))
    torch.cuda.synchronize()
    q = Q.cpu().numpy().astype(np.float64); r = R.cpu().numpy().astype(np.float64)
    print(f"planted m={m} n={n} c={cut}: R exact {np.array_equal(r, r0)} Q exact {np.array_equal(q, qt)}"
          f" maxdiff R {np.abs(r - r0).max():.2e} Q {np.abs(q - qt).max():.2e}", flush=True)
# timing at config 3
m, n = 32768, 16384
A = torch.randn(n, m, device="cuda").t()
Q = torch.empty_like(A); R = torch.empty(n, n, device="cuda").t()
for lk in (0, 1):
    tq.set_config(leaf_kernel=lk)
    for _ in range(2):
        tq.factor(A, Q, R)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tq.factor(A, Q, R)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"config3 leaf={lk}: {ms:.2f} ms  {(2*m*n*n - 2*n**3/3)/ms/1e9:.1f} TFLOP/s", flush=True)
    tq.profile_enable(True); tq.factor(A, Q, R); cl = tq.profile_read(); tq.profile_enable(False)
    print({k: (round(v["ms"], 2), v["launches"]) for k, v in cl.items() if v["launches"]}, flush=True)
