"""NEXT-4 (FP16 split) accuracy and cost against the plain FP16 path: QR metrics vs the FP64
oracle, LLS iterations at geometric kappa 1e5 / 1e6, and the config-3 factor time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1912_05508_b200 as tq
import workloads as W
from oracle.cgls import oracle_lls
from oracle.metrics import backward_error_f, orthogonality_f, r_rel_error, x_rel_error
from oracle.qr import rgs

tq.init(0)
for kind, cond in [("gaussian", 1), ("geometric", 1e2), ("arithmetic", 1e3), ("geometric", 1e3),
                   ("geometric", 1e5)]:
    a = W.make_matrix(kind, 4096, 1024, seed=31, cond=cond)
    _, r_o = rgs(a.astype(np.float64))
    A = tq.to_device_colmajor(a)
    for split in (0, 1):
        tq.set_config(fp16_split=split)
        Q, R = tq.factor(A)
        q = Q.cpu().numpy().astype(np.float64)
        r = R.cpu().numpy().astype(np.float64)
        print(f"{kind:10s} {cond:7.0e} split={split}: backward {backward_error_f(a, q, r):.2e} "
              f"orth {orthogonality_f(q):.2e} R-err {r_rel_error(r, r_o):.2e}", flush=True)
for cond in (1e5, 1e6):
    a = W.spectrum_matrix(4096, 1024, "geometric", cond, seed=37)
    b, x_true = W.consistent_rhs(a, seed=38)
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    A = tq.to_device_colmajor(a)
    B = torch.from_numpy(b).cuda()
    for split, reorth in [(0, 0), (1, 0), (0, 1), (1, 1)]:
        tq.set_config(fp16_split=split, reorth=reorth)
        x, info = tq.lls_solve(A, B, tol=1e-10, maxit=3000)
        print(f"LLS geometric {cond:.0e} split={split} reorth={reorth}: iters {info['iterations']} "
              f"converged {info['converged']} x-err vs oracle {x_rel_error(x.cpu().numpy(), x_o):.2e}",
              flush=True)
m, n = 32768, 16384
A = W.gaussian_cuda(m, n, 4)
Q = torch.empty_like(A)
R = torch.empty(n, n, device="cuda").t()
for split in (0, 1):
    tq.set_config(fp16_split=split)
    for _ in range(2):
        tq.factor(A, Q, R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tq.factor(A, Q, R)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"cfg3 split={split}: {ms:.1f} ms, {(2 * m * n * n - 2 / 3 * n ** 3) / ms / 1e9:.1f} TFLOP/s", flush=True)
tq.set_config()
