"""Sweep the restart-pass tolerance tol2 (reading R-A12) on the parity cases (development aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
from oracle.cgls import oracle_lls
tq.init(0)
cases = [(2048, 512, "arithmetic", 1e6), (2048, 256, "cluster", 1e6), (2000, 300, "geometric", 1e3),
         (4096, 1024, "geometric", 1e4), (4096, 512, "arithmetic", 1e6), (4096, 512, "cluster2", 1e4)]
data = []
for (m, n, kind, cond) in cases:
    a = W.make_matrix(kind, m, n, seed=m + n, cond=cond)
    b, xt = W.consistent_rhs(a, seed=n)
    xo, _ = oracle_lls(a.astype(np.float64), b)
    data.append((a, b, xo))
for tol2 in (1e-6, 1e-8, 1e-10):
    tq.set_config(tol2=tol2)
    for (m, n, kind, cond), (a, b, xo) in zip(cases, data):
        x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), tol=1e-10, maxit=4000)
        x = x.cpu().numpy()
        print("tol2 %.0e %s %g %dx%d err %.2e it %d/%d reason %d conv %d" % (
            tol2, kind, cond, m, n, np.linalg.norm(x - xo) / np.linalg.norm(xo), info["iterations_pass1"],
            info["iterations"], info["stop_reason"], info["converged"]), flush=True)
