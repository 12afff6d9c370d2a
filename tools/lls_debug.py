"""Print LLS info and x error for a few spectra / block-row settings (development aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
from oracle.cgls import oracle_lls
tq.init(0)
for br in (256, 1024):
    tq.set_config(panel_rows=br)
    for (m, n, kind, cond) in [(2048, 512, "arithmetic", 1e6), (2048, 256, "cluster", 1e6), (1024, 128, "gaussian", 1)]:
        a = W.make_matrix(kind, m, n, seed=m + n, cond=cond)
        b, xt = W.consistent_rhs(a, seed=n)
        x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), tol=1e-10, maxit=2000)
        xo, _ = oracle_lls(a.astype(np.float64), b)
        x = x.cpu().numpy()
        print(br, m, n, kind, cond, "err_vs_oracle %.2e" % (np.linalg.norm(x - xo) / np.linalg.norm(xo)),
              "err_vs_true %.2e" % (np.linalg.norm(x - xt) / np.linalg.norm(xt)), info)
