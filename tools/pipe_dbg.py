import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
for m in (32768, 4100, 8192):
    X = W.gaussian_cuda(m, 32, 3)
    for it in range(3):
        Xq, R = tq.panel_qr(X.clone(), br=1024)
        torch.cuda.synchronize()
        a = X.cpu().numpy().astype(np.float64)
        r0 = np.linalg.qr(a, mode='r'); r0 *= np.sign(np.diag(r0))[:, None]
        r = R.cpu().numpy().astype(np.float64)
        e = np.abs(r - r0) / np.abs(r0).max()
        bad = np.argwhere(e > 1e-4)
        print(m, it, "maxerr", e.max(), "first bad (row,col)", bad[:6].tolist(), "nbad", len(bad))
