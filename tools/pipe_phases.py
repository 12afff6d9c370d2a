"""Timestamps (us) of the pipelined panel on a 32768 x 32 block: child-0 MGS end, root steps,
apply columns (debug hook tcqr_debug_panel_timestamps)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_panel_timestamps.argtypes = [ctypes.c_void_p]
verbose = "-v" in sys.argv
for m in (32768, 4100):
    dbg = torch.zeros(256, dtype=torch.int64, device="cuda")
    L.tcqr_debug_panel_timestamps(ctypes.c_void_p(dbg.data_ptr()))
    X = W.gaussian_cuda(m, 32, 3)
    res = []
    for _ in range(5):
        dbg.zero_()
        Xq, R = tq.panel_qr(X.clone(), br=1024)
        torch.cuda.synchronize()
        d = dbg.cpu().numpy().astype(np.int64)
        t0 = d[0]
        f = lambda v: round((int(v) - int(t0)) / 1000, 2) if v else None
        res.append((f(d[1]), f(d[64]), f(d[95]), f(d[63])))
    L.tcqr_debug_panel_timestamps(None)
    print(m, "child0 mgs end / root step0 / root step31 / apply end (us):", res[-3:])
    if verbose:
        print("  root steps", [f(v) for v in d[64:96]])
        print("  apply cols", [f(v) for v in d[32:64]])
    q = Xq.cpu().numpy().astype(np.float64); r = R.cpu().numpy().astype(np.float64)
    a = X.cpu().numpy().astype(np.float64)
    print("  backward", np.linalg.norm(a - q @ r) / np.linalg.norm(a), "orth", np.linalg.norm(q.T @ q - np.eye(32)))
