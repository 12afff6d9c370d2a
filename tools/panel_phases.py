"""Phase timestamps (globaltimer, us) of one fused CAQR panel launch (debug hook of libtcqr)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1912_05508_b200 as tq  # noqa: E402
import workloads as W  # noqa: E402

tq.init(0)
L = tq.lib()
L.tcqr_debug_panel_timestamps.argtypes = [ctypes.c_void_p]
for m, br in ((32768, 1024), (32768, 256), (8192, 1024), (1024, 1024)):
    dbg = torch.zeros(128, dtype=torch.int64, device="cuda")
    L.tcqr_debug_panel_timestamps(ctypes.c_void_p(dbg.data_ptr()))
    X = W.gaussian_cuda(m, 32, 3)
    for _ in range(3):
        dbg.zero_()
        tq.panel_qr(X.clone(), br=br)
    torch.cuda.synchronize()
    d = dbg.cpu().numpy()
    t0 = int(d[0])
    print(m, br, {i: round((int(v) - t0) / 1000.0, 2) for i, v in enumerate(d[:32]) if v})
    l1 = [int(v) for v in d[32:64] if v]
    l2 = [int(v) for v in d[64:96] if v]
    print("  level-1 step us:", [round((b - a) / 1000, 2) for a, b in zip(l1, l1[1:])])
    print("  stack   step us:", [round((b - a) / 1000, 2) for a, b in zip(l2, l2[1:])])
L.tcqr_debug_panel_timestamps(None)
