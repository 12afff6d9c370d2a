import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_panel_timestamps.argtypes = [ctypes.c_void_p]
dbg = torch.zeros(192, dtype=torch.int64, device="cuda")
L.tcqr_debug_panel_timestamps(ctypes.c_void_p(dbg.data_ptr()))
X = W.gaussian_cuda(32768, 32, 3)
for _ in range(3):
    dbg.zero_()
    tq.panel_qr(X.clone(), br=1024)
torch.cuda.synchronize()
d = dbg.cpu().numpy().astype(np.int64)
t0 = d[0]
print("d0", d[0], "d1", d[1] - t0)
print("root step", [(int(v) - t0) / 1000 for v in d[64:96]])
print("root after load", [(int(v) - t0) / 1000 if v else 0 for v in d[96:128]])
print("apply", [(int(v) - t0) / 1000 for v in d[32:64]])
