import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_step_clocks.argtypes = [ctypes.c_void_p]
d = torch.zeros(16, dtype=torch.int64, device="cuda")
print("rc", L.tcqr_debug_step_clocks(ctypes.c_void_p(d.data_ptr())))
X = W.gaussian_cuda(32768, 32, 3)
for _ in range(3):
    tq.panel_qr(X.clone(), br=1024)
torch.cuda.synchronize()
v = d.cpu().numpy()
for base in (0, 8):
    print("k=%d" % (0 if base == 0 else 5), [int(v[base + i] - v[base]) for i in range(5)])
L.tcqr_debug_step_clocks(None)
