"""Phase timestamps (us) of the fused FP32 projection inside a 32768 x 128 factorization."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
tq.set_config(use_graphs=0)
L = tq.lib()
L.tcqr_debug_proj_timestamps.argtypes = [ctypes.c_void_p]
for m in (32768, 8192):
    dbg = torch.zeros(16, dtype=torch.int64, device="cuda")
    L.tcqr_debug_proj_timestamps(ctypes.c_void_p(dbg.data_ptr()))
    A = W.gaussian_cuda(m, 64, 3)    # w=64 leaf: one 32x32 projection
    for _ in range(2):
        tq.factor(A)
    torch.cuda.synchronize()
    d = dbg.cpu().numpy()
    print(m, "w=64", [round((int(v) - int(d[0])) / 1000, 2) for v in d[:9]])
    A = W.gaussian_cuda(m, 128, 3)   # last projection of a 128 leaf is 32x32; the middle one 64x64
    for _ in range(2):
        tq.factor(A)
    torch.cuda.synchronize()
    d = dbg.cpu().numpy()
    print(m, "w=128(last)", [round((int(v) - int(d[0])) / 1000, 2) for v in d[:9]])
L.tcqr_debug_proj_timestamps(None)
