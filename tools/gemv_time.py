"""Time the K5 GEMVs (A v and A' v) through the component entry point at configs[3]'s shape
(tools/, not a test)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
tq.init(0)
m, n = 32768, 8192
A = torch.randn((n, m), device="cuda").t()
vt = torch.randn(m, device="cuda", dtype=torch.float64)
vn = torch.randn(n, device="cuda", dtype=torch.float64)
for trans, v in ((False, vn), (True, vt)):
    for _ in range(3):
        tq.gemv(A, v, trans)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y = tq.gemv(A, v, trans)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    ref = (A.double().t() @ v) if trans else (A.double() @ v)
    print(f"trans={trans}: {ms*1e3:.1f} us ({4*m*n/ms/1e6:.0f} GB/s), rel err {float(torch.linalg.norm(y-ref)/torch.linalg.norm(ref)):.2e}")
