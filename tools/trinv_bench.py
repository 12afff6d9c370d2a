"""Time the FP64 explicit triangular inverse (tcqr_trinv) at n = 4096 / 8192 / 16384."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
tq.init(0)
for n in (4096, 8192, 16384):
    R = torch.triu(torch.randn(n, n, device="cuda")) + n * torch.eye(n, device="cuda")
    Rc = R.t().contiguous().t()
    tq.trinv(Rc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        tq.trinv(Rc)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"n={n}: trinv {dt*1e3:.2f} ms, {n**3/3/dt/1e12:.2f} TFLOP/s (n^3/3)")
