"""Config-4 LLS (32768 x 8192 geometric kappa=1e4, b = A x_true): warm + timed solve, per-class
profile of one more solve."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
M, n = int(os.environ.get("M", 32768)), int(os.environ.get("N", 8192))
kappa = float(os.environ.get("KAPPA", 1e4))
A = W.spectrum_cuda(M, n, "geometric", kappa, 6)
g = torch.Generator(device="cuda"); g.manual_seed(106)
xt = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
b = A.to(torch.float64) @ xt
tq.set_config(reorth=int(os.environ.get("REORTH", 0)))
for it in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, info = tq.lls_solve(A, b, tol=1e-10, maxit=4000)
    e1.record(); torch.cuda.synchronize()
    err = float(torch.linalg.norm(x - xt) / torch.linalg.norm(xt))
    print(f"solve {it}: {e0.elapsed_time(e1):.1f} ms, err {err:.2e}, {info}")
tq.profile_enable(True)
x, info = tq.lls_solve(A, b, tol=1e-10, maxit=4000)
prof = tq.profile_read()
tq.profile_enable(False)
it = info["iterations"]
for k, v in prof.items():
    if v["launches"]:
        print(f"  {k:12s} {v['ms']:9.2f} ms  launches {v['launches']:6d}  per-iter {v['ms']/max(it,1)*1e3:8.1f} us  "
              f"{v['bytes']/max(v['ms'],1e-9)/1e6:8.1f} GB/s")
