"""Kernel-class profile of one tall factorization (NEXT-3 4194304 x 128 by default, or M/N from
the environment): warm call, then one profiled call (tools/, not a test)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
m, n = int(os.environ.get("M", 4194304)), int(os.environ.get("N", 128))
A = W.gaussian_cuda(m, n, 9)
Q = tq.colmajor_empty(m, n)
R = tq.colmajor_empty(n, n)
for _ in range(2):
    tq.factor(A, Q, R)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); tq.factor(A, Q, R); e1.record(); torch.cuda.synchronize()
print(f"{m}x{n}: {e0.elapsed_time(e1):.2f} ms")
tq.profile_enable(True)
tq.factor(A, Q, R)
prof = tq.profile_read()
tq.profile_enable(False)
for k, v in prof.items():
    if v["launches"]:
        print(f"  {k:14s} {v['ms']:8.3f} ms  launches {v['launches']:5d}  {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s")
