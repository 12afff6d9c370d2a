"""One config-5 factorization (262144 x 2048 Gaussian, BASELINE configs[4]): the ncu target for the
tall-panel path (panel_pipe_kernel) and the narrow casts (tools/, not a test)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
m, n = int(os.environ.get("M", 262144)), int(os.environ.get("N", 2048))
A = W.gaussian_cuda(m, n, 8)
Q = torch.empty_like(A)
R = torch.empty(n, n, device="cuda").t()
tq.set_config(use_graphs=0)
for _ in range(2):
    tq.factor(A, Q, R)
torch.cuda.synchronize()
print("done")
