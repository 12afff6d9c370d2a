"""One m x 128 factorization (a single whole-leaf launch) repeated a few times: the ncu target
for the leaf kernel (tools/, not a test)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
A = W.gaussian_cuda(m, 128, 3)
Q = torch.empty_like(A)
R = torch.empty(128, 128, device="cuda").t()
tq.set_config(use_graphs=0)
for _ in range(4):
    tq.factor(A, Q, R)
torch.cuda.synchronize()
print("done")
