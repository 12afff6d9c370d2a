"""Run one 32768 x 128 factorization (its FP32 projections are the ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
tq.set_config(use_graphs=0)
A = W.gaussian_cuda(int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 128, 3)
for _ in range(2):
    tq.factor(A)
torch.cuda.synchronize()
