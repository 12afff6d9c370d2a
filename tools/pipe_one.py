"""One pipelined-panel launch on a 32768 x 32 block (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
X = W.gaussian_cuda(32768, 32, 3)
for _ in range(3):
    tq.panel_qr(X.clone(), br=1024)
torch.cuda.synchronize()
