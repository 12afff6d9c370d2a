"""One TN and one NN GEMM at the recursion shape h = w2 = H (env), m = 32768 (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
tq.init(0)
m = int(os.environ.get("M", 32768)); h = int(os.environ.get("H", 1024)); w2 = h
A1 = torch.randn((h, m), device="cuda", dtype=torch.float16).t()
A2 = torch.randn((w2, m), device="cuda", dtype=torch.float16).t()
B = torch.randn((w2, h), device="cuda", dtype=torch.float16).t()
C = torch.randn((w2, m), device="cuda", dtype=torch.float32).t()
for _ in range(3):
    tq.gemm_tn(A1, A2)
    tq.gemm_nn_update(C, A1, B)
torch.cuda.synchronize()
