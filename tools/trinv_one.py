"""One FP64 triangular inverse at n = 8192 (the ncu target for the trinv kernels; tools/, not a test)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_05508_b200 as tq
tq.init(0)
n = int(os.environ.get("N", 8192))
R = torch.triu(torch.randn(n, n, device="cuda")) + n * torch.eye(n, device="cuda")
Rc = R.t().contiguous().t()
for _ in range(2):
    tq.trinv(Rc)
torch.cuda.synchronize()
print("done")
