"""Time K3 (TN split-K) and K4 (NN update) at the recursion shapes of config 3 via the C ABI."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1912_05508_b200 as tq
tq.init(0)
m = int(os.environ.get("M", 32768))
shapes = [int(x) for x in os.environ.get("H", "8192,4096,2048,1024,512,256,128,64").split(",")]
print("m", m)
for h in shapes:
    w2 = h
    A1 = torch.randn((h, m), device="cuda", dtype=torch.float16).t()
    A2 = torch.randn((w2, m), device="cuda", dtype=torch.float16).t()
    B = torch.randn((w2, h), device="cuda", dtype=torch.float16).t()
    C = torch.randn((w2, m), device="cuda", dtype=torch.float32).t()
    for _ in range(2):
        tq.gemm_tn(A1, A2)
        tq.gemm_nn_update(C, A1, B)
    reps = max(1, min(20, int(2e12 / (2 * m * h * w2))))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(reps):
        tq.gemm_tn(A1, A2)
    e[1].record()
    for _ in range(reps):
        tq.gemm_nn_update(C, A1, B)
    e[2].record()
    torch.cuda.synchronize()
    fl = 2.0 * m * h * w2
    t1 = e[0].elapsed_time(e[1]) / reps
    t2 = e[1].elapsed_time(e[2]) / reps
    nb = 2.0 * m * h + 2.0 * h * w2 + 8.0 * m * w2
    tb = 2.0 * m * (h + w2)
    print(f"h=w2={h:5d}: TN {t1*1e3:8.1f} us {fl/t1/1e9:7.1f} TF/s {tb/t1/1e6:7.0f} GB/s | "
          f"NN {t2*1e3:8.1f} us {fl/t2/1e9:7.1f} TF/s {nb/t2/1e6:7.0f} GB/s")
