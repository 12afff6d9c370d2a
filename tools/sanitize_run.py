"""Small invocations of every cooperative / cluster / CTA-pair kernel for compute-sanitizer
(memcheck, racecheck, synccheck): the whole-leaf kernel K2L, the pipelined and fused CAQR panels,
the FP32 projection kernel, the tensor-core GEMMs (1-CTA and CTA-pair), the cluster cast, the
CGLS kernels and the virtual-rank collectives.  tools/, not a test."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
tq.set_config(use_graphs=0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "leaf"):
    a = W.gaussian(2048, 256, seed=1)                       # K2L leaves + 1-CTA TC GEMMs + cast
    tq.factor(tq.to_device_colmajor(a))
if which in ("all", "panel"):
    X = tq.to_device_colmajor(W.gaussian(8192, 32, seed=2))  # pipelined CAQR panel (8 x 1024 rows)
    tq.panel_qr(X, br=1024)
    X = tq.to_device_colmajor(W.gaussian(8192, 32, seed=3))  # fused / level CAQR (256-row blocks)
    tq.panel_qr(X, br=256)
if which in ("all", "proj"):
    tq.set_config(use_graphs=0, leaf_kernel=0)              # FP32 projection kernel + panels
    tq.factor(tq.to_device_colmajor(W.gaussian(4096, 128, seed=4)))
    tq.set_config(use_graphs=0)
if which in ("all", "gemm"):
    m, h = 4096, 512                                        # CTA-pair TN / NN GEMMs
    A1 = torch.randn((h, m), device="cuda", dtype=torch.float16).t()
    A2 = torch.randn((h, m), device="cuda", dtype=torch.float16).t()
    B = torch.randn((h, h), device="cuda", dtype=torch.float16).t()
    C = torch.randn((h, m), device="cuda", dtype=torch.float32).t()
    tq.gemm_tn(A1, A2)
    tq.gemm_nn_update(C, A1, B)
if which in ("all", "cgls"):
    a = W.gaussian(2048, 128, seed=5)
    b, _ = W.consistent_rhs(a, seed=6)
    tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), tol=1e-10, maxit=50)
if which in ("all", "vranks"):
    import ctypes
    a = W.gaussian(2048, 256, seed=7)
    A = tq.to_device_colmajor(a)
    Qs = [tq.colmajor_empty(1024, 256) for _ in range(2)]
    Rs = [tq.colmajor_empty(256, 256) for _ in range(2)]
    torch.cuda.synchronize()

    def fn(r):
        l = tq.lib()
        return l.tcqr_factor(1024, 256, ctypes.c_void_p(A.data_ptr() + 4 * 1024 * r), 2048,
                             ctypes.c_void_p(Qs[r].data_ptr()), ctypes.c_void_p(Rs[r].data_ptr()))

    assert tq.run_virtual_ranks(2, fn, slot_bytes=1 << 20) == [0, 0]
torch.cuda.synchronize()
print("sanitize_run", which, "done")
