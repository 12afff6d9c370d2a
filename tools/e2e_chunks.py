"""e2e (tcqr_factor_host, pinned host A/Q/R) at config 3 for several stream chunk divisors
(TCQR_STREAM_DIV is read once per process: one process per value)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, "%s")
import paper_1912_05508_b200 as tq, workloads as W
tq.init(0)
m, n = 32768, 16384
A = W.gaussian_cuda(m, n, 4)
import ctypes
P = ctypes.c_void_p
ha = torch.empty((n, m), dtype=torch.float32, pin_memory=True); ha.copy_(A.t())
hq = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
hr = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
del A; torch.cuda.empty_cache()
L = tq.lib()
def run():
    assert L.tcqr_factor_host(m, n, P(ha.data_ptr()), m, P(hq.data_ptr()), P(hr.data_ptr())) == 0
for _ in range(2): run()
s = torch.cuda.current_stream(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(s)
for _ in range(3): run()
e1.record(s); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"div=%s e2e {ms:.1f} ms {(2*m*n*n - 2/3*n**3)/ms/1e9:.1f} TFLOP/s", flush=True)
'''
for d in (sys.argv[1:] or ["8", "16", "32", "64"]):
    env = dict(os.environ, TCQR_STREAM_DIV=d)
    subprocess.run([sys.executable, "-c", code % (ROOT, d)], env=env)
