"""Run `--reps` tcqr_factor calls of a bench workload (for ncu / launch lists); no timing output."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16384)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--graphs", type=int, default=1)
ap.add_argument("--cutoff", type=int, default=128)
a = ap.parse_args()

import torch  # noqa: E402
import paper_1912_05508_b200 as tq  # noqa: E402
import workloads as W  # noqa: E402

tq.init(0)
tq.set_config(cutoff=a.cutoff, use_graphs=a.graphs)
A = W.gaussian_cuda(a.m, a.n, 4)
Q = tq.colmajor_empty(a.m, a.n)
R = tq.colmajor_empty(a.n, a.n)
for _ in range(a.reps):
    tq.factor(A, Q, R)
torch.cuda.synchronize()
print("done", a.m, a.n, a.reps)
