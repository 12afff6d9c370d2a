"""The alternate kernel paths behind the library's tuning switches (environment variables read once
per process into function-local statics, so the in-process suite only ever sees the defaults):
each group runs in its own Python process and must pass the same oracle gates as the default path
(north_star tolerances vs oracle.qr.rgs) and the planted-Hadamard bitwise pin (P2).

  group "fallbacks": TCQR_CAST_CLUSTER=0 (one-CTA-per-column / split-row casts), TCQR_TC2=0 (no
      CTA-pair GEMMs), TCQR_LOOKAHEAD_W=0 (no look-ahead), TCQR_CAST_OVERLAP=0 (casts in line),
      TCQR_NN_PRE_ALL=0 (NN epilogue with NBUF - 1 C chunks in flight), TCQR_L2_EF=0 (no L2
      evict-first hints), TCQR_TRI_N_V4=0 (one row per thread in the CGLS M p partials); every
      group also solves a small LLS
  group "variants":  TCQR_CAST_V8=0 (4096-row cluster CTAs), TCQR_TC2_NN_MINK=256 (CTA-pair NN
      from K = 256), TCQR_TN_MINKB=1 (finest split-K), TCQR_NN_SHORTK=0 (no short-K NN),
      TCQR_LOOKAHEAD_W=1024 with TCQR_LA_SMS=2 (leaf-wide deferred look-ahead blocks),
      TCQR_L2_EF=15 (evict-first hints on every operand and C tile), TCQR_LEAF_RESERVE=0 (the leaf
      beside a look-ahead block takes every SM)
  group "host":      TCQR_CAST_COL_MIN=1 (per-column cast kernel at every width), TCQR_STREAM_DIV=4
      (coarse chunks of the streamed host factorization)
"""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
from oracle.metrics import backward_error_f, orthogonality_f, r_rel_error
from oracle.qr import rgs
tq.init(0)
a = W.gaussian(4096, 1024, seed=71)
Q, R = tq.factor(tq.to_device_colmajor(a))
q, r = Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
_, r_o = rgs(a.astype(np.float64))
assert backward_error_f(a, q, r) <= 5e-3 and orthogonality_f(q) <= 5e-2
assert r_rel_error(r, r_o) <= 1e-2
for cutoff in (128, 32):
    tq.set_config(cutoff=cutoff)
    ap, qt, r0 = W.planted_hadamard(1024, 256, seed=201)
    Q, R = tq.factor(tq.to_device_colmajor(ap))
    assert np.array_equal(R.cpu().numpy().astype(np.float64), r0), cutoff
    assert np.array_equal(Q.cpu().numpy().astype(np.float64), qt), cutoff
tq.set_config()
qh, rh = tq.factor_host(a)
assert r_rel_error(rh.astype(np.float64), r_o) <= 1e-2
# LLS (the CGLS GEMVs and triangular products of the variant): x within 1e-10 of x_true
al = W.gaussian(4096, 512, seed=72)
xt = np.random.default_rng(73).standard_normal(512)
Ad = tq.to_device_colmajor(al)
b = torch.from_numpy(al.astype(np.float64) @ xt).cuda()
x, info = tq.lls_solve(Ad, b, tol=1e-10, maxit=400)
assert np.linalg.norm(x.cpu().numpy() - xt) <= 1e-10 * np.linalg.norm(xt), info
print("ok")
"""

GROUPS = {
    "fallbacks": {"TCQR_CAST_CLUSTER": "0", "TCQR_TC2": "0", "TCQR_LOOKAHEAD_W": "0",
                  "TCQR_CAST_OVERLAP": "0", "TCQR_NN_PRE_ALL": "0", "TCQR_L2_EF": "0",
                  "TCQR_TRI_N_V4": "0"},
    "variants": {"TCQR_CAST_V8": "0", "TCQR_TC2_NN_MINK": "256", "TCQR_TN_MINKB": "1",
                 "TCQR_NN_SHORTK": "0", "TCQR_LOOKAHEAD_W": "1024", "TCQR_LA_SMS": "2",
                 "TCQR_L2_EF": "15", "TCQR_LEAF_RESERVE": "0"},
    "host": {"TCQR_CAST_COL_MIN": "1", "TCQR_STREAM_DIV": "4"},
}


@pytest.mark.parametrize("group", sorted(GROUPS))
def test_env_variant_paths(group):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **GROUPS[group])
    p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), (p.stdout[-2000:],
                                                                   p.stderr[-4000:])
