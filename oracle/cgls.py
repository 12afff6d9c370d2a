"""R-preconditioned CGLS, oracle side (plain numpy/scipy, float64).

Alg. 5 "CGLS with RMGSQR as Preconditioner", with the three printed typos
corrected (reading R-A10):
  (i)   line 15 ``alpha = gamma/gamma1``  ->  alpha = gamma/delta  (gamma1 undefined at k=1;
        PAPER.md:552);
  (ii)  line 7  ``s = A'*r``              ->  s0 = R^-T (A' r)     (matches line 18's inv(R');
        PAPER.md:544);
  (iii) line 16 ``x = x + alpha*p``       ->  x = x + alpha * R^-1 p.
Line numbers follow the Verbatim numbering (line 1 = PAPER.md:538).
The convergence test "is omitted"; reading R-A11 defines it as
||s_k|| / ||s_0|| <= tol plus a windowed stagnation stop, and R-A12 the FP64 target as one
restart from the true residual with tol2 = 1e-6.

R enters only through triangular solves (Alg. 5 lines 12 and 18: inv(R)*p, inv(R')*v);
scipy.linalg.solve_triangular is the library primitive for those two steps.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import solve_triangular


@dataclass
class CglsInfo:
    iterations: int = 0
    converged: bool = False
    reason: str = "maxit"          # "tol" | "stagnation" | "maxit" | "zero_rhs"
    s0: float = 0.0
    final_rel: float = 0.0
    history: list = field(default_factory=list)   # ||s_k|| / ||s_0||


def _rinv(r, v):
    return solve_triangular(r, v, lower=False)


def _rinvt(r, v):
    return solve_triangular(r, v, lower=False, trans="T")


def pcgls(a, b, r, tol=1e-10, maxit=200, window=10, floor=1e-11, sref=None):
    """Corrected Alg. 5 from x0 = 0. Returns (x, CglsInfo)."""
    a = np.asarray(a, dtype=np.float64)
    r_fac = np.asarray(r, dtype=np.float64)
    m, n = a.shape
    x = np.zeros(n)                                   # line 5
    res = np.array(b, dtype=np.float64, copy=True)    # line 6: r = b - A*x = b
    s = _rinvt(r_fac, a.T @ res)                      # line 7 (R-A10 ii)
    p = s.copy()                                      # line 8
    gamma = float(s @ s)                              # lines 9-10
    s0 = np.sqrt(gamma)
    info = CglsInfo(s0=s0)
    if sref is None:
        sref = s0
    if s0 == 0.0:
        info.converged, info.reason = True, "zero_rhs"
        return x, info
    best, xbest, since = s0, x.copy(), 0
    for k in range(1, maxit + 1):                     # line 11
        t = _rinv(r_fac, p)                           # line 12: inv(R)*p
        q = a @ t                                     # line 12: A*(...)
        delta = float(q @ q)                          # line 14
        alpha = gamma / delta                         # line 15 (R-A10 i)
        x = x + alpha * t                             # line 16 (R-A10 iii)
        res = res - alpha * q                         # line 17
        s = _rinvt(r_fac, a.T @ res)                  # line 18
        ns = float(np.sqrt(s @ s))                    # line 20
        info.iterations = k
        info.history.append(ns / s0)
        if ns < best:
            best, xbest, since = ns, x.copy(), 0
        else:
            since += 1
        if ns / s0 <= tol:                            # R-A11 tolerance stop
            info.converged, info.reason, info.final_rel = True, "tol", ns / s0
            return x, info
        if best < floor * sref and since >= window:   # R-A11 stagnation stop
            info.converged, info.reason, info.final_rel = True, "stagnation", best / s0
            return xbest, info
        gamma1 = gamma                                # line 21
        gamma = ns * ns                               # line 22
        beta = gamma / gamma1                         # line 23
        p = s + beta * p                              # line 24
    info.final_rel = best / s0
    return xbest, info


def lls_refine(a, b, r, tol=1e-10, maxit=200, target="fp64", tol2=1e-6, window=10, floor=1e-11):
    """The LLS rule of R-A12 on a given preconditioner R: pass 1 with ``tol``; for the FP64
    target one restart from the true residual r = b - A x with tol2, stagnation floor relative
    to pass 1's s0. Returns (x, [info1, info2?])."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    x1, i1 = pcgls(a, b, r, tol, maxit, window, floor)
    if target != "fp64" or i1.reason == "zero_rhs":
        return x1, [i1]
    res = b - a @ x1
    dx, i2 = pcgls(a, res, r, tol2, maxit, window, floor, sref=i1.s0)
    return x1 + dx, [i1, i2]


def oracle_lls(a, b, maxit=50):
    """The oracle's own x* (SURVEY.md §8c.2 item 5): FP64 RGS R, then one corrected-PCGLS pass
    with tol 1e-15 and the stagnation stop. With an exact R, kappa(A R^-1) ~ 1."""
    from .qr import rgs
    _, r = rgs(np.asarray(a, dtype=np.float64))
    x, i = pcgls(a, b, r, tol=1e-15, maxit=maxit, window=10, floor=1e-11)
    return x, i


def cgls_literal(a, b, r, iters=10):
    """Alg. 5 EXACTLY as printed (incl. the typos), for the R-A10 test that
    shows the literal text does not converge. gamma1 is taken as gamma at k=1."""
    a = np.asarray(a, dtype=np.float64)
    x = np.zeros(a.shape[1])
    res = np.array(b, dtype=np.float64)
    s = a.T @ res
    p = s.copy()
    gamma = float(s @ s)
    gamma1 = gamma
    xs = []
    for _ in range(iters):
        if not np.all(np.isfinite(p)):
            xs.append(x.copy())
            continue
        q = a @ _rinv(r, p)
        delta = float(q @ q)  # noqa: F841  (computed but unused in the printed line 14)
        alpha = gamma / gamma1
        x = x + alpha * p
        res = res - alpha * q
        s = _rinvt(r, a.T @ res)
        ns = float(np.sqrt(s @ s))
        gamma1 = gamma
        gamma = ns * ns
        beta = gamma / gamma1
        p = s + beta * p
        xs.append(x.copy())
    return xs
