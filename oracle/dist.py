"""Row-partitioned (1-D block-row) decomposition of the same algorithm, over a communicator.

The paper runs on one GPU; north_star row-partitions the tall matrix across
P GPUs. In exact arithmetic the decomposition below returns the same (Q, R) and x as
``oracle.qr.rgs`` / ``oracle.cgls``:

* R12 = sum_r Q1^(r)' A2^(r)                         (Alg. 2 line 8 as an allreduce)
* panel: TSQR = Eq. (6) with the ranks as the top tree level (reading R-A26):
  local CAQR -> allgather of the P local R's -> every rank factors the stack redundantly ->
  Q^(r) <- Q^(r) Q_stack[r]
* CGLS: A'r and ||q||^2 are allreduced; R, x, s, p, t are replicated (Alg. 5).

``comm`` needs .rank, .size, .allreduce_sum(ndarray) -> ndarray, .allgather(ndarray) -> list.
"""
from __future__ import annotations

import numpy as np

from .qr import caqr, mgs, split_point, Breakdown
from .cgls import CglsInfo, _rinv, _rinvt


class SelfComm:
    rank, size = 0, 1

    def allreduce_sum(self, x):
        return np.array(x, dtype=np.float64, copy=True)

    def allgather(self, x):
        return [np.array(x, dtype=np.float64, copy=True)]


def dist_panel(a_loc, comm, br=256, col0=0):
    """TSQR panel: local Eq. (6) CAQR, then the rank level of the tree."""
    w = a_loc.shape[1]
    if comm.size == 1:
        return caqr(a_loc, br, col0=col0)
    q_loc, r_loc = caqr(a_loc, br, col0=col0, _top=False)
    stack = np.vstack(comm.allgather(r_loc))
    qst, r = caqr(stack, br, col0=col0, _top=True)
    return q_loc @ qst[comm.rank * w:(comm.rank + 1) * w], r


def dist_rgs(a_loc, comm, pw=32, br=256, col0=0):
    """Alg. 2 on this rank's rows; exact (FP64) products."""
    a_loc = np.array(a_loc, dtype=np.float64, copy=True)
    w = a_loc.shape[1]
    if w <= pw:
        return dist_panel(a_loc, comm, br, col0)
    h = split_point(w)
    q1, r11 = dist_rgs(a_loc[:, :h], comm, pw, br, col0)
    r12 = comm.allreduce_sum(q1.T @ a_loc[:, h:])
    q2, r22 = dist_rgs(a_loc[:, h:] - q1 @ r12, comm, pw, br, col0 + h)
    r = np.zeros((w, w))
    r[:h, :h], r[:h, h:], r[h:, h:] = r11, r12, r22
    return np.hstack([q1, q2]), r


def dist_pcgls(a_loc, b_loc, r, comm, tol=1e-10, maxit=200, window=10, floor=1e-11, sref=None):
    """Corrected Alg. 5 with row-partitioned A, b, residual (same stop rule as oracle.cgls)."""
    a_loc = np.asarray(a_loc, dtype=np.float64)
    n = a_loc.shape[1]
    x = np.zeros(n)
    res = np.array(b_loc, dtype=np.float64, copy=True)
    s = _rinvt(r, comm.allreduce_sum(a_loc.T @ res))
    p = s.copy()
    gamma = float(s @ s)
    s0 = np.sqrt(gamma)
    info = CglsInfo(s0=s0)
    sref = s0 if sref is None else sref
    if s0 == 0.0:
        info.converged, info.reason = True, "zero_rhs"
        return x, info
    best, xbest, since = s0, x.copy(), 0
    for k in range(1, maxit + 1):
        t = _rinv(r, p)
        q = a_loc @ t
        delta = float(comm.allreduce_sum(np.array([q @ q]))[0])
        alpha = gamma / delta
        x = x + alpha * t
        res = res - alpha * q
        s = _rinvt(r, comm.allreduce_sum(a_loc.T @ res))
        ns = float(np.sqrt(s @ s))
        info.iterations = k
        info.history.append(ns / s0)
        if ns < best:
            best, xbest, since = ns, x.copy(), 0
        else:
            since += 1
        if ns / s0 <= tol:
            info.converged, info.reason, info.final_rel = True, "tol", ns / s0
            return x, info
        if best < floor * sref and since >= window:
            info.converged, info.reason, info.final_rel = True, "stagnation", best / s0
            return xbest, info
        gamma1, gamma = gamma, ns * ns
        p = s + (gamma / gamma1) * p
    info.final_rel = best / s0
    return xbest, info


__all__ = ["SelfComm", "dist_panel", "dist_rgs", "dist_pcgls", "Breakdown", "mgs"]
