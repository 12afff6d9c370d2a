"""Brute-force Householder QR / least squares, written out in loops (oracle cross-check).

Used only on tiny inputs to pin ``oracle.qr`` (R uniqueness under diag(R) > 0, reading R-A9)
and ``oracle.cgls`` (x* of Eq. (2), via Eq. (4) x* = R^-1 Q' b,
PAPER.md:183-185, Alg. 1). Householder QR is the classical algorithm the
paper compares against; here it is only a checker.
"""
from __future__ import annotations

import numpy as np


def householder_qr(a: np.ndarray):
    """Thin QR by explicit reflectors, sign-normalized so that diag(R) > 0."""
    r = np.array(a, dtype=np.float64, copy=True)
    m, n = r.shape
    qfull = np.eye(m)
    for k in range(n):
        x = r[k:, k].copy()
        nx = 0.0
        for v in x:
            nx += v * v
        nx = np.sqrt(nx)
        if nx == 0.0:
            continue
        alpha = -nx if x[0] >= 0 else nx
        v = x
        v[0] -= alpha
        vn = np.sqrt(np.dot(v, v))
        if vn == 0.0:
            continue
        v /= vn
        for j in range(n):                       # R[k:, j] -= 2 v (v' R[k:, j])
            r[k:, j] -= 2.0 * v * np.dot(v, r[k:, j])
        for i in range(m):                       # Q[i, k:] -= 2 (Q[i, k:] v) v'
            qfull[i, k:] -= 2.0 * np.dot(qfull[i, k:], v) * v
    q = qfull[:, :n]
    r = np.triu(r[:n, :])
    d = np.where(np.diag(r) < 0, -1.0, 1.0)
    return q * d, (r.T * d).T


def back_substitution(r: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Solve R x = y for upper-triangular R by explicit back substitution."""
    n = r.shape[0]
    x = np.zeros(n)
    for i in range(n - 1, -1, -1):
        s = y[i]
        for j in range(i + 1, n):
            s -= r[i, j] * x[j]
        x[i] = s / r[i, i]
    return x


def qr_solve(q: np.ndarray, r: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Alg. 1 lines 3-4 (Eq. (4)): x = R^-1 (Q' b) for any
    thin QR (Q m x n, R n x n upper triangular), in FP64 -- the direct QR solve of NEXT-2."""
    q = np.asarray(q, dtype=np.float64)
    return back_substitution(np.asarray(r, dtype=np.float64), q.T @ np.asarray(b, dtype=np.float64))


def householder_lls(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Alg. 1 with Householder factors: x = R^-1 (Q' b)."""
    q, r = householder_qr(a)
    return qr_solve(q, r, b)


def normal_equations_lls(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Eq. (3): A'A x = A'b by Cholesky, tiny well-conditioned inputs only."""
    a = np.asarray(a, dtype=np.float64)
    g = a.T @ a
    l = np.linalg.cholesky(g)
    y = np.linalg.solve(l, a.T @ b)
    return np.linalg.solve(l.T, y)
