"""Recursive Gram-Schmidt QR, oracle side (plain numpy, float64).

Follows, in the paper's order and notation:

* ``mgs``   -- Alg. 4 "256x32 Modified Gram-Schmidt QR", PAPER.md:464-478 (lines 5-8 of the
  Verbatim: R(k,k)=norm(Q(:,k)); Q(:,k)=Q(:,k)/R(k,k); R(k,k+1:n)=Q(:,k)'*Q(:,k+1:n);
  Q(:,k+1:n)=Q(:,k+1:n)-Q(:,k)*R(k,k+1:n)).
* ``caqr``  -- the communication-avoiding panel, Eq. (6) steps 1-5, PAPER.md:403-462:
  split rows into br-row blocks (br=256 in the paper, :441-442), MGS each block, stack the
  R factors, factor the stack recursively "until the number of rows is below 256"
  (:455-456), multiply each local Q by its slice of the stack's Q (step 4, :453-455).
* ``rgs``   -- Alg. 2 "Recursive Modified Gram-Schmidt QR", PAPER.md:319-336 with the
  assembly of Eq. (5): recurse left, R12 = Q1'*A2 (line 8),
  recurse on A2 - Q1*R12 (line 9), Q=[Q1 Q2], R=[R11 R12; 0 R22].

Readings: R-A1 leaf/cutoff, R-A2 split point h = 32*ceil(w/64), R-A3/R-A4
FP16 operands and power-of-two column scaling (only in ``gemm="fp16"`` emulation mode),
R-A6 CAQR ragged blocks, R-A7 row-oriented MGS, R-A8 local zero norms, R-A9 diag(R) > 0.
"""
from __future__ import annotations

import numpy as np

from .fp16 import fl16, pow2_colscale


class Breakdown(ArithmeticError):
    """Zero or non-finite column norm at global column ``col`` (0-based)."""

    def __init__(self, col: int):
        super().__init__(f"QR breakdown at column {col}")
        self.col = col


def mgs(a: np.ndarray, allow_zero: bool = False, col0: int = 0):
    """Alg. 4. Returns (Q, R) with R upper triangular, diag(R) >= 0.

    allow_zero: reading R-A8 -- inside a CAQR block a locally zero column gets q=0, r=0.
    """
    q = np.array(a, dtype=np.float64, copy=True)
    m, n = q.shape
    r = np.zeros((n, n))
    for k in range(n):
        r[k, k] = np.sqrt(np.dot(q[:, k], q[:, k]))                    # line 5
        if not np.isfinite(r[k, k]) or (r[k, k] == 0.0 and not allow_zero):
            raise Breakdown(col0 + k)
        if r[k, k] == 0.0:
            q[:, k] = 0.0
            continue
        q[:, k] = q[:, k] / r[k, k]                                      # line 6
        r[k, k + 1:] = q[:, k] @ q[:, k + 1:]                            # line 7
        q[:, k + 1:] = q[:, k + 1:] - np.outer(q[:, k], r[k, k + 1:])    # line 8
    return q, r


def caqr_blocks(m: int, br: int, w: int):
    """Row blocks of the CAQR panel (R-A6): br-row blocks; a remainder shorter than w rows is
    folded into the previous block. Returns a list of (row0, rows)."""
    nb = max(1, -(-m // br))
    last = m - (nb - 1) * br
    if nb > 1 and last < w:
        nb -= 1
    out = [(b * br, br) for b in range(nb - 1)]
    out.append(((nb - 1) * br, m - (nb - 1) * br))
    return out


def caqr(a: np.ndarray, br: int = 256, col0: int = 0, _top: bool = True):
    """Eq. (6) CAQR panel, MGS blocks, recursive stack."""
    a = np.asarray(a, dtype=np.float64)
    m, w = a.shape
    if m <= br:
        return mgs(a, allow_zero=not _top, col0=col0)
    blocks = caqr_blocks(m, br, w)
    if len(blocks) == 1:
        return mgs(a, allow_zero=not _top, col0=col0)
    qs, rs = [], []
    for r0, rows in blocks:                                   # step 1: independent MGS
        qb, rb = mgs(a[r0:r0 + rows], allow_zero=True, col0=col0)
        qs.append(qb)
        rs.append(rb)
    stack = np.vstack(rs)                                     # step 2: stack the R's
    qst, r = caqr(stack, br, col0=col0, _top=_top)            # step 3: factor the stack
    q = np.empty_like(a)
    for b, (r0, rows) in enumerate(blocks):                   # step 4: Q_b <- Q_b Q_red[b]
        q[r0:r0 + rows] = qs[b] @ qst[b * w:(b + 1) * w]
    return q, r                                               # step 5: (Q, R)


def split_point(w: int, unit: int = 32) -> int:
    """R-A2: h = 32*ceil(w/64) (the left half gets the larger share, multiple of 32).
    ``unit`` generalizes the multiple for panel widths pw < 32 (tests only)."""
    return unit * (-(-w // (2 * unit)))


def rgs(a: np.ndarray, cutoff: int = 128, panel: str = "mgs", br: int = 256,
        gemm: str = "fp64", pw: int = 32, col0: int = 0):
    """Alg. 2 recursive Gram-Schmidt.

    cutoff : the paper's recursion cutoff (Alg. 2 line 3, n==128; reading R-A1: stop when
             w <= cutoff is reached by the FP16 split nodes; below it the recursion continues
             with FP32-class (here: exact) products down to the 32-column panel).
    panel  : "mgs" (Alg. 4 on the whole m x 32 panel) or "caqr" (Eq. 6 with br-row blocks).
    gemm   : "fp64" -- exact products at every split node (the oracle of record);
             "fp16" -- emulate the method's precision at split nodes wider than ``cutoff``:
             R12 = fl16(Q1)' fl16(A2 diag(s)) / s and A2 - fl16(Q1) fl16(R12 diag(s')) / s'
             (R-A3, R-A4), products summed exactly in float64 and rounded to float32.
    Returns (Q, R) as float64 arrays.
    """
    a = np.array(a, dtype=np.float64, copy=True)
    m, w = a.shape
    if w <= pw:
        if panel == "caqr":
            return caqr(a, br, col0=col0)
        return mgs(a, col0=col0)
    h = split_point(w, min(pw, 32))
    q1, r11 = rgs(a[:, :h], cutoff, panel, br, gemm, pw, col0)            # line 7
    a2 = a[:, h:]
    if gemm == "fp16" and w > cutoff:
        s = pow2_colscale(a2)
        r12 = (fl16(q1).T @ fl16(a2 * s)) / s                                # line 8
        r12 = r12.astype(np.float32).astype(np.float64)
        s2 = pow2_colscale(r12)
        upd = (fl16(q1) @ fl16(r12 * s2)) / s2
        upd = upd.astype(np.float32).astype(np.float64)
        a2 = (a2 - upd).astype(np.float32).astype(np.float64)               # line 9 argument
    else:
        r12 = q1.T @ a2                                                      # line 8
        a2 = a2 - q1 @ r12                                                   # line 9 argument
    q2, r22 = rgs(a2, cutoff, panel, br, gemm, pw, col0 + h)               # line 9
    q = np.hstack([q1, q2])                                                  # line 10
    r = np.zeros((w, w))                                                     # line 11, Eq. (5)
    r[:h, :h] = r11
    r[:h, h:] = r12
    r[h:, h:] = r22
    return q, r


def rgs_reorth(a: np.ndarray, **kw):
    """Re-orthogonalization (§4.1.2, NEXT-1): (Q2, R2 R1) with Q2 R2 = rgs(Q1)."""
    q1, r1 = rgs(a, **kw)
    q2, r2 = rgs(q1, **kw)
    return q2, r2 @ r1
