"""Accuracy metrics and flop conventions (oracle side, float64).

* backward error ||A - QR|| / ||A||      PAPER.md:497-499 (§3.2.1)
* orthogonality  ||I - Q'Q||             PAPER.md:500-501; normalized /N in Fig. 2, :607, :633
* LLS optimality ||A'(A x - b)||         PAPER.md:512-519 (§3.2.2)
* R relative error ||R - R_o||_F / ||R_o||_F   (north_star gate; reading R-A16)
* flops: RGS 2mn^2 executed; the reporting convention 2mn^2 - 2/3 n^3 (PAPER.md:302-304,
  :373-374; reading R-A19).
"""
from __future__ import annotations

import numpy as np


def backward_error_f(a, q, r) -> float:
    a = np.asarray(a, dtype=np.float64)
    return float(np.linalg.norm(a - np.asarray(q, np.float64) @ np.asarray(r, np.float64))
                 / np.linalg.norm(a))


def backward_error_2(a, q, r) -> float:
    a = np.asarray(a, dtype=np.float64)
    return float(np.linalg.norm(a - np.asarray(q, np.float64) @ np.asarray(r, np.float64), 2)
                 / np.linalg.norm(a, 2))


def orthogonality_f(q) -> float:
    """||Q'Q - I||_F / sqrt(n)  (north_star form)."""
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[1]
    return float(np.linalg.norm(q.T @ q - np.eye(n)) / np.sqrt(n))


def orthogonality_2_over_n(q) -> float:
    """||I - Q'Q||_2 / N  (the paper's Fig. 2 form)."""
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[1]
    return float(np.linalg.norm(np.eye(n) - q.T @ q, 2) / n)


def r_rel_error(r, r_ref) -> float:
    r = np.asarray(r, dtype=np.float64)
    r_ref = np.asarray(r_ref, dtype=np.float64)
    return float(np.linalg.norm(r - r_ref) / np.linalg.norm(r_ref))


def lls_optimality(a, x, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    return float(np.linalg.norm(a.T @ (a @ np.asarray(x, np.float64) - np.asarray(b, np.float64))))


def x_rel_error(x, x_ref) -> float:
    x_ref = np.asarray(x_ref, dtype=np.float64)
    return float(np.linalg.norm(np.asarray(x, np.float64) - x_ref) / np.linalg.norm(x_ref))


def flops_convention(m: int, n: int) -> float:
    """2mn^2 - 2/3 n^3 (the north_star reporting convention)."""
    return 2.0 * m * n * n - 2.0 / 3.0 * n ** 3


def flops_rgs_exec(m: int, n: int) -> float:
    """2mn^2: T(w) = 2T(w/2) + m w^2, T(c) = 2mc^2  =>  T(n) = 2mn^2."""
    return 2.0 * m * n * n
