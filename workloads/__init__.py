"""Seeded synthetic input generators shared by the tests, the oracle checks and bench.py.

This module holds NONE of the method's arithmetic (no Gram-Schmidt, no CGLS, no FP16
casting). It only draws inputs with the shapes and spectra of the paper's workloads:

* i.i.d. families, PAPER.md:642-645 (§4.2 items 1-2): uniform(0,1), uniform(-1,1), normal(0,1).
* prescribed singular values, PAPER.md:645-651 (§4.2 items 3-5) and the Fig. 3 captions
  PAPER.md:677-698: geometric, arithmetic, cluster; "cluster2" (undefined in the
  paper) is read as (1, 1/k, ..., 1/k)  -- DESIGN.md reading R-A18.
  A = U diag(sigma) V^T with sigma_1 = 1 and U (m x n), V (n x n) Haar-distributed
  (sign-fixed QR of Gaussian matrices; numpy's LAPACK QR is a library primitive of the
  generator, not of the method).
* the planted-Hadamard fixture: A = (H_m[:, :n] / sqrt(m)) R0 with
  Sylvester H and a small-integer upper-triangular R0, for which every step of the FP16
  method is exact.
* right-hand sides b = A x_true (consistent) or b ~ N(0,1) (large residual), DESIGN.md R-A15.

Matrices are returned as numpy float32 arrays in Fortran (column-major) order, which is the
layout the C-ABI consumes (element (i, j) at i + j*lda).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "gaussian", "uniform01", "uniform_sym", "spectrum_values", "spectrum_matrix",
    "planted_hadamard", "sylvester_hadamard_cols", "consistent_rhs", "random_rhs",
    "make_matrix", "CONFIG_SEEDS",
]

# Seeds of SURVEY.md §8(d) "Synthetic inputs".
CONFIG_SEEDS = {
    "cfg1": 1, "cfg1_x": 101, "cfg1_planted": 201,
    "cfg2": 2, "cfg2_geo": 3,
    "cfg3": 4, "cfg3_arith": 5,
    "cfg4_k1e4": 6, "cfg4_k1e6": 7, "cfg4_x_k1e4": 106, "cfg4_x_k1e6": 107,
    "cfg5": 8, "cfg5_x": 108,
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def gaussian(m: int, n: int, seed: int) -> np.ndarray:
    """i.i.d. N(0,1) entries (matrix type 3), float32, column-major."""
    a = _rng(seed).standard_normal((n, m), dtype=np.float32)  # row j = column j
    return a.T  # Fortran-ordered view, element (i, j) = a[j, i]


def uniform01(m: int, n: int, seed: int) -> np.ndarray:
    """i.i.d. uniform(0,1) (matrix type 1)."""
    a = _rng(seed).random((n, m), dtype=np.float32)
    return a.T


def uniform_sym(m: int, n: int, seed: int) -> np.ndarray:
    """i.i.d. uniform(-1,1) (matrix type 2)."""
    a = _rng(seed).random((n, m), dtype=np.float32)
    return (2.0 * a - 1.0).astype(np.float32).T


def spectrum_values(n: int, kind: str, cond: float) -> np.ndarray:
    """Singular values with sigma_1 = 1 (reading R-A18)."""
    i = np.arange(n, dtype=np.float64)
    if n == 1:
        return np.ones(1)
    if kind == "geometric":      # log sigma evenly spaced
        return cond ** (-i / (n - 1))
    if kind == "arithmetic":     # sigma evenly spaced
        return 1.0 - i / (n - 1) * (1.0 - 1.0 / cond)
    if kind == "cluster":        # all but the smallest are 1
        s = np.ones(n)
        s[-1] = 1.0 / cond
        return s
    if kind == "cluster2":       # reading: (1, 1/cond, ..., 1/cond)
        s = np.full(n, 1.0 / cond)
        s[0] = 1.0
        return s
    raise ValueError(f"unknown spectrum kind {kind!r}")


def _haar(rows: int, cols: int, rng: np.random.Generator) -> np.ndarray:
    g = rng.standard_normal((rows, cols))
    q, r = np.linalg.qr(g)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d


def spectrum_matrix(m: int, n: int, kind: str, cond: float, seed: int) -> np.ndarray:
    """A = U diag(sigma) V^T, float32 column-major (the values the method receives)."""
    rng = _rng(seed)
    u = _haar(m, n, rng)
    v = _haar(n, n, rng)
    s = spectrum_values(n, kind, cond)
    a = (u * s) @ v.T
    return np.asfortranarray(a.astype(np.float32))


def sylvester_hadamard_cols(m: int, n: int) -> np.ndarray:
    """Columns 0..n-1 of the Sylvester Hadamard matrix H_m: H[i, j] = (-1)^popcount(i & j)."""
    if m & (m - 1):
        raise ValueError("m must be a power of two")
    i = np.arange(m, dtype=np.int64)[:, None]
    j = np.arange(n, dtype=np.int64)[None, :]
    x = i & j
    pc = np.zeros_like(x)
    while np.any(x):
        pc += x & 1
        x >>= 1
    return np.where(pc % 2 == 0, 1.0, -1.0)


def planted_hadamard(m: int, n: int, seed: int, max_int: int = 3):
    """Planted fixture. Returns (A, Q_true, R0) in float64/float32.

    A = (H_m[:, :n] / sqrt(m)) R0, m a power of 4, R0 upper triangular with integer entries
    in [-max_int, max_int] and an integer diagonal in [1, max_int].
    """
    k = int(round(np.log2(m)))
    if (1 << k) != m or k % 2:
        raise ValueError("m must be a power of 4")
    rng = _rng(seed)
    r0 = np.triu(rng.integers(-max_int, max_int + 1, size=(n, n))).astype(np.float64)
    np.fill_diagonal(r0, rng.integers(1, max_int + 1, size=n))
    q = sylvester_hadamard_cols(m, n) / float(1 << (k // 2))
    a = q @ r0
    a32 = np.asfortranarray(a.astype(np.float32))
    assert np.array_equal(a32.astype(np.float64), a), "planted A must be exact in fp32"
    return a32, q, r0


def consistent_rhs(a: np.ndarray, seed: int):
    """b = A x_true in float64 with x_true ~ N(0,1) (reading R-A15). Returns (b, x_true)."""
    x = _rng(seed).standard_normal(a.shape[1])
    b = a.astype(np.float64) @ x
    return b, x


def random_rhs(m: int, seed: int) -> np.ndarray:
    """Large-residual right-hand side b ~ N(0,1) in float64."""
    return _rng(seed).standard_normal(m)


def make_matrix(kind: str, m: int, n: int, seed: int, cond: float = 1.0) -> np.ndarray:
    """Dispatch by family name: gaussian|uniform01|uniform_sym|geometric|arithmetic|cluster|cluster2."""
    if kind == "gaussian":
        return gaussian(m, n, seed)
    if kind == "uniform01":
        return uniform01(m, n, seed)
    if kind == "uniform_sym":
        return uniform_sym(m, n, seed)
    return spectrum_matrix(m, n, kind, cond, seed)


# ------------------------------------------------------------------------------------------
# Device-side generators for the full-size bench workloads (same distributions; torch's Philox
# generator seeded per call; torch.linalg is a library primitive of the GENERATOR only).
# ------------------------------------------------------------------------------------------
def gaussian_cuda(m: int, n: int, seed: int, device="cuda"):
    """i.i.d. N(0,1) float32, column-major (shape (m, n), stride (1, m)), on `device`."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((n, m), generator=g, device=device, dtype=torch.float32).t()


def spectrum_cuda(m: int, n: int, kind: str, cond: float, seed: int, device="cuda"):
    """A = U diag(sigma) V^T (float32, column-major) with Haar U, V drawn on the device."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.randn((m, n), generator=g, device=device, dtype=torch.float64)
    u, ru = torch.linalg.qr(u)
    u *= torch.sign(torch.diagonal(ru))
    del ru
    v = torch.randn((n, n), generator=g, device=device, dtype=torch.float64)
    v, rv = torch.linalg.qr(v)
    v *= torch.sign(torch.diagonal(rv))
    s = torch.from_numpy(spectrum_values(n, kind, cond)).to(device)
    a = (u * s) @ v.T
    del u, v
    out = torch.empty((n, m), device=device, dtype=torch.float32).t()
    out.copy_(a)
    return out
