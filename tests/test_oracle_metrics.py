"""Pins for oracle.metrics (the north_star gates, §3.2) and oracle.qr.rgs_reorth
(re-orthogonalization, §4.1.2). Every expected value is a hand-computed closed
form, chosen so that a plausible slip (a /n instead of /sqrt(n), a missing ||A|| or ||x_ref||
divisor, a transposed operand, a dropped factor) changes the result."""
import numpy as np
import pytest

import workloads as W
from oracle.householder import householder_qr
from oracle.metrics import (backward_error_2, backward_error_f, lls_optimality,
                            orthogonality_2_over_n, orthogonality_f, r_rel_error, x_rel_error)
from oracle.qr import rgs, rgs_reorth


def test_orthogonality_f_repeated_column():
    # Q = [e1 e1]: Q'Q - I = [[0, 1], [1, 0]], ||.||_F = sqrt(2), / sqrt(n=2) -> exactly 1
    q = np.zeros((3, 2))
    q[0, 0] = q[0, 1] = 1.0
    assert orthogonality_f(q) == pytest.approx(1.0, rel=0, abs=1e-15)


def test_orthogonality_f_scaled_identity_distinguishes_sqrt_n():
    # Q = 2 I_4: Q'Q - I = 3 I_4, ||.||_F = 3 * 2 = 6; /sqrt(4) = 3 (a /n slip would give 1.5,
    # ||Q'Q||_F - ... or a missing -I would give 8 / 2 = 4)
    q = 2.0 * np.eye(4)
    assert orthogonality_f(q) == pytest.approx(3.0, abs=1e-15)
    # orthonormal but non-square (8 x 3): exactly 0 up to rounding
    u = W.sylvester_hadamard_cols(8, 3) / np.sqrt(8.0)
    assert orthogonality_f(u) < 1e-15


def test_orthogonality_2_over_n_hand_value():
    # ||I - Q'Q||_2 / N (Fig. 2 form): Q = 2 I_4 -> ||-3 I||_2 / 4 = 0.75
    assert orthogonality_2_over_n(2.0 * np.eye(4)) == pytest.approx(0.75, abs=1e-15)
    # rank-one defect: Q = [e1 e1] -> eigenvalues of [[0,1],[1,0]] are +-1 -> 1 / 2
    q = np.zeros((3, 2))
    q[0, 0] = q[0, 1] = 1.0
    assert orthogonality_2_over_n(q) == pytest.approx(0.5, abs=1e-15)


def test_backward_error_rank_one_residual():
    # A = [diag(3, 4); 0], Q = [I; 0], R = [[3, d], [0, 4]]: A - QR = -d e1 e2', so
    # ||A - QR||_F = d and ||A||_F = 5 -> d / 5; in the 2-norm ||A||_2 = 4 -> d / 4.
    d = 0.125
    a = np.zeros((5, 2))
    a[0, 0], a[1, 1] = 3.0, 4.0
    q = np.zeros((5, 2))
    q[0, 0] = q[1, 1] = 1.0
    r = np.array([[3.0, d], [0.0, 4.0]])
    assert backward_error_f(a, q, r) == pytest.approx(d / 5.0, abs=1e-16)
    assert backward_error_2(a, q, r) == pytest.approx(d / 4.0, abs=1e-16)
    # a transposed R (R' instead of R) would put the defect at (2, 1): A - Q R' has a d at
    # position (1, 0), same norm -- so also pin the sign/position through an asymmetric case
    r2 = np.array([[3.0, 0.0], [0.0, 4.0 + d]])
    assert backward_error_f(a, q, r2) == pytest.approx(d / 5.0, abs=1e-16)
    assert backward_error_f(a, q, np.diag([3.0, 4.0])) == 0.0


def test_r_rel_error_hand_value():
    # ||R - R_o||_F / ||R_o||_F: R_o = diag(3, 4) (norm 5), R = R_o + e1 e2' -> 1/5; the
    # divisor is the reference (dividing by ||R||_F = sqrt(26) would give 0.196...)
    r_o = np.diag([3.0, 4.0])
    r = np.array([[3.0, 1.0], [0.0, 4.0]])
    assert r_rel_error(r, r_o) == pytest.approx(0.2, abs=1e-16)
    assert r_rel_error(r_o, r_o) == 0.0


def test_x_rel_error_hand_value():
    # ||x - x_ref|| / ||x_ref||: x = (3, 4), x_ref = (0, 4) -> 3 / 4 (not 3 / 5)
    assert x_rel_error(np.array([3.0, 4.0]), np.array([0.0, 4.0])) == pytest.approx(0.75,
                                                                                    abs=1e-16)


def test_lls_optimality_hand_value():
    # ||A'(A x - b)||: A = [[1, 0], [0, 2], [0, 0]], x = (1, 1), b = (1, 0, 5):
    # A x - b = (0, 2, -5), A'(.) = (0, 4) -> 4 (b's third entry is orthogonal to range(A))
    a = np.array([[1.0, 0.0], [0.0, 2.0], [0.0, 0.0]])
    assert lls_optimality(a, np.array([1.0, 1.0]), np.array([1.0, 0.0, 5.0])) == pytest.approx(
        4.0, abs=1e-15)


# ---- rgs_reorth: (Q2, R2 R1) with Q2 R2 = rgs(Q1) -------------------------

def test_reorth_planted_hadamard_exact():
    # The planted fixture A = (H/sqrt(m)) R0: the first pass is exact (Q1 = H/sqrt(m), R1 = R0),
    # so the second pass factors an exactly orthonormal Q1: Q2 = Q1 and R2 = I exactly, and the
    # product R2 R1 = R0 bitwise (also in the FP16 emulation: every cast is exact).
    a, qt, r0 = W.planted_hadamard(1024, 128, seed=201)
    for gemm in ("fp64", "fp16"):
        q, r = rgs_reorth(a, cutoff=32, panel="caqr", br=256, gemm=gemm)
        assert np.array_equal(q, qt), gemm
        assert np.array_equal(r, r0), gemm


@pytest.mark.parametrize("m,n,cond", [(256, 48, 1e2), (512, 96, 1e3)])
def test_reorth_r_equals_householder_r(m, n, cond):
    # exact products: R2 R1 is the unique R of A (diag > 0), i.e. the sign-normalized
    # Householder R, and Q2 (R2 R1) = A
    a = W.spectrum_matrix(m, n, "geometric", cond, seed=61).astype(np.float64)
    q, r = rgs_reorth(a)
    _, rh = householder_qr(a)
    assert np.allclose(np.tril(r, -1), 0.0)
    assert np.all(np.diag(r) > 0)
    assert r_rel_error(r, rh) < 1e-12
    assert backward_error_f(a, q, r) < 1e-14
    assert orthogonality_f(q) < 1e-14


def test_reorth_restores_orthogonality_of_the_fp16_method():
    # orthogonality of the FP16 method grows with kappa (Fig. 2); a second
    # pass over Q1 brings it back near the unit round-off of the second pass's own error
    # (Q1 is well conditioned), while R2 R1 keeps the backward error of the first pass.
    a = W.spectrum_matrix(1024, 256, "geometric", 1e4, seed=62).astype(np.float64)
    q1, r1 = rgs(a, cutoff=32, gemm="fp16")
    q2, r = rgs_reorth(a, cutoff=32, gemm="fp16")
    o1, o2 = orthogonality_f(q1), orthogonality_f(q2)
    assert o1 > 0.05          # A23: the single FP16 pass loses orthogonality at geometric 1e4
    assert o2 < 5e-3 and o2 < o1 / 50
    assert backward_error_f(a, q2, r) < 5e-3
    assert np.allclose(np.tril(r, -1), 0.0) and np.all(np.diag(r) > 0)
