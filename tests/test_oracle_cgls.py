"""Pins for oracle.cgls (P8, P9 of SURVEY.md §8c.4): the paper's "1 iteration with perfect QR"
(PAPER.md:575-576), CG finite termination, the linear-rate bound, the
closed-form LS solution (Eq. 2) via brute-force Householder / normal equations, and the
R-A10 reading that the literal Alg. 5 does not converge."""
import numpy as np
import pytest

import workloads as W
from conftest import golden_lines
from oracle.cgls import cgls_literal, lls_refine, oracle_lls, pcgls
from oracle.householder import back_substitution, householder_lls, householder_qr, normal_equations_lls
from oracle.metrics import lls_optimality, x_rel_error
from oracle.qr import rgs


def test_golden_trsv():
    for line in golden_lines("trsv_2x2.txt"):
        r, b, x = [np.array(t.split(), float) for t in line.split(";")]
        assert np.array_equal(back_substitution(r.reshape(2, 2), b), x)


def test_perfect_qr_one_iteration():
    # kappa(AR^-1) = 1 -> CGLS converges in 1 iteration. Golden fact file.
    facts = dict(l.split("#")[0].split("=") for l in golden_lines("paper_facts.txt"))
    want = int(facts["cgls_iterations_perfect_qr "].strip())
    a = W.spectrum_matrix(512, 128, "geometric", 1e4, seed=9).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=19)
    _, r = householder_qr(a)
    x, info = pcgls(a, b, r, tol=1e-12, maxit=50)
    # exact arithmetic: 1; floating point: the second iteration only mops up rounding.
    assert info.iterations <= want + 1 and info.history[0] < 1e-8
    assert x_rel_error(x, x_true) < 1e-9


def test_zero_projection_rhs():
    # b orthogonal to range(A) -> s0 = 0 -> x = 0, 0 iterations.
    rng = np.random.default_rng(2)
    a = rng.standard_normal((60, 10))
    q, _ = np.linalg.qr(a, mode="complete")
    b = q[:, 20]
    x, info = pcgls(a, b, householder_qr(a)[1], tol=1e-10)
    assert info.reason == "zero_rhs" or np.linalg.norm(x) < 1e-12
    assert np.linalg.norm(x) < 1e-12


def test_orthonormal_columns_identity_preconditioner():
    rng = np.random.default_rng(4)
    qa, _ = np.linalg.qr(rng.standard_normal((80, 12)))
    b = rng.standard_normal(80)
    x, info = pcgls(qa, b, np.eye(12), tol=1e-12)
    assert np.allclose(x, qa.T @ b, atol=1e-13) and info.iterations <= 2


def test_two_singular_values_finite_termination():
    # CG on A'A with two distinct eigenvalues terminates in 2 steps (SPEC.md:335 analogue).
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((200, 30)))
    v, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    a = (u * W.spectrum_values(30, "cluster", 1e3)) @ v.T        # exact two-valued spectrum (fp64)
    b = a @ rng.standard_normal(30)
    x, info = pcgls(a, b, np.eye(30), tol=1e-10, maxit=20)
    assert info.converged and info.iterations <= 3


def test_rate_bound():
    # error reduced at least by (k'-1)/(k'+1) per iteration (CG energy-norm
    # bound ||A(x_k - x*)|| <= 2 rho^k ||A x*||), kappa' = kappa(A R^-1) by dense SVD.
    a = W.spectrum_matrix(600, 100, "geometric", 1e5, seed=8).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=18)
    _, r = rgs(a, cutoff=32, gemm="fp16")          # an imperfect (FP16-method) preconditioner
    kp = np.linalg.cond(a @ np.linalg.inv(r))
    rho = (kp - 1) / (kp + 1)
    e0 = np.linalg.norm(a @ x_true)
    for k in (1, 3, 6, 10):
        xk, _ = pcgls(a, b, r, tol=0.0, maxit=k, floor=0.0)
        ek = np.linalg.norm(a @ (xk - x_true))
        assert ek <= 2 * rho ** k * e0 * (1 + 1e-6) + 1e-12


def test_literal_alg5_does_not_converge_corrected_does():
    # R-A10: as printed, Alg. 5 iterates in the preconditioned variable and never maps back.
    a = W.spectrum_matrix(300, 40, "geometric", 1e3, seed=12).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=13)
    _, r = rgs(a, cutoff=32, gemm="fp16")
    with np.errstate(all="ignore"):
        xs = cgls_literal(a, b, r, iters=15)
    last = xs[-1]
    assert (not np.all(np.isfinite(last))) or x_rel_error(last, x_true) > 1e-2
    x, info = pcgls(a, b, r, tol=1e-12)
    assert x_rel_error(x, x_true) < 1e-9


@pytest.mark.parametrize("m,n,kind,cond", [(40, 8, "gaussian", 1), (120, 30, "geometric", 1e3)])
def test_oracle_lls_matches_householder_and_ne(m, n, kind, cond):
    a = W.make_matrix(kind, m, n, seed=m, cond=cond).astype(np.float64)
    b = W.random_rhs(m, seed=n)
    x, info = oracle_lls(a, b)
    xh = householder_lls(a, b)
    assert x_rel_error(x, xh) < 1e-12 * max(cond, 1) ** 2
    assert info.iterations <= 15
    if cond <= 1e3:
        assert x_rel_error(x, np.linalg.lstsq(a, b, rcond=None)[0]) < 1e-13 * cond ** 2
    if cond == 1:
        assert x_rel_error(x, normal_equations_lls(a, b)) < 1e-12


def test_consistent_rhs_recovers_x_true():
    a = W.spectrum_matrix(400, 100, "arithmetic", 1e6, seed=21).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=22)
    x, _ = oracle_lls(a, b)
    assert x_rel_error(x, x_true) < 1e6 * 1e-15 * 50
    assert lls_optimality(a, x, b) < 1e-10 * np.linalg.norm(a.T @ b)


def test_restart_rule_reaches_fp64_with_fp16_preconditioner():
    # R-A12 [calib]: arithmetic kappa=1e6 -- pass 1 stalls near 1e-10, the restart reaches ~1e-12.
    a = W.spectrum_matrix(1024, 256, "arithmetic", 1e6, seed=31).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=32)
    _, r = rgs(a, cutoff=32, gemm="fp16")
    x_o, _ = oracle_lls(a, b)
    x2, infos = lls_refine(a, b, r, tol=1e-10, maxit=400, target="fp64")
    assert x_rel_error(x2, x_o) < 1e-10
    assert len(infos) == 2 and all(i.converged for i in infos)


def test_uniform_few_iterations():
    # uniform random -> "pretty good accuracy in 20 iterations" (desk scale).
    a = W.uniform01(2048, 512, seed=3).astype(np.float64)
    b, x_true = W.consistent_rhs(a, seed=4)
    _, r = rgs(a, cutoff=128, gemm="fp16")
    x, infos = lls_refine(a, b, r, tol=1e-10, maxit=200, target="fp64")
    assert sum(i.iterations for i in infos) <= 20
    assert x_rel_error(x, x_true) < 1e-10


# ---- NEXT-2: direct QR solve x = R^-1 Q' b (Alg. 1 lines 3-4) ----
@pytest.mark.parametrize("m,n,cond", [(60, 12, 1.0), (200, 40, 1e3)])
def test_oracle_qr_solve_is_the_least_squares_solution(m, n, cond):
    # any exact thin QR gives the LS solution (Eq. (4)): pinned against
    # numpy's SVD-based lstsq (a different algorithm) and against the normal equations' optimality
    # condition A'(b - A x) = 0.
    from oracle.householder import qr_solve
    from oracle.qr import rgs
    a = W.make_matrix("geometric" if cond > 1 else "gaussian", m, n, seed=m + n, cond=cond)
    a = a.astype(np.float64)
    b = W.random_rhs(m, seed=m)
    x_ls = np.linalg.lstsq(a, b, rcond=None)[0]
    q, r = householder_qr(a)
    x = qr_solve(q, r, b)
    assert x_rel_error(x, x_ls) < 1e-13 * cond ** 2
    g = a.T @ (b - a @ x)
    assert np.linalg.norm(g) <= 1e-12 * cond * np.linalg.norm(a) * np.linalg.norm(b)
    # the recursive Gram-Schmidt factors in FP64 give the same solution (Q'Q = I to ~cond*u)
    q2, r2 = rgs(a, cutoff=32, gemm="fp64")
    assert x_rel_error(qr_solve(q2, r2, b), x_ls) < 1e-12 * cond ** 2


def test_oracle_qr_solve_upper_triangular_hand_example():
    # R = [[2, 1], [0, 4]], Q = I (3 x 2 slice), b = [4, 8, 5]: Q'b = [4, 8], x2 = 2, x1 = 1
    from oracle.householder import qr_solve
    q = np.eye(3)[:, :2]
    r = np.array([[2.0, 1.0], [0.0, 4.0]])
    x = qr_solve(q, r, np.array([4.0, 8.0, 5.0]))
    assert np.array_equal(x, np.array([1.0, 2.0]))
