"""GPU parity of the whole hot path through the C ABI: tcqr_factor and tcqr_lls_solve against the CPU
FP64 oracle (north_star tolerances: ||A-QR||_F/||A||_F <= 5e-3, ||Q'Q-I||_F/sqrt(n) <= 5e-2,
||R-R_o||_F/||R_o||_F <= 1e-2 for kappa <= 1e3; x within 1e-10 of the oracle for the FP64 target),
plus the closed-form pins: planted Hadamard bitwise (P2), power-of-two scale equivariance bitwise
(P3), breakdown / non-finite status codes, degenerate right-hand sides."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import workloads as W  # noqa: E402
from oracle.cgls import oracle_lls  # noqa: E402
from oracle.metrics import (backward_error_f, orthogonality_f, r_rel_error,  # noqa: E402
                            x_rel_error, lls_optimality)
from oracle.qr import rgs  # noqa: E402


@pytest.fixture(scope="module")
def tq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_05508_b200 as tq
    tq.init(0)
    yield tq
    tq.set_config()


def _factor(tq, a, **cfg):
    tq.set_config(**cfg)
    A = tq.to_device_colmajor(a)
    Q, R = tq.factor(A)
    torch.cuda.synchronize()
    return Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)


def _gates(a, q, r, r_o, orth_gate=5e-2):
    be = backward_error_f(a, q, r)
    orth = orthogonality_f(q)
    re = r_rel_error(r, r_o)
    assert np.array_equal(r, np.triu(r)) and np.all(np.diag(r) > 0)
    assert be <= 5e-3, be
    assert orth <= orth_gate, orth
    assert re <= 1e-2, re
    return be, orth, re


@pytest.mark.parametrize("m,n,cutoff", [(1024, 128, 128), (1024, 128, 64), (1024, 128, 32),
                                        (1000, 100, 32), (777, 96, 64), (2048, 512, 128),
                                        (4100, 300, 64), (300, 300, 128)])
def test_factor_gaussian_gates(tq, m, n, cutoff):
    a = W.gaussian(m, n, seed=m * 7 + n)
    q, r = _factor(tq, a, cutoff=cutoff)
    _, r_o = rgs(a.astype(np.float64))
    be, orth, re = _gates(a, q, r, r_o)
    if n <= cutoff:   # no FP16 anywhere: FP32 accuracy
        assert be < 1e-5 and re < 1e-4


@pytest.mark.parametrize("kind,cond", [("geometric", 1e2), ("arithmetic", 1e3)])
def test_factor_spectrum_gates(tq, kind, cond):
    a = W.spectrum_matrix(4096, 1024, kind, cond, seed=3)
    q, r = _factor(tq, a)
    _, r_o = rgs(a.astype(np.float64))
    _gates(a, q, r, r_o)


@pytest.mark.parametrize("m,n,cutoff,br", [(1024, 128, 32, 256), (1024, 128, 128, 256),
                                           (1024, 256, 32, 256), (1024, 256, 64, 256),
                                           (4096, 256, 64, 1024), (4096, 512, 128, 1024)])
def test_factor_planted_hadamard_bitwise(tq, m, n, cutoff, br):
    a, qt, r0 = W.planted_hadamard(m, n, seed=201)
    q, r = _factor(tq, a, cutoff=cutoff, panel_rows=br)
    assert np.array_equal(r, r0)
    assert np.array_equal(q, qt)


def test_factor_scale_equivariance_bitwise(tq):
    a = W.gaussian(2048, 384, seed=11)
    q, r = _factor(tq, a, cutoff=64)
    for e in (-30, -9, 7, 20):
        qe, re_ = _factor(tq, np.ldexp(a, e).astype(np.float32), cutoff=64)
        assert np.array_equal(qe, q), e
        assert np.array_equal(re_, np.ldexp(r, e)), e


def test_factor_deterministic(tq):
    a = W.gaussian(3000, 640, seed=5)
    q1, r1 = _factor(tq, a)
    q2, r2 = _factor(tq, a)
    assert np.array_equal(q1, q2) and np.array_equal(r1, r2)


def test_factor_breakdown_and_nonfinite(tq):
    tq.set_config()
    a = W.gaussian(512, 200, seed=2)
    a[:, 150] = 0.0
    with pytest.raises(tq.TcqrError) as e:
        tq.factor(tq.to_device_colmajor(a))
    assert e.value.code == 151
    a = W.gaussian(512, 200, seed=2)
    a[7, 42] = np.inf
    with pytest.raises(tq.TcqrError) as e:
        tq.factor(tq.to_device_colmajor(a))
    assert e.value.code == 43


def test_factor_argument_errors(tq):
    A = tq.to_device_colmajor(W.gaussian(64, 32, seed=1))
    import ctypes
    lib = tq.lib()
    p = ctypes.c_void_p(A.data_ptr())
    assert lib.tcqr_factor(0, 32, p, 64, p, p) == -1
    assert lib.tcqr_factor(64, 0, p, 64, p, p) == -2
    assert lib.tcqr_factor(64, 32, None, 64, p, p) == -3
    assert lib.tcqr_factor(64, 32, p, 63, p, p) == -4
    assert lib.tcqr_factor(64, 32, p, 64, p, None) == -6
    assert lib.tcqr_factor(16, 32, p, 64, p, p) == -1     # m < n


def test_factor_host_entry_point(tq):
    tq.set_config()
    a = W.gaussian(1500, 200, seed=8)
    q, r = tq.factor_host(a)
    _, r_o = rgs(a.astype(np.float64))
    _gates(a, q.astype(np.float64), r.astype(np.float64), r_o)


@pytest.mark.parametrize("m,n,kind,cond", [(1024, 128, "gaussian", 1), (2048, 512, "arithmetic", 1e6),
                                           (2048, 256, "cluster", 1e6), (2000, 300, "geometric", 1e3)])
def test_lls_fp64_target(tq, m, n, kind, cond):
    tq.set_config()
    a = W.make_matrix(kind, m, n, seed=m + n, cond=cond)
    b, x_true = W.consistent_rhs(a, seed=n)
    x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), tol=1e-10,
                           maxit=2000)
    x = x.cpu().numpy()
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    assert info["converged"] == 1, info
    assert x_rel_error(x, x_o) <= 1e-10, (x_rel_error(x, x_o), info)


def test_lls_large_residual_optimality(tq):
    tq.set_config()
    a = W.gaussian(3000, 400, seed=4)
    b = W.random_rhs(3000, seed=5)
    x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda())
    x = x.cpu().numpy()
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    assert x_rel_error(x, x_o) <= 1e-10
    assert lls_optimality(a, x, b) <= 1e-9 * np.linalg.norm(a.astype(np.float64).T @ b)


def test_lls_zero_projection_rhs(tq):
    tq.set_config()
    rng = np.random.default_rng(2)
    a = W.gaussian(500, 50, seed=9)
    qf, _ = np.linalg.qr(a.astype(np.float64), mode="complete")
    b = qf[:, 100].copy()
    x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda())
    # In floating point A'b is rounding noise (not exactly 0, SPEC.md:327 is the exact case):
    # the solve must return x ~ 0; convergence on pure noise is not required.
    assert np.linalg.norm(x.cpu().numpy()) < 1e-10


def test_lls_host_entry_point(tq):
    tq.set_config()
    a = W.gaussian(1024, 128, seed=1)
    b, _ = W.consistent_rhs(a, seed=101)
    x, info = tq.lls_solve_host(a, b)
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    assert x_rel_error(x, x_o) <= 1e-10


def test_lls_maxit_reports_not_converged(tq):
    # SPEC.md:324-325 / :343: hitting the cap is data, not an error.
    tq.set_config()
    a = W.spectrum_matrix(2048, 256, "geometric", 1e6, seed=7)
    b, _ = W.consistent_rhs(a, seed=8)
    x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), maxit=5)
    assert info["converged"] == 0 and info["stop_reason"] == 2
    assert np.all(np.isfinite(x.cpu().numpy()))


# ---- NEXT-1: re-orthogonalization -------------------------------------------
@pytest.mark.parametrize("kind,cond", [("geometric", 1e3), ("geometric", 1e4), ("gaussian", 1)])
def test_reorth_factor(tq, kind, cond):
    a = W.make_matrix(kind, 4096, 512, seed=17, cond=cond)
    q1, r1 = _factor(tq, a)
    q2, r2 = _factor(tq, a, reorth=1)
    tq.set_config()
    _, r_o = rgs(a.astype(np.float64))
    # Q2 is orthogonal to working accuracy whatever kappa (the paper's remedy), A = Q2 (R2 R1)
    assert orthogonality_f(q2) < 5e-4
    assert orthogonality_f(q2) <= orthogonality_f(q1) + 1e-6
    assert backward_error_f(a, q2, r2) < 5e-3
    assert np.array_equal(r2, np.triu(r2)) and np.all(np.diag(r2) > 0)
    if cond <= 1e3:
        assert r_rel_error(r2, r_o) < 1e-2


def test_reorth_lls_fewer_iterations(tq):
    a = W.spectrum_matrix(4096, 1024, "geometric", 1e4, seed=23)
    b, x_true = W.consistent_rhs(a, seed=24)
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    A = tq.to_device_colmajor(a)
    B = torch.from_numpy(b).cuda()
    tq.set_config()
    x1, i1 = tq.lls_solve(A, B, tol=1e-10, maxit=4000)
    tq.set_config(reorth=1)
    x2, i2 = tq.lls_solve(A, B, tol=1e-10, maxit=4000)
    tq.set_config()
    assert i2["converged"] == 1 and x_rel_error(x2.cpu().numpy(), x_o) <= 1e-10
    assert x_rel_error(x1.cpu().numpy(), x_o) <= 1e-10
    assert i2["iterations"] * 4 < i1["iterations"], (i1["iterations"], i2["iterations"])


# ---- NEXT-2: direct QR solve x = R^-1 Q' b (Alg. 1 lines 3-4) ---------------
def test_qr_solve_matches_oracle_on_the_same_factors(tq):
    # the same FP32 factors on both sides: the oracle's FP64 back substitution of R x = Q' b vs the
    # C-ABI solve (FP64 Q' b, FP64 explicit inverse); both are FP64 on identical inputs.
    from oracle.householder import qr_solve as qr_solve_o
    a = W.spectrum_matrix(2048, 256, "geometric", 1e3, seed=31).astype(np.float64)
    q, r = np.linalg.qr(a)
    d = np.sign(np.diag(r))
    q = (q * d).astype(np.float32)
    r = np.triu((r.T * d).T).astype(np.float32)
    b = W.random_rhs(2048, seed=32)
    x = tq.qr_solve(tq.to_device_colmajor(q), tq.to_device_colmajor(r), torch.from_numpy(b).cuda())
    x_o = qr_solve_o(q.astype(np.float64), r.astype(np.float64), b)
    assert x_rel_error(x.cpu().numpy(), x_o) <= 1e-11 * 1e3


@pytest.mark.parametrize("m,n", [(4096, 512), (3000, 300)])
def test_qr_solve_after_factor_fp16_accuracy(tq, m, n):
    # Alg. 1 with the tensor-core factors: accuracy at the FP16 level, the paper's "~2 orders worse
    # than SGEQRF"; consistent right-hand side, Gaussian A (kappa ~ 5).
    tq.set_config()
    a = W.gaussian(m, n, seed=n)
    b, x_true = W.consistent_rhs(a, seed=m)
    Q, R = tq.factor(tq.to_device_colmajor(a))
    x = tq.qr_solve(Q, R, torch.from_numpy(b).cuda()).cpu().numpy()
    assert x_rel_error(x, x_true) <= 2e-2
    assert np.all(np.isfinite(x))


def test_qr_solve_breakdown_and_args(tq):
    q = tq.to_device_colmajor(np.eye(64, 8, dtype=np.float32))
    r = np.eye(8, dtype=np.float32)
    r[5, 5] = 0.0
    b = torch.ones(64, dtype=torch.float64, device="cuda")
    with pytest.raises(tq.TcqrError) as e:
        tq.qr_solve(q, tq.to_device_colmajor(r), b)
    assert e.value.code == 6
    rc = tq.lib().tcqr_qr_solve(64, 8, None, 64, None, 8, None, None)
    assert rc == -3


@pytest.mark.parametrize("kind,cond", [("gaussian", 1), ("geometric", 1e3)])
def test_lls_warm_start(tq, kind, cond):
    # CGLS from x0 = R^-1 Q' b: same FP64-target answer, fewer iterations on a well-conditioned A
    a = W.make_matrix(kind, 4096, 512, seed=41, cond=cond)
    b, x_true = W.consistent_rhs(a, seed=42)
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    A = tq.to_device_colmajor(a)
    B = torch.from_numpy(b).cuda()
    tq.set_config()
    x1, i1 = tq.lls_solve(A, B, tol=1e-10, maxit=2000)
    tq.set_config(warm_start=1)
    x2, i2 = tq.lls_solve(A, B, tol=1e-10, maxit=2000)
    tq.set_config()
    assert i2["converged"] == 1, i2
    assert x_rel_error(x2.cpu().numpy(), x_o) <= 1e-10
    if cond == 1:
        assert i2["iterations"] <= i1["iterations"], (i1, i2)


# ---- streamed host entry (H2D / compute / D2H overlapped by column chunks) ----------------------
def test_factor_host_streamed_matches_device(tq):
    # n > 2 * cutoff: tcqr_factor_host ships column chunks in and finished chunks out while the
    # recursion runs, and runs the split nodes' GEMMs per arriving column chunk (different split-K
    # partitions, so rounding-level differences from the device path).  Same gates as the device
    # entry point, close to its factors, deterministic, strictly-lower R zero on the host.
    tq.set_config()
    a = W.gaussian(4096, 1024, seed=51)
    q_h, r_h = tq.factor_host(a)
    q_h2, r_h2 = tq.factor_host(a)
    assert np.array_equal(q_h, q_h2) and np.array_equal(r_h, r_h2)
    Q, R = tq.factor(tq.to_device_colmajor(a))
    r_d = R.cpu().numpy().astype(np.float64)
    assert r_rel_error(r_h.astype(np.float64), r_d) < 1e-4
    assert np.array_equal(np.tril(r_h, -1), np.zeros_like(r_h))
    _, r_o = rgs(a.astype(np.float64))
    _gates(a, q_h.astype(np.float64), r_h.astype(np.float64), r_o)


def test_factor_host_streamed_nonfinite_column(tq):
    tq.set_config()
    a = W.gaussian(2048, 1024, seed=52)
    a[17, 901] = np.inf  # a column in a late chunk: the status names the global column
    with pytest.raises(tq.TcqrError) as e:
        tq.factor_host(a)
    assert e.value.code == 902


# ---- NEXT-4: error-compensated FP16 split (hi + lo halves, three MMAs per product) -------------
# Gates derived from the arithmetic: each split-node product carries the dropped
# lo*lo term (<= 2^-22 relative to |a||b|) and the rounding of the lo halves (<= 2^-25 absolute
# against a column max in [1, 2)), the leaves are FP32 (u = 2^-24).  Measured on B200 at
# 4096 x 1024: backward 4e-7..1.2e-6, R 4.5e-7..5.3e-6 (kappa <= 1e3), orthogonality <= 3.9e-4
# (geometric 1e3); the gates sit 8-40x above.
@pytest.mark.parametrize("kind,cond", [("gaussian", 1), ("geometric", 1e2), ("arithmetic", 1e3),
                                       ("geometric", 1e3)])
def test_fp16_split_factor_accuracy(tq, kind, cond):
    a = W.make_matrix(kind, 4096, 1024, seed=41, cond=cond)
    _, r_o = rgs(a.astype(np.float64))
    q1, r1 = _factor(tq, a)
    q2, r2 = _factor(tq, a, fp16_split=1)
    tq.set_config()
    assert np.array_equal(r2, np.triu(r2)) and np.all(np.diag(r2) > 0)
    assert backward_error_f(a, q2, r2) <= 1e-5
    assert r_rel_error(r2, r_o) <= 5e-5
    assert orthogonality_f(q2) <= 5e-3
    # the split path is at least 30x more accurate than the plain FP16 path on every metric
    assert backward_error_f(a, q2, r2) * 30 < backward_error_f(a, q1, r1)
    assert r_rel_error(r2, r_o) * 30 < r_rel_error(r1, r_o)


def test_fp16_split_planted_and_scale_bitwise(tq):
    # exact inputs have zero lo halves: the planted pin (P2) still holds bitwise, and the
    # power-of-two scale guard keeps the split path bitwise scale-equivariant (P3)
    a, q_ex, r0 = W.planted_hadamard(1024, 256, seed=201)
    q, r = _factor(tq, a, cutoff=64, panel_rows=256, fp16_split=1)
    assert np.array_equal(r, r0.astype(np.float64)) and np.array_equal(q, q_ex.astype(np.float64))
    g = W.gaussian(2048, 512, seed=43)
    q1, r1 = _factor(tq, g, fp16_split=1)
    q2, r2 = _factor(tq, (g * np.float32(2.0 ** -20)).astype(np.float32), fp16_split=1)
    tq.set_config()
    assert np.array_equal(q1, q2) and np.array_equal(r1 * 2.0 ** -20, r2)


@pytest.mark.parametrize("cond,reorth,max_iters", [(1e5, 0, 200), (1e6, 1, 60)])
def test_fp16_split_lls_ill_conditioned(tq, cond, reorth, max_iters):
    # reading R-A24: geometric kappa = 1e6 does not converge with the single FP16 R; with the split
    # (and NEXT-1) CGLS reaches the FP64 target (B200: 1e5 split 75 iterations, 1e6 split+reorth 18)
    a = W.spectrum_matrix(4096, 1024, "geometric", cond, seed=37)
    b, _ = W.consistent_rhs(a, seed=38)
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    tq.set_config(fp16_split=1, reorth=reorth)
    x, info = tq.lls_solve(tq.to_device_colmajor(a), torch.from_numpy(b).cuda(), tol=1e-10,
                           maxit=3000)
    tq.set_config()
    assert info["converged"] == 1 and info["iterations"] <= max_iters, info
    assert x_rel_error(x.cpu().numpy(), x_o) <= 1e-10


# ---- panels taller than the whole-leaf kernel holds (m > 148 * 256: the K2 panel path) ----------
@pytest.mark.parametrize("m,n,cutoff", [(70001, 128, 128), (65600, 96, 32)])
def test_tall_panel_gates(tq, m, n, cutoff):
    a = W.gaussian(m, n, seed=m % 1000 + n)
    q, r = _factor(tq, a, cutoff=cutoff)
    tq.set_config()
    _, r_o = rgs(a.astype(np.float64))
    be, orth, re = _gates(a, q, r, r_o)
    if n <= cutoff:   # leaves only: FP32 accuracy
        assert be < 1e-5 and re < 1e-4 and orth < 1e-5


def test_tall_panel_breakdown(tq):
    # (the planted pin P2 needs a power-of-4 row count at every Eq. (6) level; the tall path's
    # 8-way tree over 64 blocks has stacks of 8, so it is checked by the gates above instead)
    b = W.gaussian(40000, 64, seed=5)
    b[:, 37] = 0.0
    tq.set_config()
    with pytest.raises(tq.TcqrError) as e:
        tq.factor(tq.to_device_colmajor(b))
    assert e.value.code == 38
