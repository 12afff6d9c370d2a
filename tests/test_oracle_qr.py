"""Pins for oracle.qr (P2-P7 of SURVEY.md §8c.4). Nothing here is checked against the oracle itself:
closed forms (golden tiny cases, planted Hadamard), brute-force Householder, exact-precision
Cholesky of A'A (mpmath), invariants (Eq. 5 assembly, triu, diag > 0), and the paper's stated
trends (backward error flat vs kappa, orthogonality loss growing with kappa)."""
import mpmath
import numpy as np
import pytest

import workloads as W
from conftest import golden_lines
from oracle.householder import householder_qr
from oracle.metrics import (backward_error_f, flops_convention, flops_rgs_exec,
                            orthogonality_f, orthogonality_2_over_n, r_rel_error)
from oracle.qr import Breakdown, caqr, caqr_blocks, mgs, rgs, split_point


def _golden_qr():
    for line in golden_lines("tiny_qr.txt"):
        name, mn, a, q, r = [t.strip() for t in line.split(";")]
        m, n = map(int, mn.split())
        f = lambda s, sh: np.array(s.split(), float).reshape(sh[::-1]).T
        yield name, f(a, (m, n)), f(q, (m, n)), f(r, (n, n))


@pytest.mark.parametrize("fn", ["mgs", "caqr", "rgs32", "rgs_c1"])
def test_golden_tiny(fn):
    for name, a, q0, r0 in _golden_qr():
        if fn == "mgs":
            q, r = mgs(a)
        elif fn == "caqr":
            q, r = caqr(a, br=2)
        elif fn == "rgs32":
            q, r = rgs(a)
        else:
            q, r = rgs(a, pw=1)
        assert np.allclose(q, q0, atol=1e-15) and np.allclose(r, r0, atol=1e-15), name


def test_orthogonal_columns_give_diagonal_r():
    # columns [3e, 4f] for orthonormal e, f -> R = diag(3, 4)
    rng = np.random.default_rng(3)
    e, _ = np.linalg.qr(rng.standard_normal((40, 2)))
    a = np.column_stack([3 * e[:, 0], 4 * e[:, 1]])
    q, r = rgs(a)
    assert np.allclose(r, np.diag([3.0, 4.0]), atol=1e-14)


def test_mgs_is_row_oriented_alg4():
    # Alg. 4 line 7 uses the already-updated trailing columns (R-A7). On a 3-column example the
    # CGS and MGS R(2,3) entries differ in floating point for nearly dependent columns; check
    # the MGS-specific orthogonality advantage against Householder on a Lauchli-type matrix.
    eps = 1e-6
    a = np.array([[1, 1, 1], [eps, 0, 0], [0, eps, 0], [0, 0, eps]], float)
    q, r = mgs(a)
    # MGS: |q2'q3| ~ eps/sqrt(2)*... stays O(1e-11); CGS gives ~0.5 on this example.
    assert abs(q[:, 1] @ q[:, 2]) < 1e-9


@pytest.mark.parametrize("m,n", [(64, 16), (300, 40), (257, 96)])
def test_rgs_matches_householder(m, n):
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    qh, rh = householder_qr(a)
    for kw in [dict(), dict(panel="caqr", br=64), dict(pw=8), dict(panel="caqr", br=32, pw=16)]:
        q, r = rgs(a, **kw)
        assert r_rel_error(r, rh) < 1e-12, kw
        assert np.max(np.abs(q - qh)) < 1e-12, kw
        assert np.array_equal(r, np.triu(r)) and np.all(np.diag(r) > 0)
        assert backward_error_f(a, q, r) < 1e-14                    # Eq. (5) assembly


def test_rgs_r_is_cholesky_of_gram_mpmath():
    # R'R = A'A with diag(R) > 0 => R = chol(A'A); computed at 50 digits (P5).
    rng = np.random.default_rng(7)
    a = rng.standard_normal((12, 5))
    mpmath.mp.dps = 50
    g = mpmath.matrix(a.T.tolist()) * mpmath.matrix(a.tolist())
    l = mpmath.cholesky(g)
    rc = np.array([[float(l[j, i]) for j in range(5)] for i in range(5)])  # R = L'
    _, r = rgs(a, pw=2)
    assert r_rel_error(r, rc) < 1e-14


def test_caqr_blocks_ragged():
    assert caqr_blocks(1024, 256, 32) == [(0, 256), (256, 256), (512, 256), (768, 256)]
    assert caqr_blocks(300, 256, 32) == [(0, 256), (256, 44)]
    assert caqr_blocks(270, 256, 32) == [(0, 270)]               # remainder 14 < 32 folded
    assert caqr_blocks(530, 256, 32) == [(0, 256), (256, 274)]
    assert caqr_blocks(100, 256, 32) == [(0, 100)]


@pytest.mark.parametrize("m", [256, 300, 1024, 4096])
def test_caqr_equals_full_panel_mgs(m):
    # SPEC.md:509 acceptance 9 / Eq. (6) product-of-orthogonals
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, 32))
    q0, r0 = mgs(a)
    q, r = caqr(a, br=256)
    if m <= 256:
        assert np.array_equal(q, q0) and np.array_equal(r, r0)     # single block == Alg. 4
    assert r_rel_error(r, r0) < 1e-13
    assert orthogonality_f(q) < 1e-14
    assert backward_error_f(a, q, r) < 1e-14


def test_caqr_local_zero_block_rank_ok():
    # R-A8: a locally zero block (rows of zeros) is not an error when A has full rank.
    rng = np.random.default_rng(5)
    a = rng.standard_normal((1024, 32))
    a[256:512] = 0.0
    q, r = caqr(a, br=256)
    assert orthogonality_f(q) < 1e-14 and np.all(np.diag(r) > 0)
    with pytest.raises(Breakdown) as e:
        b = a.copy()
        b[:, 7] = 0.0
        caqr(b, br=256)
    assert e.value.col == 7


def test_rgs_breakdown_reports_global_column():
    rng = np.random.default_rng(6)
    a = rng.standard_normal((200, 100))
    a[:, 77] = 0.0
    with pytest.raises(Breakdown) as e:
        rgs(a)
    assert e.value.col == 77


def test_split_point():
    assert [split_point(w) for w in (64, 96, 128, 160, 16384, 4097)] == [32, 64, 64, 96, 8192, 2080]


@pytest.mark.parametrize("cutoff,n", [(32, 128), (128, 128), (32, 256), (128, 256)])
def test_planted_hadamard_fp16_bitwise(cutoff, n):
    # P2: every FP16 cast, dot and norm is exact -> R == R0 and Q == H/sqrt(m) bitwise.
    a, qt, r0 = W.planted_hadamard(1024, n, seed=201)
    q, r = rgs(a, cutoff=cutoff, panel="caqr", br=256, gemm="fp16")
    assert np.array_equal(r, r0)
    assert np.array_equal(q, qt)


def test_planted_hadamard_128_row_blocks_not_exact():
    # [calib]: with 128-row blocks (not a power of 4) the local norms are irrational.
    a, qt, r0 = W.planted_hadamard(1024, 64, seed=201)
    _, r = rgs(a, cutoff=32, panel="caqr", br=128, gemm="fp16")
    assert not np.array_equal(r, r0)
    assert r_rel_error(r, r0) < 1e-12


def test_scale_equivariance_fp16_bitwise():
    # P3: with power-of-two column scaling the FP16 method is exactly scale-equivariant.
    a = W.gaussian(512, 128, seed=11).astype(np.float64)
    q, r = rgs(a, cutoff=32, gemm="fp16")
    for e in (-30, -7, 5, 20):
        qe, re = rgs(np.ldexp(a, e), cutoff=32, gemm="fp16")
        assert np.array_equal(qe, q) and np.array_equal(re, np.ldexp(r, e)), e


def test_fp16_emulation_accuracy_gaussian():
    # north_star gates on the emulated method (the GPU must meet the same gates).
    a = W.gaussian(2048, 512, seed=1).astype(np.float64)
    q, r = rgs(a, cutoff=128, gemm="fp16")
    _, ro = rgs(a)
    assert backward_error_f(a, q, r) < 5e-3
    assert orthogonality_f(q) < 5e-2
    assert r_rel_error(r, ro) < 1e-2


def test_backward_error_flat_orthogonality_grows():
    # PAPER.md:503-510 and :607-608 (Fig. 2 trends); SPEC.md:501-502 acceptance 1-2.
    be, orth = [], []
    for k, cond in enumerate([1e1, 1e2, 1e3, 1e4, 1e5, 1e6]):
        a = W.spectrum_matrix(1024, 256, "arithmetic", cond, seed=40 + k).astype(np.float64)
        q, r = rgs(a, cutoff=32, gemm="fp16")
        be.append(backward_error_f(a, q, r))
        orth.append(orthogonality_2_over_n(q))
    assert max(be) < 1e-3 and max(be) / min(be) < 10
    assert orth[-1] / orth[0] > 10
    for i in range(1, len(orth)):
        assert orth[i] >= orth[i - 1] / 3


def test_flops_match_paper_and_survey_table():
    for line in golden_lines("flops_configs.txt"):
        m, n, conv, exe = line.split()
        m, n = int(m), int(n)
        assert abs(flops_convention(m, n) / float(conv) - 1) < 5e-3
        assert abs(flops_rgs_exec(m, n) / float(exe) - 1) < 5e-3


def test_flops_exec_is_count_of_split_tree():
    # Count multiply-adds of the actual recursion (split nodes: R12 2mhw2 + update 2mhw2;
    # panels: MGS ~2mw^2) and compare with 2mn^2 for power-of-two n.
    def count(m, w, pw=32):
        if w <= pw:
            return 2 * m * w * w
        h = split_point(w)
        return count(m, h, pw) + 4 * m * h * (w - h) + count(m, w - h, pw)
    for m, n in [(1024, 128), (32768, 16384), (262144, 2048)]:
        assert count(m, n) == flops_rgs_exec(m, n)
