"""GPU parity of the individual hot-path kernels through the C ABI.

Each kernel is compared element by element with a plain float64 reference built from the SAME
rounded inputs (oracle.fp16 for the FP16 rounding), at sizes spanning several tiles and ragged
edges. Tolerances: FP16 cast bitwise; tensor-core GEMMs within the FP32-accumulation envelope
|gpu - ref| <= k 2^-22 ||row|| ||col||; FP32 panel within 1e-5 of the FP64 oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import workloads as W  # noqa: E402
from oracle.fp16 import fl16, pow2_colscale  # noqa: E402
from oracle.metrics import orthogonality_f, r_rel_error  # noqa: E402
from oracle.qr import caqr, mgs  # noqa: E402


@pytest.fixture(scope="module")
def tq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_05508_b200 as tq
    tq.init(0)
    return tq


def _h2np(xh):
    return xh.float().cpu().numpy().astype(np.float64)


# (20000, 3): five 4096-row CTAs per cluster with a ragged last one; (40000, 2): the 8192-row
# cluster variant; (70000, 2): past the cluster path (memset + colmax + cast_pass2)
@pytest.mark.parametrize("m,w", [(1000, 7), (4096, 33), (37, 3), (20000, 3), (32768, 4),
                                 (40000, 2), (70000, 2)])
def test_cast_scale_bitwise(tq, m, w):
    rng = np.random.default_rng(m)
    x = (rng.standard_normal((m, w)) * np.exp2(rng.integers(-30, 20, w))).astype(np.float32)
    x[:, 1] = 0.0
    X = tq.to_device_colmajor(x)
    Xh, inv_s = tq.cast_scale(X, scaling=True)
    s = pow2_colscale(x.astype(np.float64))
    ref = fl16(x.astype(np.float64) * s)
    assert np.array_equal(_h2np(Xh), ref)
    assert np.array_equal(inv_s.cpu().numpy().astype(np.float64), 1.0 / s)
    Xh2, _ = tq.cast_scale(X, scaling=False)
    with np.errstate(over="ignore"):
        assert np.array_equal(_h2np(Xh2), fl16(x.astype(np.float64)))


def test_cast_flags_nonfinite(tq):
    x = np.ones((300, 5), np.float32)
    x[17, 3] = np.nan
    X = tq.to_device_colmajor(x)
    with pytest.raises(tq.TcqrError) as e:
        tq.cast_scale(X)
    assert e.value.code == 4


def test_cast_flags_nonfinite_late_chunk(tq):
    """Non-finite entry in the last row chunk of a multi-CTA column (cluster cast path)."""
    x = np.ones((32768, 3), np.float32)
    x[30001, 2] = np.inf
    X = tq.to_device_colmajor(x)
    with pytest.raises(tq.TcqrError) as e:
        tq.cast_scale(X)
    assert e.value.code == 3


def _fp16_operand(rng, m, k, scale=1.0):
    return fl16(rng.standard_normal((m, k)) * scale)


@pytest.mark.parametrize("m,h,w2", [(64, 128, 128), (1000, 96, 200), (4160, 128, 384),
                                    (8192, 300, 130), (262144, 128, 128),
                                    # h, w2 >= 256: the CTA-pair (cta_group::2) kernel, with
                                    # ragged 256-tiles and split-K / no split
                                    (8192, 512, 384), (4104, 300, 640), (16384, 2048, 1024),
                                    (96, 256, 256)])
def test_gemm_tn_envelope(tq, m, h, w2):
    rng = np.random.default_rng(h + w2)
    a1 = _fp16_operand(rng, m, h)
    a2 = _fp16_operand(rng, m, w2)
    mult = np.exp2(rng.integers(-3, 3, w2)).astype(np.float32)
    A1 = tq.to_device_colmajor(a1, dtype=torch.float16)
    A2 = tq.to_device_colmajor(a2, dtype=torch.float16)
    C = tq.gemm_tn(A1, A2, torch.from_numpy(mult).cuda()).cpu().numpy().astype(np.float64)
    ref = (a1.T @ a2) * mult
    env = 8 * 2.0 ** -22 * np.outer(np.linalg.norm(a1, axis=0), np.linalg.norm(a2, axis=0)) * mult
    err = np.abs(C - ref)
    assert np.all(err <= env + 1e-30), float(np.max(err / env))


@pytest.mark.parametrize("m,h,w2", [(128, 64, 128), (1000, 96, 200), (4160, 256, 384),
                                    (3000, 512, 64),
                                    # K = h <= 256: the two-CTAs-per-SM short-K variant, with more
                                    # tiles than CTA slots (persistent loop) and ragged rows/columns
                                    (40000, 128, 256), (33000, 200, 130), (70000, 256, 128),
                                    # K = h in (512, 1024]: the short-K variant with a long K loop
                                    (20000, 1000, 200), (8192, 1024, 1024),
                                    # h > 2048, w2 >= 256: the CTA-pair kernel (ragged tiles)
                                    (4104, 2304, 320), (704, 4096, 256)])
def test_gemm_nn_update_envelope(tq, m, h, w2):
    rng = np.random.default_rng(m + h)
    qh = _fp16_operand(rng, m, h, 0.05)
    bh = _fp16_operand(rng, h, w2)
    c = rng.standard_normal((m, w2)).astype(np.float32)
    mult = np.exp2(rng.integers(-3, 3, w2)).astype(np.float32)
    Q = tq.to_device_colmajor(qh, dtype=torch.float16)
    B = tq.to_device_colmajor(bh, dtype=torch.float16)
    C = tq.to_device_colmajor(c)
    tq.gemm_nn_update(C, Q, B, torch.from_numpy(mult).cuda())
    got = C.cpu().numpy().astype(np.float64)
    ref = c.astype(np.float64) - (qh @ bh) * mult
    env = 8 * 2.0 ** -22 * np.outer(np.linalg.norm(qh, axis=1), np.linalg.norm(bh, axis=0)) * mult \
        + 2.0 ** -23 * np.abs(ref) * 2
    assert np.all(np.abs(got - ref) <= env + 1e-30), float(np.max(np.abs(got - ref) / env))


def test_gemm_exact_small_integers(tq):
    # FP16 small integers: products and sums exact in FP32 -> bitwise (SPEC.md:58 analogue).
    rng = np.random.default_rng(5)
    a1 = rng.integers(-3, 4, (512, 128)).astype(np.float64)
    a2 = rng.integers(-3, 4, (512, 256)).astype(np.float64)
    A1 = tq.to_device_colmajor(a1, dtype=torch.float16)
    A2 = tq.to_device_colmajor(a2, dtype=torch.float16)
    C = tq.gemm_tn(A1, A2).cpu().numpy().astype(np.float64)
    assert np.array_equal(C, a1.T @ a2)


@pytest.mark.parametrize("m,w,br", [(256, 32, 256), (300, 32, 256), (1024, 32, 256),
                                    (4096, 32, 256), (70000, 32, 256), (5000, 17, 128),
                                    (33, 32, 64), (32768, 32, 1024), (5000, 17, 1024),
                                    (70000, 32, 1024), (1000, 32, 1024), (200000, 32, 1024)])
def test_panel_vs_oracle(tq, m, w, br):
    a = W.gaussian(m, w, seed=m + w)
    X = tq.to_device_colmajor(a)
    Xq, R = tq.panel_qr(X, br=br)
    q, r = Xq.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    _, r_o = mgs(a.astype(np.float64))
    assert np.array_equal(r, np.triu(r)) and np.all(np.diag(r) > 0)
    assert r_rel_error(r, r_o) < 1e-5
    assert orthogonality_f(q) < 1e-5
    assert np.linalg.norm(a - q @ r) / np.linalg.norm(a) < 1e-6


@pytest.mark.parametrize("m,br", [(1024, 256), (4096, 1024), (1024, 1024), (16384, 1024)])
def test_panel_planted_hadamard_bitwise(tq, m, br):
    # block rows, rank-local rows and the number of stacked R's are powers of 4
    a, qt, r0 = W.planted_hadamard(m, 32, seed=201)
    X = tq.to_device_colmajor(a)
    Xq, R = tq.panel_qr(X, br=br)
    assert np.array_equal(R.cpu().numpy().astype(np.float64), r0)
    assert np.array_equal(Xq.cpu().numpy().astype(np.float64), qt)


def test_trinv_and_gemv(tq):
    rng = np.random.default_rng(9)
    n = 300
    r = np.linalg.qr(rng.standard_normal((2 * n, n)))[1]       # well-conditioned triangle
    r = (r * np.sign(np.diag(r))[:, None]).astype(np.float32)
    M = tq.trinv(tq.to_device_colmajor(r)).cpu().numpy()
    res = np.linalg.norm(r.astype(np.float64) @ M - np.eye(n)) / np.sqrt(n)
    assert res < 1e-12
    a = rng.standard_normal((1000, n)).astype(np.float32)
    A = tq.to_device_colmajor(a)
    v = rng.standard_normal(n)
    y = tq.gemv(A, torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.allclose(y, a.astype(np.float64) @ v, rtol=1e-12, atol=1e-10)
    u = rng.standard_normal(1000)
    z = tq.gemv(A, torch.from_numpy(u).cuda(), trans=True).cpu().numpy()
    assert np.allclose(z, a.astype(np.float64).T @ u, rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("n", [300, 1000, 2100])
def test_trinv_large_tiles(tq, n):
    # the 128 x 128 FP64 pair-GEMM path (b >= 128) against the FP64 residual R M - I
    rng = np.random.default_rng(n)
    r = np.linalg.qr(rng.standard_normal((2 * n, n)))[1]
    r = (r * np.sign(np.diag(r))[:, None]).astype(np.float32)
    M = tq.trinv(tq.to_device_colmajor(r)).cpu().numpy()
    assert np.array_equal(M, np.triu(M))
    assert np.linalg.norm(r.astype(np.float64) @ M - np.eye(n)) / np.sqrt(n) < 1e-12


def test_reorth_product_is_r2_r1(tq):
    # tcqr_factor with reorth: A = Q2 (R2 R1); R2 R1 upper triangular (trmm kernel), n >= 512 path
    a = W.gaussian(2048, 640, seed=3)
    tq.set_config(reorth=1)
    A = tq.to_device_colmajor(a)
    Q, R = tq.factor(A)
    tq.set_config()
    q, r = Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    assert np.array_equal(r, np.triu(r))
    assert np.linalg.norm(a - q @ r) / np.linalg.norm(a) < 5e-3
    assert orthogonality_f(q) < 5e-4      # FP16-GEMM level: the second pass cannot go below it


def test_panel_nonfinite_data_does_not_stall(tq):
    # the pipelined panel hands values over through a sentinel bit pattern; a NaN/Inf in the data
    # must flow through (and be reported by the status), never be taken for "not yet written"
    X = W.gaussian_cuda(32768, 32, 61)
    X[1234, 7] = float("nan")
    X[99, 20] = float("inf")
    with pytest.raises(tq.TcqrError):
        tq.panel_qr(X, br=1024)
    # the next panel on clean data still works (sentinels were reset)
    X2 = W.gaussian_cuda(32768, 32, 62)
    Xq, R = tq.panel_qr(X2.clone(), br=1024)
    q = Xq.double().cpu().numpy()
    assert np.linalg.norm(q.T @ q - np.eye(32)) < 1e-4
