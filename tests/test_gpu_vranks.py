"""GPU parity of the ROW-PARTITIONED product path on one device through
the virtual-rank test seam (include/tcqr.h "Virtual ranks"): P host threads, each with its own
library context and its own row block, run tcqr_factor / tcqr_lls_solve / tcqr_qr_solve with the
same collectives, in the same order, as the NCCL build (R12 / A'r / ||q||^2 allreduces, per-leaf
TSQR allgather = Eq. (6) with the ranks as the top tree level, reading R-A26).

Checked against the CPU oracle: the gathered Q and the replicated R against oracle.qr.rgs (the
north_star gates) and against oracle.dist.dist_rgs run over the same row partition; R and x
bit-identical on every rank; x within 1e-10 of oracle_lls and of oracle.dist.dist_pcgls; the
planted Hadamard fixture (zero-padded ranks, reading R-A8) bitwise; collective counts; and that a
rank failing on its arguments aborts the group instead of hanging it."""
import ctypes
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import workloads as W  # noqa: E402
from oracle.cgls import oracle_lls  # noqa: E402
from oracle.dist import dist_pcgls, dist_rgs  # noqa: E402
from oracle.metrics import (backward_error_f, orthogonality_f, r_rel_error,  # noqa: E402
                            x_rel_error)
from oracle.qr import rgs  # noqa: E402


@pytest.fixture(scope="module")
def tq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_05508_b200 as tq
    tq.init(0)
    yield tq


class ThreadComm:
    """In-process communicator for oracle.dist over P Python threads (numpy, FP64)."""

    def __init__(self, shared, rank):
        self.shared, self.rank, self.size = shared, rank, shared["P"]

    def _exchange(self, x):
        sh = self.shared
        sh["barrier"].wait()
        sh["buf"][self.rank] = np.array(x, dtype=np.float64, copy=True)
        sh["barrier"].wait()
        out = [b.copy() for b in sh["buf"]]
        sh["barrier"].wait()
        return out

    def allreduce_sum(self, x):
        parts = self._exchange(x)
        acc = parts[0]
        for p in parts[1:]:
            acc = acc + p
        return acc

    def allgather(self, x):
        return self._exchange(x)


def _oracle_dist(a, b, bounds, tol=1e-12):
    P = len(bounds) - 1
    shared = {"P": P, "barrier": threading.Barrier(P), "buf": [None] * P}
    out = [None] * P

    def work(r):
        comm = ThreadComm(shared, r)
        lo, hi = bounds[r], bounds[r + 1]
        q, rr = dist_rgs(a[lo:hi], comm, br=256)
        x = None
        if b is not None:
            x, _ = dist_pcgls(a[lo:hi], b[lo:hi], rr, comm, tol=tol, maxit=50)
        out[r] = (q, rr, x)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def _bounds(m, P):
    # contiguous row blocks in rank order, multiples of 4 rows (16-byte aligned sub-views)
    step = -(-m // (4 * P)) * 4
    return [min(r * step, m) for r in range(P)] + [m]


def _cfg(tq, **kw):
    c = tq.default_config()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _vfactor(tq, a, P, **cfg):
    """Factor the rows of a (float32, column-major) across P virtual ranks. Returns per-rank
    (Q_r, R_r, collectives)."""
    m, n = a.shape
    A = tq.to_device_colmajor(a)
    bounds = _bounds(m, P)
    Qs = [tq.colmajor_empty(bounds[r + 1] - bounds[r], n) for r in range(P)]
    Rs = [tq.colmajor_empty(n, n) for _ in range(P)]
    torch.cuda.synchronize()
    c = _cfg(tq, **cfg)

    def fn(r):
        l = tq.lib()
        assert l.tcqr_set_config(ctypes.byref(c)) == 0
        mr = bounds[r + 1] - bounds[r]
        a_ptr = ctypes.c_void_p(A.data_ptr() + 4 * bounds[r])
        rc = l.tcqr_factor(mr, n, a_ptr, m, ctypes.c_void_p(Qs[r].data_ptr()),
                           ctypes.c_void_p(Rs[r].data_ptr()))
        return rc, l.tcqr_last_collective_count()

    res = tq.run_virtual_ranks(P, fn, slot_bytes=max(4 * n * n, 8 << 20))
    torch.cuda.synchronize()
    return ([q.cpu().numpy().astype(np.float64) for q in Qs],
            [r.cpu().numpy().astype(np.float64) for r in Rs], res, bounds)


def _leaves_and_splits(n, c=128):
    if n <= c:
        return 1, 0
    h = 32 * (-(-n // 64))
    l1, s1 = _leaves_and_splits(h, c)
    l2, s2 = _leaves_and_splits(n - h, c)
    return l1 + l2, s1 + s2 + 1


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("leaf_kernel", [1, 2])
def test_vranks_factor_matches_oracle(tq, P, leaf_kernel):
    # leaf_kernel=1: replicated leaves (P x 4096/P rows fit one whole-leaf grid of the rank's SM
    # share); leaf_kernel=2: per-leaf TSQR
    m, n = 4096, 512
    a = W.gaussian(m, n, seed=900 + P)
    qs, rs, res, bounds = _vfactor(tq, a, P, leaf_kernel=leaf_kernel)
    assert all(rc == 0 for rc, _ in res), res
    for r in rs[1:]:
        assert np.array_equal(r, rs[0])                 # R replicated bitwise on all ranks
    q = np.vstack(qs)
    r = rs[0]
    a64 = a.astype(np.float64)
    _, r_o = rgs(a64)
    assert np.array_equal(r, np.triu(r)) and np.all(np.diag(r) > 0)
    assert backward_error_f(a64, q, r) <= 5e-3
    assert orthogonality_f(q) <= 5e-2
    assert r_rel_error(r, r_o) <= 1e-2
    # the same row partition through the FP64 distributed oracle
    od = _oracle_dist(a64, None, bounds)
    assert r_rel_error(r, od[0][1]) <= 1e-2
    q_od = np.vstack([o[0] for o in od])
    assert np.linalg.norm(q - q_od) / np.linalg.norm(q_od) <= 1e-2
    # one allgather per leaf (the leaf's rows, or the local R's), one R12 allreduce per split
    # node, one status
    leaves, splits = _leaves_and_splits(n)
    assert all(cnt == leaves + splits + 1 for _, cnt in res), (res, leaves, splits)


def _chunked_collectives(n, chunk, c=128):
    """Collectives of one factor with the R12 allreduce in column chunks of `chunk` (nodes whose
    right part has >= 2 chunks): leaves + per split node max(1, ceil(w2 / chunk)) + 1 status."""
    def rec(w):
        if w <= c:
            return 1
        h = 32 * (-(-w // 64))
        w2 = w - h
        k = -(-w2 // chunk) if w2 >= 2 * chunk else 1
        return rec(h) + rec(w2) + k
    return rec(n) + 1


def test_vranks_chunked_r12_allreduce(tq, monkeypatch):
    # the R12 allreduce in 64-column chunks on the communication stream, overlapping the TN and NN
    # products (TCQR_AR_CHUNK, read when the virtual contexts are created)
    monkeypatch.setenv("TCQR_AR_CHUNK", "64")
    m, n, P = 4096, 512, 4
    a = W.gaussian(m, n, seed=990)
    qs, rs, res, bounds = _vfactor(tq, a, P)
    assert all(rc == 0 for rc, _ in res), res
    for r in rs[1:]:
        assert np.array_equal(r, rs[0])
    q, r = np.vstack(qs), rs[0]
    a64 = a.astype(np.float64)
    _, r_o = rgs(a64)
    assert backward_error_f(a64, q, r) <= 5e-3
    assert orthogonality_f(q) <= 5e-2
    assert r_rel_error(r, r_o) <= 1e-2
    want = _chunked_collectives(n, 64)
    assert all(cnt == want for _, cnt in res), (res, want)


@pytest.mark.parametrize("P,leaf_kernel,cutoff", [(2, 0, 128), (4, 0, 64), (8, 1, 32)])
def test_vranks_factor_panel_paths(tq, P, leaf_kernel, cutoff):
    # leaf_kernel=0: per-panel TSQR (allgather per 32-column panel) + FP32 intra-leaf allreduces;
    # cutoff 32: tensor-core split nodes down to w = 64 with per-leaf TSQR of 32-column leaves
    m, n = 2048, 256
    a = W.gaussian(m, n, seed=950 + P)
    qs, rs, res, _ = _vfactor(tq, a, P, leaf_kernel=leaf_kernel, cutoff=cutoff)
    assert all(rc == 0 for rc, _ in res), res
    for r in rs[1:]:
        assert np.array_equal(r, rs[0])
    q, r = np.vstack(qs), rs[0]
    a64 = a.astype(np.float64)
    _, r_o = rgs(a64)
    assert backward_error_f(a64, q, r) <= 5e-3
    assert orthogonality_f(q) <= 5e-2
    assert r_rel_error(r, r_o) <= 1e-2


@pytest.mark.parametrize("P,leaf_kernel,cutoff", [(2, 1, 128), (4, 1, 32), (2, 0, 64),
                                                  (4, 0, 128)])
def test_vranks_planted_hadamard_zero_padded_bitwise(tq, P, leaf_kernel, cutoff):
    # P2 with zero padding: rank 0 holds the 1024 Hadamard rows, the other ranks
    # zeros (locally zero blocks, reading R-A8) -> R == R0 and Q == [H/sqrt(m); 0] bitwise
    mh, n = 1024, 256
    a0, qt, r0 = W.planted_hadamard(mh, n, seed=201)
    m = mh * P
    a = np.zeros((m, n), dtype=np.float32, order="F")
    a[:mh] = a0
    # 256-row CAQR blocks on the per-panel path (powers of 4 keep every norm exact, P2)
    qs, rs, res, bounds = _vfactor(tq, a, P, leaf_kernel=leaf_kernel, cutoff=cutoff,
                                   panel_rows=256)
    assert bounds[1] == mh
    assert all(rc == 0 for rc, _ in res), res
    for r in rs:
        assert np.array_equal(r, r0)
    assert np.array_equal(qs[0], qt)
    for q in qs[1:]:
        assert not np.any(q)


def test_vranks_planted_hadamard_replicated_leaves_bitwise(tq):
    # P2 through the replicated leaves: 4 x 1024 Hadamard rows gathered into one 4096-row leaf
    # (128-row K2L blocks, 64-row MGS blocks: powers of 4) -> R == R0 and Q == H / sqrt(m)
    # bitwise on every rank, and Q identical to the one-GPU factorization
    m, n, P = 4096, 256, 4
    a, qt, r0 = W.planted_hadamard(m, n, seed=205)
    qs, rs, res, bounds = _vfactor(tq, a, P, leaf_kernel=1)
    assert all(rc == 0 for rc, _ in res), res
    for r in rs:
        assert np.array_equal(r, r0)
    assert np.array_equal(np.vstack(qs), qt)


def test_vranks_planted_hadamard_all_ranks_bitwise(tq):
    # P2 at 16384 = 4 x 4096 rows, every rank holding Hadamard rows (no padding): each rank's
    # 256-row K2L blocks, 64-row MGS blocks and its 64-block local stack, and the 4-rank stack, are
    # all powers of 4 -> R == R0 and Q == H / sqrt(m) bitwise on every rank
    m, n, P = 16384, 256, 4
    a, qt, r0 = W.planted_hadamard(m, n, seed=204)
    qs, rs, res, bounds = _vfactor(tq, a, P)
    assert all(rc == 0 for rc, _ in res), res
    for r in rs:
        assert np.array_equal(r, r0)
    assert np.array_equal(np.vstack(qs), qt)


def _vlls(tq, a, b, P, tol=1e-10, maxit=200, **cfg):
    m, n = a.shape
    A = tq.to_device_colmajor(a)
    B = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).cuda()
    bounds = _bounds(m, P)
    X = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
    torch.cuda.synchronize()
    c = _cfg(tq, **cfg)

    def fn(r):
        l = tq.lib()
        assert l.tcqr_set_config(ctypes.byref(c)) == 0
        info = tq.TcqrLlsInfo()
        mr = bounds[r + 1] - bounds[r]
        rc = l.tcqr_lls_solve(mr, n, ctypes.c_void_p(A.data_ptr() + 4 * bounds[r]), m,
                              ctypes.c_void_p(B.data_ptr() + 8 * bounds[r]),
                              ctypes.c_void_p(X[r].data_ptr()), tol, maxit, ctypes.byref(info))
        return rc, info.as_dict()

    res = tq.run_virtual_ranks(P, fn, slot_bytes=max(4 * n * n, 8 << 20))
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in X], res, bounds


@pytest.mark.parametrize("P", [2, 4, 8])
def test_vranks_lls_fp64_target(tq, P):
    m, n = 4096, 256
    a = W.gaussian(m, n, seed=960 + P)
    b, _ = W.consistent_rhs(a, seed=961 + P)
    xs, res, bounds = _vlls(tq, a, b, P)
    assert all(rc == 0 for rc, _ in res), res
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])                 # x replicated bitwise
    assert all(info["converged"] == 1 for _, info in res)
    a64 = a.astype(np.float64)
    x_o, _ = oracle_lls(a64, b)
    assert x_rel_error(xs[0], x_o) <= 1e-10
    od = _oracle_dist(a64, b, bounds, tol=1e-14)
    assert x_rel_error(xs[0], od[0][2]) <= 1e-10


def test_vranks_lls_ill_conditioned(tq):
    # arithmetic kappa = 1e3 (Fig. 2 family), FP64 target through the restart rule (R-A12)
    m, n, P = 4096, 256, 4
    a = W.spectrum_matrix(m, n, "arithmetic", 1e3, seed=970)
    b, _ = W.consistent_rhs(a, seed=971)
    xs, res, _ = _vlls(tq, a, b, P)
    assert all(rc == 0 for rc, _ in res), res
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])
    x_o, _ = oracle_lls(a.astype(np.float64), b)
    assert x_rel_error(xs[0], x_o) <= 1e-10


def test_vranks_qr_solve(tq):
    # NEXT-2 at P > 1: x = R^-1 (Q'b) with Q'b allreduced; equals the direct solve on the
    # gathered factors
    m, n, P = 2048, 128, 4
    a = W.gaussian(m, n, seed=980)
    b, _ = W.consistent_rhs(a, seed=981)
    qs, rs, res, bounds = _vfactor(tq, a, P)
    Qd = [tq.to_device_colmajor(q.astype(np.float32)) for q in qs]
    Rd = tq.to_device_colmajor(rs[0].astype(np.float32))
    Bd = torch.from_numpy(b).cuda()
    X = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
    torch.cuda.synchronize()

    def fn(r):
        l = tq.lib()
        mr = bounds[r + 1] - bounds[r]
        return l.tcqr_qr_solve(mr, n, ctypes.c_void_p(Qd[r].data_ptr()), mr,
                               ctypes.c_void_p(Rd.data_ptr()), n,
                               ctypes.c_void_p(Bd.data_ptr() + 8 * bounds[r]),
                               ctypes.c_void_p(X[r].data_ptr()))

    rcs = tq.run_virtual_ranks(P, fn)
    assert rcs == [0] * P
    xs = [x.cpu().numpy() for x in X]
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])
    q, r = np.vstack(qs), rs[0]
    x_ref = np.linalg.solve(r, q.T @ b)
    assert x_rel_error(xs[0], x_ref) <= 1e-9


def test_vranks_bad_argument_aborts_group(tq):
    # rank 1 passes lda < m: it returns -4 at once and aborts the group; rank 0, already inside
    # its factorization, gets an error from its first collective instead of waiting forever
    m, n, P = 1024, 256, 2
    a = W.gaussian(m, n, seed=990)
    A = tq.to_device_colmajor(a)
    Q = tq.colmajor_empty(m, n)
    R = [tq.colmajor_empty(n, n) for _ in range(P)]
    torch.cuda.synchronize()

    def fn(r):
        l = tq.lib()
        lda = m if r == 0 else 4
        return l.tcqr_factor(m // 2, n, ctypes.c_void_p(A.data_ptr() + 4 * r * (m // 2)), lda,
                             ctypes.c_void_p(Q.data_ptr() + 4 * r * (m // 2)),
                             ctypes.c_void_p(R[r].data_ptr()))

    rcs = tq.run_virtual_ranks(P, fn, timeout=300)
    assert rcs[1] == -4
    assert rcs[0] != 0
