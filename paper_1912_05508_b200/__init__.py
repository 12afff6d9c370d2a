"""paper_1912_05508_b200 -- thin Python binding of libtcqr.so (include/tcqr.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of the C-ABI
library. PyTorch provides device memory, the current stream and torch.distributed (to broadcast
the NCCL unique id); it never computes any part of the method. There is no CPU fallback: if the
library is missing or the device is not sm_100, every call raises.

Matrices are column-major (the C ABI's layout): an m x n matrix is a torch tensor of shape (m, n)
with stride (1, ld), e.g. ``colmajor_empty(m, n)`` == ``torch.empty(n, m).t()``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtcqr.so")

_lib = None


class TcqrError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} returned {code}")
        self.code = code


class TcqrConfig(ctypes.Structure):
    _fields_ = [("cutoff", ctypes.c_int), ("panel_rows", ctypes.c_int),
                ("col_scaling", ctypes.c_int), ("restart", ctypes.c_int),
                ("tol2", ctypes.c_double), ("stag_window", ctypes.c_int),
                ("stag_floor", ctypes.c_double), ("use_graphs", ctypes.c_int),
                ("reorth", ctypes.c_int), ("warm_start", ctypes.c_int),
                ("leaf_kernel", ctypes.c_int), ("fp16_split", ctypes.c_int)]


class TcqrLlsInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("iterations_pass1", ctypes.c_int),
                ("outer_passes", ctypes.c_int), ("converged", ctypes.c_int),
                ("stop_reason", ctypes.c_int), ("s0", ctypes.c_double),
                ("final_rel", ctypes.c_double), ("qr_ms", ctypes.c_double),
                ("cgls_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_SIGS = {
    "tcqr_init": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int]),
    "tcqr_nccl_unique_id": (ctypes.c_int, [_P]),
    "tcqr_finalize": (ctypes.c_int, []),
    "tcqr_default_config": (None, [ctypes.POINTER(TcqrConfig)]),
    "tcqr_set_config": (ctypes.c_int, [ctypes.POINTER(TcqrConfig)]),
    "tcqr_workspace_size": (ctypes.c_int, [_I64, _I64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "tcqr_set_workspace": (ctypes.c_int, [_P, ctypes.c_size_t]),
    "tcqr_factor": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _P]),
    "tcqr_lls_solve": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _P, ctypes.c_double, ctypes.c_int,
                                      ctypes.POINTER(TcqrLlsInfo)]),
    "tcqr_factor_host": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _P]),
    "tcqr_lls_solve_host": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _P, ctypes.c_double,
                                           ctypes.c_int, ctypes.POINTER(TcqrLlsInfo)]),
    "tcqr_cast_scale": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _I64, _P, ctypes.c_int]),
    "tcqr_gemm_tn": (ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "tcqr_gemm_nn_update": (ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "tcqr_panel_qr": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _I64, ctypes.c_int]),
    "tcqr_trinv": (ctypes.c_int, [_I64, _P, _I64, _P, _I64]),
    "tcqr_qr_solve": (ctypes.c_int, [_I64, _I64, _P, _I64, _P, _I64, _P, _P]),
    "tcqr_gemv": (ctypes.c_int, [ctypes.c_int, _I64, _I64, _P, _I64, _P, _P]),
    "tcqr_version": (ctypes.c_char_p, []),
    "tcqr_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tcqr_profile_read": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_int)]),
    "tcqr_last_launch_count": (ctypes.c_int, []),
    "tcqr_last_collective_count": (ctypes.c_int, []),
    "tcqr_vgroup_create": (ctypes.c_void_p, [ctypes.c_int, ctypes.c_size_t]),
    "tcqr_init_virtual": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int]),
    "tcqr_vgroup_destroy": (ctypes.c_int, [_P]),
}
PROFILE_CLASSES = ["copy", "k1_cast", "k3_tn", "k3_finalize", "k4_nn", "k2_mgs", "k2_apply",
                   "k2b_tn", "k2b_nn", "k5_gemv", "k6_tri", "k7_scalar", "trinv", "k2_leaf"]
EXPORTS = tuple(_SIGS)


def lib():
    """Load libtcqr.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C csrc)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _check(fn, rc):
    if rc != 0:
        raise TcqrError(fn, rc)


# ------------------------------------------------------------------------------------------
# torch helpers (memory only)
# ------------------------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def colmajor_empty(m, n, dtype=None, device="cuda"):
    torch = _torch()
    return torch.empty((n, m), dtype=dtype or torch.float32, device=device).t()


def to_device_colmajor(a_np, dtype=None, device="cuda"):
    """numpy (any order) m x n -> column-major CUDA tensor (shape (m, n), stride (1, m))."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(a_np).T))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device).t()


def _ld(x):
    """Leading dimension of a column-major (m, n) tensor; rejects other layouts."""
    m, n = x.shape
    if x.stride(0) != 1 and not (n == 1 or m == 1):
        raise ValueError(f"expected a column-major view (stride (1, ld)), got stride {x.stride()}")
    return x.stride(1) if n > 1 else max(m, 1)


def _ptr(x):
    return ctypes.c_void_p(x.data_ptr())


def _need(x, what, dtype, shape, device=None, ld=None):
    """Validate a tensor argument before it reaches the C ABI (which trusts sizes and layouts):
    CUDA residency, dtype, shape, and for matrices the column-major leading dimension."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if x.dtype != dtype:
        raise ValueError(f"{what}: expected {dtype}, got {x.dtype}")
    if tuple(x.shape) != tuple(shape):
        raise ValueError(f"{what}: expected shape {tuple(shape)}, got {tuple(x.shape)}")
    if device is not None and x.device != device:
        raise ValueError(f"{what}: on {x.device}, expected {device}")
    if len(shape) == 1:
        if x.numel() > 1 and x.stride(0) != 1:
            raise ValueError(f"{what}: expected a contiguous vector, got stride {x.stride()}")
    elif ld is not None and _ld(x) != ld:
        raise ValueError(f"{what}: expected leading dimension {ld}, got {_ld(x)}")


_state = {"inited": False, "device": None, "ws": None}


def init(device=0, stream=None, nccl_id=None, rank=0, nranks=1):
    """tcqr_init on `device` with torch's current stream (or `stream`)."""
    torch = _torch()
    torch.cuda.set_device(device)
    if stream is None:
        stream = torch.cuda.current_stream(device)
    sp = ctypes.c_void_p(stream.cuda_stream)
    idp = None
    if nccl_id is not None:
        idp = ctypes.cast(ctypes.create_string_buffer(bytes(nccl_id), 128), ctypes.c_void_p)
    _check("tcqr_init", lib().tcqr_init(device, sp, idp, rank, nranks))
    _state.update(inited=True, device=device, ws=None)


def init_distributed():
    """One process per GPU under torchrun: rank 0 makes the NCCL id, torch.distributed broadcasts
    it, every rank calls tcqr_init(local_rank, ...). torch.distributed must be initialized."""
    torch = _torch()
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        raw = ctypes.create_string_buffer(128)
        _check("tcqr_nccl_unique_id", lib().tcqr_nccl_unique_id(raw))
        buf = torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8).clone()
    if dist.get_backend() == "nccl":
        buf = buf.cuda(local)
    dist.broadcast(buf, 0)
    init(device=local, nccl_id=bytes(buf.cpu().numpy().tobytes()), rank=rank, nranks=world)


def finalize():
    lib().tcqr_finalize()
    _state.update(inited=False, ws=None)


def _ensure():
    if not _state["inited"]:
        init(0)


def default_config() -> TcqrConfig:
    c = TcqrConfig()
    lib().tcqr_default_config(ctypes.byref(c))
    return c


def set_config(**kw):
    _ensure()
    c = default_config()
    for k, v in kw.items():
        setattr(c, k, v)
    _check("tcqr_set_config", lib().tcqr_set_config(ctypes.byref(c)))


def reserve_workspace(m, n, op=1):
    """Allocate the library workspace as a torch tensor (torch owns device memory)."""
    torch = _torch()
    _ensure()
    nb = ctypes.c_size_t(0)
    _check("tcqr_workspace_size", lib().tcqr_workspace_size(m, n, op, ctypes.byref(nb)))
    cur = _state["ws"]
    if cur is None or cur.numel() < nb.value:
        ws = torch.empty(nb.value + 1024, dtype=torch.uint8, device=f"cuda:{_state['device']}")
        _check("tcqr_set_workspace", lib().tcqr_set_workspace(_ptr(ws), ws.numel()))
        _state["ws"] = ws
    return _state["ws"]


# ------------------------------------------------------------------------------------------
# Hot-path entry points
# ------------------------------------------------------------------------------------------
def factor(A, Q=None, R=None, in_place=False):
    """A = QR (tcqr_factor). A: CUDA float32 column-major (m, n). Returns (Q, R)."""
    torch = _torch()
    _ensure()
    m, n = A.shape
    _need(A, "A", torch.float32, (m, n))
    lda = _ld(A)
    if in_place:
        if lda != m:
            raise ValueError("in_place needs A with leading dimension m")
        Q = A
    elif Q is None:
        Q = colmajor_empty(m, n, device=A.device)
    if R is None:
        R = colmajor_empty(n, n, device=A.device)
    _need(Q, "Q", torch.float32, (m, n), A.device, ld=m)
    _need(R, "R", torch.float32, (n, n), A.device, ld=n)
    reserve_workspace(m, n, op=0)
    _check("tcqr_factor", lib().tcqr_factor(m, n, _ptr(A), lda, _ptr(Q), _ptr(R)))
    return Q, R


def lls_solve(A, b, tol=1e-10, maxit=200, x=None):
    """min ||Ax - b|| (tcqr_lls_solve). A CUDA float32 column-major, b CUDA float64 (m,).
    Returns (x, info dict)."""
    torch = _torch()
    _ensure()
    m, n = A.shape
    _need(A, "A", torch.float32, (m, n))
    _need(b, "b", torch.float64, (m,), A.device)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=A.device)
    _need(x, "x", torch.float64, (n,), A.device)
    info = TcqrLlsInfo()
    reserve_workspace(m, n, op=1)
    _check("tcqr_lls_solve", lib().tcqr_lls_solve(m, n, _ptr(A), _ld(A), _ptr(b), _ptr(x),
                                                  float(tol), int(maxit), ctypes.byref(info)))
    return x, info.as_dict()


def qr_solve(Q, R, b, x=None):
    """NEXT-2, Alg. 1 lines 3-4: x = R^-1 (Q' b) (tcqr_qr_solve). Q CUDA
    float32 m x n column-major, R float32 n x n column-major, b float64 (m,). Returns x (n,)."""
    torch = _torch()
    _ensure()
    m, n = Q.shape
    _need(Q, "Q", torch.float32, (m, n))
    _need(R, "R", torch.float32, (n, n), Q.device)
    _need(b, "b", torch.float64, (m,), Q.device)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=Q.device)
    _need(x, "x", torch.float64, (n,), Q.device)
    _check("tcqr_qr_solve", lib().tcqr_qr_solve(m, n, _ptr(Q), _ld(Q), _ptr(R), _ld(R), _ptr(b),
                                                _ptr(x)))
    return x


def factor_host(A_np):
    """End-to-end variant on host numpy arrays (H2D and D2H copies inside the call)."""
    _ensure()
    a = np.asfortranarray(A_np, dtype=np.float32)
    m, n = a.shape
    q = np.empty((m, n), dtype=np.float32, order="F")
    r = np.empty((n, n), dtype=np.float32, order="F")
    _check("tcqr_factor_host", lib().tcqr_factor_host(
        m, n, a.ctypes.data_as(_P), m, q.ctypes.data_as(_P), r.ctypes.data_as(_P)))
    return q, r


def lls_solve_host(A_np, b_np, tol=1e-10, maxit=200):
    _ensure()
    a = np.asfortranarray(A_np, dtype=np.float32)
    b = np.ascontiguousarray(b_np, dtype=np.float64)
    m, n = a.shape
    x = np.empty(n, dtype=np.float64)
    info = TcqrLlsInfo()
    _check("tcqr_lls_solve_host", lib().tcqr_lls_solve_host(
        m, n, a.ctypes.data_as(_P), m, b.ctypes.data_as(_P), x.ctypes.data_as(_P), float(tol),
        int(maxit), ctypes.byref(info)))
    return x, info.as_dict()


# ------------------------------------------------------------------------------------------
# Component entry points (parity tests of each step)
# ------------------------------------------------------------------------------------------
def cast_scale(X, scaling=True):
    """K1: returns (Xh as torch.float16 column-major, inv_s float32)."""
    torch = _torch()
    _ensure()
    m, w = X.shape
    ldh = (m + 7) // 8 * 8
    Xh = torch.empty((w, ldh), dtype=torch.float16, device=X.device).t()[:m]
    inv_s = torch.empty(w, dtype=torch.float32, device=X.device)
    rc = lib().tcqr_cast_scale(m, w, _ptr(X), _ld(X), _ptr(Xh), ldh, _ptr(inv_s), int(scaling))
    _check("tcqr_cast_scale", rc)
    return Xh, inv_s


def _h_ld(Xh):
    return Xh.stride(1)


def gemm_tn(A1h, A2h, col_mult=None):
    """K3: C = A1h' A2h diag(col_mult) (FP16 in, FP32 out)."""
    torch = _torch()
    _ensure()
    m, h = A1h.shape
    _, w2 = A2h.shape
    C = colmajor_empty(h, w2, device=A1h.device)
    cm = _ptr(col_mult) if col_mult is not None else None
    _check("tcqr_gemm_tn", lib().tcqr_gemm_tn(m, h, w2, _ptr(A1h), _h_ld(A1h), _ptr(A2h),
                                              _h_ld(A2h), _ptr(C), h, cm))
    return C


def gemm_nn_update(C, Qh, Bh, col_mult=None):
    """K4: C -= (Qh Bh) diag(col_mult), in place; returns C."""
    _ensure()
    m, h = Qh.shape
    _, w2 = Bh.shape
    cm = _ptr(col_mult) if col_mult is not None else None
    _check("tcqr_gemm_nn_update", lib().tcqr_gemm_nn_update(
        m, h, w2, _ptr(Qh), _h_ld(Qh), _ptr(Bh), _h_ld(Bh), _ptr(C), _ld(C), cm))
    return C


def panel_qr(X, br=256):
    """K2: CAQR-MGS panel in place on X (m, w<=32); returns (X, R)."""
    _ensure()
    m, w = X.shape
    R = colmajor_empty(w, w, device=X.device)
    _check("tcqr_panel_qr", lib().tcqr_panel_qr(m, w, _ptr(X), _ld(X), _ptr(R), w, int(br)))
    return X, R


def trinv(R):
    """K6 set-up: M = inv(R) in FP64 (R float32 upper triangular, column-major)."""
    torch = _torch()
    _ensure()
    n = R.shape[0]
    M = colmajor_empty(n, n, dtype=torch.float64, device=R.device)
    _check("tcqr_trinv", lib().tcqr_trinv(n, _ptr(R), _ld(R), _ptr(M), n))
    return M


def gemv(A, v, trans=False):
    """K5: y = A v or A' v (A float32 column-major, v float64)."""
    torch = _torch()
    _ensure()
    m, n = A.shape
    y = torch.empty(n if trans else m, dtype=torch.float64, device=A.device)
    _check("tcqr_gemv", lib().tcqr_gemv(int(trans), m, n, _ptr(A), _ld(A), _ptr(v), _ptr(y)))
    return y


def profile_enable(on=True):
    _ensure()
    _check("tcqr_profile_enable", lib().tcqr_profile_enable(int(on)))


def profile_read():
    """{class: {ms, flops, bytes, launches}} accumulated since profile_enable()."""
    out = {}
    for i, name in enumerate(PROFILE_CLASSES):
        ms, fl, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _check("tcqr_profile_read", lib().tcqr_profile_read(
            i, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by), ctypes.byref(n)))
        out[name] = {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": n.value}
    return out


def last_launch_count():
    return lib().tcqr_last_launch_count()


def last_collective_count():
    return lib().tcqr_last_collective_count()


def run_virtual_ranks(nranks, fn, slot_bytes=64 << 20, device=0, timeout=600):
    """Test seam (include/tcqr.h "Virtual ranks"): run ``fn(rank)`` on ``nranks`` host threads,
    each bound to its own library context (tcqr_init_virtual) on ``device`` with its own CUDA
    stream, sharing one virtual group whose collectives stand in for NCCL. ``fn`` calls the
    C ABI through ``lib()`` directly (the module-level helpers use the process context).
    Returns the list of fn's results; re-raises the first exception of any rank."""
    import threading
    torch = _torch()
    l = lib()
    torch.cuda.set_device(device)
    g = l.tcqr_vgroup_create(int(nranks), int(slot_bytes))
    if not g:
        raise TcqrError("tcqr_vgroup_create", -1)
    results, errors = [None] * nranks, []

    def worker(r):
        try:
            torch.cuda.set_device(device)
            stream = torch.cuda.Stream(device=device)
            _check("tcqr_init_virtual", l.tcqr_init_virtual(device, ctypes.c_void_p(
                stream.cuda_stream), ctypes.c_void_p(g), r))
            try:
                with torch.cuda.stream(stream):
                    results[r] = fn(r)
                stream.synchronize()
            finally:
                l.tcqr_finalize()
        except BaseException as e:  # noqa: BLE001 -- re-raised in the caller
            errors.append((r, e))

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    hung = [i for i, t in enumerate(threads) if t.is_alive()]
    if not hung:
        l.tcqr_vgroup_destroy(ctypes.c_void_p(g))
    if hung:
        raise TimeoutError(f"virtual ranks {hung} still running after {timeout} s")
    if errors:
        r, e = sorted(errors, key=lambda x: x[0])[0]
        raise RuntimeError(f"virtual rank {r}: {e!r}") from e
    return results


def version():
    return lib().tcqr_version().decode()


@dataclass
class FlopModel:
    m: int
    n: int

    @property
    def convention(self):
        """2mn^2 - 2/3 n^3 (north_star reporting convention)."""
        return 2.0 * self.m * self.n ** 2 - 2.0 / 3.0 * self.n ** 3

    @property
    def executed(self):
        return 2.0 * self.m * self.n ** 2
