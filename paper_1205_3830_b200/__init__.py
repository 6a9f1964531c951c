"""paper_1205_3830_b200 — randomized interpolative decomposition (arXiv 1205.3830) on B200.

Thin Python binding over the C ABI of ``include/rid.h`` (``librid.so``, built in-tree by
``paper_1205_3830_b200.build``). Argument marshalling only: every step of the method runs in the
CUDA kernels of ``csrc/``. There is no CPU fallback — if the library is missing or no GPU is
visible, calls raise.

Matrices are complex128 and column-major: a torch tensor of shape (rows, cols) with
``stride(0) == 1`` (e.g. ``torch.empty((cols, rows), dtype=torch.complex128).T``) or a numpy
array in Fortran order. Tensors on the GPU are used in place; host tensors / numpy arrays go
through the library's own host staging (the "e2e" path of bench.py).
"""
from __future__ import annotations

import ctypes
import os
import warnings
from dataclasses import dataclass

import numpy as np

__all__ = [
    "RidError", "Context", "Diag", "lib", "colmajor_empty", "generate", "sketch", "decompose",
    "error_estimate", "error_bound", "normal_fill", "qrcp", "factor_solve", "shard_range",
    "STREAM_R", "STREAM_R_RETRY",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librid.so")
STREAM_R, STREAM_R_RETRY = 4, 20

RID_OK, RID_EINVAL, RID_ERANK, RID_ESINGULAR, RID_ENOMEM, RID_ECUDA, RID_ENCCL = range(7)
_STATUS = {0: "RID_OK", 1: "RID_EINVAL", 2: "RID_ERANK", 3: "RID_ESINGULAR", 4: "RID_ENOMEM",
           5: "RID_ECUDA", 6: "RID_ENCCL"}


class RidError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Diag(ctypes.Structure):
    """rid_diag (include/rid.h)."""

    _fields_ = [("t_rgen", ctypes.c_double), ("t_sketch", ctypes.c_double),
                ("t_gather", ctypes.c_double), ("t_qrcp", ctypes.c_double),
                ("t_solve", ctypes.c_double), ("t_total", ctypes.c_double),
                ("t_h2d", ctypes.c_double), ("t_d2h", ctypes.c_double),
                ("retries", ctypes.c_int), ("rank_achieved", ctypes.c_int),
                ("tie_margin_min", ctypes.c_double), ("resid_last", ctypes.c_double),
                ("launches", ctypes.c_int),
                ("t_sketch_tc", ctypes.c_double), ("sketch_engine", ctypes.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
EXPORTS = ["rid_create", "rid_destroy", "rid_last_error", "rid_version", "rid_comm_id_bytes",
           "rid_comm_get_id", "rid_comm_init", "rid_comm_info", "rid_generate", "rid_sketch",
           "rid_decompose", "rid_error_estimate", "rid_error_bound", "rid_normal_fill",
           "rid_qrcp", "rid_factor_solve", "rid_sketch_splits", "rid_sketch_srft",
           "rid_set_sketch", "rid_sketch_mults", "rid_sketch_cols", "rid_set_qr",
           "rid_set_stream", "rid_comm_init_local", "rid_set_qr_dist", "rid_sketch_strassen",
           "rid_set_sketch_engine", "rid_sketch_engine_of", "rid_crt_plan", "rid_crt_moduli"]
SKETCH_GAUSSIAN, SKETCH_SRFT = 0, 1
QR_HOUSEHOLDER, QR_CGS2 = 0, 1
QR_REPLICATED, QR_SHARDED = 0, 1
ENGINE_AUTO, ENGINE_FP64_DMMA, ENGINE_INT8_CRT = 0, 1, 2
_ENGINES = {"auto": ENGINE_AUTO, "fp64_dmma": ENGINE_FP64_DMMA, "int8_crt": ENGINE_INT8_CRT}
_QR_DIST = {"replicated": QR_REPLICATED, "sharded": QR_SHARDED}
_QR_KINDS = {"householder": QR_HOUSEHOLDER, "cgs2": QR_CGS2}


def lib():
    """Load librid.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_1205_3830_b200.build` "
                           "(the CUDA path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    p, i64, u64, u32, d, ci = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                               ctypes.c_double, ctypes.c_int)
    sig = {
        "rid_create": ([ctypes.POINTER(p), ci, p], ci),
        "rid_destroy": ([p], None),
        "rid_set_stream": ([p, p], ci),
        "rid_comm_init_local": ([ctypes.POINTER(p), ci], ci),
        "rid_last_error": ([p], ctypes.c_char_p),
        "rid_version": ([], ctypes.c_char_p),
        "rid_comm_id_bytes": ([], ctypes.c_size_t),
        "rid_comm_get_id": ([p], ci),
        "rid_comm_init": ([p, p, ci, ci], ci),
        "rid_comm_info": ([p, ctypes.POINTER(ci), ctypes.POINTER(ci)], ci),
        "rid_generate": ([p, u64, i64, i64, i64, d, i64, i64, p, i64], ci),
        "rid_sketch": ([p, u64, u32, i64, p, i64, i64, i64, i64, p, i64], ci),
        "rid_sketch_splits": ([p, i64, i64, i64], ci),
        "rid_sketch_mults": ([], ci),
        "rid_sketch_strassen": ([p, i64, i64, i64], ci),
        "rid_sketch_cols": ([p, u64, u32, i64, p, i64, i64, i64, i64, i64, p, i64], ci),
        "rid_sketch_srft": ([p, u64, ci, i64, p, i64, i64, i64, i64, p, i64], ci),
        "rid_set_sketch": ([p, ci], ci),
        "rid_set_qr": ([p, ci], ci),
        "rid_set_qr_dist": ([p, ci], ci),
        "rid_set_sketch_engine": ([p, ci], ci),
        "rid_sketch_engine_of": ([p, i64, i64, i64], ci),
        "rid_crt_plan": ([i64, i64, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.POINTER(ci),
                          ctypes.POINTER(i64), ctypes.POINTER(ci), ctypes.POINTER(d)], ci),
        "rid_crt_moduli": ([ctypes.POINTER(ci), ci], ci),
        "rid_decompose": ([p, p, i64, i64, i64, i64, i64, i64, i64, u64, p, p, i64, p], ci),
        "rid_error_estimate": ([p, p, i64, i64, i64, i64, i64, p, i64, p, i64, ci, u64, p, p], ci),
        "rid_error_bound": ([i64, i64, i64, d, d], d),
        "rid_normal_fill": ([p, u64, u32, i64, i64, i64, i64, p, i64], ci),
        "rid_qrcp": ([p, p, i64, i64, i64, i64, p, p, i64, p, p, p], ci),
        "rid_factor_solve": ([p, p, i64, i64, i64, i64, i64, i64, p, p, i64, p], ci),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


# ------------------------------------------------------------------------------ buffers ---------
def _torch():
    import torch

    return torch


def colmajor_empty(rows: int, cols: int, device="cuda", dtype=None, pin_memory=False):
    """Empty column-major (rows, cols) tensor (stride (1, rows))."""
    torch = _torch()
    dtype = dtype or torch.complex128
    if str(device) == "cpu":
        t = torch.empty((cols, rows), dtype=dtype, pin_memory=pin_memory)
    else:
        t = torch.empty((cols, rows), dtype=dtype, device=device)
    return t.T


class _Buf:
    """(pointer, leading dimension, keep-alive) for a complex128 column-major matrix.

    Rejects (ValueError) any layout librid cannot address as (pointer, ld >= rows): a column stride
    below the row count (broadcast / overlapping views), a stride that is not a whole number of
    elements, and a CUDA tensor on another device than the context's."""

    def __init__(self, a, rows: int, cols: int, name: str, ctx: "Context | None" = None):
        self.obj = a
        if isinstance(a, np.ndarray):
            if a.dtype != np.complex128:
                raise TypeError(f"{name}: need complex128, got {a.dtype}")
            if a.ndim == 1:
                a = a.reshape(-1, 1)
            if a.shape != (rows, cols):
                raise ValueError(f"{name}: shape {a.shape} != {(rows, cols)}")
            if cols > 1 and not a.flags.f_contiguous and a.strides[0] != 16:
                raise ValueError(f"{name}: numpy array must be column-major (Fortran order)")
            if cols > 1 and (a.strides[1] % 16 != 0 or a.strides[1] // 16 < rows):
                raise ValueError(f"{name}: column stride {a.strides[1]} B is not a leading "
                                 f"dimension >= {rows} complex128 elements")
            self.ptr = a.ctypes.data
            self.ld = a.strides[1] // 16 if cols > 1 else rows
            self.obj = a
        else:
            torch = _torch()
            if a.dtype != torch.complex128:
                raise TypeError(f"{name}: need torch.complex128, got {a.dtype}")
            if a.dim() == 1:
                a = a.reshape(-1, 1)
            if tuple(a.shape) != (rows, cols):
                raise ValueError(f"{name}: shape {tuple(a.shape)} != {(rows, cols)}")
            if a.stride(0) != 1 and rows > 1:
                raise ValueError(f"{name}: tensor must be column-major (stride(0) == 1)")
            if cols > 1 and a.stride(1) < rows:
                raise ValueError(f"{name}: column stride {a.stride(1)} < {rows} rows "
                                 "(broadcast or overlapping view)")
            if ctx is not None and a.is_cuda and a.device.index != ctx.device:
                raise ValueError(f"{name}: tensor on {a.device}, context on cuda:{ctx.device}")
            self.ptr = a.data_ptr()
            self.ld = a.stride(1) if cols > 1 else max(rows, 1)
            self.obj = a
        self.ld = max(self.ld, rows)


def _ptr_i64(a):
    if isinstance(a, np.ndarray):
        if a.dtype != np.int64 or not a.flags.c_contiguous:
            raise TypeError("J must be a contiguous int64 array")
        return a.ctypes.data
    torch = _torch()
    if a.dtype != torch.int64 or not a.is_contiguous():
        raise TypeError("J must be a contiguous int64 tensor")
    return a.data_ptr()


# ------------------------------------------------------------------------------ context ---------
class Context:
    """A librid context (rid_ctx) bound to one CUDA device and stream."""

    def __init__(self, device: int = 0, stream=None):
        L = lib()
        self._L = L
        self.device = device
        h = ctypes.c_void_p()
        sp = None
        if stream is not None:
            sp = ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
        st = L.rid_create(ctypes.byref(h), device, sp)
        if st != RID_OK:
            raise RidError(st, f"rid_create(device={device}) failed (is a B200 visible?)")
        self.h = h
        self._stream = sp.value if sp is not None else None

    def set_stream(self, stream):
        """Order subsequent calls on `stream` (a torch.cuda.Stream or a raw cudaStream_t)."""
        s = stream if isinstance(stream, int) or stream is None else stream.cuda_stream
        if s != self._stream:
            self.check(self._L.rid_set_stream(self.h, ctypes.c_void_p(s)), "rid_set_stream")
            self._stream = s

    def close(self):
        if getattr(self, "h", None):
            self._L.rid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int, what: str):
        if st != RID_OK:
            msg = self._L.rid_last_error(self.h).decode(errors="replace")
            raise RidError(st, f"{what}: {msg}")

    # communicator ------------------------------------------------------------------------------
    def comm_init(self, id_bytes: bytes, rank: int, nranks: int):
        buf = ctypes.create_string_buffer(id_bytes, len(id_bytes))
        self.check(self._L.rid_comm_init(self.h, buf, rank, nranks), "rid_comm_init")

    def set_qr_dist(self, mode: str):
        """'replicated' (all-gather Y, whole-sketch QR on every rank; default) or 'sharded'
        (NEXT-3: the ranks factor their blocks together; in-process communicator only)."""
        self.check(self._L.rid_set_qr_dist(self.h, _QR_DIST[mode]), "rid_set_qr_dist")

    def set_sketch_engine(self, engine: str):
        """Arithmetic of the Gaussian sketch: 'auto' (default: 'int8_crt' when l m n >= 2^34),
        'fp64_dmma' (DMMA tensor pipe) or 'int8_crt' (exact modular products on tcgen05)."""
        self.check(self._L.rid_set_sketch_engine(self.h, _ENGINES[engine]), "rid_set_sketch_engine")

    def comm_info(self):
        r, n = ctypes.c_int(), ctypes.c_int()
        self.check(self._L.rid_comm_info(self.h, ctypes.byref(r), ctypes.byref(n)), "rid_comm_info")
        return r.value, n.value


def comm_init_local(ctxs) -> None:
    """Join the contexts `ctxs` (one process, one device) into an in-process communicator, context
    r as rank r (rid_comm_init_local). Each rank's calls must then run concurrently on its own
    thread (tests/test_gpu_multirank.py): the G > 1 data path on one GPU."""
    L = lib()
    arr = (ctypes.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    st = L.rid_comm_init_local(arr, len(ctxs))
    if st != RID_OK:
        raise RidError(st, "rid_comm_init_local: " +
                       L.rid_last_error(ctxs[0].h).decode(errors="replace"))


def comm_get_id() -> bytes:
    L = lib()
    nb = L.rid_comm_id_bytes()
    buf = ctypes.create_string_buffer(nb)
    st = L.rid_comm_get_id(buf)
    if st != RID_OK:
        raise RidError(st, "rid_comm_get_id")
    return buf.raw


_default = {}


def default_context(device=None) -> Context:
    """The per-device context of calls made without ctx=, ordered on torch's CURRENT stream of
    that device at each call (re-bound with rid_set_stream whenever it changes)."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _default:
        _default[dev] = Context(dev, torch.cuda.current_stream(dev))
    ctx = _default[dev]
    ctx.set_stream(torch.cuda.current_stream(dev))
    return ctx


def shard_range(n: int, rank: int, world: int):
    """Columns [col0, col0 + n_loc) of rank `rank` (contiguous equal blocks; n % world == 0)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n % world:
        raise ValueError(f"n={n} is not divisible by world={world}")
    n_loc = n // world
    return rank * n_loc, n_loc


# ------------------------------------------------------------------------------ the method ------
def generate(seed: int, m: int, n: int, k: int, noise: float, col0: int = 0, n_loc=None,
             out=None, ctx: Context | None = None, device="cuda"):
    """A[:, col0:col0+n_loc] = X Y0 + noise E (docs/RNG.md §5), bit-identical to the oracle."""
    ctx = ctx or default_context()
    n_loc = n - col0 if n_loc is None else n_loc
    if out is None:
        out = colmajor_empty(m, n_loc, device=device)
    b = _Buf(out, m, n_loc, "A", ctx)
    ctx.check(lib().rid_generate(ctx.h, seed, m, n, k, float(noise), col0, n_loc, b.ptr, b.ld),
              "rid_generate")
    return out


def sketch(A, seed: int, l: int, stream: int = STREAM_R, out=None, n: int | None = None,
           col0: int = 0, ctx: Context | None = None):
    """Y = R A with R(r, i) = N(seed, stream, r, i) on the DMMA pipe. A may be the column block
    [col0, col0 + width) of an n-column matrix (n defaults to A's own width); (n, col0) fix the
    kernel plan (K split, wave tail), so a block's columns match the whole matrix's bit for bit."""
    ctx = ctx or default_context()
    m, n_loc = A.shape
    n = n_loc if n is None else n
    a = _Buf(A, m, n_loc, "A", ctx)
    if out is None:
        out = colmajor_empty(l, n_loc, device=A.device if hasattr(A, "device") else "cpu") \
            if not isinstance(A, np.ndarray) else np.zeros((l, n_loc), np.complex128, order="F")
    y = _Buf(out, l, n_loc, "Y", ctx)
    ctx.check(lib().rid_sketch_cols(ctx.h, seed, stream, l, a.ptr, m, n, col0, n_loc, a.ld, y.ptr,
                                    y.ld), "rid_sketch")
    return out


def sketch_srft(A, seed: int, l: int, retry: bool = False, out=None, n: int | None = None,
                ctx: Context | None = None):
    """Y = S F D A, the paper's SRFT randomisation; m a power of two >= 16."""
    ctx = ctx or default_context()
    m, n_loc = A.shape
    n = n_loc if n is None else n
    a = _Buf(A, m, n_loc, "A", ctx)
    if out is None:
        out = colmajor_empty(l, n_loc, device=A.device if hasattr(A, "device") else "cpu") \
            if not isinstance(A, np.ndarray) else np.zeros((l, n_loc), np.complex128, order="F")
    y = _Buf(out, l, n_loc, "Y", ctx)
    ctx.check(lib().rid_sketch_srft(ctx.h, seed, int(retry), l, a.ptr, m, n, n_loc, a.ld, y.ptr,
                                    y.ld), "rid_sketch_srft")
    return out


def sketch_splits(m: int, l: int, n: int, ctx: Context | None = None) -> int:
    """K slices of the sketch of an m x n matrix."""
    ctx = ctx or default_context()
    return lib().rid_sketch_splits(ctx.h, m, l, n)


def sketch_strassen(m: int, l: int, n: int, ctx: Context | None = None) -> bool:
    """True when the sketch of an m x n matrix runs one Strassen level over Gauss's three products
    (then column blocks must be 64-aligned)."""
    ctx = ctx or default_context()
    return bool(lib().rid_sketch_strassen(ctx.h, m, l, n))


def sketch_engine(m: int, l: int, n: int, ctx: Context | None = None) -> str:
    """'fp64_dmma' or 'int8_crt': the engine the Gaussian sketch of an m x n matrix runs on."""
    ctx = ctx or default_context()
    e = lib().rid_sketch_engine_of(ctx.h, m, l, n)
    if e not in (ENGINE_FP64_DMMA, ENGINE_INT8_CRT):
        raise RidError(1, f"rid_sketch_engine_of: bad shape (m={m}, l={l}, n={n})")
    return {ENGINE_FP64_DMMA: "fp64_dmma", ENGINE_INT8_CRT: "int8_crt"}[e]


def crt_plan(l: int, m: int) -> dict:
    """The INT8_CRT engine's plan for an l x m sketch matrix (host arithmetic, no GPU)."""
    T, b, ks, nc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    Kp, lg = ctypes.c_int64(), ctypes.c_double()
    st = lib().rid_crt_plan(l, m, ctypes.byref(T), ctypes.byref(b), ctypes.byref(ks),
                            ctypes.byref(Kp), ctypes.byref(nc), ctypes.byref(lg))
    if st != 0:
        raise RidError(st, "rid_crt_plan: bad arguments")
    return {"T": T.value, "b": b.value, "kslices": ks.value, "Kp": Kp.value, "nc": nc.value,
            "log2M": lg.value}


def crt_moduli() -> list:
    """The moduli of the INT8_CRT engine, in the order used."""
    buf = (ctypes.c_int * 32)()
    n = lib().rid_crt_moduli(buf, 32)
    return [buf[i] for i in range(n)]


def sketch_mults() -> int:
    """3: Gauss's three-multiplication sketch (default); 4: the ordered real embedding
    (RID_SKETCH_4M=1), bit-identical to the oracle's chain when sketch_splits(...) == 1."""
    return lib().rid_sketch_mults()


@dataclass
class IdResult:
    J: object
    P: object
    diag: dict


def _set_qr(ctx, qr: str):
    ctx.check(lib().rid_set_qr(ctx.h, _QR_KINDS[qr]), "rid_set_qr")


def decompose(A, k: int, l: int, seed: int, n: int | None = None, col0: int = 0, J=None, P=None,
              ctx: Context | None = None, sketch: str = "gaussian",
              qr: str = "householder") -> IdResult:
    """The whole ID of the (shard of the) matrix A: J (k, global ids) and P_loc.
    sketch: 'gaussian' (north star, default) or 'srft' (the paper's Y = S F D A); qr:
    'householder' (default) or 'cgs2' (the paper's CGS with iteration)."""
    ctx = ctx or default_context()
    kind = {"gaussian": SKETCH_GAUSSIAN, "srft": SKETCH_SRFT}[sketch]
    ctx.check(lib().rid_set_sketch(ctx.h, kind), "rid_set_sketch")
    _set_qr(ctx, qr)
    m, n_loc = A.shape
    n = n_loc if n is None else n
    a = _Buf(A, m, n_loc, "A", ctx)
    host = isinstance(A, np.ndarray) or (hasattr(A, "device") and A.device.type == "cpu")
    if J is None:
        J = np.zeros(k, np.int64) if isinstance(A, np.ndarray) else _torch().empty(
            k, dtype=_torch().int64, device=A.device)
    if P is None:
        P = np.zeros((k, n_loc), np.complex128, order="F") if isinstance(A, np.ndarray) else \
            colmajor_empty(k, n_loc, device="cpu" if host else A.device,
                           pin_memory=host and _torch().cuda.is_available())
    p = _Buf(P, k, n_loc, "P", ctx)
    d = Diag()
    ctx.check(lib().rid_decompose(ctx.h, a.ptr, m, n, col0, n_loc, a.ld, k, l, seed, _ptr_i64(J),
                                  p.ptr, p.ld, ctypes.byref(d)), "rid_decompose")
    if k > 1 and d.tie_margin_min < 1e-9:
        # reading R18: below ~1e-9 the pivot choice is decided by rounding; the blocked QR's
        # downdated norms (R11') may then pick another (equally valid) column than the
        # exact-norm kernels or the oracle
        warnings.warn(f"rid.decompose: near-tie pivot step (top-2 margin {d.tie_margin_min:.3g} "
                      "< 1e-9); J is not uniquely determined at this precision", RuntimeWarning)
    return IdResult(J, P, d.as_dict())


def error_estimate(A, J, P, q: int, seed: int, n: int | None = None, col0: int = 0,
                   ctx: Context | None = None) -> float:
    """Compensated power-iteration estimate of ||A - A[:, J] P||_2 (Table 5)."""
    ctx = ctx or default_context()
    m, n_loc = A.shape
    k = P.shape[0]
    n = n_loc if n is None else n
    a = _Buf(A, m, n_loc, "A", ctx)
    p = _Buf(P, k, n_loc, "P", ctx)
    est = ctypes.c_double()
    d = Diag()
    ctx.check(lib().rid_error_estimate(ctx.h, a.ptr, m, n, col0, n_loc, a.ld, _ptr_i64(J), k, p.ptr,
                                       p.ld, int(q), seed, ctypes.byref(est), ctypes.byref(d)),
              "rid_error_estimate")
    return est.value


def error_bound(m: int, n: int, k: int, eps: float, sigma_kp1: float) -> float:
    """Eq. (3) right-hand side."""
    return lib().rid_error_bound(m, n, k, eps, sigma_kp1)


def normal_fill(seed: int, s: int, rows: int, cols: int, row0: int = 0, col0: int = 0, out=None,
                ctx: Context | None = None, device="cuda"):
    ctx = ctx or default_context()
    if out is None:
        out = colmajor_empty(rows, cols, device=device)
    b = _Buf(out, rows, cols, "out", ctx)
    ctx.check(lib().rid_normal_fill(ctx.h, seed, s, rows, cols, row0, col0, b.ptr, b.ld),
              "rid_normal_fill")
    return out


def qrcp(Y, k: int, ctx: Context | None = None, want_R: bool = True, qr: str = "householder"):
    """Pivoted QR of a full sketch: (J, R (k x n) or None, resid, margin, diag). qr:
    'householder' (default) or 'cgs2'."""
    torch = _torch()
    ctx = ctx or default_context()
    _set_qr(ctx, qr)
    l, n = Y.shape
    y = _Buf(Y, l, n, "Y", ctx)
    dev = Y.device
    J = torch.empty(k, dtype=torch.int64, device=dev)
    R = colmajor_empty(k, n, device=dev) if want_R else None
    resid = torch.empty(k, dtype=torch.float64, device=dev)
    margin = torch.empty(k, dtype=torch.float64, device=dev)
    d = Diag()
    st = lib().rid_qrcp(ctx.h, y.ptr, l, n, y.ld, k, J.data_ptr(),
                        R.data_ptr() if R is not None else None, k if R is not None else k,
                        resid.data_ptr(), margin.data_ptr(), ctypes.byref(d))
    if st == RID_ERANK:
        raise RidError(st, f"rank {d.rank_achieved} < k = {k}")
    ctx.check(st, "rid_qrcp")
    return J, R, resid, margin, d.as_dict()


def factor_solve(Y, k: int, col0: int, n_loc: int, ctx: Context | None = None,
                 qr: str = "householder"):
    """(J, P_loc) from a full sketch Y: factorisation + solve for one column shard."""
    torch = _torch()
    ctx = ctx or default_context()
    _set_qr(ctx, qr)
    l, n = Y.shape
    y = _Buf(Y, l, n, "Y", ctx)
    J = torch.empty(k, dtype=torch.int64, device=Y.device)
    P = colmajor_empty(k, n_loc, device=Y.device)
    p = _Buf(P, k, n_loc, "P", ctx)
    d = Diag()
    ctx.check(lib().rid_factor_solve(ctx.h, y.ptr, l, n, y.ld, k, col0, n_loc, J.data_ptr(), p.ptr,
                                     p.ld, ctypes.byref(d)), "rid_factor_solve")
    return J, P, d.as_dict()
