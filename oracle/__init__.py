"""CPU ORACLE for the randomized interpolative decomposition (arXiv 1205.3830).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package. The product path
(``paper_1205_3830_b200``) never imports it and shares no code with it.

Thin ctypes/numpy marshalling over ``oracle/rid_oracle.c`` (plain C, fp64, naive loops); every
step of the method is in the C file, whose header cites the PAPER.md passage each function
follows. Matrices are numpy complex128 arrays in Fortran (column-major) order.

Parity pins: tests/test_oracle_*.py. Parity is pinned for every function here (see DESIGN.md
"Oracle pins"); nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rid_oracle.c")
_LIB = os.path.join(_HERE, "librid_oracle.so")

RID_OK, RID_EINVAL, RID_ERANK, RID_ESINGULAR, RID_ENOMEM = 0, 1, 2, 3, 4
STREAM_X, STREAM_Y0, STREAM_E, STREAM_R, STREAM_X0, STREAM_R_RETRY = 1, 2, 3, 4, 5, 20
STREAM_PHASE, STREAM_SAMPLE, STREAM_PHASE_RETRY, STREAM_SAMPLE_RETRY = 6, 7, 22, 23


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def _cpu_has_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " fma " in f.read()
    except OSError:
        return False


def build(force: bool = False) -> str:
    """Compile rid_oracle.c -> librid_oracle.so (gcc -O2 -ffp-contract=off -fopenmp)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
           "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
    if _cpu_has_fma():
        cmd.insert(1, "-mfma")  # explicit fma() calls become one instruction; no contraction
    subprocess.check_call(cmd)
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i64, u32, u64, p = (ctypes.c_double, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                               ctypes.c_void_p)
        L.orc_philox4x32_10.argtypes = [p, p, p]
        L.orc_philox4x32_10.restype = None
        L.orc_rid_ln.argtypes = [d]
        L.orc_rid_ln.restype = d
        L.orc_rid_sincos2pi.argtypes = [d, p, p]
        L.orc_rid_sincos2pi.restype = None
        L.orc_normal.argtypes = [u64, u32, u32, u32, p]
        L.orc_normal.restype = None
        L.orc_normal_matrix.argtypes = [u64, u32, i64, i64, i64, i64, p, i64]
        L.orc_normal_matrix.restype = None
        L.orc_generate.argtypes = [u64, i64, i64, i64, d, i64, i64, p, i64]
        L.orc_generate.restype = ctypes.c_int
        L.orc_sketch.argtypes = [u64, u32, i64, i64, i64, p, i64, p, i64]
        L.orc_sketch.restype = ctypes.c_int
        L.orc_pivoted_cgs2.argtypes = [i64, i64, i64, p, i64, p, p, i64, p, p, p]
        L.orc_pivoted_cgs2.restype = ctypes.c_int
        L.orc_backsolve.argtypes = [i64, i64, p, i64, p, p, i64, p]
        L.orc_backsolve.restype = ctypes.c_int
        L.orc_error_estimate.argtypes = [i64, i64, p, i64, p, i64, p, i64, ctypes.c_int, u64, p]
        L.orc_error_estimate.restype = ctypes.c_int
        L.orc_error_bound.argtypes = [i64, i64, i64, d, d]
        L.orc_error_bound.restype = d
        L.orc_noise_floor.argtypes = [i64, i64, d]
        L.orc_noise_floor.restype = d
        L.orc_srft_plan.argtypes = [u64, u32, u32, i64, i64, p, p]
        L.orc_srft_plan.restype = ctypes.c_int
        L.orc_srft_apply.argtypes = [p, p, i64, i64, i64, p, i64, p, i64]
        L.orc_srft_apply.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def set_threads(n: int = 0) -> int:
    """Set the OpenMP thread count (0 = leave) and return the current maximum."""
    return lib().orc_set_threads(int(n))


def _fortran_c128(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


# ---------------------------------------------------------------- RNG (docs/RNG.md) -----------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def rid_ln(u: float) -> float:
    return lib().orc_rid_ln(float(u))


def rid_sincos2pi(u: float):
    c = ctypes.c_double()
    s = ctypes.c_double()
    lib().orc_rid_sincos2pi(float(u), ctypes.byref(c), ctypes.byref(s))
    return c.value, s.value


def normal(seed: int, s: int, i: int, j: int) -> complex:
    out = np.zeros(2, dtype=np.float64)
    lib().orc_normal(seed, s, i, j, _ptr(out))
    return complex(out[0], out[1])


def normal_matrix(seed: int, s: int, rows: int, cols: int, row0: int = 0, col0: int = 0):
    out = np.zeros((rows, cols), dtype=np.complex128, order="F")
    lib().orc_normal_matrix(seed, s, rows, cols, row0, col0, _ptr(out), rows)
    return out


# ---------------------------------------------------------------- the method ------------------
def generate(seed: int, m: int, n: int, k: int, noise: float, col0: int = 0, n_loc=None):
    """A[:, col0:col0+n_loc] of A = X·Y0 + noise·E (docs/RNG.md §5)."""
    n_loc = n - col0 if n_loc is None else n_loc
    A = np.zeros((m, n_loc), dtype=np.complex128, order="F")
    st = lib().orc_generate(seed, m, n, k, float(noise), col0, n_loc, _ptr(A), m)
    if st:
        raise OracleError(st, "generate")
    return A


def sketch(A, seed: int, l: int, stream: int = STREAM_R):
    """Y = R·A with R(r, i) = N(seed, stream, r, i)."""
    A = _fortran_c128(A)
    m, n_loc = A.shape
    Y = np.zeros((l, n_loc), dtype=np.complex128, order="F")
    st = lib().orc_sketch(seed, stream, l, m, n_loc, _ptr(A), m, _ptr(Y), l)
    if st:
        raise OracleError(st, "sketch")
    return Y


@dataclass
class QrResult:
    status: int
    J: np.ndarray
    R: np.ndarray
    resid_norms: np.ndarray
    tie_margins: np.ndarray
    rank_achieved: int


def pivoted_qr(Y, k: int) -> QrResult:
    """Pivoted CGS2: J (pivot order), R = Q^H Y (k x n)."""
    Y = _fortran_c128(Y)
    l, n = Y.shape
    J = np.zeros(k, dtype=np.int64)
    R = np.zeros((k, n), dtype=np.complex128, order="F")
    rn = np.zeros(k, dtype=np.float64)
    tm = np.zeros(k, dtype=np.float64)
    ra = ctypes.c_int64(0)
    st = lib().orc_pivoted_cgs2(l, n, k, _ptr(Y), l, _ptr(J), _ptr(R), k, _ptr(rn), _ptr(tm),
                                ctypes.byref(ra))
    if st not in (RID_OK, RID_ERANK):
        raise OracleError(st, "pivoted_qr")
    return QrResult(st, J, R, rn, tm, ra.value)


def backsolve(R, J, k: int):
    """P = [I T] in original column order, T = R11^{-1} R12 (Eqs. 10-11)."""
    R = _fortran_c128(R)
    n = R.shape[1]
    Jc = np.ascontiguousarray(J, dtype=np.int64)
    P = np.zeros((k, n), dtype=np.complex128, order="F")
    si = ctypes.c_int64(-1)
    st = lib().orc_backsolve(k, n, _ptr(R), R.shape[0], _ptr(Jc), _ptr(P), k, ctypes.byref(si))
    if st:
        raise OracleError(st, f"backsolve (singular index {si.value})")
    return P


@dataclass
class Decomposition:
    J: np.ndarray
    P: np.ndarray
    Y: np.ndarray
    retries: int
    resid_norms: np.ndarray
    tie_margins: np.ndarray
    extra: dict = field(default_factory=dict)


def srft_plan(seed: int, m: int, l: int, retry: bool = False):
    """SRFT plan (docs/RNG.md §7): phases d (m complex, |d| = 1) and row samples s (l ints)."""
    d = np.zeros(m, np.complex128)
    s = np.zeros(l, np.int64)
    sp, ss = (STREAM_PHASE_RETRY, STREAM_SAMPLE_RETRY) if retry else (STREAM_PHASE, STREAM_SAMPLE)
    st = lib().orc_srft_plan(seed, sp, ss, m, l, _ptr(d), _ptr(s))
    if st:
        raise OracleError(st, "srft_plan")
    return d, s


def srft_apply(d, s, A):
    """Y = S F D A for an explicit plan (Eqs. 4-7), direct ascending sums."""
    A = _fortran_c128(A)
    m, n_loc = A.shape
    d = np.ascontiguousarray(d, np.complex128)
    s = np.ascontiguousarray(s, np.int64)
    l = s.size
    Y = np.zeros((l, n_loc), np.complex128, order="F")
    st = lib().orc_srft_apply(_ptr(d), _ptr(s), l, m, n_loc, _ptr(A), m, _ptr(Y), l)
    if st:
        raise OracleError(st, "srft_apply")
    return Y


def srft_sketch(A, seed: int, l: int, retry: bool = False):
    A = _fortran_c128(A)
    d, s = srft_plan(seed, A.shape[0], l, retry)
    return srft_apply(d, s, A)


def decompose(A, k: int, l: int, seed: int, sketch_kind: str = "gaussian") -> Decomposition:
    """The whole ID: sketch -> pivoted CGS2 (one retry: stream 20, or 22/23 for the SRFT) ->
    back-substitution. sketch_kind 'gaussian' (north star) or 'srft'."""
    A = _fortran_c128(A)
    retries = 0
    mk = (lambda retry: sketch(A, seed, l, STREAM_R_RETRY if retry else STREAM_R)) \
        if sketch_kind == "gaussian" else (lambda retry: srft_sketch(A, seed, l, retry))
    Y = mk(False)
    qr = pivoted_qr(Y, k)
    if qr.status == RID_ERANK:  # PAPER.md:80 re-randomise once
        retries = 1
        Y = mk(True)
        qr = pivoted_qr(Y, k)
        if qr.status == RID_ERANK:
            raise OracleError(RID_ERANK, f"decompose (rank {qr.rank_achieved})")
    P = backsolve(qr.R, qr.J, k)
    return Decomposition(qr.J, P, Y, retries, qr.resid_norms, qr.tie_margins)


def error_estimate(A, J, P, q: int, seed: int) -> float:
    """Compensated power-iteration estimate of ||A - A[:, J] P||_2 (Table 5, R15/R16)."""
    A = _fortran_c128(A)
    P = _fortran_c128(P)
    m, n = A.shape
    k = P.shape[0]
    Jc = np.ascontiguousarray(J, dtype=np.int64)
    est = ctypes.c_double(0.0)
    st = lib().orc_error_estimate(m, n, _ptr(A), m, _ptr(Jc), k, _ptr(P), k, int(q), seed,
                                  ctypes.byref(est))
    if st:
        raise OracleError(st, "error_estimate")
    return est.value


def error_bound(m: int, n: int, k: int, eps: float, sigma_kp1: float) -> float:
    """Eq. (3) right-hand side."""
    return lib().orc_error_bound(m, n, k, eps, sigma_kp1)


def noise_floor(m: int, n: int, delta: float = 1e-16) -> float:
    """sqrt(2 min(m, n)) * delta."""
    return lib().orc_noise_floor(m, n, delta)
