"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``O`` — the plain-C restatement (oracle/qpack_oracle.c), built on demand
  with gcc (present both here and on the GPU box).
* ``R`` — the unmodified reference compiled from /root/reference by
  oracle/Makefile into oracle/_ref/libqpack_ref.so.  It can only be BUILT in
  the build container; the prebuilt .so travels to the GPU box with the repo
  snapshot.  ``ref()`` returns None when it is absent.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package.  The product path (paper_0710_0510_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libqpack_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqpack_ref.so")
REF_SRC = os.environ.get("QPACK_REFERENCE", "/root/reference/proj")

_lock = threading.Lock()
_oracle = None
_ref = None

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
U64, U32, I, D, VP = C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_void_p
PU64, PU32, PD = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when the reference sources are present,
    the reference library (oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(os.path.join(REF_SRC, "src")):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


def oracle():
    global _oracle
    with _lock:
        if _oracle is None:
            src = os.path.join(HERE, "qpack_oracle.c")
            if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
                subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
            lib = C.CDLL(ORACLE_SO)
            _sig(lib, "qo_last_error", C.c_char_p, [])
            _sig(lib, "qo_splitmix_at", U64, [U64, U64])
            _sig(lib, "qo_draws_u8", None, [U64, U64, U64, U64, u8p])
            _sig(lib, "qo_premul_floor_bound", I, [D, PU64])
            _sig(lib, "qo_reciprocal", I, [U64, PD, PU64])
            _sig(lib, "qo_floor_div_premul", I, [U64, D, U64, PU64])
            _sig(lib, "qo_is_prime", I, [U64])
            _sig(lib, "qo_validate", I, [U64, U64, U32, U32, U32])
            _sig(lib, "qo_qadic_for_degree", I, [U64, U32, U32, PU64, PU32, PU32])
            _sig(lib, "qo_correction_table", I, [U64, U64, U32, I, U64, C.POINTER(PU64), PU64, PU64])
            _sig(lib, "qo_redq_run_f64", I, [U64, U64, U32, I, U32, I, f64p, U64, u8p])
            _sig(lib, "qo_redq_run_u64", I, [U64, U64, U32, I, U32, I, u64p, U64, u64p])
            _sig(lib, "qo_redq_run_u128", I, [U64, U64, U32, I, U32, I, u64p, U64, u64p])
            _sig(lib, "qo_redq_trace", I, [U64, U64, U32, U64, U64, PU64, PU64, u64p, u64p])
            _sig(lib, "qo_polymul_batch", I, [U64, U32, u8p, u8p, U64, u8p])
            _sig(lib, "qo_fqt_mul", I, [U64, U32, U64, U32, u64p, U64, u64p, U64, u64p, u64p])
            _sig(lib, "qo_fqt_mul_m", I, [U64, U32, U64, U32, U32, u64p, U64, u64p, U64, u64p, u64p])
            _sig(lib, "qo_field_build", VP, [U64, U32, U64, I])
            _sig(lib, "qo_field_free", None, [VP])
            _sig(lib, "qo_field_mul", U32, [VP, U32, U32])
            _sig(lib, "qo_field_add", U32, [VP, U32, U32])
            _sig(lib, "qo_fgdp_dot", U32, [VP, u32p, u32p, U64, U64, u64p])
            _sig(lib, "qo_rep_to_bytes", None, [VP, U32, u8p])
            _sig(lib, "qo_gfq_mul_batch", I, [VP, u8p, u8p, U64, u8p, I])
            _sig(lib, "qo_gfq_matmul", I, [VP, u8p, u8p, U64, U64, U64, U64, U64, u8p, I])
            _sig(lib, "qo_gfq_freivalds", I, [VP, u8p, u8p, u8p, U64, U64, U64, U64, I])
            _sig(lib, "qo_poly_mod", I, [u64p, U64, u64p, U32, U64, u64p])
            _sig(lib, "qo_naive_gfq_dot", I, [u64p, u64p, U64, U32, u64p, U64, u64p])
            _sig(lib, "qo_fold_checksum_u8", U64, [u8p, U64, U64])
            _sig(lib, "qo_fold_checksum_u64", U64, [u64p, U64])
            _oracle = lib
    return _oracle


def ref():
    """The unmodified reference library, or None if it was never built."""
    global _ref
    with _lock:
        if _ref is None and os.path.exists(REF_SO):
            lib = C.CDLL(REF_SO)
            _sig(lib, "ref_last_error", C.c_char_p, [])
            _sig(lib, "ref_draws_u8", I, [U64, U64, U64, u8p])
            _sig(lib, "ref_splitmix_next", U64, [U64, U64])
            _sig(lib, "ref_reciprocal", I, [U64, PD, PU64])
            _sig(lib, "ref_premul_floor_bound", I, [D, PU64])
            _sig(lib, "ref_floor_div_premul", I, [U64, U64, PU64])
            _sig(lib, "ref_qadic_for_degree", I, [U64, U32, U32, PU64, PU32, PU32])
            _sig(lib, "ref_validate", I, [U64, U64, U32, U32, U32])
            _sig(lib, "ref_correction_table", I, [U64, U64, U32, I, u64p, U64, PU64, PU64])
            _sig(lib, "ref_redq_batch", I, [U64, U64, U32, I, U32, I, f64p, U64, u8p, I, PU64, u64p])
            _sig(lib, "ref_redq_batch_u64", I, [U64, U64, U32, I, U32, I, u64p, U64, u64p])
            _sig(lib, "ref_redq_trace", I, [U64, U64, U32, U64, U64, PU64, PU64, u64p, u64p, PU64, PU64])
            _sig(lib, "ref_polymul_batch", I, [U64, U32, u8p, u8p, U64, u8p, I, I, PU64, u64p])
            _sig(lib, "ref_fqt_mul", I, [U64, U32, U64, U32, u64p, U64, u64p, U64, u64p, u64p])
            _sig(lib, "ref_fqt_mul_m", I, [U64, U32, U64, U32, U32, u64p, U64, u64p, U64, u64p, u64p])
            _sig(lib, "ref_field_build", VP, [U64, U32, U64, I])
            _sig(lib, "ref_field_free", None, [VP])
            _sig(lib, "ref_field_info", I, [VP, u64p, u64p, PU32, PU64, C.c_char_p, U64])
            _sig(lib, "ref_field_tables", I, [VP, u64p, f64p, u32p])
            _sig(lib, "ref_field_op", I, [VP, I, u32p, u32p, U64, u32p])
            _sig(lib, "ref_gfq_mul_batch", I, [VP, u8p, u8p, U64, u8p, I, I, PU64, u64p])
            _sig(lib, "ref_gfq_matmul", I, [VP, u8p, u8p, U64, U64, U64, U64, U64, u8p, I, I, PU64, u64p])
            _sig(lib, "ref_gfq_matmul_rep", I, [VP, u32p, u32p, U64, U64, U64, u32p, u64p])
            _sig(lib, "ref_fgdp_dot", I, [VP, u32p, u32p, U64, PU32, u64p])
            _sig(lib, "ref_fold_checksum", U64, [u64p, U64])
            _ref = lib
    return _ref


def _chk(lib, rc, prefix="qo"):
    if rc != 0:
        msg = (lib.qo_last_error() if prefix == "qo" else lib.ref_last_error()).decode()
        raise OracleError(rc, msg)


# ---------------------------------------------------------------- helpers
FNV_OFFSET = 0xCBF29CE484222325


def checksum_u8(arr: np.ndarray, state: int = FNV_OFFSET) -> int:
    a = np.ascontiguousarray(arr, dtype=np.uint8).reshape(-1)
    return int(oracle().qo_fold_checksum_u8(a, a.size, state))


def draws(seed: int, count: int, bound: int, start: int = 0) -> np.ndarray:
    out = np.empty(count, np.uint8)
    oracle().qo_draws_u8(seed, start, count, bound, out)
    return out


def redq_f64(p, q, d, words, float_mode=True, window=0, binary_shift=False):
    w = np.ascontiguousarray(words, np.float64)
    out = np.empty(w.size * (d + 1), np.uint8)
    lib = oracle()
    _chk(lib, lib.qo_redq_run_f64(p, q, d, int(float_mode), window, int(binary_shift), w, w.size, out))
    return out.reshape(w.size, d + 1)


def redq_u64(p, q, d, words, float_mode=False, window=0, binary_shift=False):
    w = np.ascontiguousarray(words, np.uint64)
    out = np.empty(w.size * (d + 1), np.uint64)
    lib = oracle()
    _chk(lib, lib.qo_redq_run_u64(p, q, d, int(float_mode), window, int(binary_shift), w, w.size, out))
    return out.reshape(w.size, d + 1)


def redq_u128(p, q, d, words, float_mode=False, window=0, binary_shift=False):
    """words: (n, 2) uint64 (lo, hi) halves of u128 words."""
    w = np.ascontiguousarray(words, np.uint64).reshape(-1, 2)
    out = np.empty(w.shape[0] * (d + 1), np.uint64)
    lib = oracle()
    _chk(lib, lib.qo_redq_run_u128(p, q, d, int(float_mode), window, int(binary_shift), w.reshape(-1), w.shape[0],
                                   out))
    return out.reshape(w.shape[0], d + 1)


def polymul_batch(p, d, a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    n = a.shape[0]
    out = np.empty((n, 2 * d + 1), np.uint8)
    lib = oracle()
    _chk(lib, lib.qo_polymul_batch(p, d, a, b, n, out))
    return out


def fqt_mul(p, d, q, n_q, a, b, m=53):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    out = np.zeros(max(a.size + b.size - 1, 1), np.uint64)
    cost = np.zeros(4, np.uint64)
    lib = oracle()
    _chk(lib, lib.qo_fqt_mul_m(p, d, q, n_q, m, a, a.size, b, b.size, out, cost))
    return out[: a.size + b.size - 1] if a.size and b.size else out[:0], cost


class Field:
    """Restated GfqField (gfq.cpp:132-258)."""

    def __init__(self, p, k, q, binary_shift=False):
        lib = oracle()
        self.h = lib.qo_field_build(p, k, q, int(binary_shift))
        if not self.h:
            raise OracleError(-1, lib.qo_last_error().decode())
        self.p, self.k, self.q = p, k, q

    def __del__(self):
        if getattr(self, "h", None):
            oracle().qo_field_free(self.h)
            self.h = None

    def mul_batch(self, a, b, algo=0):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        out = np.empty_like(a)
        _chk(oracle(), oracle().qo_gfq_mul_batch(self.h, a, b, a.shape[0], out, algo))
        return out

    def matmul_rows(self, A, B, row_lo, row_hi, threads=os.cpu_count() or 1):
        """Rows [row_lo,row_hi) of A*B; A is m x K x k, B is K x n x k (uint8)."""
        A = np.ascontiguousarray(A, np.uint8)
        B = np.ascontiguousarray(B, np.uint8)
        m, K, k = A.shape
        n = B.shape[1]
        C_ = np.zeros((m, n, k), np.uint8)
        _chk(oracle(), oracle().qo_gfq_matmul(self.h, A, B, m, K, n, row_lo, row_hi, C_, threads))
        return C_[row_lo:row_hi]

    def freivalds(self, A, B, Cm, seed=12345, trials=4):
        A = np.ascontiguousarray(A, np.uint8)
        B = np.ascontiguousarray(B, np.uint8)
        Cm = np.ascontiguousarray(Cm, np.uint8)
        m, K, _ = A.shape
        n = B.shape[1]
        return bool(oracle().qo_gfq_freivalds(self.h, A, B, Cm, m, K, n, seed, trials))

    def dot(self, v1, v2):
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        cost = np.zeros(4, np.uint64)
        r = oracle().qo_fgdp_dot(self.h, v1, v2, v1.size, 1, cost)
        return int(r), cost

    def rep_to_coeffs(self, rep):
        c = np.zeros(self.k, np.uint8)
        oracle().qo_rep_to_bytes(self.h, rep, c)
        return c.tolist()


class RefField:
    """The reference GfqField, through ref_shim.cpp."""

    def __init__(self, p, k, q, binary_shift=False):
        lib = ref()
        if lib is None:
            raise OracleError(-1, "reference library not built (oracle/_ref)")
        self.h = lib.ref_field_build(p, k, q, int(binary_shift))
        if not self.h:
            raise OracleError(-1, lib.ref_last_error().decode())
        self.p, self.k, self.q = p, k, q

    def __del__(self):
        if getattr(self, "h", None) and ref() is not None:
            ref().ref_field_free(self.h)
            self.h = None

    def info(self):
        mod = np.zeros(self.k + 1, np.uint64)
        gen = np.zeros(self.k, np.uint64)
        nq = C.c_uint32()
        mem = C.c_uint64()
        buf = C.create_string_buffer(512)
        ref().ref_field_info(self.h, mod, gen, C.byref(nq), C.byref(mem), buf, 512)
        return dict(modulus=mod.tolist(), generator=gen.tolist(), n_q=nq.value,
                    memory_entries=mem.value, describe=buf.value.decode())

    def tables(self):
        order = self.p ** self.k
        to_index = np.zeros(order, np.uint64)
        fval = np.zeros(order, np.float64)
        from_index = np.zeros(order, np.uint32)
        ref().ref_field_tables(self.h, to_index, fval, from_index)
        return to_index, fval, from_index

    def mul_batch(self, a, b, algo=0, threads=1, out=None):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        out = np.empty_like(a) if out is None else out
        ns = C.c_uint64()
        cost = np.zeros(4, np.uint64)
        _chk(ref(), ref().ref_gfq_mul_batch(self.h, a, b, a.shape[0], out, algo, threads, C.byref(ns), cost), "ref")
        return out, ns.value, cost

    def matmul(self, A, B, row_lo=0, row_hi=None, algo=1, threads=os.cpu_count() or 1, out=None):
        """out: optional (m, n, k) uint8 buffer (rows [row_lo, row_hi) are written)."""
        A = np.ascontiguousarray(A, np.uint8)
        B = np.ascontiguousarray(B, np.uint8)
        m, K, k = A.shape
        n = B.shape[1]
        row_hi = m if row_hi is None else row_hi
        C_ = np.zeros((m, n, k), np.uint8) if out is None else out
        ns = C.c_uint64()
        cost = np.zeros(4, np.uint64)
        _chk(ref(), ref().ref_gfq_matmul(self.h, A, B, m, K, n, row_lo, row_hi, C_, algo, threads,
                                         C.byref(ns), cost), "ref")
        return C_[row_lo:row_hi], ns.value, cost

    def op(self, op, a, b=None):
        a = np.ascontiguousarray(a, np.uint32)
        bb = np.ascontiguousarray(b if b is not None else a, np.uint32)
        out = np.empty_like(a)
        _chk(ref(), ref().ref_field_op(self.h, op, a, bb, a.size, out), "ref")
        return out

    def dot(self, v1, v2):
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        out = C.c_uint32()
        cost = np.zeros(4, np.uint64)
        _chk(ref(), ref().ref_fgdp_dot(self.h, v1, v2, v1.size, C.byref(out), cost), "ref")
        return out.value, cost

    def matmul_rep(self, A, B):
        A = np.ascontiguousarray(A, np.uint32)
        B = np.ascontiguousarray(B, np.uint32)
        m, K = A.shape
        n = B.shape[1]
        out = np.empty((m, n), np.uint32)
        cost = np.zeros(4, np.uint64)
        _chk(ref(), ref().ref_gfq_matmul_rep(self.h, A, B, m, K, n, out, cost), "ref")
        return out, cost


def ref_redq_f64(p, q, d, words, float_mode=True, window=0, binary_shift=False, threads=1, out=None):
    w = np.ascontiguousarray(words, np.float64)
    out = np.empty((w.size, d + 1), np.uint8) if out is None else out
    ns = C.c_uint64()
    cost = np.zeros(4, np.uint64)
    lib = ref()
    _chk(lib, lib.ref_redq_batch(p, q, d, int(float_mode), window, int(binary_shift), w, w.size, out, threads,
                                 C.byref(ns), cost), "ref")
    return out, ns.value, cost


def ref_polymul_batch(p, d, a, b, algo=0, threads=1, out=None):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    n = a.shape[0]
    out = np.empty((n, 2 * d + 1), np.uint8) if out is None else out
    ns = C.c_uint64()
    cost = np.zeros(4, np.uint64)
    lib = ref()
    _chk(lib, lib.ref_polymul_batch(p, d, a, b, n, out, algo, threads, C.byref(ns), cost), "ref")
    return out, ns.value, cost
