"""qpack-b200: the q-adic transform pipeline of arXiv 0710.0510 on B200.

Python face of the C-ABI in include/qpack_b200.h (libqpack_b200.so, built
in-tree by ``paper_0710_0510_b200.build``).  Names follow the reference's
C++ API (proj/include/qpack): RedqPlan, GfqField, fgdp_dot, gfq_matmul ...;
batched calls take either numpy arrays (host memory, synchronous: the
``*_host`` C entry points) or CUDA torch tensors (device memory, asynchronous
on torch's current stream).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .configs import CONFIGS, C1, C2, C3, C4, C5, Config, scaled  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libqpack_b200.so")
if os.environ.get("QPK_DEV_LIB"):  # development: load a variant build (scripts/)
    LIB_PATH = os.path.abspath(os.environ["QPK_DEV_LIB"])

# ---------------------------------------------------------------- errors
QPK_OK, QPK_ERR_INVALID_ARGUMENT, QPK_ERR_DOMAIN, QPK_ERR_LENGTH = 0, 1, 2, 3
QPK_ERR_OUT_OF_RANGE, QPK_ERR_OVERFLOW, QPK_ERR_RUNTIME, QPK_ERR_LOGIC, QPK_ERR_CUDA = 4, 5, 6, 7, 8


class QpackError(RuntimeError):
    status = -1


class InvalidArgument(QpackError, ValueError):  # std::invalid_argument
    status = QPK_ERR_INVALID_ARGUMENT


class DomainError(QpackError, ValueError):  # std::domain_error
    status = QPK_ERR_DOMAIN


class LengthError(QpackError, ValueError):  # std::length_error
    status = QPK_ERR_LENGTH


class OutOfRange(QpackError, IndexError):  # std::out_of_range
    status = QPK_ERR_OUT_OF_RANGE


class OverflowErr(QpackError, OverflowError):  # std::overflow_error
    status = QPK_ERR_OVERFLOW


class RuntimeErr(QpackError):  # std::runtime_error
    status = QPK_ERR_RUNTIME


class LogicErr(QpackError):  # std::logic_error
    status = QPK_ERR_LOGIC


class CudaError(QpackError):  # device failure / no device
    status = QPK_ERR_CUDA


_ERRORS = {c.status: c for c in (InvalidArgument, DomainError, LengthError, OutOfRange, OverflowErr, RuntimeErr,
                                 LogicErr, CudaError)}

# ---------------------------------------------------------------- library
_lib = None
VP, U64, U32, I, D = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
PU64, PU32, PD = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_double)


class Cost(C.Structure):
    """CostReport (counters.hpp:20-33)."""

    _fields_ = [("mul_add", C.c_uint64), ("divisions", C.c_uint64), ("table_accesses", C.c_uint64),
                ("reduction_calls", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


PCost = C.POINTER(Cost)

# name -> (restype, argtypes); every symbol declared in include/qpack_b200.h
SIGNATURES = {
    "qpk_last_error": (C.c_char_p, []),
    "qpk_abi_version": (I, []),
    "qpk_device_info": (I, [C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
    "qpk_redq_plan_create": (I, [U64, U64, U32, I, C.POINTER(VP)]),
    "qpk_redq_plan_attach_table": (I, [VP, U32, I]),
    "qpk_redq_plan_attach_table_bytes": (I, [VP, VP, U64]),
    "qpk_redq_plan_destroy": (None, [VP]),
    "qpk_redq_residues_f64": (I, [VP, VP, U64, VP, VP]),
    "qpk_redq_residues_f64_host": (I, [VP, VP, U64, VP, PCost]),
    "qpk_redq_residues_u64": (I, [VP, VP, U64, VP, VP]),
    "qpk_redq_residues_u64_host": (I, [VP, VP, U64, VP, PCost]),
    "qpk_redq_residues_u128": (I, [VP, VP, U64, VP, VP]),
    "qpk_redq_residues_u128_host": (I, [VP, VP, U64, VP, PCost]),
    "qpk_redq_sync": (I, [VP, VP]),
    "qpk_redq_cost": (I, [VP, U64, PCost]),
    "qpk_polymul_plan_create": (I, [U64, U64, U32, U32, C.POINTER(VP)]),
    "qpk_polymul_plan_create_m": (I, [U64, U64, U32, U32, U32, C.POINTER(VP)]),
    "qpk_polymul_plan_destroy": (None, [VP]),
    "qpk_polymul_batch": (I, [VP, VP, VP, U64, VP, VP]),
    "qpk_polymul_batch_host": (I, [VP, VP, VP, U64, VP, PCost]),
    "qpk_polymul_sync": (I, [VP, VP]),
    "qpk_field_create": (I, [U64, U32, U64, I, C.POINTER(VP)]),
    "qpk_field_destroy": (None, [VP]),
    "qpk_field_info": (I, [VP, VP, VP, PU32, PU64]),
    "qpk_field_describe": (I, [VP, C.c_char_p, U64]),
    "qpk_field_tables": (I, [VP, VP, VP, VP, VP, VP, VP]),
    "qpk_field_op": (I, [VP, I, VP, VP, U64, VP]),
    "qpk_field_op1": (I, [VP, I, U32, U32, C.POINTER(C.c_uint32)]),
    "qpk_field_sync": (I, [VP, VP]),
    "qpk_fgdp_dot": (I, [VP, VP, VP, U64, PU32, PCost]),
    "qpk_gfq_mul_batch": (I, [VP, VP, VP, U64, VP, I, VP]),
    "qpk_gfq_mul_batch_host": (I, [VP, VP, VP, U64, VP, I]),
    "qpk_gfq_mul_rep_host": (I, [VP, VP, VP, U64, VP]),
    "qpk_gfq_matmul": (I, [VP, VP, VP, U64, U64, U64, U32, VP, VP]),
    "qpk_gfq_matmul_host": (I, [VP, VP, VP, U64, U64, U64, U32, VP, PCost]),
    "qpk_gfq_matmul_repack": (I, [VP, VP, VP, U64, U64, U64, U32, U32, VP, VP]),
    "qpk_gfq_matmul_repack_host": (I, [VP, VP, VP, U64, U64, U64, U32, U32, VP, PCost]),
    "qpk_gfq_matmul_rep": (I, [VP, VP, VP, U64, U64, U64, VP, VP]),
    "qpk_gfq_matmul_rep_host": (I, [VP, VP, VP, U64, U64, U64, VP, PCost]),
    "qpk_gfq_gemv": (I, [VP, VP, VP, U64, U64, VP, VP, VP]),
    "qpk_fqt_mul": (I, [VP, VP, U64, VP, U64, VP, VP]),
    "qpk_fqt_mul_host": (I, [VP, VP, U64, VP, U64, VP, PCost]),
    "qpk_fqt_mul_u64": (I, [VP, VP, U64, VP, U64, VP, VP]),
    "qpk_fqt_mul_u64_host": (I, [VP, VP, U64, VP, U64, VP, PCost]),
    "qpk_gfq_gemv_host": (I, [VP, VP, VP, U64, U64, VP, VP, PCost]),
    "qpk_gen_draws": (I, [U64, U64, U64, U32, VP, VP]),
    "qpk_gen_words": (I, [U64, U64, U64, U64, U32, VP, VP]),
    "qpk_gen_pairs": (I, [U64, U64, U32, U32, VP, VP, VP]),
    "qpk_probe_fp64": (I, [I, I, PD]),
}


def lib():
    """Load libqpack_b200.so (raises ImportError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"qpack-b200: {LIB_PATH} missing; run `python -m paper_0710_0510_b200.build`")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype, f.argtypes = res, args
        _lib = h
    return _lib


def _check(rc):
    if rc != QPK_OK:
        msg = lib().qpk_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, QpackError)(msg)


def build():
    from .build import build as _b
    return _b()


# ----------------------------------------------------------- buffer helpers
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return x.data_ptr()
    return x.ctypes.data


def _stream(x=None):
    import torch
    return torch.cuda.current_stream().cuda_stream


def _host(x, dtype):
    a = np.ascontiguousarray(x, dtype=dtype)
    return a


def _dev(t, dtypes, name, numel=None):
    """A device-path tensor argument: a CUDA tensor, contiguous, of one of
    `dtypes` (torch dtype names), holding at least `numel` elements; anything
    else raises InvalidArgument before a pointer reaches the C-ABI."""
    if not _is_torch(t):
        raise InvalidArgument(f"{name}: expected a CUDA tensor (the other operands are on the device)")
    if str(t.dtype).replace("torch.", "") not in dtypes:
        raise InvalidArgument(f"{name}: dtype {t.dtype} (expected {' / '.join(dtypes)})")
    if not t.is_contiguous():
        raise InvalidArgument(f"{name}: tensor is not contiguous")
    if t.device.type != "cuda":
        raise InvalidArgument(f"{name}: tensor is on {t.device}, not a CUDA device")
    if numel is not None and t.numel() < numel:
        raise InvalidArgument(f"{name}: {t.numel()} elements, needs {numel}")
    return t


def _out_host(out, dtype, numel, name="out"):
    """A caller's host output buffer: a C-contiguous numpy array of `dtype`
    with at least `numel` elements (results are written through its pointer)."""
    if not isinstance(out, np.ndarray) or out.dtype != np.dtype(dtype):
        raise InvalidArgument(f"{name}: expected a numpy {np.dtype(dtype)} array")
    if not out.flags.c_contiguous or not out.flags.writeable:
        raise InvalidArgument(f"{name}: array is not C-contiguous and writeable")
    if out.size < numel:
        raise InvalidArgument(f"{name}: {out.size} elements, needs {numel}")
    return out


def _records(a, b, k, name):
    """n records of k bytes in two equally sized operands."""
    na, nb = (a.numel(), b.numel()) if _is_torch(a) else (a.size, b.size)
    if na != nb or na % k:
        raise InvalidArgument(f"{name}: operands of {na} and {nb} bytes are not the same n records of {k} bytes")
    return na // k


# ----------------------------------------------------------------- REDQ
BASE_P, BINARY_SHIFT = 0, 1
INTEGER, FLOAT_PREMUL = 0, 1


class RedqPlan:
    """RedqPlan (redq.hpp:46-61) with its device mirror."""

    def __init__(self, p, q, d, mode=INTEGER):
        h = VP()
        _check(lib().qpk_redq_plan_create(p, q, d, mode, C.byref(h)))
        self._h, self.p, self.q, self.d, self.mode = h, p, q, d, mode
        self.window = 0

    @classmethod
    def build(cls, p, q, d, mode=INTEGER):
        return cls(p, q, d, mode)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.qpk_redq_plan_destroy(self._h)
            self._h = None

    def attach_correction(self, window, indexing=BASE_P):
        _check(lib().qpk_redq_plan_attach_table(self._h, window, indexing))
        self.window = window
        return self

    def attach_table_bytes(self, blob: bytes):
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib().qpk_redq_plan_attach_table_bytes(self._h, C.cast(buf, VP), len(blob)))
        return self

    def residues(self, words, out=None):
        """redq_residues_into over a batch: words (n,) float64 -> (n, d+1) uint8;
        (n,) uint64 / int64 integer words, (n, 2) uint64 / int64 u128 words as
        (lo, hi) pairs.
        numpy in -> host path (synchronous); CUDA tensor in -> device path on
        torch's current stream (call .sync() to surface data errors)."""
        nd = self.d + 1
        if _is_torch(words):
            import torch
            _dev(words, ("float64", "int64", "uint64"), "words")
            wide = words.dtype in (torch.int64, torch.uint64) and words.dim() == 2 and words.shape[-1] == 2
            n = words.shape[0] if wide else words.numel()  # u128 words as (lo, hi) pairs
            if out is None:
                out = torch.empty((n, nd), dtype=torch.uint8, device=words.device)
            _dev(out, ("uint8",), "out", n * nd)
            if wide:
                _check(lib().qpk_redq_residues_u128(self._h, _ptr(words), n, _ptr(out), _stream()))
            elif words.dtype in (torch.int64, torch.uint64):  # integer words (two's-complement bits as u64)
                _check(lib().qpk_redq_residues_u64(self._h, _ptr(words), n, _ptr(out), _stream()))
            else:
                _check(lib().qpk_redq_residues_f64(self._h, _ptr(words), n, _ptr(out), _stream()))
            return out
        if isinstance(words, np.ndarray) and words.dtype == np.uint64 and words.ndim == 2 and words.shape[1] == 2:
            w = np.ascontiguousarray(words)  # u128 words as (lo, hi) pairs
            out = np.empty((w.shape[0], nd), np.uint8) if out is None else _out_host(out, np.uint8, w.shape[0] * nd)
            cost = Cost()
            _check(lib().qpk_redq_residues_u128_host(self._h, _ptr(w), w.shape[0], _ptr(out), C.byref(cost)))
            self.last_cost = cost.as_dict()
            return out
        if isinstance(words, np.ndarray) and words.dtype == np.uint64:
            w = np.ascontiguousarray(words).reshape(-1)
            out = np.empty((w.size, nd), np.uint8) if out is None else _out_host(out, np.uint8, w.size * nd)
            cost = Cost()
            _check(lib().qpk_redq_residues_u64_host(self._h, _ptr(w), w.size, _ptr(out), C.byref(cost)))
            self.last_cost = cost.as_dict()
            return out
        w = _host(words, np.float64).reshape(-1)
        out = np.empty((w.size, nd), np.uint8) if out is None else _out_host(out, np.uint8, w.size * nd)
        cost = Cost()
        _check(lib().qpk_redq_residues_f64_host(self._h, _ptr(w), w.size, _ptr(out), C.byref(cost)))
        self.last_cost = cost.as_dict()
        return out

    def sync(self):
        _check(lib().qpk_redq_sync(self._h, _stream()))

    def cost(self, n):
        c = Cost()
        _check(lib().qpk_redq_cost(self._h, n, C.byref(c)))
        return c.as_dict()


class PolymulPlan:
    """Batched dqt_mul_poly / single-chunk fqt_mul (dqt.hpp:46, polymul.hpp:42)."""

    def __init__(self, p, q, k, n_q=1, m=53):
        """m > 53: integer (u128) words for fqt_mul, the reference's integer mode."""
        h = VP()
        _check(lib().qpk_polymul_plan_create_m(p, q, k, n_q, m, C.byref(h)))
        self._h, self.p, self.q, self.k, self.m = h, p, q, k, m

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.qpk_polymul_plan_destroy(self._h)
            self._h = None

    def __call__(self, a, b, out=None):
        ko = 2 * self.k - 1
        if _is_torch(a):
            import torch
            _dev(a, ("uint8",), "a")
            _dev(b, ("uint8",), "b")
            n = _records(a, b, self.k, "polymul_batch")
            if out is None:
                out = torch.empty((n, ko), dtype=torch.uint8, device=a.device)
            _dev(out, ("uint8",), "out", n * ko)
            _check(lib().qpk_polymul_batch(self._h, _ptr(a), _ptr(b), n, _ptr(out), _stream()))
            return out
        a = _host(a, np.uint8)
        b = _host(b, np.uint8)
        n = _records(a, b, self.k, "polymul_batch")
        out = np.empty((n, ko), np.uint8) if out is None else _out_host(out, np.uint8, n * ko)
        cost = Cost()
        _check(lib().qpk_polymul_batch_host(self._h, _ptr(a), _ptr(b), n, _ptr(out), C.byref(cost)))
        self.last_cost = cost.as_dict()
        return out

    def sync(self):
        _check(lib().qpk_polymul_sync(self._h, _stream()))

    def _fqt_mul_u64(self, a, b, out=None):
        if _is_torch(a):
            import torch
            _dev(a, ("int64", "uint64"), "a")
            _dev(b, ("int64", "uint64"), "b")
            na, nb = a.numel(), b.numel()
            no = na + nb - 1 if na and nb else 0
            if out is None:
                out = torch.empty((no,), dtype=torch.int64, device=a.device)
            _dev(out, ("int64", "uint64"), "out", no)
            _check(lib().qpk_fqt_mul_u64(self._h, _ptr(a), na, _ptr(b), nb, _ptr(out), _stream()))
            return out
        a = _host(a, np.uint64).reshape(-1)
        b = _host(b, np.uint64).reshape(-1)
        no = a.size + b.size - 1 if a.size and b.size else 0
        out = np.empty((no,), np.uint64) if out is None else _out_host(out, np.uint64, no)
        cost = Cost()
        _check(lib().qpk_fqt_mul_u64_host(self._h, _ptr(a), a.size, _ptr(b), b.size, _ptr(out), C.byref(cost)))
        self.last_cost = cost.as_dict()
        return out

    def fqt_mul(self, a, b, out=None):
        """One product of two long polynomials (chunked FQT, fqt_mul
        polymul.cpp:81-147): len(a)+len(b)-1 coefficients mod p.  uint8
        coefficients for p <= 256; uint64 operands (numpy or CUDA tensors)
        take the u64 entry points (any p)."""
        if (_is_torch(a) and str(a.dtype) in ("torch.int64", "torch.uint64")) or \
                (isinstance(a, np.ndarray) and a.dtype in (np.uint64, np.int64)) or self.p > 256:
            return self._fqt_mul_u64(a, b, out)
        if _is_torch(a):
            import torch
            _dev(a, ("uint8",), "a")
            _dev(b, ("uint8",), "b")
            na, nb = a.numel(), b.numel()
            if out is None:  # an empty operand gives the empty product (polymul.cpp:81-88)
                out = torch.empty((na + nb - 1 if na and nb else 0,), dtype=torch.uint8, device=a.device)
            _dev(out, ("uint8",), "out", na + nb - 1 if na and nb else 0)
            _check(lib().qpk_fqt_mul(self._h, _ptr(a), na, _ptr(b), nb, _ptr(out), _stream()))
            return out
        a = _host(a, np.uint8).reshape(-1)
        b = _host(b, np.uint8).reshape(-1)
        no = a.size + b.size - 1 if a.size and b.size else 0
        out = np.empty((no,), np.uint8) if out is None else _out_host(out, np.uint8, no)
        cost = Cost()
        _check(lib().qpk_fqt_mul_host(self._h, _ptr(a), a.size, _ptr(b), b.size, _ptr(out), C.byref(cost)))
        self.last_cost = cost.as_dict()
        return out


# ------------------------------------------------------------- GF(p^k)
PACKED, DLOG, LINEAR = 0, 1, 2


class GfqField:
    """GfqField (gfq.hpp:30-90) with its device mirror."""

    def __init__(self, p, k, q, indexing=BASE_P):
        h = VP()
        _check(lib().qpk_field_create(p, k, q, indexing, C.byref(h)))
        self._h, self.p, self.k, self.q, self.indexing = h, p, k, q, indexing
        self.order = p ** k

    @classmethod
    def build(cls, p, k, q, indexing=BASE_P):
        return cls(p, k, q, indexing)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.qpk_field_destroy(self._h)
            self._h = None

    @property
    def zero(self):
        return self.order - 1

    def sync(self):
        """Wait for torch's current stream and raise what the field's device
        launches latched (OutOfRange: a rep outside the field)."""
        _check(lib().qpk_field_sync(self._h, _stream()))

    def info(self):
        mod = np.zeros(self.k + 1, np.uint64)
        gen = np.zeros(self.k, np.uint64)
        nq = C.c_uint32()
        mem = C.c_uint64()
        _check(lib().qpk_field_info(self._h, _ptr(mod), _ptr(gen), C.byref(nq), C.byref(mem)))
        return dict(modulus=mod.tolist(), generator=gen.tolist(), n_q=nq.value, memory_entries=mem.value)

    def describe(self):
        buf = C.create_string_buffer(1024)
        _check(lib().qpk_field_describe(self._h, buf, 1024))
        return buf.value.decode()

    def tables(self):
        o = self.order
        lh = self.p if self.indexing == BASE_P else 1 << (self.p - 1).bit_length()
        t = dict(log=np.zeros(o, np.uint32), antilog=np.zeros(o, np.uint64), plus1=np.zeros(o, np.uint32),
                 fval=np.zeros(o, np.float64), low=np.zeros(lh ** self.k, np.uint32),
                 high=np.zeros(lh ** self.k, np.uint32))
        _check(lib().qpk_field_tables(self._h, *(_ptr(t[k]) for k in ("log", "antilog", "plus1", "fval", "low",
                                                                        "high"))))
        return t

    @property
    def n_q(self):
        return self.info()["n_q"]

    def to_coeffs(self, rep):
        """to_coeffs (gfq.cpp:296-314): coefficient list of a rep, low first."""
        if rep == self.order - 1:
            return [0] * self.k
        if getattr(self, "_antilog", None) is None:
            self._antilog = self.tables()["antilog"]
        idx, out = int(self._antilog[rep]), []
        for _ in range(self.k):
            out.append(idx % self.p)
            idx //= self.p
        return out

    def op(self, op, a, b=None):
        """n elements on the device (qpk_field_op)."""
        a = _host(a, np.uint32).reshape(-1)
        bb = _host(b, np.uint32).reshape(-1) if b is not None else None
        out = np.empty_like(a)
        _check(lib().qpk_field_op(self._h, op, _ptr(a), _ptr(bb), a.size, _ptr(out)))
        return out

    def op1(self, op, a, b=0):
        """One element through the reference's scalar call (host)."""
        r = C.c_uint32()
        _check(lib().qpk_field_op1(self._h, op, int(a), int(b), C.byref(r)))
        return r.value

    def mul(self, a, b):
        return self.op(0, a, b)

    def add(self, a, b):
        return self.op(1, a, b)

    def fgdp_dot(self, v1, v2):
        v1 = _host(v1, np.uint32).reshape(-1)
        v2 = _host(v2, np.uint32).reshape(-1)
        if v1.size != v2.size:
            raise InvalidArgument("fgdp_dot: vector length mismatch")  # gfq.cpp:337
        out = C.c_uint32()
        cost = Cost()
        _check(lib().qpk_fgdp_dot(self._h, _ptr(v1), _ptr(v2), v1.size, C.byref(out), C.byref(cost)))
        return out.value, cost.as_dict()

    def mul_batch(self, a, b, path=PACKED, out=None):
        """Elementwise products of k-byte coefficient records."""
        if _is_torch(a):
            import torch
            _dev(a, ("uint8",), "a")
            _dev(b, ("uint8",), "b")
            n = _records(a, b, self.k, "gfq_mul_batch")
            if out is None:
                out = torch.empty((n, self.k), dtype=torch.uint8, device=a.device)
            _dev(out, ("uint8",), "out", n * self.k)
            _check(lib().qpk_gfq_mul_batch(self._h, _ptr(a), _ptr(b), n, _ptr(out), path, _stream()))
            return out
        a = _host(a, np.uint8)
        b = _host(b, np.uint8)
        n = _records(a, b, self.k, "gfq_mul_batch")
        out = np.empty((n, self.k), np.uint8) if out is None else _out_host(out, np.uint8, n * self.k)
        _check(lib().qpk_gfq_mul_batch_host(self._h, _ptr(a), _ptr(b), n, _ptr(out), path))
        return out

    def mul_rep_batch(self, a, b):
        a = _host(a, np.uint32).reshape(-1)
        b = _host(b, np.uint32).reshape(-1)
        out = np.empty_like(a)
        _check(lib().qpk_gfq_mul_rep_host(self._h, _ptr(a), _ptr(b), a.size, _ptr(out)))
        return out

    def matmul(self, A, B, m, K, n, chunk=0, out=None, repack="redq", counters=False):
        """C = A*B on coefficient records (A m x K x k, B K x n x k).
        repack: "redq" (delayed REDQ re-pack, the default) or "fold"
        (GF(3^3) at q = 2^10 only; same C).  counters=True (host buffers):
        self.last_cost gets the reference's gfq_matmul counters, the
        data-dependent Zech reads included (an extra device pass, K7)."""
        if repack not in ("redq", "fold"):
            raise InvalidArgument(f"gfq_matmul: unknown re-pack mode {repack!r}")
        mode = {"redq": 0, "fold": 1}[repack]
        k = self.k
        if _is_torch(A):
            import torch
            _dev(A, ("uint8",), "A", m * K * k)
            _dev(B, ("uint8",), "B", K * n * k)
            if out is None:
                out = torch.empty((m, n, self.k), dtype=torch.uint8, device=A.device)
            _dev(out, ("uint8",), "out", m * n * k)
            _check(lib().qpk_gfq_matmul_repack(self._h, _ptr(A), _ptr(B), m, K, n, chunk, mode, _ptr(out),
                                               _stream()))
            return out
        A = _host(A, np.uint8)
        B = _host(B, np.uint8)
        if A.size < m * K * k or B.size < K * n * k:
            raise InvalidArgument("gfq_matmul: A or B holds fewer than m*K or K*n records")
        out = np.empty((m, n, self.k), np.uint8) if out is None else _out_host(out, np.uint8, m * n * k)
        cost = Cost()
        _check(lib().qpk_gfq_matmul_repack_host(self._h, _ptr(A), _ptr(B), m, K, n, chunk, mode, _ptr(out),
                                                C.byref(cost) if counters else None))
        self.last_cost = cost.as_dict() if counters else None
        return out

    def gemv(self, A, x, coeffs=False, out=None, counters=True):
        """y = A x on reps (A m x K, x K): each y_i = fgdp_dot(A[i,:], x) on
        the GPU.  Returns reps (m,) or, with coeffs=True, coefficients (m, k)."""
        if _is_torch(A):
            import torch
            _dev(A, ("int32", "uint32"), "A")
            if A.dim() != 2:
                raise InvalidArgument("gfq_gemv: A must be an m x K tensor")
            m, K = A.shape
            _dev(x, ("int32", "uint32"), "x")
            if x.numel() != K:
                raise InvalidArgument("gfq_gemv: x length differs from the columns of A")
            if out is None:
                out = (torch.empty((m, self.k), dtype=torch.uint8, device=A.device) if coeffs
                       else torch.empty((m,), dtype=torch.int32, device=A.device))
            _dev(out, ("uint8",) if coeffs else ("int32", "uint32"), "out", m * (self.k if coeffs else 1))
            _check(lib().qpk_gfq_gemv(self._h, _ptr(A), _ptr(x), m, K, None if coeffs else _ptr(out),
                                      _ptr(out) if coeffs else None, _stream()))
            return out
        A = _host(A, np.uint32)
        x = _host(x, np.uint32).reshape(-1)
        if A.ndim == 1:
            A = A.reshape(1, -1)
        m, K = A.shape
        if x.size != K:
            raise InvalidArgument("gfq_gemv: x length differs from the columns of A")
        if out is None:
            out = np.empty((m, self.k), np.uint8) if coeffs else np.empty((m,), np.uint32)
        else:
            _out_host(out, np.uint8 if coeffs else np.uint32, m * (self.k if coeffs else 1))
        cost = Cost()
        _check(lib().qpk_gfq_gemv_host(self._h, _ptr(A), _ptr(x), m, K, None if coeffs else _ptr(out),
                                       _ptr(out) if coeffs else None, C.byref(cost) if counters else None))
        self.last_cost = cost.as_dict() if counters else None
        return out

    def fgdp_dot_gpu(self, v1, v2):
        """fgdp_dot of two long rep vectors on the GPU; (rep, counters)."""
        v1 = _host(v1, np.uint32).reshape(-1)
        v2 = _host(v2, np.uint32).reshape(-1)
        if v1.size != v2.size:
            raise InvalidArgument("fgdp_dot: vector length mismatch")  # gfq.cpp:337
        y = self.gemv(v1.reshape(1, -1), v2)
        return int(y[0]), self.last_cost

    def matmul_rep(self, A, B, out=None, counters=False):
        """The reference gfq_matmul on GfqMatrix data (reps in, reps out);
        counters=True (host buffers): self.last_cost = the reference's
        CostReport, data-dependent Zech reads included (K7)."""
        if _is_torch(A):
            import torch
            _dev(A, ("int32", "uint32"), "A")
            _dev(B, ("int32", "uint32"), "B")
            if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
                raise InvalidArgument("gfq_matmul: inner dimensions differ")  # gfq.cpp:391
            m, K = A.shape
            n = B.shape[1]
            if out is None:
                out = torch.empty((m, n), dtype=torch.int32, device=A.device)
            _dev(out, ("int32", "uint32"), "out", m * n)
            _check(lib().qpk_gfq_matmul_rep(self._h, _ptr(A), _ptr(B), m, K, n, _ptr(out), _stream()))
            return out
        A = _host(A, np.uint32)
        B = _host(B, np.uint32)
        if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
            raise InvalidArgument("gfq_matmul: inner dimensions differ")  # gfq.cpp:391
        m, K = A.shape
        n = B.shape[1]
        out = np.empty((m, n), np.uint32) if out is None else _out_host(out, np.uint32, m * n)
        cost = Cost()
        _check(lib().qpk_gfq_matmul_rep_host(self._h, _ptr(A), _ptr(B), m, K, n, _ptr(out),
                                             C.byref(cost) if counters else None))
        self.last_cost = cost.as_dict() if counters else None
        return out


# ------------------------------------------------------ synthetic inputs
def gen_draws(seed, count, bound, out, start=0):
    _check(lib().qpk_gen_draws(seed, start, count, bound, _ptr(out), _stream()))
    return out


def gen_words(seed, n, q, d, out, first=0):
    _check(lib().qpk_gen_words(seed, first, n, q, d, _ptr(out), _stream()))
    return out


def gen_pairs(seed, n, k, bound, a, b):
    _check(lib().qpk_gen_pairs(seed, n, k, bound, _ptr(a), _ptr(b), _stream()))
    return a, b


def probe_fp64(which, iters=4096):
    t = C.c_double()
    _check(lib().qpk_probe_fp64(which, iters, C.byref(t)))
    return t.value


def device_info():
    sms, ma, mi = I(), I(), I()
    _check(lib().qpk_device_info(C.byref(sms), C.byref(ma), C.byref(mi)))
    return dict(sms=sms.value, cc=(ma.value, mi.value))
