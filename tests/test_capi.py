"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/qpack_b200.h declares, and its host-side logic (plan building, field
construction, Zech arithmetic, fgdp_dot, error classes) matches the reference.
"""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qpack_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"QPK_API\s+[\w\s\*]+?\b(qpk_\w+)\s*\(", text)))


def test_header_declares_the_surface():
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in ("qpk_redq_residues_f64", "qpk_gfq_matmul", "qpk_gfq_mul_batch", "qpk_polymul_batch"):
        assert s in syms


def test_library_exports_every_declared_symbol(qpk):
    out = subprocess.run(["nm", "-D", "--defined-only", qpk.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r"\bT (qpk_\w+)", out.stdout))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # the Python binding types every one of them
    assert sorted(qpk.SIGNATURES) == declared_symbols()
    assert qpk.lib().qpk_abi_version() == 1


def test_library_does_not_link_the_oracle(qpk):
    out = subprocess.run(["nm", "-D", qpk.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "qo_" not in out and "ref_" not in re.sub(r"\w+ref_\w*", "", out)
    ldd = subprocess.run(["ldd", qpk.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "qpack_ref" not in ldd


FIELDS = [(7, 3, 256, 0), (3, 2, 1 << 16, 0), (3, 3, 1 << 10, 0), (3, 2, 64, 1), (5, 2, 1 << 17, 1),
          (2, 3, 1 << 10, 0), (2, 1, 1 << 26, 0), (13, 2, 1000, 0), (11, 3, 1 << 10, 1)]


@pytest.mark.parametrize("p,k,q,bs", FIELDS)
def test_field_construction_matches_oracle(qpk, orc, p, k, q, bs):
    f = qpk.GfqField(p, k, q, bs)
    o = orc.Field(p, k, q, bs)
    t = f.tables()
    rng = np.random.default_rng(p + k)
    order = p ** k
    a = rng.integers(0, order, 3000).astype(np.uint32)
    b = rng.integers(0, order, 3000).astype(np.uint32)
    lib = orc.oracle()
    assert all(f.op1(0, x, y) == lib.qo_field_mul(o.h, int(x), int(y)) for x, y in zip(a[:300], b[:300]))
    assert all(f.op1(1, x, y) == lib.qo_field_add(o.h, int(x), int(y)) for x, y in zip(a[:300], b[:300]))
    for n in (0, 1, 5, 100, 301):
        got, cost = f.fgdp_dot(a[:n], b[:n])
        want, wcost = o.dot(a[:n], b[:n])
        assert got == want
        assert [cost["mul_add"], cost["divisions"], cost["reduction_calls"]] == [int(wcost[0]), int(wcost[1]),
                                                                                int(wcost[3])]
    assert t["log"].size == order


@pytest.mark.skipif(__import__("oracle").ref() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("p,k,q,bs", FIELDS)
def test_field_construction_matches_reference(qpk, orc, p, k, q, bs):
    f = qpk.GfqField(p, k, q, bs)
    r = orc.RefField(p, k, q, bs)
    fi, ri = f.info(), r.info()
    for key in ("modulus", "generator", "n_q", "memory_entries"):
        assert fi[key] == ri[key], key
    assert f.describe() == ri["describe"]
    to_index, fval, from_index = r.tables()
    t = f.tables()
    reps = np.arange(p ** k)
    assert (np.where(reps == p ** k - 1, 0, t["antilog"]) == to_index).all()
    assert (t["fval"] == fval).all() and (t["log"] == from_index).all()
    rng = np.random.default_rng(1)
    a = rng.integers(0, p ** k, 4000).astype(np.uint32)
    b = rng.integers(0, p ** k, 4000).astype(np.uint32)
    for op in (0, 1, 2):  # the scalar calls here; the batched device op in tests/test_gpu_parity.py
        want = r.op(op, a[:500], b[:500])
        assert all(f.op1(op, x, y) == w for x, y, w in zip(a[:500], b[:500], want))
    nz = a[a != p ** k - 1][:500]
    assert all(f.op1(3, x) == w for x, w in zip(nz, r.op(3, nz)))
    for n in (1, 7, 8, 85, 86, 1000):
        got, cost = f.fgdp_dot(a[:n], b[:n])
        want, wcost = r.dot(a[:n], b[:n])
        assert got == want and list(cost.values()) == wcost.tolist()


def test_error_classes_match_the_reference(qpk):
    with pytest.raises(qpk.DomainError):
        qpk.GfqField(4, 2, 64)                    # composite p (test_gfq.cpp:280)
    with pytest.raises(qpk.LengthError):
        qpk.GfqField(3, 30, 1 << 16)              # table cap (test_gfq.cpp:281)
    with pytest.raises(qpk.InvalidArgument):
        qpk.RedqPlan(3, 1 << 20, 3, qpk.FLOAT_PREMUL)  # float bound (test_redq.cpp:88)
    with pytest.raises(qpk.InvalidArgument):
        qpk.RedqPlan(1, 128, 6)
    with pytest.raises(qpk.LengthError):
        qpk.RedqPlan(251, 1 << 20, 4).attach_correction(4)  # 251^4 > 2^26 budget
    with pytest.raises(qpk.InvalidArgument):
        qpk.RedqPlan(5, 128, 6).attach_correction(1)
    with pytest.raises(qpk.RuntimeErr):
        qpk.RedqPlan(5, 128, 6).attach_table_bytes(b"not a table")
    f = qpk.GfqField(3, 2, 1 << 16)
    with pytest.raises(qpk.DomainError):
        f.op1(3, f.zero)                          # zero has no inverse
    with pytest.raises(qpk.InvalidArgument):
        f.fgdp_dot([1, 2], [1])


def qpkt_bytes(p, q, w, tag, entries):
    """The reference's serialized table layout (redq.cpp:285-297)."""
    import struct
    return (b"QPKT" + struct.pack("<IQQI", 1, p, q, w) + bytes([tag, 0, 0, 0]) + struct.pack("<Q", len(entries))
            + b"".join(struct.pack("<Q", e) for e in entries))


def test_serialized_tables_attach(qpk, orc):
    import ctypes as C
    ent = C.POINTER(C.c_uint64)()
    n, radix = C.c_uint64(), C.c_uint64()
    orc.oracle().qo_correction_table(5, 128, 4, 0, 1 << 26, C.byref(ent), C.byref(n), C.byref(radix))
    blob = qpkt_bytes(5, 128, 4, 0, [ent[i] for i in range(n.value)])
    assert blob[:4] == b"QPKT" and blob[8] == 5 and blob[16] == 128 and blob[24] == 4  # test_redq.cpp:237-247
    plan = qpk.RedqPlan(5, 128, 6).attach_table_bytes(blob)
    assert plan.cost(10)["table_accesses"] == 20
    with pytest.raises(qpk.InvalidArgument):       # table for another q
        qpk.RedqPlan(5, 256, 6).attach_table_bytes(blob)
    with pytest.raises(qpk.RuntimeErr):            # truncated stream
        qpk.RedqPlan(5, 128, 6).attach_table_bytes(blob[:-3])


def test_closed_form_counters(qpk):
    plan = qpk.RedqPlan(5, 128, 6, qpk.FLOAT_PREMUL).attach_correction(4)
    assert plan.cost(1 << 26) == dict(mul_add=0, divisions=1 << 26, table_accesses=2 << 26, reduction_calls=1 << 26)
    plan = qpk.RedqPlan(5, 10000, 4)  # p | q: identity correction, no table accesses
    assert plan.cost(7)["table_accesses"] == 0


def test_compute_entry_points_fail_loudly_without_a_device(qpk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    plan = qpk.RedqPlan(5, 128, 6, qpk.FLOAT_PREMUL)
    with pytest.raises(qpk.CudaError):
        plan.residues(np.zeros(16))
    with pytest.raises(qpk.CudaError):
        qpk.GfqField(3, 2, 1 << 16).matmul(np.zeros((2, 2, 2), np.uint8), np.zeros((2, 2, 2), np.uint8), 2, 2, 2)
    with pytest.raises(qpk.CudaError):
        qpk.PolymulPlan(3, 32, 4, 1)
    with pytest.raises(qpk.CudaError):
        qpk.GfqField(3, 3, 1 << 10).gemv(np.zeros((2, 8), np.uint32), np.zeros(8, np.uint32))


def test_to_coeffs_matches_oracle(qpk, orc):
    f = qpk.GfqField(7, 3, 256)
    of = orc.Field(7, 3, 256)
    for rep in (0, 1, 5, 100, 341, 342):
        assert f.to_coeffs(rep) == of.rep_to_coeffs(rep)


class _QoField(__import__("ctypes").Structure):
    """oracle/qpack_oracle.h qo_field (the C restatement's field tables)."""
    import ctypes as C
    _fields_ = [("p", C.c_uint64), ("q", C.c_uint64), ("order", C.c_uint64), ("group", C.c_uint64),
                ("lh_radix", C.c_uint64), ("lh_size", C.c_uint64), ("k", C.c_uint32), ("n_q", C.c_uint32),
                ("binary_shift", C.c_int), ("modulus", C.c_uint64 * 33), ("generator_index", C.c_uint64),
                ("log", C.POINTER(C.c_uint32)), ("antilog", C.POINTER(C.c_uint64)), ("plus1", C.POINTER(C.c_uint32)),
                ("fval", C.POINTER(C.c_double)), ("ltab", C.POINTER(C.c_uint32)), ("htab", C.POINTER(C.c_uint32)),
                ("inv_p", C.c_double), ("r_max", C.c_uint64)]


def _default_q(p, k):  # widest power-of-two radix with 2k-1 digits below 2^53 (gfq_default_q)
    return 1 << (52 // (2 * k - 1))


SWEEP_FIELDS = [(p, k, q, bs)
                for (p, k, q) in [(2, 1, 1 << 20), (2, 2, 64), (2, 5, 0), (2, 6, 0), (2, 7, 0), (2, 8, 9),
                                  (3, 1, 1 << 20), (3, 3, 1 << 10), (3, 5, 0), (3, 6, 25), (5, 2, 1 << 12), (5, 4, 0),
                                  (7, 3, 256), (7, 4, 145), (11, 2, 1 << 12), (13, 3, 10 ** 3), (31, 2, 1 << 14),
                                  (101, 2, 1 << 17), (257, 2, 131073), (1009, 1, 1 << 26), (65537, 1, 1 << 40),
                                  (3, 2, 10 ** 4), (5, 3, 999)]
                for bs in (0, 1)]
SWEEP_FIELDS = [(p, k, q or _default_q(p, k), bs) for (p, k, q, bs) in SWEEP_FIELDS]


@pytest.mark.parametrize("p,k,q,bs", SWEEP_FIELDS)
def test_field_tables_match_the_restatement(qpk, orc, p, k, q, bs):
    """Every table of the drop-in's GfqField (log, antilog, Zech, q-adic
    evaluation and both half-window tables) against the C restatement's,
    entry by entry, over 40 fields (k = 1..10, both indexings)."""
    import ctypes as C
    try:
        f = qpk.GfqField(p, k, q, bs)
    except qpk.QpackError:
        pytest.skip("field outside the 2^20-entry table budget")
    o = orc.Field(p, k, q, bs)
    of = C.cast(C.c_void_p(o.h) if isinstance(o.h, int) else o.h, C.POINTER(_QoField)).contents
    t = f.tables()
    order = p ** k
    assert of.order == order and list(of.modulus[:k + 1]) == f.info()["modulus"]
    assert (t["log"] == np.ctypeslib.as_array(of.log, (order,))).all()
    assert (t["antilog"][:order - 1] == np.ctypeslib.as_array(of.antilog, (order,))[:order - 1]).all()
    assert (t["plus1"] == np.ctypeslib.as_array(of.plus1, (order,))).all()
    assert (t["fval"] == np.ctypeslib.as_array(of.fval, (order,))).all()
    assert t["low"].size == of.lh_size
    assert (t["low"] == np.ctypeslib.as_array(of.ltab, (of.lh_size,))).all()
    assert (t["high"] == np.ctypeslib.as_array(of.htab, (of.lh_size,))).all()
