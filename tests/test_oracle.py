"""Pin the C restatement oracle (oracle/qpack_oracle.c) before trusting it.

1. Known-answer vectors copied (as values, with citations) from the
   reference's own tests.
2. The committed golden fixtures, produced by the UNMODIFIED reference
   (tests/golden/make_golden.py).
3. The reference library itself (oracle/_ref) when it is present.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import load_small


def _u64(x):
    return C.c_uint64(x)


# ----------------------------------------------------------- known answers
def test_premul_floor_bound_known(orc):
    o = orc.oracle()
    out = C.c_uint64()
    # test_fpdiv.cpp:31-36
    for eps, want in [(2.0 ** -53, (1 << 52) - 1), (0.5, 0), (2.0 ** -24, (1 << 23) - 1), (2.0 ** -52, (1 << 51) - 1)]:
        assert o.qo_premul_floor_bound(eps, C.byref(out)) == 0
        assert out.value == want
    assert o.qo_premul_floor_bound(0.0, C.byref(out)) != 0
    assert o.qo_premul_floor_bound(1.0, C.byref(out)) != 0
    # survey probe: r_max = bound(3 eps) = 1501199875790165
    inv, rmax = C.c_double(), C.c_uint64()
    o.qo_reciprocal(3, C.byref(inv), C.byref(rmax))
    assert rmax.value == 1501199875790165


def test_premul_division_exhaustive_small_grid(orc):
    # test_fpdiv.cpp:68-73
    o = orc.oracle()
    inv, rmax, out = C.c_double(), C.c_uint64(), C.c_uint64()
    for p in range(1, 41):
        o.qo_reciprocal(p, C.byref(inv), C.byref(rmax))
        for r in list(range(0, 5001, 7)) + [rmax.value, rmax.value - 1]:
            o.qo_floor_div_premul(r, inv.value, rmax.value, C.byref(out))
            assert out.value == r // p


def test_redq_worked_examples(orc):
    # acceptance.cpp:70-80 / test_redq.cpp:26-33: p | q, correction is identity
    r = 40013002800270018
    mu = orc.redq_u64(5, 10000, 4, [r])
    assert mu[0].tolist() == [3, 2, 3, 3, 4]
    # acceptance.cpp:82-88 / test_redq.cpp:35-46: p = 23, q = 10^6, d = 3
    r = 1234005678009123004567
    rop_lo, rop_hi = C.c_uint64(), C.c_uint64()
    u = np.zeros(4, np.uint64)
    mu = np.zeros(4, np.uint64)
    assert orc.oracle().qo_redq_trace(23, 10 ** 6, 3, r & (2 ** 64 - 1), r >> 64, C.byref(rop_lo), C.byref(rop_hi),
                                      u, mu) == 0
    assert (rop_hi.value << 64) | rop_lo.value == 53652420783005348024
    assert u.tolist() == [15, 8, 18, 15]
    assert mu.tolist() == [13, 15, 20, 15]
    word = sum(int(m) * 10 ** (6 * i) for i, m in enumerate(mu))
    assert word == 15000020000015000013


def test_correction_table_sizes(orc):
    # test_redq.cpp:161-167
    o = orc.oracle()
    ent = C.POINTER(C.c_uint64)()
    n, radix = C.c_uint64(), C.c_uint64()
    for p, q, w, bs, size in [(5, 10000, 3, 0, 125), (23, 1000000, 2, 0, 529), (5, 10000, 3, 1, 512)]:
        assert o.qo_correction_table(p, q, w, bs, 1 << 26, C.byref(ent), C.byref(n), C.byref(radix)) == 0
        assert n.value == size
    assert o.qo_correction_table(251, 1 << 20, 4, 0, 1 << 20, C.byref(ent), C.byref(n), C.byref(radix)) == 3


def test_dqt_worked_product(orc):
    # acceptance.cpp:61-68: (X+1)(X+2) over F_3 at q = 100 -> X^2 + 2
    out, cost = orc.fqt_mul(3, 1, 100, 1, [1, 1], [2, 1])
    assert out.tolist() == [2, 0, 1]
    # test_polymul.cpp: squaring X+1 mod 3 with degree-1 chunks at q = 32
    out, _ = orc.fqt_mul(3, 1, 32, 1, [1, 1], [1, 1])
    assert out.tolist() == [1, 2, 1]


def test_gf9_known_answers(orc):
    # test_gfq.cpp:23-36 and test_oracle.cpp:118-128
    f = orc.Field(3, 2, 1 << 17)
    modulus = np.zeros(3, np.uint64)
    o = orc.oracle()
    # naive dot [[1,1],[0,2]] . [[2,1],[0,1]] = [2,0] over F3[X]/(X^2+1)
    out = np.zeros(2, np.uint64)
    o.qo_naive_gfq_dot(np.array([1, 1, 0, 2], np.uint64), np.array([2, 1, 0, 1], np.uint64), 2, 2,
                       np.array([1, 0, 1], np.uint64), 3, out)
    assert out.tolist() == [2, 0]
    # X * X = 2 in GF(9): coefficient records [0,1] x [0,1] -> [2,0]
    got = f.mul_batch(np.array([[0, 1]], np.uint8), np.array([[0, 1]], np.uint8), 0)
    assert got.tolist() == [[2, 0]]
    del modulus


def test_checksum_restatement(orc):
    data = np.arange(1000, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    want = int(orc.oracle().qo_fold_checksum_u64(data, data.size))
    if orc.ref() is not None:
        assert int(orc.ref().ref_fold_checksum(data, data.size)) == want
    b = (np.arange(777) % 251).astype(np.uint8)
    assert orc.checksum_u8(b) == int(orc.oracle().qo_fold_checksum_u64(b.astype(np.uint64), b.size))
    # chaining
    assert orc.checksum_u8(b[300:], orc.checksum_u8(b[:300])) == orc.checksum_u8(b)


# ------------------------------------------------------- golden fixtures
def test_oracle_c1_golden(orc):
    g = load_small(1)
    assert (orc.polymul_batch(3, 3, g["a"], g["b"]) == g["out"]).all()


def test_oracle_c2_golden(orc):
    g = load_small(2)
    for fm in (True, False):
        for win in (0, 2, 3, 4):
            assert (orc.redq_f64(5, 128, 6, g["words"], float_mode=fm, window=win) == g["out"]).all()


def test_oracle_c3_golden(orc):
    g = load_small(3)
    f = orc.Field(7, 3, 256)
    assert (f.mul_batch(g["a"], g["b"], 0) == g["out"]).all()
    assert (f.mul_batch(g["a"], g["b"], 1) == g["out"]).all()


@pytest.mark.parametrize("cid,k,q", [(4, 2, 1 << 16), (5, 3, 1 << 10)])
def test_oracle_matmul_golden(orc, cid, k, q):
    g = load_small(cid)
    n = int(g["n"])
    f = orc.Field(3, k, q)
    assert (f.matmul_rows(g["A"], g["B"], 0, n) == g["out"]).all()
    assert f.freivalds(g["A"], g["B"], g["out"])


def test_golden_inputs_follow_the_pinned_seed_protocol(orc, golden):
    # draw streams of the small fixtures equal the oracle's counter-based draws
    from paper_0710_0510_b200.configs import C1, C2, C3, C4, C5
    g1 = load_small(1)
    dr = orc.draws(C1.seed, 4096 * 8, 3).reshape(4096, 8)
    assert (dr[:, :4] == g1["a"]).all() and (dr[:, 4:] == g1["b"]).all()
    g2 = load_small(2)
    dr = orc.draws(C2.seed, 4096 * 7, 128).reshape(4096, 7).astype(np.uint64)
    w = np.zeros(4096, np.uint64)
    for j in range(7):
        w = w * np.uint64(128) + dr[:, j]
    assert (w.astype(np.float64) == g2["words"]).all()
    g3 = load_small(3)
    dr = orc.draws(C3.seed, 4096 * 6, 7).reshape(4096, 6)
    assert (dr[:, :3] == g3["a"]).all()
    for cfg, cid in ((C4, 4), (C5, 5)):
        g = load_small(cid)
        n = int(g["n"])
        dr = orc.draws(cfg.seed, 2 * n * n * cfg.k, 3)
        assert (dr[: n * n * cfg.k].reshape(n, n, cfg.k) == g["A"]).all()
    # full-size input checksums (first draws of each full stream)
    assert golden["c2"]["n"] == C2.n and golden["c5"]["n"] == C5.n


@pytest.mark.parametrize("cid,bound,per", [(1, 3, 8), (2, 128, 7), (3, 7, 6)])
def test_full_size_input_draw_checksums(orc, golden, cid, bound, per):
    from paper_0710_0510_b200.configs import CONFIGS
    cfg = CONFIGS[cid]
    dr = orc.draws(cfg.seed, cfg.n * per, bound)
    assert f"{orc.checksum_u8(dr):016x}" == golden[f"c{cid}"]["input_draws_checksum"]


# ------------------------------------------------------ against _ref
need_ref = pytest.mark.skipif(__import__("oracle").ref() is None, reason="oracle/_ref not built")


@need_ref
def test_oracle_vs_reference_redq_sweep(orc):
    # acceptance.cpp:106-151 parameter grid (subset) on seeded words
    rng = np.random.default_rng(407)
    for p in (2, 3, 5, 7, 23, 251):
        for q in (1 << 5, 1 << 10, 1 << 16, 10000, 1000000):
            for d in range(0, 8):
                if q ** (d + 1) > (1 << 53):
                    continue
                words = np.floor(rng.random(300) * q ** (d + 1)).astype(np.uint64)
                want = np.empty((300, d + 1), np.uint64)
                orc.ref().ref_redq_batch_u64(p, q, d, 0, 0, 0, words, 300, want)
                assert (orc.redq_u64(p, q, d, words) == want).all(), (p, q, d)


@need_ref
def test_oracle_vs_reference_fields(orc):
    for p, k, q in [(7, 3, 256), (3, 2, 1 << 16), (3, 3, 1 << 10), (5, 2, 1 << 17), (2, 4, 64), (13, 2, 1000)]:
        f, r = orc.Field(p, k, q), orc.RefField(p, k, q)
        rng = np.random.default_rng(p * k)
        a = rng.integers(0, p, (2000, k)).astype(np.uint8)
        b = rng.integers(0, p, (2000, k)).astype(np.uint8)
        assert (f.mul_batch(a, b, 0) == r.mul_batch(a, b, 0)[0]).all()
        v1 = rng.integers(0, p ** k, 300).astype(np.uint32)
        v2 = rng.integers(0, p ** k, 300).astype(np.uint32)
        assert f.dot(v1, v2)[0] == r.dot(v1, v2)[0]


@need_ref
@pytest.mark.skipif(__import__("oracle").ref() is None, reason="oracle/_ref not built")
def test_oracle_vs_reference_fqt_u128_words(orc):
    # the reference's integer mode: u128 words up to m = 128 (polymul.cpp u128 MAC)
    rng = np.random.default_rng(128)
    for p, d, q, nq, m in [(5, 2, 10000, 1, 128), (3, 3, 1 << 16, 1000, 128), (251, 1, 1 << 40, 1000, 128),
                           (7, 2, 10 ** 7, 5000, 128), (3, 1, 1 << 30, 7, 96), (2, 7, 1 << 8, 3, 128)]:
        for n in (1, 10, 57):
            a = rng.integers(0, p, n + 1).astype(np.uint64)
            b = rng.integers(0, p, n + 3).astype(np.uint64)
            got, cost = orc.fqt_mul(p, d, q, nq, a, b, m)
            want = np.zeros(2 * n + 3, np.uint64)
            rc = np.zeros(4, np.uint64)
            assert orc.ref().ref_fqt_mul_m(p, d, q, nq, m, a, a.size, b, b.size, want, rc) == 0
            assert (got == want).all() and cost.tolist() == rc.tolist()


def test_oracle_vs_reference_chunked_fqt(orc):
    # acceptance.cpp:154-170 style: multi-chunk FQT products, counters too
    rng = np.random.default_rng(408)
    for p, d, q, nq in [(3, 4, 32, 1), (2, 6, 8, 1), (3, 1, 1 << 13, 409), (2, 3, 1 << 7, 18)]:
        for n in (1, 10, 57):
            a = rng.integers(0, p, n + 1).astype(np.uint64)
            b = rng.integers(0, p, n + 1).astype(np.uint64)
            got, cost = orc.fqt_mul(p, d, q, nq, a, b)
            want = np.zeros(2 * n + 1, np.uint64)
            rc = np.zeros(4, np.uint64)
            assert orc.ref().ref_fqt_mul(p, d, q, nq, a, a.size, b, b.size, want, rc) == 0
            assert (got == want).all()
            assert cost.tolist() == rc.tolist()
