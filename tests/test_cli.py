"""The reference CLI surface (proj/tools/qpack.cpp, README "CSV schema"):
tools/qpack_b200.cpp prints the reference's stdout lines and appends CSV rows
in the reference schema with the same seeded inputs, closed-form counters and
FNV-1a checksums.  The expected rows are computed here with the oracle (and
the reference itself when oracle/_ref is built)."""
import csv
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_0710_0510_b200", "bin", "qpack_b200")
HEADER = "algo,p,q,k,d,N,n_q,n_d,mul_add,divisions,table_accesses,wall_time_ns,checksum"


def run(*args, env=None):
    if not os.path.exists(TOOL):
        pytest.skip("qpack_b200 tool not built")
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, env=e, timeout=300)


def rows(path):
    with open(path) as f:
        assert f.readline().strip() == HEADER
    with open(path) as f:
        return list(csv.DictReader(f))


def mulpoly_inputs(orc, p, n, seed):
    d = orc.draws(seed, 2 * (n + 1), p)
    return d[: n + 1].astype(np.uint64), d[n + 1:].astype(np.uint64)


def fold(orc, v):
    v = np.ascontiguousarray(v, np.uint64)
    return int(orc.oracle().qo_fold_checksum_u64(v, v.size))


def test_usage_and_error_exit_codes():
    assert run().returncode == 1
    assert run("bogus").returncode == 1
    r = run("mulpoly", "--p", "3", "--n", "4", "--algo", "delayed")
    assert r.returncode == 2 and "error:" in r.stderr
    assert run("mulpoly", "--p", "4", "--n", "4").returncode == 2  # not prime (best_qadic)


def test_dump_field_is_the_fixture(qpk):
    r = run("gfq", "--p", "3", "--k", "2", "--dump-field")
    assert r.returncode == 0
    q = qpk.GfqField(3, 2, 1 << 17).describe()  # gfq_default_q(3, 2) = 2^17
    assert r.stdout == q
    assert "modulus 1 0 1" in r.stdout and "generator 1 1" in r.stdout  # test_gfq.cpp:23-30


def test_oracle_rows_match_reference_checksum(orc, tmp_path):
    p, n, seed = 3, 300, 7
    path = tmp_path / "rows.csv"
    r = run("mulpoly", "--p", p, "--n", n, "--algo", "oracle", "--seed", seed, "--repeat", 2, "--csv", path)
    assert r.returncode == 0, r.stderr
    a, b = mulpoly_inputs(orc, p, n, seed)
    want = np.convolve(a.astype(np.int64), b.astype(np.int64)) % p
    rs = rows(path)
    assert len(rs) == 2 and rs[0]["algo"] == "oracle"
    assert int(rs[0]["checksum"], 16) == fold(orc, want)
    assert rs[0]["N"] == str(n) and rs[0]["mul_add"] == "0"
    # rep 1 draws the next inputs from the same stream
    d = orc.draws(seed, 4 * (n + 1), p)
    a2, b2 = d[2 * (n + 1): 3 * (n + 1)], d[3 * (n + 1):]
    assert int(rs[1]["checksum"], 16) == fold(orc, np.convolve(a2.astype(np.int64), b2.astype(np.int64)) % p)


def test_table_cache_writes_the_reference_layout(orc, tmp_path):
    import ctypes as C
    from test_capi import qpkt_bytes
    cache = tmp_path / "cache"
    # best_qadic(3, 53, 1) packs k = 5 at q = 32; the FQT plan (d = 8) uses the
    # window-4 base-p table (qpack.cpp:80-98 names the file)
    r = run("mulpoly", "--p", "3", "--n", "20", env={"QPACK_TABLE_CACHE": str(cache)})
    f = cache / "redq_p3_q32_w4_basep.tbl"
    assert f.exists(), r.stderr
    ent = C.POINTER(C.c_uint64)()
    n, radix = C.c_uint64(), C.c_uint64()
    orc.oracle().qo_correction_table(3, 32, 4, 0, 1 << 26, C.byref(ent), C.byref(n), C.byref(radix))
    assert f.read_bytes() == qpkt_bytes(3, 32, 4, 0, [ent[i] for i in range(n.value)])
    # a corrupted cache is loaded as is (the reference trusts it); a
    # truncated one is rejected with the reference's runtime_error
    f.write_bytes(f.read_bytes()[:-5])
    r = run("mulpoly", "--p", "3", "--n", "20", env={"QPACK_TABLE_CACHE": str(cache)})
    assert r.returncode == 2 and "error:" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("p,n,d", [(3, 1000, None), (3, 4000, 3), (5, 777, 1), (2, 2500, None), (7, 64, 2)])
def test_mulpoly_fqt_rows_match_reference(orc, tmp_path, p, n, d):
    path = tmp_path / "rows.csv"
    args = ["mulpoly", "--p", p, "--n", n, "--seed", 11, "--csv", path]
    if d is not None:
        args += ["--d", d]
    r = run(*args)
    assert r.returncode == 0, r.stderr
    assert "verified=ok" in r.stdout
    row = rows(path)[0]
    assert row["algo"] == "fqt_b200"
    pp, dd, q, nq = int(row["p"]), int(row["d"]), int(row["q"]), int(row["n_q"])
    a, b = mulpoly_inputs(orc, p, n, 11)
    want, cost = orc.fqt_mul(pp, dd, q, nq, a, b)
    assert int(row["checksum"], 16) == fold(orc, want)
    assert [int(row[k]) for k in ("mul_add", "divisions", "table_accesses")] == [int(cost[0]), int(cost[1]),
                                                                               int(cost[2])]
    if orc.ref() is not None and n <= 1000:
        w2 = np.zeros(2 * n + 1, np.uint64)
        rc = np.zeros(4, np.uint64)
        assert orc.ref().ref_fqt_mul(pp, dd, q, nq, a, a.size, b, b.size, w2, rc) == 0
        assert int(row["checksum"], 16) == int(orc.ref().ref_fold_checksum(w2, w2.size))
        assert int(row["mul_add"]) == int(rc[0]) and int(row["divisions"]) == int(rc[1])


@pytest.mark.gpu
def test_paper_examples_and_fault_injection():
    r = run("paper-examples")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all examples reproduced" in r.stdout and "device residues == host: yes" in r.stdout
    r = run("paper-examples", "--inject-fault")
    assert r.returncode == 4 and "MISMATCHES FOUND" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("p,k,op,n", [(3, 2, "dot", 1000), (3, 3, "dot", 100000), (7, 3, "dot", 513),
                                      (3, 2, "matmul", 24), (5, 2, "matmul", 17)])
def test_gfq_rows(orc, tmp_path, p, k, op, n):
    path = tmp_path / "rows.csv"
    r = run("gfq", "--p", p, "--k", k, "--op", op, "--len" if op == "dot" else "--size", n, "--csv", path)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "agreement=ok" in r.stdout
    packed, naive = rows(path)
    assert packed["algo"] == "fgdp_b200" and naive["algo"] == "naive_dot"
    assert packed["checksum"] == naive["checksum"]
    nq = int(packed["n_q"])
    if op == "dot":
        assert int(packed["divisions"]) == -(-n // nq)
        assert int(packed["mul_add"]) == n
    else:
        assert int(packed["divisions"]) == n * n * -(-n // nq)
