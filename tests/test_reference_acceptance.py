"""The reference's own acceptance binary (acceptance.cpp:413-452, compiled
unchanged by tests/cpp/build_acceptance.py) run against include/qpack +
libqpack_b200.so.  Criteria 1-3, 7, 8, 10 exercise the host drop-in;
4 (fqt_mul) and 9 (GfqField, fgdp_dot, gfq_matmul) run on the device.
Criteria 5 and 6 need the out-of-scope delayed_mul / cost_model."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "qpack_acceptance_dropin")


def run_criterion(c):
    if not os.path.exists(BIN):
        pytest.skip("acceptance binary not built (needs /root/reference at build time: tests/cpp/build_acceptance.py)")
    r = subprocess.run([BIN, "--criterion", str(c)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and f"PASS criterion {c}" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("c", [1, 2, 3, 7, 8, 10])
def test_reference_acceptance_host_criteria(qpk, c):
    run_criterion(c)


@pytest.mark.gpu
@pytest.mark.parametrize("c", [4, 9])
def test_reference_acceptance_device_criteria(qpk, torch_cuda, c):
    run_criterion(c)
