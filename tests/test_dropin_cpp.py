"""Build tests/cpp/test_dropin.cpp against include/qpack + libqpack_b200.so
and run it: the reference's C++ API used exactly as a reference client would."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")


@pytest.fixture(scope="module")
def binary(qpk, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dropin") / "test_dropin")
    libdir = os.path.dirname(qpk.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
                    "-L", libdir, "-lqpack_b200", f"-Wl,-rpath,{libdir}"], check=True)
    return out


def test_dropin_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


@pytest.mark.gpu
def test_dropin_gpu_api(binary, torch_cuda):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
