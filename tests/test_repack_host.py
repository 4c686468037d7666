"""The canonical re-pack of the C5 matrix product (gfq_matmul.cuh
repack_canon3_bits) against the digit-wise definition, on the host."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")


@pytest.mark.skipif(not (os.path.exists(NVCC) or shutil.which("nvcc")), reason="nvcc not available")
def test_canonical_repack_matches_digitwise_mod_p(tmp_path):
    exe = str(tmp_path / "test_repack_host")
    nvcc = NVCC if os.path.exists(NVCC) else "nvcc"
    subprocess.run([nvcc, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", os.path.join(ROOT, "paper_0710_0510_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "test_repack_host.cu"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout
