"""Build the reference's own acceptance binary against the drop-in.

/root/reference/proj/tests/acceptance.cpp is compiled UNCHANGED, with
include/qpack (the drop-in headers) first on the include path, so every
qpack/*.hpp it includes is ours except qpack/oracle.hpp (the reference's
brute-force namespace, out of scope, test infrastructure).  It links
against libqpack_b200.so plus the reference's src/oracle.cpp as a test-only
object; tests/cpp/acceptance_oos.hpp supplies throwing stubs for the
out-of-scope delayed_mul / cost_model (criteria 5 and 6 are not run).

Output: tests/cpp/_bin/qpack_acceptance_dropin (git-ignored, travels to the
GPU box with the repo snapshot like oracle/_ref).  Only where
/root/reference exists (this build container); nothing is copied out of it.
    python tests/cpp/build_acceptance.py
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
OUT = os.path.join(HERE, "_bin", "qpack_acceptance_dropin")


def build(lib_dir: str | None = None) -> str | None:
    if not os.path.isfile(os.path.join(REF, "tests", "acceptance.cpp")):
        return None
    lib_dir = lib_dir or os.path.join(ROOT, "paper_0710_0510_b200", "lib")
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(REF, "include")]
    cmd = ["g++", "-std=c++20", "-O2", *inc, "-include", os.path.join(HERE, "acceptance_oos.hpp"),
           os.path.join(REF, "tests", "acceptance.cpp"), os.path.join(REF, "src", "oracle.cpp"),
           "-L", lib_dir, "-lqpack_b200", "-Wl,-rpath,$ORIGIN/../../../paper_0710_0510_b200/lib", "-o", OUT]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build() or "reference sources absent: not built")
    sys.exit(0)
