"""Build libqpack_b200.so in-tree (sm_100a) with ninja.

    python -m paper_0710_0510_b200.build          # incremental
    python -m paper_0710_0510_b200.build --clean

The heavy template translation units (stream_inst.cu, gfq_matmul_inst.cu) are
compiled once per -DQPK_INST value so nvcc/ptxas run in parallel.  Output:
paper_0710_0510_b200/lib/libqpack_b200.so (git-ignored; travels to the GPU box
with the repo snapshot).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "lib", "libqpack_b200.so")
TOOL = os.path.join(PKG, "bin", "qpack_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = "-gencode arch=compute_100a,code=sm_100a"

NVCC_FLAGS = f"{ARCH} -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I{CSRC} -I{ROOT}/include --expt-relaxed-constexpr"
CXX_FLAGS = f"-std=c++20 -O2 -fPIC -Wall -Wextra -I{CSRC} -I{ROOT}/include -I{CUDA}/include"

CU_UNITS = [("stream_main.cu", None), ("gfq_matmul_main.cu", None), ("gfq_gemv.cu", None), ("fqt_conv.cu", None),
            ("probe.cu", None), ("gfq_count.cu", None), ("gfq_wide.cu", None)]
CU_UNITS += [("stream_inst.cu", i) for i in range(1, 9)]
CU_UNITS += [("fqt_conv_inst.cu", nd) for nd in range(1, 16, 2)]
CU_UNITS += [("gfq_matmul_inst.cu", (k, 0)) for k in range(1, 5)] + [("gfq_matmul_inst.cu", (k, 1)) for k in (2, 3)]
CXX_UNITS = ["capi.cpp"] + [f"host/{f}" for f in
                            ("common.cpp", "params.cpp", "fpdiv.cpp", "dqt.cpp", "redq.cpp", "polymul.cpp",
                             "gfq.cpp", "gpu_api.cpp")]


def _ninja_text() -> str:
    lines = [
        f"nvcc = {NVCC}",
        f"nvflags = {NVCC_FLAGS}",
        f"cxxflags = {CXX_FLAGS}",
        "rule nvcc",
        "  command = $nvcc $nvflags $defs -MD -MF $out.d -c $in -o $out",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = NVCC $out",
        "rule cxx",
        "  command = g++ $cxxflags -MMD -MF $out.d -c $in -o $out",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = CXX $out",
        "rule link",
        f"  command = $nvcc {ARCH} -shared -Xcompiler -fPIC -cudart static $in -o $out -lpthread -ldl -lrt",
        "  description = LINK $out",
    ]
    objs = []
    for src, inst in CU_UNITS:
        if isinstance(inst, tuple):
            tag, defs = f"_{inst[0]}_v{inst[1]}", f"-DQPK_INST={inst[0]} -DQPK_VARIANT={inst[1]}"
        else:
            tag, defs = (f"_{inst}", f"-DQPK_INST={inst}") if inst else ("", "")
        obj = os.path.join(BUILD, os.path.splitext(src)[0] + tag + ".o")
        lines.append(f"build {obj}: nvcc {os.path.join(CSRC, src)}")
        if defs:
            lines.append(f"  defs = {defs}")
        objs.append(obj)
    for src in CXX_UNITS:
        obj = os.path.join(BUILD, src.replace("/", "_").replace(".cpp", ".o"))
        lines.append(f"build {obj}: cxx {os.path.join(CSRC, src)}")
        objs.append(obj)
    lines.append(f"build {LIB}: link {' '.join(objs)}")
    # the reference CLI surface (tools/qpack_b200.cpp) over the library
    lines += [
        "rule tool",
        f"  command = g++ $cxxflags -MMD -MF $out.d $in -o $out -L{os.path.dirname(LIB)} -lqpack_b200 "
        "-Wl,-rpath,'$$ORIGIN/../lib'",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = TOOL $out",
        f"build {TOOL}: tool {os.path.join(ROOT, 'tools', 'qpack_b200.cpp')} | {LIB}",
    ]
    lines.append(f"default {LIB} {TOOL}")
    return "\n".join(lines) + "\n"


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    os.makedirs(os.path.dirname(TOOL), exist_ok=True)
    nf = os.path.join(BUILD, "build.ninja")
    text = _ninja_text()
    if not os.path.exists(nf) or open(nf).read() != text:
        with open(nf, "w") as f:
            f.write(text)
    cmd = ["ninja", "-f", nf, "-j", str(max(os.cpu_count() or 1, 1))]
    if verbose:
        cmd.append("-v")
    subprocess.run(cmd, check=True, cwd=BUILD)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args(argv)
    if args.clean:
        shutil.rmtree(BUILD, ignore_errors=True)
        if os.path.exists(LIB):
            os.remove(LIB)
    print(build(args.verbose))


if __name__ == "__main__":
    sys.exit(main())
