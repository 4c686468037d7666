"""Development: relink libqpack_b200.so with one translation unit rebuilt
under extra -D flags (tile-geometry sweeps).  Load it with QPK_DEV_LIB.

    python scripts/build_variant.py NAME UNIT_OBJ SRC "-DQPK_INST=3 -DQPK_GFE_R=8"
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import importlib  # noqa: E402

B = importlib.import_module("paper_0710_0510_b200.build")

name, unit_obj, src, defs = sys.argv[1:5]

out_dir = os.path.join(B.ROOT, "scripts", "variants")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, name + ".o")
subprocess.run(f"{B.NVCC} {B.NVCC_FLAGS} {defs} -c {os.path.join(B.CSRC, src)} -o {obj}", shell=True, check=True)
objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(o) != unit_obj] + [obj]
lib = os.path.join(out_dir, f"lib_{name}.so")
subprocess.run(f"{B.NVCC} {B.ARCH} -shared -Xcompiler -fPIC -cudart static {' '.join(objs)} -o {lib} -lpthread -ldl -lrt",
               shell=True, check=True)
print(lib)
