"""Development: relink libqpack_b200.so with stream_inst (QPK_INST=3) and the
host gpu_api rebuilt under extra -D flags (QPK_DLOG_COPIES / QPK_GFE_* sweeps):
    python scripts/build_variant_dlog.py NAME "-DQPK_DLOG_COPIES=16"
Load it with QPK_DEV_LIB."""
import glob, os, subprocess, sys
sys.path.insert(0, "/root/repo")
import importlib
B = importlib.import_module("paper_0710_0510_b200.build")
name, defs = sys.argv[1], sys.argv[2]
out = os.path.join(B.ROOT, "scripts", "variants"); os.makedirs(out, exist_ok=True)
inst = int(os.environ.get("VARIANT_INST", "3"))  # the stream_inst slice rebuilt (3: C3, 4: C1, 7: C2)
o1 = os.path.join(out, name + f"_s{inst}.o"); o2 = os.path.join(out, name + "_api.o")
subprocess.run(f"{B.NVCC} {B.NVCC_FLAGS} -DQPK_INST={inst} {defs} -c {B.CSRC}/stream_inst.cu -o {o1}", shell=True, check=True)
subprocess.run(f"g++ {B.CXX_FLAGS} {defs} -c {B.CSRC}/host/gpu_api.cpp -o {o2}", shell=True, check=True)
objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(o) not in (f"stream_inst_{inst}.o", "host_gpu_api.o")] + [o1, o2]
lib = os.path.join(out, f"lib_{name}.so")
subprocess.run(f"{B.NVCC} {B.ARCH} -shared -Xcompiler -fPIC -cudart static {' '.join(objs)} -o {lib} -lpthread -ldl -lrt", shell=True, check=True)
print(lib)
