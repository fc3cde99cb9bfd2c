"""Build an in-tree variant of libstkde.so with extra -D flags (development A/B aid).
    python scripts/build_variant.py NAME -DFOO=1 ...   -> paper_1705_09366_b200/libstkde_NAME.so"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1705_09366_b200")
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(PKG, "libstkde_%s.so" % name)
objdir = os.path.join(PKG, "build", name)
os.makedirs(objdir, exist_ok=True)
arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
objs = []
for src in sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu"))):
    o = os.path.join(objdir, os.path.basename(src) + ".o")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc"] + arch + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")] + defs + ["-c", src, "-o", o])
    objs.append(o)
subprocess.check_call(["/usr/local/cuda/bin/nvcc"] + arch + ["-shared", "-o", out] + objs + ["-cudart", "static"])
print(out)
