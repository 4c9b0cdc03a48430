"""Build liblemix_<tag>.so: the main build's objects with lemix_fast.cu
recompiled under extra -D flags (A/B experiments on the fast kernel).
Usage: python tools/build_fast_variant.py TAG [-DNAME=VAL ...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_21276_b200")
CSRC = os.path.join(PKG, "csrc")
tag, defs = sys.argv[1], sys.argv[2:]
bdir = os.path.join(PKG, "build", "liblemix")
vdir = os.path.join(PKG, "build", "var_" + tag)
os.makedirs(vdir, exist_ok=True)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
obj = os.path.join(vdir, "lemix_fast.o")
r = subprocess.run(["/usr/local/cuda/bin/nvcc", *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I",
                    os.path.join(ROOT, "include"), "-lineinfo", "--fmad=false", "-Xptxas", "-v", *defs, "-c",
                    os.path.join(CSRC, "lemix_fast.cu"), "-o", obj], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
lines = r.stdout.splitlines() + r.stderr.splitlines()
for k, ln in enumerate(lines):   # the bench instantiation's resources
    if "ILi2ELi4E" in ln and "Function properties" in ln:
        print(tag, "LEAN" if "Lb1E" in ln else "full", lines[k + 1].strip(), "|", lines[k + 2].strip())
objs = [o for o in glob.glob(os.path.join(bdir, "*.o")) if not o.endswith("lemix_fast.o")] + [obj]
subprocess.run(["/usr/local/cuda/bin/nvcc", *ARCH, "-shared", *objs, "-o", os.path.join(PKG, f"liblemix_{tag}.so"),
                "-lcudart", "-ldl"], check=True)
