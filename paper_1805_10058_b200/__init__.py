"""B200-native IgA curl-div solver (arXiv 1805.10058 hot path).

The compute path is libigacd.so (hand-written sm_100a CUDA, C ABI in include/igacd.h);
``paper_1805_10058_b200.igacd`` is its thin ctypes binding.  ``build`` compiles it.
"""
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
LIB = os.path.join(_HERE, "lib", "libigacd.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def build(verbose=False, jobs=8):
    """Compile every csrc/*.cu for sm_100a (parallel, one object per file) and link libigacd.so."""
    srcs = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    objdir = os.path.join(_HERE, "lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for f in srcs:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f[:-3] + ".o")
        objs.append(obj)
        deps = [src, os.path.join(CSRC, "internal.cuh"), os.path.join(_HERE, "..", "include", "igacd.h")]
        if os.path.exists(obj) and all(os.path.getmtime(obj) >= os.path.getmtime(d) for d in deps):
            continue
        cmd = ["nvcc", *NVCC_FLAGS, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        if len([p for _, p in procs if p.poll() is None]) >= jobs:
            procs[0][1].wait()
    for cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: %s\n%s" % (" ".join(cmd), out))
        if verbose and out.strip():
            print(out)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    subprocess.check_call(cmd)
    return LIB
