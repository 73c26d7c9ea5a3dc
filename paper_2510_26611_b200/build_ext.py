"""Build librsdock.so in-tree with nvcc for sm_100a (no torch extension machinery: the
library is torch-free, its C ABI is include/rs_dock.h)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "librsdock.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) +
                  glob.glob(os.path.join(PKG, "csrc", "*.cpp")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(PKG, "csrc", "*.h")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
        [os.path.join(ROOT, "include", "rs_dock.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile every csrc/ source and link librsdock.so (or `out`, with extra -D defines)."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    objdir = os.path.join(ROOT, "build", "obj" + ("_" + os.path.basename(lib) if out else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
                   *[f"-D{d}" for d in defines],
                   "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-c", src, "-o", obj]
        else:
            cmd = [NVCC, "-O3", "-std=c++17", *[f"-D{d}" for d in defines], "-Xcompiler",
                   "-fPIC,-O3,-fopenmp,-ffp-contract=off", "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out.decode())
    link = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fopenmp", "-lgomp",
            "-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    subprocess.check_call(link)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
