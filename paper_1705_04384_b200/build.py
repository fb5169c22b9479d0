"""Build libfdiga.so in-tree with nvcc for sm_100a (B200).  No JIT cache: the .so lives next to
the package so it travels with the repository snapshot to the GPU box."""
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# FDIGA_CSRC / FDIGA_LIBDIR: experiment builds of a copied source tree into another directory
CSRC = os.environ.get("FDIGA_CSRC") or os.path.join(PKG, "csrc")
LIBDIR = os.environ.get("FDIGA_LIBDIR") or os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libfdiga.so")
SOURCES = ["ctx.cu", "comm.cu", "fd_gemm.cu", "fd.cu", "stencil.cu", "krylov.cu", "bicgstab.cu", "matfree.cu", "wq.cu", "oz.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "fdiga.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def nccl_include():
    """Directory of nccl.h (types only: libnccl.so.2 is dlopen'ed at run time, the copy torch loads)."""
    import glob
    for cand in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include")) + \
            ["/usr/include"]:
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    raise RuntimeError("nccl.h not found")


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    nvcc = nvcc_path()
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                     "-I", nccl_include()]
    build_dir = os.path.join(LIBDIR, "build") if os.environ.get("FDIGA_LIBDIR") else os.path.join(PKG, "build")
    os.makedirs(build_dir, exist_ok=True)
    cmds = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        cmds.append([nvcc] + common + ["-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(run, cmds))
    tmp = LIB + ".tmp"
    cmd = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcusolver", "-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
