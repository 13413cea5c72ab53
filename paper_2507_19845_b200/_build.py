"""Build the sm_100a shared library in-tree (nvcc, no JIT cache): libmegascan.so next to this file."""
from __future__ import annotations

import glob
import importlib.util
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmegascan.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]
FLAGS += os.environ.get("MS_NVCC_EXTRA", "").split()  # experiments only (e.g. -DMS_FT_NT=256)


def nccl_paths() -> tuple[str, str]:
    """(include dir, lib dir) of the NCCL torch ships (same libnccl.so.2 the process loads)."""
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        root = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(root, "include"), os.path.join(root, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(HERE, "..", "include", "megascan", "scan.h")]


def headers():
    return glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(HERE, "..", "include", "megascan", "scan.h")]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def obj_stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *headers()])


def _flags_changed(objdir: str) -> bool:
    """True if the compile flags differ from the ones the objects were built with (then rebuild all)."""
    stamp = os.path.join(objdir, "flags.txt")
    cur = " ".join(ARCH + FLAGS)
    old = open(stamp).read() if os.path.exists(stamp) else None
    if old != cur:
        os.makedirs(objdir, exist_ok=True)
        with open(stamp, "w") as f:
            f.write(cur)
        return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    objdir = os.path.join(HERE, "build")
    force = _flags_changed(objdir) or force
    if not force and not stale():
        return SO
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    inc, lib = nccl_paths()
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not obj_stale(src, obj):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-I", inc, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
    for p, src in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out}")
        if verbose and out:
            sys.stderr.write(out)
    tmp = SO + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", f"-L{lib}", "-l:libnccl.so.2",
                           f"-Xlinker=-rpath={lib}"])
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
