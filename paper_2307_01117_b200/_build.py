"""Build libheat1d.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

    python -m paper_2307_01117_b200._build           # incremental
    python -m paper_2307_01117_b200._build --force

The .so lands next to this file so it travels to the GPU box with the repo
snapshot.  NCCL headers and libnccl.so.2 come from the nvidia-nccl wheel that
torch itself loads (2.28.x), so one libnccl is in the process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libheat1d.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl wheel not found (needed for nccl.h / libnccl.so.2)")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(INCLUDE, "heat1d.h"), os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = "", defines=()) -> str:
    """Compile libheat1d.so (or, for measurement builds, `out` with extra -D`defines`)."""
    target = out or LIB
    if not out and not force and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC,-fvisibility=hidden", "-DHEAT1D_BUILD", "-I", INCLUDE, "-I", CSRC, "-I", inc,
              *["-D" + d for d in defines]]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".%d.%d.o" % (os.getpid(), abs(hash(target)) % 10000))
        cmd = common + ["-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return obj, " ".join(cmd) + "\n" + res.stdout + res.stderr, res.returncode

    # one nvcc per translation unit, in parallel (the pass-kernel instantiations dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(sources())) as ex:
        results = list(ex.map(compile_one, sources()))
    log = "".join(r[1] for r in results)
    tmp = target + ".tmp%d" % os.getpid()
    ok = all(r[2] == 0 for r in results)
    if ok:
        cmd = [nvcc, *ARCH, "-shared", *[r[0] for r in results], "-o", tmp,
               "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log += " ".join(cmd) + "\n" + res.stdout + res.stderr
        ok = res.returncode == 0
    for r in results:
        if os.path.exists(r[0]):
            os.remove(r[0])
    os.makedirs(objdir, exist_ok=True)
    with open(os.path.join(objdir, "build.log" if not out else os.path.basename(out) + ".log"), "w") as f:
        f.write(log)
    if not ok:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed (see paper_2307_01117_b200/build/build.log)")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
