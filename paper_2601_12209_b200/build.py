"""Build libdfft.so (sm_100a) and inputs/libdfft_inputs.so with nvcc — in tree, no JIT cache."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-std=c++17", "--expt-relaxed-constexpr", "-lineinfo", "-Xcompiler", "-fPIC",
                 "-I" + os.path.join(ROOT, "include")]


def nccl_dir() -> str:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL wheel (nvidia/nccl) not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib_name: str = "libdfft.so") -> str:
    """defines / lib_name: dev A/B variants (e.g. -DDFFT_STRIDED_W0=128 -> libdfft_w16.so)."""
    global BUILD
    if defines:
        BUILD = os.path.join(ROOT, "build", lib_name.replace(".so", ""))
    os.makedirs(BUILD, exist_ok=True)
    nccl = nccl_dir()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "dfft.h"))
    units = ["kernels_f32.cu", "kernels_f64.cu", "dfft.cu"]
    objs, jobs = [], []
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
        for u in units:
            src = os.path.join(CSRC, u)
            obj = os.path.join(BUILD, u.replace(".cu", ".o"))
            objs.append(obj)
            if force or _stale(obj, [src] + headers):
                cmd = [NVCC] + CFLAGS + list(defines) + ["-I" + os.path.join(nccl, "include"), "-Xptxas", "-v", "-c",
                                                         src, "-o", obj]
                jobs.append(ex.submit(_run, cmd))
        for j in jobs:
            out = j.result()
            if verbose:
                print(out)
    lib = os.path.join(PKG, lib_name)
    if force or _stale(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs +
             ["-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")])
    gen_src = os.path.join(ROOT, "inputs", "gen.cu")
    gen_lib = os.path.join(ROOT, "inputs", "libdfft_inputs.so")
    if force or _stale(gen_lib, [gen_src]):
        _run([NVCC] + CFLAGS + ["-shared", gen_src, "-o", gen_lib])
    return lib


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    names = [a for a in sys.argv[1:] if a.endswith(".so")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs,
                lib_name=names[0] if names else "libdfft.so"))
