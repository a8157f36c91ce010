"""In-tree build of libtnrd.so (sm_100a) with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libtnrd.so")
BUILD = os.path.join(ROOT, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    import nvidia.nccl  # torch's NCCL (2.28.x); headers ship with the wheel
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include")


def nccl_library() -> str:
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "lib", "libnccl.so.2")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    srcs = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in srcs)


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Compile libtnrd.so (`defines`/`out`: experiment variants, never the product)."""
    if out == OUT and not defines and not force and not _stale():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_include()]
    common = ["nvcc", "-std=c++17", "-O3", "-Xcompiler", "-fPIC,-fvisibility=hidden"] + inc
    objs = []
    ptxas_log = []
    for src, extra in [("tnrd_kernels.cu", ARCH + ["-lineinfo", "-fmad=false", "-Xptxas", "-v"] + ["-D" + d for d in defines]),
                       ("tnrd_tc.cu", ARCH + ["-lineinfo", "-fmad=false", "-Xptxas", "-v"] + ["-D" + d for d in defines]),
                       ("tnrd_grad.cu", ARCH + ["-lineinfo", "-Xptxas", "-v"] + ["-D" + d for d in defines]),
                       ("tnrd_data.cu", ARCH + ["-lineinfo"]),
                       ("tnrd_api.cpp", [])]:
        obj = os.path.join(BUILD, src + ("." + "_".join(defines) if defines else "") + ".o")
        cmd = common + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        ptxas_log.append(r.stderr)
        objs.append(obj)
    cmd = ["nvcc", "-shared"] + ARCH + ["-o", out] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    with open(os.path.join(BUILD, "ptxas.log"), "w") as fh:
        fh.write("".join(ptxas_log))
    if verbose:
        print("".join(ptxas_log))
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
