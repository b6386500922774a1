"""Build libspecformer.so in-tree for sm_100a (nvcc; no torch JIT, no cache outside the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspecformer.so")
SOURCES = ["gemm.cu", "kernels.cu", "attn_fd.cu", "specformer.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """The NCCL that ships with the torch wheel (nvidia/nccl: include/nccl.h, lib/libnccl.so.2)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    except Exception:
        roots = []
    for r in roots:
        if os.path.exists(os.path.join(r, "include", "nccl.h")) and os.path.exists(os.path.join(r, "lib", "libnccl.so.2")):
            return r
    return None


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "specformer.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    odir = os.path.join(HERE, "_obj")
    os.makedirs(odir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(odir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if NCCL and src == "specformer.cu":
            cmd[1:1] = ["-DSF_WITH_NCCL", "-I" + os.path.join(NCCL, "include")]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
        if verbose and out:
            print(out)
    tmp = LIB + ".tmp"
    # shared CUDA runtime: the library binds to the process's libcudart.so.12 (torch's, when torch is
    # loaded first) instead of carrying a static copy of the whole runtime
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared", "-o", tmp, *objs,
           "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    if NCCL:
        lib = os.path.join(NCCL, "lib")
        cmd += ["-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
