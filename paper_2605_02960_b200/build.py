"""Build libasyncep.so in-tree with nvcc for sm_100a (explicit -gencode, -lineinfo).

Objects compile in parallel; the shared library is linked with the static CUDA runtime
(cudaStream_t / cudaEvent_t are driver objects, shared with torch's runtime) and -ldl
(NCCL is resolved at run time inside the caller's process)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libasyncep.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["asyncep.cu", "router.cu", "permute.cu", "gemm_simt.cu", "gemm_tc.cu", "combine.cu", "pack.cu",
           "attn.cu", "admission.cpp"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def _inputs():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "asyncep.h"))
    return deps


def _compile(src: str, build_dir: str = BUILD, defines=()) -> str:
    obj = os.path.join(build_dir, os.path.splitext(src)[0] + ".o")
    dep_mtime = max(os.path.getmtime(d) for d in _inputs())
    if os.path.exists(obj) and os.path.getmtime(obj) >= dep_mtime:
        return obj
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c",
           os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Build the library.  defines / out: a variant (extra -D macros) for same-box A/B runs,
    linked to another path (loaded with ASYNCEP_LIB=path); the default build is LIB."""
    build_dir = BUILD if not defines else os.path.join(BUILD, "v_" + "_".join(defines).replace("=", ""))
    os.makedirs(build_dir, exist_ok=True)
    if force:
        for f in os.listdir(build_dir):
            if f.endswith(".o"):
                os.remove(os.path.join(build_dir, f))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda f: _compile(f, build_dir, defines), SOURCES))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
        tmp = out + f".tmp{os.getpid()}"
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               *objs, "-o", tmp, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, out)
        if verbose:
            print("built", out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="variant macro NAME=VALUE")
    ap.add_argument("--out", default=LIB)
    a = ap.parse_args()
    build(force=a.force, verbose=True, defines=tuple(a.defines), out=a.out)
