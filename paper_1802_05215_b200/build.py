"""Build libsliceeig_cuda.so in-tree (sm_100a only).

    python -m paper_1802_05215_b200.build [--force]

Every translation unit in csrc/ is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (host code through the host compiler),
then linked into ``paper_1802_05215_b200/libsliceeig_cuda.so`` against cuSOLVER / cudart.
Object files go to ``paper_1802_05215_b200/_build`` (git-ignored); the .so travels with the repo
snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsliceeig_cuda.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "sliceeig_cuda.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, src + ".o")
    path = os.path.join(CSRC, src)
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(path), _headers_mtime())):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", path, "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-warn-spills"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if (force or not os.path.exists(LIB)
            or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, f"-L{os.path.join(CUDA, 'lib64')}",
               "-lcusolver", "-lcudart",
               "-Xlinker", f"-rpath={os.path.join(CUDA, 'lib64')}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cli(force)
    if verbose:
        print(f"built {LIB}")
    return LIB


CLI_SRC = os.path.join(ROOT, "tools", "sliceeig_b200_main.cpp")
CLI = os.path.join(ROOT, "tools", "sliceeig_b200")


def build_cli(force: bool = False) -> str:
    """tools/sliceeig_b200: the C++ command-line caller (host code over the facade + the .so)."""
    deps = [CLI_SRC, os.path.join(ROOT, "tools", "json_out.hpp"), LIB,
            *[os.path.join(ROOT, "include", "sliceeig", f)
              for f in os.listdir(os.path.join(ROOT, "include", "sliceeig"))]]
    if not force and os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(d) for d in deps):
        return CLI
    cmd = ["g++", "-O2", "-std=c++17", "-pthread", f"-I{os.path.join(ROOT, 'include')}",
           f"-I{os.path.join(CUDA, 'include')}", CLI_SRC, "-o", CLI, f"-L{PKG}", "-lsliceeig_cuda",
           "-Wl,-rpath,$ORIGIN/../paper_1802_05215_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv)
