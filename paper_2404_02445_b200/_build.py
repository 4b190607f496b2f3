"""Build libprnet.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box).  Each .cu compiles to its own
object under build/obj (in parallel, reused while newer than its inputs), then
one nvcc -shared link."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libprnet.so")
OBJ = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "prnet.h")]


def _inputs():
    return sources() + _headers()


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def _compile(src: str, extra: list[str], tag: str, verbose: bool) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + tag + ".o")
    newest = max(os.path.getmtime(p) for p in [src, *_headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) > newest and not extra:
        return obj
    tmp = obj + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-Xptxas=-v"] if verbose else []), *extra, "-I",
           os.path.join(ROOT, "include"), "-c", src, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          extra: dict[str, list[str]] | None = None) -> str:
    """extra: {source basename: [nvcc flags]} (A/B builds into `out`)."""
    lib = out or LIB
    if not force and not extra and out is None and not needs_build():
        return LIB
    extra = extra or {}
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(
            s, extra.get(os.path.basename(s), []),
            ".x" + str(abs(hash(tuple(extra.get(os.path.basename(s), []))))) if extra.get(
                os.path.basename(s)) else "", verbose), sources()))
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    args = [a for a in sys.argv[1:] if a != "-v"]
    if args:   # python _build.py OUT.so file.cu:-DFLAG ...  (A/B variant builds)
        ex: dict[str, list[str]] = {}
        for a in args[1:]:
            f, flag = a.split(":", 1)
            ex.setdefault(f, []).append(flag)
        print(build(force=True, verbose="-v" in sys.argv, out=os.path.join(PKG, args[0]), extra=ex))
    else:
        print(build(force=True, verbose="-v" in sys.argv))
