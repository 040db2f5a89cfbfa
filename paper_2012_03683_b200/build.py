"""In-tree build of the native engine: paper_2012_03683_b200/libkreg_b200.so.

nvcc cross-compiles for sm_100a only (no multi-arch, no JIT fallback):
    python -m paper_2012_03683_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libkreg_b200.so")
OBJ_DIR = os.path.join(HERE, "_build")

SOURCES = ["kernels.cu", "dense.cu", "ingest.cu", "ply.cu", "engine_host.cu", "solver.cpp", "capi.cpp", "nccl_coll.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB, obj_dir: str = OBJ_DIR) -> str:
    """Compile and link; `defines` (e.g. ["KREG_UNIT_STEPS=4"]) select kernel
    variants for A/B measurements (written to `lib` / `obj_dir`)."""
    os.makedirs(obj_dir, exist_ok=True)
    extra = ["-D" + d for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "kreg_b200.h"))
    nvcc = _nvcc()
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(obj_dir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-x", "cu" if src.endswith(".cu") else "c++", "-c", path, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [nvcc, *NVCC_FLAGS, *extra, "-x", "c++", "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}")
            with open(obj + ".log", "w") as f:
                f.write(r.stdout + r.stderr)
    if force or _stale(lib, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib


def build_variant(name: str, defines) -> str:
    """Experimental kernel variant: paper_2012_03683_b200/_variants/<name>.so."""
    vdir = os.path.join(HERE, "_variants")
    return build(force=False, defines=defines, lib=os.path.join(vdir, name + ".so"),
                 obj_dir=os.path.join(vdir, name + "_obj"))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
