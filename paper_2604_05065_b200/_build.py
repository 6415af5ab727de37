"""In-tree build of libapc_b200.so (sm_100a) -- no JIT cache, the .so travels
with the repo snapshot to the GPU box.

The CUDA translation units on the CUR index path (cur.cu: sketch, E^row,
E^col, LUPP, core factor and solves, rho probes; rng_dev.cu) are compiled with
``-fmad=false`` and all host code with ``-ffp-contract=off``: the indices must
round exactly like the reference's SSE2 build
(/root/reference/proj/CMakeLists.txt:3-11).  The LSQR, operator,
preconditioner and residual kernels do not decide indices and
keep FMA contraction.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INC = ROOT / "include"
OUT_DIR = PKG / "_lib"
OBJ_DIR = ROOT / "build" / "apc_obj"
LIB = OUT_DIR / "libapc_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v",
]
EXACT_CU = {"cur.cu", "rng_dev.cu"}  # the index path: no FMA contraction
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function"]


def _nccl_link_args() -> list[str]:
    for d in ("/usr/lib/x86_64-linux-gnu", "/usr/local/lib"):
        if Path(d, "libnccl.so.2").exists() or Path(d, "libnccl.so").exists():
            return [f"-L{d}", "-l:libnccl.so.2"]
    return ["-lnccl"]


def _run(cmd: list[str]) -> str:
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p.stderr


def _compile(src: Path) -> tuple[Path, str]:
    obj = OBJ_DIR / (src.name + ".o")
    deps = [src, Path(__file__)] + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list(INC.glob("*.h"))
    if obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return obj, ""
    inc = [f"-I{INC}", f"-I{CSRC}"]
    if src.suffix == ".cu":
        exact = ["-fmad=false"] if src.name in EXACT_CU else []
        cmd = [NVCC, *CU_FLAGS, *exact, *inc, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXX_FLAGS, *inc, "-I/usr/local/cuda/include", "-c", str(src), "-o", str(obj)]
    return obj, _run(cmd)


def build(verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        results = list(ex.map(_compile, srcs))
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    objs = [str(o) for o, _ in results]
    newest = max(Path(o).stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, *_nccl_link_args(), "-L/usr/local/cuda/lib64",
              "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-lpthread"])
        shutil.move(str(tmp), str(LIB))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
