"""Build a variant of libapc_b200.so with extra nvcc defines (kernel A/B tests).

usage: python scripts/build_variant.py NAME -DAPC_S4_ROWS=4 [...]
writes _variants/libapc_NAME.so (git-ignored, travels with gpurun); select it
with APC_LIB_PATH=<that path>.  Only sources mentioning a defined macro are
recompiled (every .cu file when a macro appears in a header)."""
import shutil
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_05065_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = B.ROOT / "_variants"
obj_dir = out / f"obj_{name}"
obj_dir.mkdir(parents=True, exist_ok=True)
B.build()  # objects of the default build
objs = []
for src in sorted(B.CSRC.glob("*.cu")) + sorted(B.CSRC.glob("*.cpp")):
    obj = B.OBJ_DIR / (src.name + ".o")
    macros = [d[2:].split("=")[0] for d in defs if d.startswith("-D")]
    in_header = any(mc in h.read_text() for mc in macros for h in list(B.CSRC.glob("*.cuh")) + list(B.CSRC.glob("*.hpp")))
    if src.suffix == ".cu" and (in_header or any(mc in src.read_text() for mc in macros)):
        obj = obj_dir / (src.name + ".o")
        exact = ["-fmad=false"] if src.name in B.EXACT_CU else []
        B._run([B.NVCC, *B.CU_FLAGS, *exact, *defs, f"-I{B.INC}", f"-I{B.CSRC}", "-c", str(src), "-o", str(obj)])
    objs.append(str(obj))
lib = out / f"libapc_{name}.so"
B._run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *objs, *B._nccl_link_args(), "-L/usr/local/cuda/lib64",
        "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-lpthread"])
print(lib)
