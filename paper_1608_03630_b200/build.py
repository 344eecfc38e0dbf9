"""Build libdiffreg.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
CHECK = os.environ.get("DR_CHECK", "0") == "1"  # bounds-checked debug variant (device asserts)
LIB = os.path.join(PKG, "libdiffreg_check.so" if CHECK else "libdiffreg.so")
SOURCES = [os.path.join(CSRC, "diffreg.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + [
    os.path.join(ROOT, "include", "diffreg.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# --split-compile (parallel device compilation, 2x faster builds) measured slower code: the fp32 x2 pass
# 82 -> 93 us, the TMA middle pass 122 -> 149 us at 256^3; opt-in for quick experiments only
SPLIT = ["--split-compile=0"] if os.environ.get("DR_SPLIT") == "1" else []
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr", *SPLIT,
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-ldl"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-DDR_CHECK"] if CHECK else []), "-o", tmp, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build_check.log" if CHECK else "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, LIB)
    if verbose:
        print(r.stderr[-4000:])
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """A/B experiment build: the same sources with extra -D flags into libdiffreg_<name>.so (selected at
    run time with DR_LIB_VARIANT=<name>); never the product library."""
    out = os.path.join(PKG, f"libdiffreg_{name}.so")
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(PKG, f"build_{name}.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for variant {name}")
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        build(force="--force" in sys.argv, verbose=True)
        print(LIB)
