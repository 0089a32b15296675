"""Builds libgss_b200.so in-tree with nvcc for sm_100a (and the oracle checkers under oracle/_ref).

The product library is compiled with IEEE div/sqrt and -fmad=false: the reference's arithmetic
is reproduced op for op (no contraction) so cull ids, forward pixels and Adam updates are
bit-identical to the CPU reference.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libgss_b200.so"
SOURCES = ["cull.cu", "adam.cu", "raster.cu", "engine.cu", "densify.cu", "synth.cu", "ply.cu", "abi.cu"]
HEADERS = ["common.cuh", "gss_math.cuh"]

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2,-ffp-contract=off", "-I", str(ROOT / "include"), "-I", str(CSRC),
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + [CSRC / h for h in HEADERS] + [ROOT / "include" / "gss_b200.h", Path(__file__)]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def _compile(src: str, build: Path = BUILD, defines: tuple = ()) -> Path:
    s = CSRC / src
    o = build / (src + ".o")
    if _stale(o, s):
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(s), "-o", str(o)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if r.stderr.strip():
            sys.stderr.write(r.stderr)
    return o


def build_lib(verbose: bool = False, variant: str = "", defines: tuple = ()) -> Path:
    """Builds the product library; with `variant`, a copy compiled with extra -D `defines` into
    _build/var_<variant>/libgss_b200.so (load it with GSS_LIB=...; experiments only)."""
    build = BUILD / f"var_{variant}" if variant else BUILD
    lib = build / "libgss_b200.so" if variant else LIB
    build.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda src: _compile(src, build, defines), SOURCES))
    if not lib.exists() or any(o.stat().st_mtime > lib.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {lib}")
    return lib


def build_oracle(with_ref: bool | None = None) -> None:
    """Test-infrastructure checkers: oracle/_ref/libgss_oracle.so always; libgss_ref.so (the
    reference headers behind a C shim) only where /root/reference exists (this container)."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = Path("/root/reference/proj/include/gss").is_dir()
    if with_ref:
        targets += ["ref", "dropin"]
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), *targets], check=True)


if __name__ == "__main__":
    build_lib(verbose=True)
    build_oracle()
