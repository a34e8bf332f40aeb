"""Build the sm_100a shared library in-tree (paper_1910_01304_b200/lib/).

    python -m paper_1910_01304_b200.build [--force]
    python -m paper_1910_01304_b200.build --variant NAME -DMACRO=V ...   (exp/NAME/)

Each translation unit is compiled in parallel with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` with ``--fmad=false`` (the
reference's float64 traversal has no fused multiply-add; see
csrc/hrpp_device.cuh) and ``-lineinfo`` (ncu source view), then linked
into ``lib/libhrpp_b200.so`` with the static CUDA runtime.
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
OBJ = PKG / "build_obj"
LIB = PKG / "lib" / "libhrpp_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-warn-spills",
              f"-I{ROOT / 'include'}", f"-I{CSRC}"]
SOURCES = ["k_hash_trace.cu", "k_table.cu", "k_consult.cu", "k_fast.cu", "k_spawn.cu", "k_shard.cu",
           "capi.cu", "bvh_build.cpp"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def _deps(src: Path):
    return [src, CSRC / "hrpp_device.cuh", CSRC / "hrpp_internal.h",
            ROOT / "include" / "hrpp_b200.h"]


def _compile(src: Path, verbose: bool, objdir: Path = OBJ, defines=()):
    obj = objdir / (src.name + ".o")
    if obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime for d in _deps(src)
                            if d.exists()):
        return obj, ""
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *defines, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [nvcc(), *NVCC_FLAGS, *defines, "-x", "c++", "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v") if src.suffix == ".cu" else None
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-6000:]}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), variant: str | None = None
          ) -> Path:
    """Build lib/libhrpp_b200.so; with ``variant`` build an experiment copy
    with extra ``-D`` flags into exp/<variant>/ (never the shipped library)."""
    objdir, lib = OBJ, LIB
    if variant:
        objdir = ROOT / "exp" / variant / "obj"
        lib = ROOT / "exp" / variant / "libhrpp_b200.so"
        force = True
    objdir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    if force:
        for o in objdir.glob("*.o"):
            o.unlink()
    srcs = [CSRC / s for s in SOURCES]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, objdir, defines), srcs))
    objs = [r[0] for r in results]
    logs = "".join(r[1] for r in results)
    if logs and verbose:
        sys.stderr.write(logs)
    if lib.exists() and not force and all(lib.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return lib
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return lib


if __name__ == "__main__":
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else None
    print(build(force="--force" in argv, verbose="-v" in argv,
                defines=[a for a in argv if a.startswith("-D")], variant=var))
