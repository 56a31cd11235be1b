"""Build the engine's shared library in-tree with nvcc (sm_100a only).

    python -m paper_2504_15303_b200.build

Produces paper_2504_15303_b200/libhetserve_b200.so.  Flags: -fmad=false so
nvcc never contracts a*b+c (CPython rounds every operation separately);
-lineinfo for ncu source correlation; cudart linked statically so the .so
is self-contained on the GPU box.
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libhetserve_b200.so"
SOURCES = ["capi.cu", "search.cu", "replay.cu", "topk.cu", "sort.cu", "rng.cu", "scheduler.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, force: bool = False, timers: bool = False, defines=(), out=None) -> pathlib.Path:
    """defines / out: diagnostic variants (e.g. -DHS_REPLAY_MIN_BLOCKS_MULTI=5 into a
    separate .so, loaded with HS_LIB=...); the product library takes neither."""
    lib = pathlib.Path(out).resolve() if out else (PKG / "libhetserve_b200_timers.so" if timers else LIB)
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps += list((PKG.parent / "include").glob("*.h"))
    if not force and lib.exists() and all(lib.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return lib
    flags = [*ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
             "-Xptxas", "-v" if verbose else "-O3", *(["-DHS_TIMERS"] if timers else []), *defines]
    objdir = PKG / "build" / (lib.stem if out else ("timers" if timers else "release"))
    objdir.mkdir(parents=True, exist_ok=True)
    # one nvcc per translation unit, in parallel, then one link
    cmds = [[nvcc(), *flags, "-c", str(CSRC / s), "-o", str(objdir / (s + ".o"))] for s in SOURCES]
    if verbose:
        for c in cmds:
            print(" ".join(c))
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, cwd=CSRC, capture_output=not verbose, text=True), cmds):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed:\n{r.stderr}")
    link = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(lib) + ".tmp",
            *[str(objdir / (s + ".o")) for s in SOURCES]]
    subprocess.run(link, check=True, cwd=CSRC)
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, timers="--timers" in sys.argv))
