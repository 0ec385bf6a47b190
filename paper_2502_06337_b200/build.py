"""Builds the sm_100a shared library of the voting path (in-tree, no JIT cache).

Output: paper_2502_06337_b200/_lib/librotavote_b200.so (git-ignored; travels to the GPU box).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
if os.environ.get("RV_LIB_OUT"):  # dev A/B builds of kernel variants (tools/ab_vote.py)
    LIB_DIR = Path(os.environ["RV_LIB_OUT"]).resolve()
LIB = LIB_DIR / "librotavote_b200.so"
INCLUDE = PKG.parent / "include"
SOURCES = ["rv_prep.cu", "rv_vote.cu", "rv_peaks.cu", "rv_refine.cu", "rv_coop.cu", "rv_io.cu", "rv_api.cpp",
           "rv_multi.cpp"]
# translation units whose device arithmetic must follow the host op order exactly
NO_FMAD = {"rv_coop.cu"}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp"))
    deps.append(INCLUDE / "rotavote_b200.h")
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    common = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
    extra = os.environ.get("RV_NVCC_EXTRA", "").split()  # dev A/B sweeps only (e.g. -DRV_BCAST_REDUX=0)
    common += extra
    jobs = []
    for src in SOURCES:
        obj = obj_dir / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *common, *(["-fmad=false"] if src in NO_FMAD else []),
               *(["-Xptxas", "-v"] if verbose else []), "-x",
               "cu" if src.endswith(".cu") else "c++", "-c", str(CSRC / src), "-o", str(obj)]
        if src.endswith(".cpp"):
            cmd = [nvcc(), *ARCH, *[a for a in common if a != "--expt-relaxed-constexpr"], "-x", "c++", "-c",
                   str(CSRC / src), "-o", str(obj)]
        jobs.append((src, cmd, str(obj)))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[1], capture_output=True, text=True), jobs))
    objs = []
    for (src, _, obj), res in zip(jobs, results):
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
