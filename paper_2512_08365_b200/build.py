"""Build libdwb200.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

    python -m paper_2512_08365_b200.build       # or __graft_entry__.build()

The library lands at paper_2512_08365_b200/_lib/libdwb200.so: git-ignored, but
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libdwb200.so"
SOURCES = ["capi.cu", "attribute.cu", "split.cu", "replay.cu", "diff.cu", "pack.cu", "ingest.cu", "tensor.cu", "exchange.cu", "align.cu"]
HEADERS = ["dw_common.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",              # no FMA contraction: fp64 sums must match the reference bit for bit
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    deps.append(PKG.parent / "include" / "dwb200.h")
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> Path:
    """Diagnostic variants, never the product library (scripts/probe_attr.py):
    "prof" -- per-phase clock64 counters in the tile kernel (-DDW_PHASE_PROF,
    dw_phase_prof()); "skip" -- consumers release every stage unprocessed
    (-DDW_SKIP_CONSUMERS), the staging pipeline's own speed."""
    lib = LIB if not variant else OUT_DIR / f"libdwb200_{variant}.so"
    extra = {"prof": ["-DDW_PHASE_PROF"], "skip": ["-DDW_SKIP_CONSUMERS"]}.get(variant.split("_")[0], [])[:]
    if variant:  # experiment knobs for diagnostic builds only (e.g. -DDW_PREFETCH=0)
        extra += os.environ.get("DWB200_NVCC_EXTRA", "").split()
    if not variant and not force and not _stale():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    jobs = []
    for src in SOURCES:
        if not (CSRC / src).exists():
            continue
        obj = OUT_DIR / (Path(src).stem + variant + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(PKG.parent / "include"), "-c", str(CSRC / src),
               "-o", str(obj)]
        jobs.append((src, obj, cmd))
    # the translation units are independent: compile them side by side
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[2], capture_output=True, text=True), jobs))
    objs = []
    log = []
    for (src, obj, _), r in zip(jobs, results):
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        objs.append(str(obj))
    tmp = OUT_DIR / (lib.name + ".tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
           *objs, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    if not variant:
        (OUT_DIR / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose=True, variant=var))
