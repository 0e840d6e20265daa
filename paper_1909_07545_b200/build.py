"""Build libfsb200.so (the C-ABI of include/fsb200.h) in-tree with nvcc for sm_100a.

    python -m paper_1909_07545_b200.build [--force] [--verbose]

Translation units with fp64 geometry/setup math are compiled with -fmad=false so
their rounding sequence follows NumPy's (no FMA contraction); the fp32 hot-path
units keep contraction on.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libfsb200.so"
# checked build (-DFSB_CHECKED: NaN-poisoned shared memory + index asserts), loaded
# instead of LIB when FSB_LIB=checked
BUILD_CHECKED = PKG / "_build_checked"
LIB_CHECKED = PKG / "libfsb200_checked.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", str(ROOT / "include")]
# (source, extra flags)
UNITS = [
    ("fields.cu", ["-fmad=false"]),
    ("rasters.cu", ["-fmad=false"]),
    ("setup.cu", ["-fmad=false"]),
    ("pd.cu", []),
    ("pd_block.cu", []),
    ("pd_pair.cu", []),
    ("pd_tma.cu", []),
    ("pd_cluster.cu", []),
    ("pd64.cu", ["-fmad=false"]),
    ("pd64_block.cu", ["-fmad=false"]),
    ("pd64_tile.cu", []),
    ("pd64_tma.cu", []),
    ("pd64_ctile.cu", []),
    ("pd64_level.cu", []),
    ("sample64.cu", ["-fmad=false"]),
    ("solver.cu", []),
    ("synth.cu", ["-fmad=false"]),
    ("depth.cu", ["-fmad=false"]),
    ("evaluate.cu", ["-fmad=false"]),
]
HEADERS = [*sorted(CSRC.glob("*.cuh")), ROOT / "include" / "fsb200.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
          checked: bool = False) -> Path:
    bdir, lib = (BUILD_CHECKED, LIB_CHECKED) if checked else (BUILD, LIB)
    bdir.mkdir(exist_ok=True)
    objs, jobs = [], []
    for src, extra in UNITS:
        s = CSRC / src
        o = bdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *HEADERS, Path(__file__)]):
            cmd = [nvcc(), *ARCH, *COMMON, *extra, *(["-DFSB_CHECKED"] if checked else []),
                   "-c", str(s), "-o", str(o)]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            jobs.append(cmd)
    if jobs:  # translation units compile independently: run them in parallel
        from concurrent.futures import ThreadPoolExecutor
        workers = max(1, min(len(jobs), os.cpu_count() or 1))
        with ThreadPoolExecutor(workers) as ex:
            for f in [ex.submit(subprocess.run, cmd, check=True) for cmd in jobs]:
                f.result()
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print ptxas register/smem usage")
    ap.add_argument("--checked", action="store_true",
                    help="build libfsb200_checked.so (NaN-poisoned shared memory, index asserts)")
    a = ap.parse_args(argv)
    out = build(force=a.force, verbose=a.verbose, ptxas_verbose=a.ptxas, checked=a.checked)
    print(out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
