"""Build libdsv.so in-tree: every csrc/*.cu compiled by nvcc for sm_100a.

The library links the CUDA runtime statically and resolves driver entry points
(cuTensorMapEncodeTiled) at run time, so it loads on hosts without a GPU
driver (the CPU test tier checks its exported symbols there).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG.parent / "build" / "dsv"
LIB = PKG / "libdsv.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-Xptxas", "-v", "-DDSV_WATCHDOG", "-I", str(PKG.parent / "include"),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the DSV CUDA library cannot be built")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps_mtime() -> float:
    files = list(CSRC.glob("*")) + [PKG.parent / "include" / "dsv.h", Path(__file__)]
    return max(f.stat().st_mtime for f in files if f.exists())


def up_to_date() -> bool:
    return LIB.exists() and LIB.stat().st_mtime >= _deps_mtime()


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """defines: extra -D flags for a variant library written to `out` (tools only)."""
    lib = Path(out) if out is not None else LIB
    if not force and not defines and up_to_date():
        return LIB
    nvcc = _nvcc()
    bdir = BUILD if not defines else BUILD.parent / ("dsv_" + "_".join(d.split("=")[0].lower() for d in defines))
    bdir.mkdir(parents=True, exist_ok=True)
    objs = []

    def compile_one(src: Path):
        obj = bdir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        (bdir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for obj, log in ex.map(compile_one, _sources()):
            objs.append(obj)
            if verbose:
                sys.stderr.write(log)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [-DNAME=VAL ... --out path/libvariant.so]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=out))
