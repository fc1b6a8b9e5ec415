"""In-tree build of the B200 planner library (paper_2409_03365_b200/lib/libwsgpu.so).

Device code: nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``),
``-fmad=false`` so every double matches the reference bit for bit,
``-lineinfo`` for ncu source attribution.  Host C++: g++ with
``-ffp-contract=off``.  nvcc cross-compiles without a GPU, so this runs in the
build container; the resulting .so travels to the GPU box in-tree.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
BUILD = PKG / "lib" / "obj"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-I", str(ROOT / "include")] + ARCH
# nlohmann/json (header-only; the same library the reference's workload_from_json uses)
JSON_DIR = Path(os.environ.get("WSGPU_JSON_DIR", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/"
                                                 "cudnn_frontend/thirdparty/nlohmann"))
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-sign-compare",
             "-I", str(ROOT / "include"), "-I", str(CUDA / "include"), "-I", str(JSON_DIR)]

LIBNAME = LIB / "libwsgpu.so"


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: list[str] | None = None,
          name: str | None = None, extra_nvcc: list[str] | None = None) -> Path:
    """Compile host + device sources and link libwsgpu.so; returns its path.
    `defines`/`name` build a tuning variant (e.g. ["WS_PLACE_MINB=6"], "libwsgpu_v6.so")
    with its own object directory."""
    libname = LIB / name if name else LIBNAME
    build_dir = BUILD if not name else LIB / ("obj_" + Path(name).stem)
    dflags = [f"-D{d}" for d in (defines or [])]
    build_dir.mkdir(parents=True, exist_ok=True)
    headers = (list((ROOT / "include").rglob("*.h*")) + list((CSRC / "device").glob("*.cuh")) +
               list((CSRC / "host").glob("*.h*")))
    objs, jobs = [], []
    for src in sorted((CSRC / "device").glob("*.cu")):  # the long nvcc compile first
        obj = build_dir / (src.stem + ".cu.o")
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC, *NVCC_FLAGS, *dflags, *(extra_nvcc or []), "-Xptxas", "-v" if verbose else "-O3",
                         "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    for src in sorted((CSRC / "host").glob("*.cpp")):
        obj = build_dir / (src.stem + ".o")
        if force or _stale(obj, [src] + headers):
            jobs.append(["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    # independent translation units compile concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as pool:
        list(pool.map(lambda cmd: _run(cmd, verbose), jobs))
    if force or _stale(libname, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(libname), *map(str, objs), "-cudart", "static",
              "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], verbose)
    return libname


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIBNAME)
