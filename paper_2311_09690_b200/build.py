"""Build libtpcb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2311_09690_b200.build          # incremental
    python -m paper_2311_09690_b200.build --force  # rebuild everything

Each .cu is compiled to an object under build/ (relocatable device code off:
every kernel is self-contained), then linked into one shared library next to
this file so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "tpcb200"
LIB = PKG / "libtpcb200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> Path:
    """NCCL 2.28 shipped with torch (nvidia-nccl wheel), same image on every box."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL) not found")
    return Path(list(spec.submodule_search_locations)[0])
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT / 'include'}",
              f"-I{_nccl_dir() / 'include'}", "-diag-suppress", "128,177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _deps(src: Path) -> list[Path]:
    return [src] + sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").glob("*.h"))


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    obj = BUILD / (src.stem + ".o")
    if not force and obj.exists():
        newest = max(p.stat().st_mtime for p in _deps(src))
        if obj.stat().st_mtime >= newest:
            return obj, ""
    extra = os.environ.get("TPCB_NVCC_EXTRA", "").split()  # debug builds, e.g. -DTPCB_TRACE_PHASES
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj, res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, len(sources))) as ex:
        results = list(ex.map(lambda s: _compile(s, force), sources))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        nccl_lib = _nccl_dir() / "lib"
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               f"-L{nccl_lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
