"""In-tree build of libmgb.so (all sm_100a kernels + the C-ABI declared in include/mgb.h).

nvcc cross-compiles here without a GPU; the built .so travels to the B200 box with the repo
snapshot.  Objects are rebuilt only when a source or header is newer than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
OUT_DIR = PKG_DIR / "_lib"
LIB_PATH = OUT_DIR / "libmgb.so"
REPO = PKG_DIR.parent

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=default",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
    f"-I{REPO / 'include'}",
    f"-I{CSRC}",
]


CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-g", "-pthread", "-I/usr/local/cuda/include", f"-I{REPO / 'include'}"]


def _sources() -> list[Path]:
    # *.cu: device code for sm_100a; *.cpp: host code (the CPU attention path), compiled by g++
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted((REPO / "include").glob("*.h"))


def _stale(obj: Path, src: Path, headers: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in headers)


def _compile(src: Path, obj: Path, verbose: bool) -> str:
    if src.suffix == ".cpp":
        cmd = [CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [NVCC, *ARCH_FLAGS, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (obj.with_suffix(".ptxas.log")).write_text(log)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{log}")
    if verbose:
        print(f"[mgb-build] compiled {src.name}", file=sys.stderr)
    return log


def build(force: bool = False, verbose: bool = True) -> Path:
    """Compile every csrc/*.cu for sm_100a and link libmgb.so (returns its path)."""
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    srcs = _sources()
    objs = [OUT_DIR / (s.name.replace(".", "_") + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, s, headers)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            list(ex.map(lambda so: _compile(so[0], so[1], verbose), todo))
    if todo or force or not LIB_PATH.exists():
        tmp = LIB_PATH.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"link failed:\n{proc.stdout}{proc.stderr}")
        os.replace(tmp, LIB_PATH)
        if verbose:
            print(f"[mgb-build] linked {LIB_PATH}", file=sys.stderr)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv)
