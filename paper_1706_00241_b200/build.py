"""Build recipe for the in-tree CUDA library ``libdefcg_b200.so``.

Every ``csrc/*.cu`` is compiled for sm_100a only (``-gencode
arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's source page maps
to the kernels, and linked with a static CUDA runtime into one shared object
that exports the C ABI of ``include/defcg_b200.h``.  The library is loaded with
ctypes; it shares the primary CUDA context (and therefore device pointers and
streams) with PyTorch.

Usage:  python -m paper_1706_00241_b200.build [--force]
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
LIB = PKG / "libdefcg_b200.so"
OBJ = PKG / "_build"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "-diag-suppress",
    "186",
    f"-I{INCLUDE}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA library cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out_dir: Path | None = None,
          defines: tuple = ()) -> Path:
    """Compile csrc/*.cu and link the library (in-tree, or a tuning variant
    with extra -D defines into out_dir)."""
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    srcs = sources()
    obj_dir = OBJ if out_dir is None else Path(out_dir) / "_build"
    lib = LIB if out_dir is None else Path(out_dir) / LIB.name
    obj_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        if force or _stale(obj, [src] + headers):
            cmd = [cc, *NVCC_FLAGS, *defines, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), flush=True)
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    if force or _stale(lib, objs):
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out_dir = None
    if "--variant" in args:
        out_dir = Path(args[args.index("--variant") + 1])
    out = build(force="--force" in args, verbose=True, out_dir=out_dir,
                defines=tuple(a for a in args if a.startswith("-D")))
    print(out)
