"""Build recipe for librsa_b200.so (sm_100a only), in-tree.

    python -m paper_2511_19835_b200.build          # or __graft_entry__.build()

nvcc compiles each csrc/*.cu with -gencode arch=compute_100a,code=sm_100a and
-lineinfo, then links one shared library next to this file.  Incremental: a
source is recompiled only when it (or a header) is newer than its object.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "librsa_b200.so"
TORCH_LIB = PKG / "librsa_b200_torch.so"   # TORCH_LIBRARY registration (csrc/torch_ops.cpp)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# RSA_EXTRA_NVCC: extra -D flags for A/B builds
NVCC_FLAGS = ["-O3", *os.environ.get("RSA_EXTRA_NVCC", "").split(), "-std=c++17", "-lineinfo", "-Xcompiler",
              "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build librsa_b200.so")


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    headers = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in headers])
    if obj.exists() and obj.stat().st_mtime >= newest:
        return obj
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = OBJ / (src.stem + ".ptxas.log")
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr[-6000:]}")
    if verbose:
        print(f"[build] {src.name}")
    return obj


def build_torch_ops(verbose: bool = True) -> Path:
    """g++ the TORCH_LIBRARY layer (host C++ only) against torch's headers and
    librsa_b200.so (found next to it through an $ORIGIN rpath)."""
    import torch
    from torch.utils.cpp_extension import include_paths, library_paths
    src = CSRC / "torch_ops.cpp"
    deps = [src, LIB, ROOT / "include" / "rsa_b200.h"]
    if TORCH_LIB.exists() and TORCH_LIB.stat().st_mtime >= max(p.stat().st_mtime for p in deps):
        return TORCH_LIB
    cuda_home = Path(nvcc()).resolve().parent.parent
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    tmp = TORCH_LIB.with_suffix(".so.tmp")
    cmd = [shutil.which("g++") or "g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           "-I", str(ROOT / "include"), *[f"-I{p}" for p in include_paths()], "-I", str(cuda_home / "include"),
           str(src), "-L", str(PKG), "-lrsa_b200", *[f"-L{p}" for p in library_paths()],
           "-lc10", "-lc10_cuda", "-ltorch_cpu", "-ltorch_cuda", "-L", str(cuda_home / "lib64"), "-lcudart",
           "-Wl,-rpath,$ORIGIN", "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed on torch_ops.cpp:\n{res.stderr[-6000:]}")
    os.replace(tmp, TORCH_LIB)
    if verbose:
        print(f"[build] linked {TORCH_LIB}")
    return TORCH_LIB


def build(verbose: bool = True) -> Path:
    _build_lib(verbose)
    build_torch_ops(verbose)
    return LIB


def _build_lib(verbose: bool) -> Path:
    OBJ.mkdir(exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), sources))
    if LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"[build] linked {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose="-q" not in sys.argv)
