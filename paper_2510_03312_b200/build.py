"""Build the sm_100a C-ABI library ``libubs_b200.so`` in-tree with nvcc.

The library is plain CUDA C++ behind ``extern "C"`` entry points declared in
``include/ubs_b200.h`` (no torch headers), loaded by ``_lib.py`` with ctypes.
Objects are compiled in parallel; ``-Xptxas -v`` output goes to
``build/ptxas.log`` for register/spill inspection.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libubs_b200.so"
TORCH_OUT = PKG / "libubs_torch.so"  # TORCH_LIBRARY(ubs) operators over the C ABI (csrc_torch/)
BUILD = ROOT / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", f"-I{ROOT / 'include'}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "ubs_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


CHECKED_OUT = PKG / "libubs_b200_checked.so"  # -DUBS_CHECKED: device bounds guards (tests/test_gpu_checked.py)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> Path:
    """nvcc every csrc/*.cu for sm_100a and link the shared library.
    ``variant="checked"`` builds the bounds-checked variant
    (libubs_b200_checked.so, -DUBS_CHECKED) from the same sources."""
    out = CHECKED_OUT if variant == "checked" else OUT
    defines = ["-DUBS_CHECKED"] if variant == "checked" else []
    if not force and out.exists() and not (variant == "" and needs_build()) and \
            not (variant and any(p.stat().st_mtime > out.stat().st_mtime for p in CSRC.glob("*"))):
        return out
    bdir = BUILD / variant if variant else BUILD
    bdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: Path):
        obj = bdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, *defines, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr[-6000:]}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    (bdir / "ptxas.log").write_text("".join(log for _, log in results))
    tmp = out.with_suffix(f".{os.getpid()}.tmp.so")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, out)
    if verbose:
        print(f"built {out}")
    return out


def torch_ops_need_build() -> bool:
    if not TORCH_OUT.exists():
        return True
    t = TORCH_OUT.stat().st_mtime
    deps = list((PKG / "csrc_torch").glob("*")) + [ROOT / "include" / "ubs_b200.h", OUT, Path(__file__)]
    return any(p.exists() and p.stat().st_mtime > t for p in deps)


def build_torch_ops(force: bool = False, verbose: bool = False) -> Path:
    """g++ the TORCH_LIBRARY(ubs) extension (csrc_torch/ubs_torch.cpp) in-tree,
    linked against libubs_b200.so (rpath $ORIGIN) and the installed torch."""
    if not force and not torch_ops_need_build():
        return TORCH_OUT
    build(verbose=verbose)
    import torch
    import torch.utils.cpp_extension as ce
    inc = ce.include_paths(device_type="cuda") if "device_type" in ce.include_paths.__code__.co_varnames \
        else ce.include_paths(cuda=True)
    libs = ce.library_paths(device_type="cuda") if "device_type" in ce.library_paths.__code__.co_varnames \
        else ce.library_paths(cuda=True)
    abi = 1 if torch.compiled_with_cxx11_abi() else 0
    tmp = TORCH_OUT.with_suffix(f".{os.getpid()}.tmp.so")
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           str(PKG / "csrc_torch" / "ubs_torch.cpp"), "-o", str(tmp), f"-I{ROOT / 'include'}",
           *[f"-I{d}" for d in inc], *[f"-L{d}" for d in libs], f"-L{PKG}", "-lubs_b200", "-ltorch",
           "-ltorch_cpu", "-ltorch_cuda", "-lc10", "-lc10_cuda", "-Wl,-rpath,$ORIGIN",
           *[f"-Wl,-rpath,{d}" for d in libs]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch ops build failed:\n{r.stderr[-6000:]}")
    os.replace(tmp, TORCH_OUT)
    if verbose:
        print(f"built {TORCH_OUT}")
    return TORCH_OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_torch_ops(force="--force" in sys.argv, verbose=True)
