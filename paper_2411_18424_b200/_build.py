"""In-tree native build: libkvswap.so (sm_100a) and the oracle's C restatement.

Both artefacts land next to their sources so gpurun snapshots carry them to
the GPU box (they are git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libkvswap.so"
CU_SRC = PKG / "csrc" / "kvswap.cu"
HDR = ROOT / "include" / "kvswap.h"
HDR_WL = ROOT / "include" / "kvswap_workload.h"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libkvswap")


def _stale(target: Path, *deps: Path) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_kvswap(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/kvswap.cu into PKG/libkvswap.so for sm_100a (static cudart)."""
    if not force and not _stale(LIB_PATH, CU_SRC, HDR, HDR_WL, Path(__file__)):
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [
        nvcc(), *ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17",
        "-shared", "-Xcompiler", "-fPIC",
        "-cudart", "static",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", str(ROOT / "include"),
        "-o", str(tmp), str(CU_SRC),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        print(res.stderr)
    tmp.replace(LIB_PATH)
    return LIB_PATH


def build_oracle(force: bool = False) -> Path:
    """Compile the oracle's C restatement (test/bench checker only)."""
    src = ROOT / "oracle" / "kvswap_oracle.c"
    out = ROOT / "oracle" / "liboracle.so"
    if not force and not _stale(out, src):
        return out
    tmp = out.with_suffix(".so.tmp")
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-shared", "-fPIC", "-pthread",
           "-o", str(tmp), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed ({res.returncode}):\n{res.stderr}")
    tmp.replace(out)
    return out


def build_kvctrl(force: bool = False) -> Path:
    """Compile the native control plane (host C++): the C ABI library
    PKG/libkvctrl.so (csrc/ctrlplane.cpp, include/kvctrl.h) and the CPython
    extension PKG/_kvctrl<EXT_SUFFIX> (csrc/kvctrl_py.cpp, same C++)."""
    import sysconfig

    src = PKG / "csrc" / "ctrlplane.cpp"
    py_src = PKG / "csrc" / "kvctrl_py.cpp"
    hdr = ROOT / "include" / "kvctrl.h"
    lib = PKG / "libkvctrl.so"
    ext = PKG / ("_kvctrl" + sysconfig.get_config_var("EXT_SUFFIX"))
    base = ["g++", "-O3", "-std=c++17", "-Wall", "-Wextra", "-shared", "-fPIC",
            "-I", str(ROOT / "include")]
    jobs = [(lib, [src], base),
            (ext, [py_src], base + ["-I", sysconfig.get_paths()["include"]])]
    for out, srcs, cmd in jobs:
        if not force and not _stale(out, src, py_src, hdr, Path(__file__)):
            continue
        tmp = out.with_name(out.name + ".tmp")
        res = subprocess.run(cmd + ["-o", str(tmp)] + [str(x) for x in srcs],
                             capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"g++ failed ({res.returncode}):\n{res.stderr}")
        tmp.replace(out)
    return ext


def build_all(force: bool = False) -> None:
    build_kvswap(force=force)
    build_kvctrl(force=force)
    build_oracle(force=force)
