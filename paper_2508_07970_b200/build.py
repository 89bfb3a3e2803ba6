"""Build the sm_100a shared library ``libyatt_b200.so`` in-tree.

Every CUDA/C++ source under ``csrc/`` is compiled by nvcc for
``-gencode arch=compute_100a,code=sm_100a`` with ``-lineinfo`` (ncu source
view) and linked into one shared object next to this file, so it travels to
the GPU box with the repo snapshot.  Object files are cached by content hash
of the source + flags under ``build/``.
"""
from __future__ import annotations

import hashlib
import re
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "yatt_b200"
LIB = PKG / "libyatt_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT / 'include'}",
]
CXX_FLAGS = ["-O2", "-fPIC", "-fopenmp", "-std=c++20", f"-I{ROOT / 'include'}",
             "-I/usr/local/cuda/include"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _digest(path: Path, flags: list[str]) -> str:
    h = hashlib.sha256()
    h.update(path.read_bytes())
    for inc in re.findall(r'#include "(\w+\.cu)"', path.read_text(errors="ignore")):
        h.update((path.parent / inc).read_bytes())  # e.g. token_stats_small.cu
    for dep in sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "yatt_cuda.h"]:
        h.update(dep.read_bytes())
    for dep in sorted((ROOT / "include" / "yatt").glob("*.hpp")):
        h.update(dep.read_bytes())
    h.update(" ".join(flags).encode())
    return h.hexdigest()[:16]


def _compile(src: Path, verbose: bool, extra: tuple = ()) -> Path:
    is_cu = src.suffix == ".cu"
    flags = (NVCC_FLAGS if is_cu else CXX_FLAGS) + list(extra)
    obj = BUILD / f"{src.stem}.{_digest(src, flags)}.o"
    if obj.exists():
        return obj
    cmd = ([nvcc(), "-c", str(src), "-o", str(obj)] + flags) if is_cu else \
        (["g++", "-c", str(src), "-o", str(obj)] + flags)
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = BUILD / f"{src.stem}.log"
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}{res.stderr}")
    if verbose:
        sys.stderr.write(f"[build] {src.name}\n")
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    link_key = hashlib.sha256("".join(sorted(o.name for o in objs)).encode()).hexdigest()[:16]
    stamp = BUILD / "link.stamp"
    if LIB.exists() and stamp.exists() and stamp.read_text() == link_key:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-o", str(tmp)] + ARCH + [str(o) for o in objs] + [
        "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lcudart_static", "-lrt", "-ldl", "-lpthread",
        "-lgomp", "-Xlinker", "--no-undefined"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}{res.stderr}")
    os.replace(tmp, LIB)
    stamp.write_text(link_key)
    return LIB


def build_variant(name: str, defines: dict) -> Path:
    """Experiment build: every source recompiled with -D overrides (knobs are
    namespaced, e.g. YATT_A1_*, YATT_GAE_*), linked into
    _variants/libyatt_b200_<name>.so (load it with YATT_B200_LIB=...)."""
    BUILD.mkdir(parents=True, exist_ok=True)
    extra = tuple(f"-D{k}={v}" for k, v in sorted(defines.items()))
    objs = []
    for src in sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")):
        objs.append(_compile(src, False, extra if src.suffix == ".cu" else ()))
    out = PKG / "_variants" / f"libyatt_b200_{name}.so"
    out.parent.mkdir(exist_ok=True)
    cmd = [nvcc(), "-shared", "-o", str(out)] + ARCH + [str(o) for o in objs] + [
        "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lcudart_static", "-lrt", "-ldl", "-lpthread", "-lgomp"]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "variant":
        print(build_variant(sys.argv[2], dict(a.split("=") for a in sys.argv[3:])))
    else:
        print(build(verbose=True))
