"""Builds every native artefact in-tree (they travel to the GPU box with gpurun):

  paper_2603_15023_b200/libpac.so   libpac, sm_100a (the product)
  datagen/libdatagen.so             device-side synthetic input generator
  oracle/liboracle.so               CPU oracle (plain C, host compiler; test infrastructure)

Usage: python build.py [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]

TARGETS = {
    "libpac": (os.path.join(ROOT, "paper_2603_15023_b200", "libpac.so"),
               sorted(glob.glob(os.path.join(ROOT, "paper_2603_15023_b200", "csrc", "*.cu"))),
               glob.glob(os.path.join(ROOT, "paper_2603_15023_b200", "csrc", "*.cuh"))
               + [os.path.join(ROOT, "include", "pac.h")]),
    "datagen": (os.path.join(ROOT, "datagen", "libdatagen.so"),
                [os.path.join(ROOT, "datagen", "csrc", "datagen.cu")], []),
}


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _includes(src, seen=None):
    """src plus every local header it includes, recursively (#include "...")."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', open(src).read(), flags=re.M):
        _includes(os.path.normpath(os.path.join(os.path.dirname(src), inc)), seen)
    return seen


def build_cuda(name: str, force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu of the target to an object in parallel, then link the .so."""
    out, srcs, hdrs = TARGETS[name]
    if not (force or _stale(out, srcs + hdrs)):
        return out
    objdir = os.path.join(ROOT, "build", name)
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and not _stale(obj, _includes(src)):
            return src, obj, None  # object newer than the source and every header it includes
        cmd = [NVCC] + ARCH + NVFLAGS + ["-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(os.cpu_count() or 8, len(srcs))) as ex:
        results = list(ex.map(compile_one, srcs))
    for src, obj, r in results:
        if r is None:
            continue
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [NVCC] + ARCH + ["-shared", "-o", out] + [o for _, o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"link failed for {name}")
    return out


def build_all(force: bool = False, verbose: bool = False):
    sys.path.insert(0, ROOT)
    out = [build_cuda("libpac", force, verbose), build_cuda("datagen", force, verbose)]
    import oracle
    out.append(oracle.build(force))
    return out


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv, verbose="--verbose" in sys.argv):
        print(p)
