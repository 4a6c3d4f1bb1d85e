"""Build the in-tree C-ABI library ``liborth.so`` for sm_100a with nvcc.

``python paper_2601_13776_b200/build.py`` (or ``__graft_entry__.build()``).  This
file is loaded by path, not as a package module: importing the package itself
requires the built library (no fallback).
Objects go to ``paper_2601_13776_b200/_build``; the library next to this file.
Rebuilds only what changed (source or any header newer than its object); a change of the compile
flags (ORTH_EXPERIMENTAL, ORTH_NVCC_FLAGS) rebuilds everything.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "liborth.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
FLAGS += os.environ.get("ORTH_NVCC_FLAGS", "").split()   # diagnostics builds only (e.g. -DORTH_NSP_TRACE)
if os.environ.get("ORTH_EXPERIMENTAL") == "1":   # opt-in kernels that measured no faster (conv_tma, conv_pair)
    FLAGS.append("-DORTH_EXPERIMENTAL")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(OBJ, exist_ok=True)
    stamp = os.path.join(OBJ, "flags.txt")
    flags = " ".join(ARCH + FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
        with open(stamp, "w") as f:
            f.write(flags)
    hdr_t = max([os.path.getmtime(h) for h in _headers()] + [0.0])
    procs, objs = [], []
    for src in _sources():
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
            continue
        extra = ["-Xptxas", "-v"] if verbose and src.endswith(".cu") else []
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        if len(procs) >= jobs:
            _drain(procs, verbose)
    _drain(procs, verbose)
    lib_t = os.path.getmtime(LIB) if os.path.exists(LIB) else -1.0
    if lib_t < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if r.returncode:
            raise RuntimeError("link failed:\n" + r.stdout)
    return LIB


def _drain(procs, verbose):
    errs = []
    for cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode:
            errs.append(" ".join(cmd) + "\n" + out)
        elif verbose and out:
            print(out)
    procs.clear()
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
