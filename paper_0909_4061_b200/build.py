"""Build liblowrank_b200.so in-tree with nvcc for sm_100a.

    python -m paper_0909_4061_b200.build [--force] [--verbose]

Each csrc/*.cu is compiled to an object (in parallel), then linked into a
shared library next to this file with a static CUDA runtime, so the .so has
no dependency beyond the driver (torch's own runtime is not needed by it).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "liblowrank_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps(src):
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + [
        os.path.join(ROOT, "include", "lowrank_b200.h"), src, __file__]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, extra=(), out=None, obj=None):
    """extra: additional nvcc flags (e.g. -D tuning macros); out/obj: build a
    variant library elsewhere (development sweeps; LR_LIB selects it)."""
    OUT = out or globals()["OUT"]
    OBJ = obj or globals()["OBJ"]
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    cc = nvcc()
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, _deps(s)):
            cmd = [cc, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
            jobs.append((s, cmd))

    def run(job):
        s, cmd = job
        if verbose:
            print(" ".join(cmd), flush=True)
        p = subprocess.run(cmd, capture_output=True, text=True)
        return s, p

    failed = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s, p in ex.map(run, jobs):
            if p.returncode != 0:
                failed.append((s, p.stderr))
            elif verbose and p.stderr.strip():
                print(p.stderr, flush=True)
    if failed:
        msg = "\n".join(f"--- {s}\n{err}" for s, err in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    if force or jobs or _stale(OUT, objs):
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
