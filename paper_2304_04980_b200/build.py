"""Build libgridlq_b200.so in-tree with nvcc for sm_100a (no torch extension machinery).

``python -m paper_2304_04980_b200.build`` or ``__graft_entry__.build()``.  Objects are
rebuilt only when a source or header is newer; translation units compile in parallel.
"""

from __future__ import annotations

import glob
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libgridlq_b200.so")
OBJDIR = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{INCLUDE}", f"-I{CSRC}"]


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + glob.glob(os.path.join(INCLUDE, "*.h"))
    hdr_time = _newest(headers)
    jobs = []
    objs = []
    for src in sources:
        obj = os.path.join(OBJDIR, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), hdr_time):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{res.stdout}\n{res.stderr}")
        return res

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    for job in jobs:
        lint_sass(job[-1])
    if force or jobs or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread"])
    return LIB


# LDGSTS whose shared destination ptxas split as [R + UR] (emitted next to an L2 cache-policy
# operand) faults with "illegal instruction" on B200; refuse to ship such code.
_BAD_LDGSTS = re.compile(r"LDGSTS[^;]*\[R\d+\+UR\d+")


def lint_sass(obj: str) -> None:
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    res = subprocess.run([cuobjdump, "-sass", obj], capture_output=True, text=True)
    if res.returncode != 0:
        return
    func, bad = None, {}
    for line in res.stdout.splitlines():
        if "Function :" in line:
            func = line.split("Function :")[1].strip()
        elif _BAD_LDGSTS.search(line):
            bad[func] = bad.get(func, 0) + 1
    if bad:
        os.remove(obj)
        raise RuntimeError(f"{os.path.basename(obj)}: LDGSTS [R+UR] forms (fault on B200) in "
                           + ", ".join(f"{k} x{v}" for k, v in bad.items()))


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
