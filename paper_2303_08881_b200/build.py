"""Builds libddilu_b200.so in-tree with nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_2303_08881_b200.build [--force] [-v]
    DDILU_EXPERIMENTS=1 python -m paper_2303_08881_b200.build     # + csrc/experiments/*.cu, -DDDILU_EXPERIMENTS

The default build is the product: the C ABI of include/ddilu_b200.h.  The experiments build adds the
measured-slower alternative kernels, tuning knobs and diagnostics declared in include/ddilu_b200_experiments.h
(used by scripts/probe_*.py and by the tests that keep those kernels bit-exact; they skip without it)."""

from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
LIB = os.path.join(PKG, "libddilu_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    # the reference never fuses a*b+c (numba, no fastmath): keep every product rounded
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
]


def experiments_enabled() -> bool:
    return os.environ.get("DDILU_EXPERIMENTS", "0") == "1"


def sources(experiments: bool = False):
    out = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    if experiments:
        exp = os.path.join(CSRC, "experiments")
        out += sorted(os.path.join(exp, f) for f in os.listdir(exp) if f.endswith(".cu"))
    return out


def _stale(out, deps):
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    exp = experiments_enabled()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    objdir = os.path.join(PKG, "build_exp" if exp else "build")      # one object directory per flavour
    os.makedirs(objdir, exist_ok=True)
    flags = NVCC_FLAGS + (["-DDDILU_EXPERIMENTS"] if exp else [])
    jobs = []
    objs = []
    for src in sources(exp):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc] + flags + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj]
            jobs.append(cmd)
    if jobs:
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
                if verbose or res.returncode:
                    sys.stderr.write(res.stdout + res.stderr)
                if res.returncode:
                    raise RuntimeError("nvcc failed: " + " ".join(cmd))
    stamp = LIB + ".flavour"
    flavour = "experiments" if exp else "product"
    built = open(stamp).read().strip() if os.path.exists(stamp) else ""
    if force or jobs or _stale(LIB, objs) or built != flavour:
        subprocess.check_call([nvcc, "-shared", "-o", LIB] + objs + ["-gencode", "arch=compute_100a,code=sm_100a"])
        with open(stamp, "w") as fh:
            fh.write(flavour + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
