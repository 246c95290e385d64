"""Iteration counts of the BASELINE-sized configurations, from the CPU oracle.

    python tests/golden/make_iterations_large.py [case ...]      (no case = all)

The oracle (oracle/ddilu_oracle.{c,py}) is pinned bit for bit to the reference
on every fixture of tests/golden (tests/test_oracle_golden.py), and reproduces
SURVEY.md Appendix B's reference-measured counts at 128^3; the reference itself
(Python + numba, per-row validation loop in csr_from_arrays) needs hours for
256^3, the C port minutes.  Each case runs the reference pipeline of
bench.py:108-140 (partition -> classify -> setup -> fgmres(50), rtol 1e-8,
inner 3, b = A*1) once and merges its record into
tests/golden/iterations_large.json: iteration count, final relative residual,
the whole residual history (hex floats), setup / solve seconds and the host
it ran on.  bench.py reads `its` from there (`its_oracle`), the gpu tests
assert |its_gpu - its| <= 1.
"""

from __future__ import annotations

import fcntl
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ddilu_oracle as orc  # noqa: E402

EPS = (1.0, 1.0, 0.01)
OUT = os.path.join(HERE, "iterations_large.json")

# name -> (kind, n per axis, p, precond, fill)
CASES = {
    # BASELINE config 2: 128^3 block-Jacobi ILU(0), 1/2/4/8 subdomains (190/233/244/244)
    "aniso3d_128_bj_p1": ("aniso3d", 128, 1, "bj", "ilu0"),
    "aniso3d_128_bj_p2": ("aniso3d", 128, 2, "bj", "ilu0"),
    "aniso3d_128_bj_p4": ("aniso3d", 128, 4, "bj", "ilu0"),
    "aniso3d_128_bj_p8": ("aniso3d", 128, 8, "bj", "ilu0"),
    # 128^3 p=8 two-level (App. B: 191 / 182 / 138)
    "aniso3d_128_schur_p8": ("aniso3d", 128, 8, "schur", "ilu0"),
    "aniso3d_128_rap_p8": ("aniso3d", 128, 8, "rap", "ilu0"),
    "aniso3d_128_rap-milu_p8": ("aniso3d", 128, 8, "rap-milu", "ilu0"),
    # BASELINE config 3 (the headline) and 4
    "aniso3d_256_schur_p8": ("aniso3d", 256, 8, "schur", "ilu0"),
    "aniso3d_256_rap-milu_p8": ("aniso3d", 256, 8, "rap-milu", "ilu0"),
    "aniso3d_256_rap_p8": ("aniso3d", 256, 8, "rap", "ilu0"),
    "aniso3d_256_bj_p8": ("aniso3d", 256, 8, "bj", "ilu0"),
    # BASELINE config 5 shapes the oracle finishes quickly, and the full one
    "convdiff27_48_schur_p8": ("convdiff27", 48, 8, "schur", "ilut:0.001,20"),
    "convdiff27_48_schur_p1": ("convdiff27", 48, 1, "schur", "ilut:0.001,20"),
    "convdiff27_96_schur_p8": ("convdiff27", 96, 8, "schur", "ilut:0.001,20"),
    "convdiff27_192_schur_p8": ("convdiff27", 192, 8, "schur", "ilut:0.001,20"),
}


def build(kind, n):
    dims = (n, n, n)
    if kind == "aniso3d":
        return orc.aniso(dims, EPS), dims
    if kind == "convdiff27":
        return orc.convdiff27(n, n, n, (10.0, 10.0, 10.0)), dims
    raise ValueError(kind)


def run_case(name):
    kind, n, p, precond, fill = CASES[name]
    a, dims = build(kind, n)
    t0 = time.perf_counter()
    rec, rep, x = orc.run(a, dims, p, precond, orc.Rule.parse(fill))
    wall = time.perf_counter() - t0
    err = float(np.max(np.abs(x - 1.0)))          # b = A*1: the exact solution is the ones vector
    return {
        "kind": kind, "dims": list(dims), "p": p, "precond": precond, "fill": fill,
        "param": list(EPS) if kind == "aniso3d" else [10.0, 10.0, 10.0],
        "its": int(rep.iterations), "converged": bool(rep.converged), "final_relres": float(rep.final_relres),
        "final_relres_hex": float(rep.final_relres).hex(),
        "history_hex": [float(v).hex() for v in rep.residual_history],
        "max_abs_error_vs_ones": err,
        "setup_s": float(rec["setup_s"]), "solve_s": float(rec["solve_s"]), "wall_s": wall,
        "host": {"cpu": platform.processor() or platform.machine(), "cores_used": 1, "cores": os.cpu_count()},
        "source": "oracle/ddilu_oracle (C port of the reference, -O2 -ffp-contract=off), restart 50, rtol 1e-8, "
                  "inner_iters 3, b = A*1",
    }


def main():
    orc.build()
    names = sys.argv[1:] or list(CASES)
    for name in names:
        rec = run_case(name)
        with open(OUT + ".lock", "w") as lock:          # several cases may run side by side
            fcntl.flock(lock, fcntl.LOCK_EX)
            data = {}
            if os.path.exists(OUT):
                with open(OUT) as fh:
                    data = json.load(fh)
            data[name] = rec
            with open(OUT + ".tmp", "w") as fh:
                json.dump(data, fh, indent=1, sort_keys=True)
            os.replace(OUT + ".tmp", OUT)
        print(name, rec["its"], rec["final_relres"], f"setup {rec['setup_s']:.1f}s solve {rec['solve_s']:.1f}s", flush=True)


if __name__ == "__main__":
    main()
