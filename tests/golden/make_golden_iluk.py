"""Golden fixtures for the level-of-fill factorisation (iluk), written by the UNMODIFIED reference.

Run in the build container only (the GPU box has no /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_iluk.py

Writes tests/golden/iluk.npz: for each small matrix the reference's iluk(level) factors, its
partial_ilu with an iluk rule (blocks + Schur factors), and the iteration counts of schur / bj
preconditioned FGMRES with iluk:1 on box partitions.  Matrices are stored with the results.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import ddilu  # noqa: E402
from ddilu import factor as rfac  # noqa: E402
from ddilu import problems as rprob  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = {}


def put(key, val):
    assert key not in OUT, key
    OUT[key] = np.asarray(val)


def put_csr(key, m):
    put(key + ".shape", np.array([m.n_rows, m.n_cols], dtype=np.int64))
    put(key + ".row_ptr", m.row_ptr)
    put(key + ".col_idx", m.col_idx)
    put(key + ".values", m.values)


def aniso(dims, eps):
    return rprob._stencil_csr(dims, [(-float(e), -float(e)) for e in eps], 2.0 * float(sum(eps)))


def random_sparse(n, density, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    mask[3, 3] = False            # one structurally missing diagonal
    rows, cols = np.nonzero(mask)
    vals = rng.standard_normal(len(rows))
    vals[rows == cols] += 4.0
    return ddilu.csr_from_coo(n, n, rows, cols, vals)


def main():
    mats = {
        "poisson2d_9x7": ddilu.poisson2d(9, 7),
        "aniso3d_6x5x4": aniso((6, 5, 4), (1.0, 1.0, 0.01)),
        "convdiff3d_5": ddilu.convdiff3d(5, 5, 5, (3.0, -2.0, 1.0)),
        "random_40": random_sparse(40, 0.08, 11),
    }
    put("names", np.array(sorted(mats)))
    for name, a in sorted(mats.items()):
        put_csr(f"{name}.a", a)
        for level in (1, 2, 3):
            f = ddilu.iluk(a, level)
            put_csr(f"{name}.k{level}.lower", f.lower)
            put_csr(f"{name}.k{level}.upper", f.upper)
        n1 = (2 * a.n_rows) // 3
        for level in (1, 2):
            pf = ddilu.partial_ilu(a, n1, ddilu.FillRule("iluk", level=level))
            key = f"{name}.partial{level}"
            put(key + ".n1", n1)
            put_csr(key + ".l_b", pf.interior.lower)
            put_csr(key + ".u_b", pf.interior.upper)
            put_csr(key + ".w", pf.w_block)
            put_csr(key + ".z", pf.z_block)
            put_csr(key + ".s_tilde", pf.s_tilde)
            put_csr(key + ".schur_l", pf.schur.lower)
            put_csr(key + ".schur_u", pf.schur.upper)
    # pipeline: iteration counts with an iluk rule
    dims = (12, 12, 12)
    a = aniso(dims, (1.0, 1.0, 0.01))
    b = ddilu.default_rhs(a)
    put_csr("pipe.a", a)
    put("pipe.dims", np.array(dims))
    for pc in ("bj", "schur"):
        for p in (1, 8):
            layout = ddilu.classify_and_order(a, ddilu.partition(a, p, dims), p)
            m = ddilu.make_preconditioner(pc, a, layout, ddilu.FillRule("iluk", level=1))
            x, rep = ddilu.fgmres(a, b, m=m.apply)
            put(f"pipe.{pc}.p{p}.its", rep.iterations)
            put(f"pipe.{pc}.p{p}.x", x)
            put(f"pipe.{pc}.p{p}.apply", m.apply(b))
    np.savez_compressed(os.path.join(HERE, "iluk.npz"), **OUT)
    print("wrote", len(OUT), "arrays")


if __name__ == "__main__":
    main()
