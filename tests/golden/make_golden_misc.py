"""Golden fixtures for `sparse_matmul`, written by the UNMODIFIED reference.

Run in the build container only (the GPU box has no /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_misc.py

Writes tests/golden/misc.npz: operand pairs (random rectangular, a stencil squared, a pair whose products
cancel exactly) with the reference's product (pattern and values).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from ddilu import problems as rprob  # noqa: E402
from ddilu import sparse as rsp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = {}


def put_csr(key, m):
    OUT[key + ".shape"] = np.array([m.n_rows, m.n_cols], dtype=np.int64)
    OUT[key + ".row_ptr"] = np.asarray(m.row_ptr)
    OUT[key + ".col_idx"] = np.asarray(m.col_idx)
    OUT[key + ".values"] = np.asarray(m.values)


def random_csr(rng, m, n, density):
    d = rng.standard_normal((m, n))
    d[rng.random((m, n)) > density] = 0.0
    return rsp.csr_from_dense(d)


def main():
    rng = np.random.default_rng(20231)
    cases = {
        "rect": (random_csr(rng, 23, 17, 0.3), random_csr(rng, 17, 31, 0.25)),
        "dense_rows": (random_csr(rng, 9, 40, 0.9), random_csr(rng, 40, 12, 0.8)),
        "stencil2": (rprob.poisson3d(5, 4, 3), rprob.poisson3d(5, 4, 3)),
        "cancel": (rsp.csr_from_dense(np.array([[1.0, 1.0], [1.0, 1.0]])),
                   rsp.csr_from_dense(np.array([[1.0, 1.0], [-1.0, -1.0]]))),
        "empty_b": (random_csr(rng, 4, 3, 0.7), rsp.csr_from_coo(3, 5, np.array([], dtype=np.int64),
                                                                np.array([], dtype=np.int64), np.array([]))),
    }
    OUT["spgemm.names"] = np.array(sorted(cases))
    for name, (a, b) in cases.items():
        put_csr(f"spgemm.{name}.a", a)
        put_csr(f"spgemm.{name}.b", b)
        put_csr(f"spgemm.{name}.c", rsp.sparse_matmul(a, b))
    np.savez_compressed(os.path.join(HERE, "misc.npz"), **OUT)
    print("wrote misc.npz:", len(OUT), "arrays")


if __name__ == "__main__":
    main()
