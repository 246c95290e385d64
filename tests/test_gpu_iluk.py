"""GPU parity of the level-of-fill factorisation: patterns and values of iluk / partial_ilu with an
iluk rule bit for bit against fixtures written by the unmodified reference
(tests/golden/make_golden_iluk.py), and the iteration counts of iluk-preconditioned FGMRES."""

import os

import numpy as np
import pytest

from _golden import same_csr

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(HERE, "golden", "iluk.npz"))


def csr(P, g, key):
    nr, nc = (int(v) for v in g[key + ".shape"])
    return P.CsrMatrix(nr, nc, g[key + ".row_ptr"].copy(), g[key + ".col_idx"].copy(), g[key + ".values"].copy())


def test_iluk_factors_bit_exact(P, g):
    for name in g["names"]:
        a = csr(P, g, f"{name}.a")
        for level in (1, 2, 3):
            f = P.iluk(a, level)
            assert f.kind == f"iluk:{level}"
            same_csr(f.lower, g, f"{name}.k{level}.lower")
            same_csr(f.upper, g, f"{name}.k{level}.upper")
        assert np.array_equal(P.iluk(a, 0).upper.values, P.ilu0(a).upper.values)
    with pytest.raises(ValueError):
        P.iluk(csr(P, g, "poisson2d_9x7.a"), -1)


def test_iluk_partial_bit_exact(P, g):
    for name in g["names"]:
        a = csr(P, g, f"{name}.a")
        for level in (1, 2):
            key = f"{name}.partial{level}"
            pf = P.partial_ilu(a, int(g[key + ".n1"]), P.FillRule("iluk", level=level))
            same_csr(pf.interior.lower, g, key + ".l_b")
            same_csr(pf.interior.upper, g, key + ".u_b")
            same_csr(pf.w_block, g, key + ".w")
            same_csr(pf.z_block, g, key + ".z")
            same_csr(pf.s_tilde, g, key + ".s_tilde")
            same_csr(pf.schur.lower, g, key + ".schur_l")
            same_csr(pf.schur.upper, g, key + ".schur_u")


def test_iluk_small_row_cap_retries(P, g):
    """A working row that outgrows the slab capacity makes the driver retry with a larger one."""
    from paper_2303_08881_b200 import _iluk
    a = csr(P, g, "random_40.a")
    old = _iluk.MIN_ROW_CAP
    _iluk.MIN_ROW_CAP = 4          # forces the first attempts to overflow
    try:
        f = P.iluk(a, 2)
    finally:
        _iluk.MIN_ROW_CAP = old
    same_csr(f.lower, g, "random_40.k2.lower")
    same_csr(f.upper, g, "random_40.k2.upper")


def test_iluk_pipeline(P, g):
    a = csr(P, g, "pipe.a")
    dims = tuple(int(v) for v in g["pipe.dims"])
    b = P.default_rhs(a)
    for pc in ("bj", "schur"):
        for p in (1, 8):
            layout = P.classify_and_order(a, P.partition(a, p, dims), p)
            m = P.make_preconditioner(pc, a, layout, P.FillRule("iluk", level=1))
            z = m.apply(b)
            ref = g[f"pipe.{pc}.p{p}.apply"]
            if pc == "bj":
                assert np.array_equal(z, ref), (pc, p)
            else:
                assert np.allclose(z, ref, rtol=1e-9, atol=1e-12), (pc, p)
            x, rep = P.fgmres(a, b, m=m.apply)
            assert abs(rep.iterations - int(g[f"pipe.{pc}.p{p}.its"])) <= 1, (pc, p, rep.iterations)
            assert rep.converged and np.max(np.abs(x - g[f"pipe.{pc}.p{p}.x"])) < 1e-6
