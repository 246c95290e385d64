"""The oracle's level-of-fill factorisation (iluk symbolic + prefill + numeric on the pattern)
against fixtures written by the unmodified reference (tests/golden/make_golden_iluk.py):
patterns and values bit for bit, iteration counts of iluk-preconditioned FGMRES."""

import os

import numpy as np
import pytest

from oracle import ddilu_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(HERE, "golden", "iluk.npz"))


def csr(g, key):
    nr, nc = (int(v) for v in g[key + ".shape"])
    return orc.Csr(nr, nc, g[key + ".row_ptr"].copy(), g[key + ".col_idx"].copy(), g[key + ".values"].copy())


def same(m, g, key):
    return (np.array_equal(m.row_ptr, g[key + ".row_ptr"]) and np.array_equal(m.col_idx, g[key + ".col_idx"])
            and np.array_equal(m.values, g[key + ".values"]))


def test_iluk_factors_bit_exact(g):
    for name in g["names"]:
        a = csr(g, f"{name}.a")
        for level in (1, 2, 3):
            f = orc.iluk(a, level)
            assert same(f.lower, g, f"{name}.k{level}.lower"), (name, level)
            assert same(f.upper, g, f"{name}.k{level}.upper"), (name, level)


def test_iluk_partial_bit_exact(g):
    for name in g["names"]:
        a = csr(g, f"{name}.a")
        for level in (1, 2):
            key = f"{name}.partial{level}"
            pf = orc.partial_ilu(a, int(g[key + ".n1"]), orc.Rule("iluk", level=level))
            assert same(pf.interior.lower, g, key + ".l_b") and same(pf.interior.upper, g, key + ".u_b"), key
            assert same(pf.w_block, g, key + ".w") and same(pf.z_block, g, key + ".z"), key
            assert same(pf.s_tilde, g, key + ".s_tilde"), key
            assert same(pf.schur.lower, g, key + ".schur_l") and same(pf.schur.upper, g, key + ".schur_u"), key


def test_iluk_level0_is_ilu0(g):
    a = csr(g, "poisson2d_9x7.a")
    f0, f = orc.ilu0(a), orc.iluk(a, 0)
    assert np.array_equal(f0.lower.values, f.lower.values) and np.array_equal(f0.upper.values, f.upper.values)


def test_iluk_pipeline_iterations(g):
    a = csr(g, "pipe.a")
    dims = tuple(int(v) for v in g["pipe.dims"])
    b = orc.default_rhs(a)
    for pc in ("bj", "schur"):
        for p in (1, 8):
            layout = orc.classify_and_order(a, orc.partition(a, p, dims), p)
            m = orc.make_preconditioner(pc, a, layout, orc.Rule("iluk", level=1))
            assert np.array_equal(m.apply(b), g[f"pipe.{pc}.p{p}.apply"]), (pc, p)
            x, rep = orc.fgmres(a, b, m=m.apply)
            assert rep.iterations == int(g[f"pipe.{pc}.p{p}.its"]), (pc, p)
            assert np.array_equal(x, g[f"pipe.{pc}.p{p}.x"]), (pc, p)
