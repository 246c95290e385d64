"""The properties the reference's own test-suite states for this path, asked of the CUDA implementation through
the public API (pkg/tests/test_krylov.py, test_precond.py, test_acceptance.py:46-230): dense numpy algebra is the
judge, tiny unstructured matrices drive the general (untiled) kernels, the block sweep on blocks of one or two
rows, empty interfaces and the reference's early exits.  Tolerances are the reference's."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 20240817


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)


# ---------------------------------------------------------------------------
# dense judges and generators (plain numpy, nothing of the package's kernels)


def lu_without_pivoting(a):
    u = np.array(a, dtype=np.float64)
    n = len(u)
    lo = np.eye(n)
    for k in range(n - 1):
        lo[k + 1:, k] = u[k + 1:, k] / u[k, k]
        u[k + 1:, k:] -= np.outer(lo[k + 1:, k], u[k, k:])
        u[k + 1:, k] = 0.0
    return lo, u


def schur_complement(a, n1):
    return a[n1:, n1:] - a[n1:, :n1] @ np.linalg.solve(a[:n1, :n1], a[:n1, n1:])


def spd(rng, n):
    g = rng.standard_normal((n, n))
    return g @ g.T + n * np.eye(n)


def symmetric_pattern_matrix(P, rng, n):
    """Random values on a symmetric pattern with a dominant diagonal (no pivot comes near zero)."""
    d = np.zeros((n, n))
    i, j = rng.integers(0, n, 2 * n), rng.integers(0, n, 2 * n)
    keep = i != j
    d[i[keep], j[keep]] = rng.standard_normal(int(keep.sum()))
    hole = ((d != 0) | (d.T != 0)) & (d == 0)
    d[hole] = rng.standard_normal(int(hole.sum()))
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, np.abs(d).sum(axis=1) + rng.uniform(1.0, 2.0, n))
    return P.csr_from_dense(d)


def chain(P, n):
    d = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    return P.csr_from_dense(d)


def torus_laplacian(P, nx, ny):
    n = nx * ny
    d = np.zeros((n, n))
    for y in range(ny):
        for x in range(nx):
            i = x + nx * y
            d[i, i] = 4.0
            for xx, yy in (((x + 1) % nx, y), ((x - 1) % nx, y), (x, (y + 1) % ny), (x, (y - 1) % ny)):
                d[i, xx + nx * yy] += -1.0
    return P.csr_from_dense(d)


def dense_blocks(P, rng, sizes, bridges):
    """Dense diagonal blocks (level-0 factorisation of a block is exact) joined by a few symmetric couplings."""
    n = sum(sizes)
    d = np.zeros((n, n))
    s = 0
    for k in sizes:
        blk = rng.uniform(-1.0, 1.0, (k, k))
        d[s:s + k, s:s + k] = blk + blk.T
        s += k
    for i, j in bridges:
        d[i, j] = d[j, i] = -rng.uniform(0.2, 1.0)
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, np.abs(d).sum(axis=1) + rng.uniform(1.0, 2.0, n))
    return P.csr_from_dense(d), np.repeat(np.arange(len(sizes)), sizes)


def layout_of(P, a, owner):
    return P.classify_and_order(a, np.asarray(owner, dtype=np.int64))


def one_domain(P, a):
    return layout_of(P, a, np.zeros(a.n_rows, dtype=np.int64))


def rhs_of_ones(P, a):
    return P.spmv(a, np.ones(a.n_cols))


# ---------------------------------------------------------------------------
# restarted GMRES / FGMRES (pkg/tests/test_krylov.py:12-153)


def test_krylov_config(P):
    cfg = P.KrylovConfig()
    assert (cfg.restart, cfg.rtol, cfg.max_iters, cfg.record_history) == (50, 1e-8, 20000, True)
    for bad in ({"restart": 0}, {"rtol": 0.0}, {"rtol": -1e-8}, {"max_iters": 0}):
        with pytest.raises(ValueError):
            P.KrylovConfig(**bad)


def test_gmres_small_and_degenerate_cases(P, rng):
    b = np.array([1.0, -2.0, 3.0])
    x, rep = P.gmres(P.csr_identity(3), b)
    assert rep.iterations == 1 and rep.converged and np.max(np.abs(x - b)) < 1e-14
    d = spd(rng, 2)
    b2 = rng.standard_normal(2)
    x, rep = P.gmres(P.csr_from_dense(d), b2, cfg=P.KrylovConfig(rtol=1e-12))
    assert rep.iterations <= 2 and np.max(np.abs(d @ x - b2)) < 1e-10 * np.max(np.abs(b2))
    a = P.poisson2d(4, 4)
    ones = np.ones(16)
    x, rep = P.gmres(a, P.spmv(a, ones), x0=ones)           # exact initial guess: no iteration, x returned as is
    assert rep.iterations == 0 and rep.converged and np.array_equal(x, ones)
    for solver in (P.gmres, P.fgmres):
        x, rep = solver(P.poisson2d(3, 3), np.zeros(9))     # zero right-hand side
        assert rep.iterations == 0 and rep.converged and np.array_equal(x, np.zeros(9))
    a = P.poisson2d(16, 16)
    x, rep = P.gmres(a, rhs_of_ones(P, a), cfg=P.KrylovConfig(max_iters=5))
    assert not rep.converged and rep.iterations == 5        # reported, never raised


def test_gmres_with_ilu0_and_operator_forms(P):
    a = P.poisson2d(16, 16)
    b = rhs_of_ones(P, a)
    f = P.ilu0(a)
    x, rep = P.gmres(a, b, m=f.solve)
    assert rep.converged and rep.iterations <= 40
    assert P.vnorm2(b - P.spmv(a, x)) <= 1e-8 * P.vnorm2(b) * 1.01
    xf, rf = P.fgmres(a, b, m=f.solve)                      # fixed preconditioner: FGMRES = GMRES
    assert rf.iterations == rep.iterations
    assert np.max(np.abs(xf - x)) <= 1e-12 * max(np.max(np.abs(x)), 1.0)
    a6 = P.poisson2d(6, 6)
    b6 = rhs_of_ones(P, a6)
    x1, r1 = P.gmres(a6, b6)
    x2, r2 = P.gmres(lambda v: P.spmv(a6, v), b6)           # any callable is an operator
    assert r1.iterations == r2.iterations and np.array_equal(x1, x2)


def test_gmres_history_and_reported_residual(P):
    a = P.poisson2d(20, 20)
    b = rhs_of_ones(P, a)
    m = 30
    x, rep = P.gmres(a, b, cfg=P.KrylovConfig(restart=m))
    h = rep.residual_history
    assert rep.converged and len(h) == rep.iterations + 1
    for i in range(2, len(h)):
        if (i - 1) % m:                                      # inside a cycle the estimate never grows
            assert h[i] <= h[i - 1] * (1.0 + 1e-12)
    fresh = P.vnorm2(b - P.spmv(a, x)) / P.vnorm2(b)
    assert abs(rep.final_relres - fresh) <= 1e-10           # test_acceptance.py:198-210
    a8 = P.poisson2d(8, 8)
    x, rep = P.gmres(a8, rhs_of_ones(P, a8), cfg=P.KrylovConfig(record_history=False))
    assert len(rep.residual_history) == 0 and rep.iterations > 0 and rep.converged
    a12 = P.poisson2d(12, 12)
    b12 = rhs_of_ones(P, a12)
    (x1, r1), (x2, r2) = P.gmres(a12, b12), P.gmres(a12, b12)
    assert np.array_equal(x1, x2) and r1.iterations == r2.iterations and r1.final_relres == r2.final_relres


def test_final_relres_is_the_recomputed_residual(P):
    """krylov.py:168-172: convergence is declared on the recomputed true residual; the reported number is that
    residual (device reductions: equal to the public vnorm2 / spmv composition to rounding)."""
    a = P.poisson2d(10, 10)
    b = rhs_of_ones(P, a)
    for x, rep in (P.gmres(a, b), P.fgmres(a, b, m=P.ilu0(a).solve)):
        fresh = P.vnorm2(b - P.spmv(a, x)) / P.vnorm2(b)
        assert abs(rep.final_relres - fresh) <= 1e-13 * max(fresh, 1e-300) + 1e-22


def test_fgmres_with_exact_preconditioner(P, rng):
    d = spd(rng, 12)
    inv = np.linalg.inv(d)
    x, rep = P.fgmres(P.csr_from_dense(d), rng.standard_normal(12), m=lambda v: inv @ v)
    assert rep.iterations == 1 and rep.converged


# ---------------------------------------------------------------------------
# fixed-iteration inner GMRES (pkg/tests/test_krylov.py:156-200): also the device-side arithmetic's early exits


def test_fixed_gmres_properties(P, rng):
    d = spd(rng, 10)
    a = P.csr_from_dense(d)
    b = rng.standard_normal(10)
    x = P.fixed_gmres(lambda v: P.spmv(a, v), b, 10)         # the full space is a direct solve
    assert np.max(np.abs(d @ x - b)) <= 1e-10 * np.max(np.abs(b))
    assert np.array_equal(P.fixed_gmres(lambda v: v, np.ones(4), 0), np.zeros(4))
    assert np.array_equal(P.fixed_gmres(lambda v: v, np.zeros(4), 3), np.zeros(4))
    assert P.fixed_gmres(lambda v: v, np.zeros(0), 3).shape == (0,)
    d8 = spd(rng, 8)
    a8 = P.csr_from_dense(d8)
    b8 = rng.standard_normal(8)
    inv = np.linalg.inv(d8)
    x = P.fixed_gmres(lambda v: P.spmv(a8, v), b8, 5, apply_m=lambda v: inv @ v)   # breakdown after one step
    assert np.all(np.isfinite(x)) and np.max(np.abs(d8 @ x - b8)) <= 1e-10 * np.max(np.abs(b8))
    d20 = spd(rng, 20)
    a20 = P.csr_from_dense(d20)
    b20 = rng.standard_normal(20)
    r2 = np.linalg.norm(d20 @ P.fixed_gmres(lambda v: P.spmv(a20, v), b20, 2) - b20)
    r20 = np.linalg.norm(d20 @ P.fixed_gmres(lambda v: P.spmv(a20, v), b20, 20) - b20)
    assert r20 < r2
    g = P.poisson2d(8, 8)
    bb = rng.standard_normal(64)
    assert np.array_equal(P.fixed_gmres(lambda v: P.spmv(g, v), bb, 7), P.fixed_gmres(lambda v: P.spmv(g, v), bb.copy(), 7))


# ---------------------------------------------------------------------------
# factorisation identities (pkg/tests/test_acceptance.py:46-102)


def test_ilu0_residual_vanishes_on_the_pattern(P, rng):
    worst = 0.0
    for _ in range(40):
        n = int(rng.integers(5, 31))
        a = symmetric_pattern_matrix(P, rng, n)
        d = a.to_dense()
        f = P.ilu0(a)
        resid = d - (f.lower.to_dense() + np.eye(n)) @ f.upper.to_dense()
        worst = max(worst, np.max(np.abs(resid[d != 0.0])) / np.max(np.abs(d)))
    assert worst <= 1e-12


def test_tridiagonal_factors_are_the_dense_lu(P):
    a = chain(P, 12)
    lo_ref, up_ref = lu_without_pivoting(a.to_dense())
    for f in (P.ilu0(a), P.milu0(a), P.ilut(a, 0.0, 2)):
        assert np.max(np.abs(f.lower.to_dense() + np.eye(12) - lo_ref)) <= 1e-12
        assert np.max(np.abs(f.upper.to_dense() - up_ref)) <= 1e-12


def test_milu_hits_its_target_vectors(P, rng):
    worst = 0.0
    for _ in range(40):
        n = int(rng.integers(4, 25))
        a = symmetric_pattern_matrix(P, rng, n)
        y = rng.uniform(0.5, 2.0, n) * rng.choice([-1.0, 1.0], n)
        w = rng.standard_normal(n)
        f = P.milu0(a, P.MiluVectors(y=y, z=np.empty(0), w=w))
        want = P.spmv(a, y) - w
        worst = max(worst, np.max(np.abs(f.lu_matvec(y) - want)) / max(np.max(np.abs(want)), 1.0))
    assert worst <= 1e-11


def test_partial_factorisation_without_dropping_gives_the_schur_complement(P, rng):
    worst = 0.0
    for _ in range(25):
        n = int(rng.integers(6, 41))
        d = spd(rng, n)
        ni = int(rng.integers(1, n))
        pf = P.partial_ilu(P.csr_from_dense(d), ni, P.FillRule("ilut", tau=0.0, maxfill=n))
        worst = max(worst, np.max(np.abs(pf.s_tilde.to_dense() - schur_complement(d, ni))) / np.max(np.abs(d)))
    assert worst <= 1e-11


# ---------------------------------------------------------------------------
# block Jacobi (pkg/tests/test_precond.py:48-105)


def test_block_jacobi_properties(P, rng):
    a = P.poisson2d(5, 5)
    r = rng.standard_normal(25)
    assert np.array_equal(P.bj_setup(a, one_domain(P, a), use_rcm=False).apply(r), P.ilu0(a).solve(r))
    diag = np.array([2.0, 3.0, 4.0, 5.0])
    m = P.bj_setup(P.csr_from_dense(np.diag(diag)), layout_of(P, P.csr_from_dense(np.diag(diag)), [0, 0, 1, 1]))
    rr = np.array([2.0, 6.0, 8.0, 15.0])
    assert np.array_equal(m.apply(rr), rr / diag)
    a6 = P.poisson2d(6, 6)
    lay = layout_of(P, a6, P.partition(a6, 4, grid_hint=(6, 6)))
    m = P.bj_setup(a6, lay)
    r1, r2 = rng.standard_normal(36), rng.standard_normal(36)
    lhs, rhs = m.apply(2.0 * r1 - 0.5 * r2), 2.0 * m.apply(r1) - 0.5 * m.apply(r2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(np.max(np.abs(rhs)), 1.0)
    assert np.array_equal(m.apply(np.zeros(36)), np.zeros(36))
    m = P.bj_setup(a6, layout_of(P, a6, P.partition(a6, 2, grid_hint=(6, 6))), rule=P.FillRule("iluk", level=1))
    assert all(f.kind == "iluk:1" for f in m.factors)


def test_l1_block_jacobi(P, rng):
    a = chain(P, 6)
    m = P.bj_setup(a, layout_of(P, a, [0, 0, 0, 1, 1, 1]), rule=P.FillRule("ilut", tau=0.0, maxfill=6), l1=True,
                   use_rcm=False)
    r = rng.standard_normal(6)
    b0 = np.array([[2.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 3.0]])   # the cut edge lands on the diagonal
    b1 = np.array([[3.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 2.0]])
    want = np.concatenate([np.linalg.solve(b0, r[:3]), np.linalg.solve(b1, r[3:])])
    assert np.max(np.abs(m.apply(r) - want)) < 1e-12
    g = P.poisson2d(4, 4)
    rr = rng.standard_normal(16)
    assert np.array_equal(P.bj_setup(g, one_domain(P, g)).apply(rr), P.bj_setup(g, one_domain(P, g), l1=True).apply(rr))


# ---------------------------------------------------------------------------
# two-level Schur preconditioner (pkg/tests/test_precond.py:107-196)


def test_schur_reduces_to_block_jacobi_and_to_the_identity(P, rng):
    a = P.poisson2d(5, 5)
    r = rng.standard_normal(25)
    lay = one_domain(P, a)
    assert np.array_equal(P.schur_setup(a, lay).apply(r), P.bj_setup(a, lay).apply(r))
    # two tridiagonal blocks joined by an explicitly STORED zero: the pattern couples them, the values do not
    rows = [0, 0, 1, 1, 1, 2, 2, 3, 3, 4, 4, 4, 5, 5, 2, 3]
    cols = [0, 1, 0, 1, 2, 1, 2, 3, 4, 3, 4, 5, 4, 5, 3, 2]
    vals = [2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0, 2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0, 0.0, 0.0]
    z = P.csr_from_coo(6, 6, np.array(rows), np.array(cols), np.array(vals))
    lay = layout_of(P, z, [0, 0, 0, 1, 1, 1])
    assert lay.n_exterior == 2
    m = P.schur_setup(z, lay)
    y = rng.standard_normal(2)
    assert np.array_equal(m.reduced_matvec(y), y) and np.array_equal(P.schur_matvec(m, y), y)
    a6 = P.poisson2d(6, 6)
    lay = layout_of(P, a6, P.partition(a6, 2, grid_hint=(6, 6)))
    m = P.schur_setup(a6, lay)
    assert np.array_equal(m.reduced_matvec(np.zeros(lay.n_exterior)), np.zeros(lay.n_exterior))
    assert np.array_equal(m.apply(np.zeros(36)), np.zeros(36))


def test_schur_apply_is_the_dense_two_level_solve(P, rng):
    """precond.py:221-267 written out with dense algebra: exact block factors, 2 interface unknowns, 2 inner steps
    (= the whole interface space)."""
    a, owner = dense_blocks(P, rng, [3, 3], [(2, 3)])
    lay = layout_of(P, a, owner)
    m = P.schur_setup(a, lay, inner_iters=2, use_rcm=False)
    r = rng.standard_normal(6)
    d = a.to_dense()
    ints, exts = [lay.interior_of[0], lay.interior_of[1]], [2, 3]
    s_glob, ghat = np.zeros((2, 2)), np.zeros(2)
    for k in range(2):
        b = d[np.ix_(ints[k], ints[k])]
        e = d[np.ix_([exts[k]], ints[k])]
        f = d[np.ix_(ints[k], [exts[k]])]
        s_glob[k, k] = d[exts[k], exts[k]] - (e @ np.linalg.solve(b, f))[0, 0]
        ghat[k] = r[exts[k]] - (e @ np.linalg.solve(b, r[ints[k]]))[0]
    s_glob[0, 1], s_glob[1, 0] = d[2, 3], d[3, 2]
    y = np.linalg.solve(s_glob, ghat)
    want = np.empty(6)
    for k in range(2):
        b = d[np.ix_(ints[k], ints[k])]
        want[ints[k]] = np.linalg.solve(b, r[ints[k]] - d[np.ix_(ints[k], [exts[k]])][:, 0] * y[k])
        want[exts[k]] = y[k]
    assert np.max(np.abs(m.apply(r) - want)) <= 1e-11 * max(np.max(np.abs(want)), 1.0)


def test_schur_with_exact_factors_inverts_the_matrix(P, rng):
    a, owner = dense_blocks(P, rng, [4, 4, 4], [(3, 4), (7, 8)])
    lay = layout_of(P, a, owner)
    m = P.schur_setup(a, lay, rule=P.FillRule("ilut", tau=0.0, maxfill=12), inner_iters=lay.n_exterior)
    r = rng.standard_normal(12)
    want = np.linalg.solve(a.to_dense(), r)
    assert np.max(np.abs(m.apply(r) - want)) <= 1e-10 * max(np.max(np.abs(want)), 1.0)


def test_schur_options_reach_the_factors(P, rng):
    a = P.poisson2d(10, 10)
    lay = layout_of(P, a, P.partition(a, 4, grid_hint=(10, 10)))
    full = P.schur_setup(a, lay, rule=P.FillRule("iluk", level=2))
    thin = P.schur_setup(a, lay, rule=P.FillRule("iluk", level=2), schur_drop_tol=0.3)
    assert sum(pf.s_tilde.nnz for pf in thin.partial) < sum(pf.s_tilde.nnz for pf in full.partial)
    a16 = P.poisson2d(16, 16)
    lay = layout_of(P, a16, P.partition(a16, 4, grid_hint=(16, 16)))
    r = rng.standard_normal(256)
    assert not np.array_equal(P.schur_setup(a16, lay, inner_iters=1).apply(r), P.schur_setup(a16, lay, inner_iters=3).apply(r))


# ---------------------------------------------------------------------------
# interface coarse correction (pkg/tests/test_precond.py:197-330, test_acceptance.py:105-196)


def test_rap_single_domain_and_zero(P, rng):
    a = P.poisson2d(5, 5)
    lay = one_domain(P, a)
    r = rng.standard_normal(25)
    base = P.bj_setup(a, lay).apply(r)
    for modified in (False, True):
        assert np.array_equal(P.rap_setup(a, lay, modified=modified).apply(r), base)
    a6 = P.poisson2d(6, 6)
    lay = layout_of(P, a6, P.partition(a6, 4, grid_hint=(6, 6)))
    for modified in (False, True):
        assert np.array_equal(P.rap_setup(a6, lay, modified=modified).apply(np.zeros(36)), np.zeros(36))


def test_rap_detached_interface_is_the_exterior_block(P, rng):
    rows = [0, 0, 1, 1, 4, 4, 5, 5, 2, 2, 3, 3]
    cols = [0, 1, 0, 1, 4, 5, 4, 5, 2, 3, 2, 3]
    vals = [2.0, -1.0, -1.0, 2.0, 2.0, -1.0, -1.0, 2.0, 2.0, -1.0, -1.0, 2.0]
    a = P.csr_from_coo(6, 6, np.array(rows), np.array(cols), np.array(vals))
    lay = layout_of(P, a, [0, 0, 0, 1, 1, 1])
    assert lay.n_exterior == 2
    m = P.rap_setup(a, lay, modified=False)
    ext = np.arange(4, 6)
    v = rng.standard_normal(2)
    assert np.array_equal(P.rap_matvec(m, v), P.spmv(P.take_submatrix(m.a_perm, ext, ext), v))


def test_rap_coarse_operator_is_the_dense_schur_complement(P, rng):
    for _ in range(4):
        a, owner = dense_blocks(P, rng, [4, 4, 4], [(3, 4), (7, 8)])
        lay = layout_of(P, a, owner)
        m = P.rap_setup(a, lay, modified=False)
        s = schur_complement(m.a_perm.to_dense(), lay.n_interior)
        v = rng.standard_normal(lay.n_exterior)
        assert np.max(np.abs(P.rap_matvec(m, v) - s @ v)) <= 1e-10 * np.max(np.abs(s)) * np.max(np.abs(v))
    # the additive (Schur) and the multiplicative (R A P) interface operators are the same matrix without dropping
    a, owner = dense_blocks(P, rng, [4, 4, 4], [(3, 4), (7, 8)])
    lay = layout_of(P, a, owner)
    sc = P.schur_setup(a, lay, rule=P.FillRule("ilut", tau=0.0, maxfill=12))
    ra = P.rap_setup(a, lay, modified=False)
    ne, st = lay.n_exterior, lay.exterior_starts
    s_add = np.zeros((ne, ne))
    for k, pf in enumerate(sc.partial):
        s_add[st[k]:st[k + 1], st[k]:st[k + 1]] = pf.s_tilde.to_dense()
    s_add += sc.coupling.to_dense()
    for _ in range(3):
        y = rng.standard_normal(ne)
        assert np.max(np.abs(s_add @ y - P.rap_matvec(ra, y))) <= 1e-10 * np.max(np.abs(s_add)) * np.max(np.abs(y))


def test_rap_disconnected_domains_are_solved_exactly(P, rng):
    d = np.zeros((8, 8))
    d[:4, :4] = chain(P, 4).to_dense() + np.eye(4)
    d[4:, 4:] = chain(P, 4).to_dense() + np.eye(4)
    a = P.csr_from_dense(d)
    lay = layout_of(P, a, [0, 0, 0, 0, 1, 1, 1, 1])
    assert lay.n_exterior == 0
    r = rng.standard_normal(8)
    want = np.linalg.solve(d, r)
    assert np.max(np.abs(P.rap_setup(a, lay).apply(r) - want)) <= 1e-12 * np.max(np.abs(want))


def _coarse_row_sum_gap(P, m, a):
    """test_precond.py:254-294: R_d A_d P_d 1 against (L_S U_S) 1, per domain."""
    worst = 0.0
    for dom, blk in zip(m.domains, m.blocks):
        local = P.take_submatrix(a, dom.nodes, dom.nodes)
        n1 = len(dom.interior_nodes)
        ones = np.ones(len(dom.nodes) - n1)
        pv = np.concatenate([-np.linalg.solve(blk.interior.upper.to_dense(), P.spmv(blk.z_tilde, ones)), ones])
        t = P.spmv(local, pv)
        lo = blk.interior.lower.to_dense() + np.eye(n1)
        rt = t[n1:] - P.spmv(blk.w_tilde, np.linalg.solve(lo, t[:n1]))
        worst = max(worst, np.max(np.abs(rt - blk.schur.lu_matvec(ones))))
    return worst


def test_modified_coarse_factors_preserve_constants(P):
    a = torus_laplacian(P, 16, 16)
    lay = layout_of(P, a, P.partition(a, 4, grid_hint=(16, 16)))
    assert _coarse_row_sum_gap(P, P.rap_setup(a, lay, modified=True), a) <= 1e-10
    assert _coarse_row_sum_gap(P, P.rap_setup(a, lay, modified=False), a) > 1e-6     # plain factors do not
    g = P.poisson2d(8, 8)
    lay = layout_of(P, g, P.partition(g, 4, grid_hint=(8, 8)))
    plain, milu = P.rap_setup(g, lay, modified=False), P.rap_setup(g, lay, modified=True)
    assert not np.array_equal(plain.blocks[0].interior.upper.values, milu.blocks[0].interior.upper.values)
    assert np.array_equal(plain.smoother[0].upper.values, milu.smoother[0].upper.values)


# ---------------------------------------------------------------------------
# factory and collapse (pkg/tests/test_precond.py:356-400, test_acceptance.py:121-132)


def test_one_domain_collapses_every_preconditioner(P, rng):
    for a in (P.poisson2d(8, 8), P.poisson2d(16, 16)):
        lay = one_domain(P, a)
        r = rng.standard_normal(a.n_rows)
        base = P.make_preconditioner("bj", a, lay).apply(r)
        for name in ("l1bj", "schur", "rap", "rap-milu"):
            assert np.array_equal(P.make_preconditioner(name, a, lay).apply(r), base), name


def test_factory(P):
    a = P.poisson2d(6, 6)
    lay = layout_of(P, a, P.partition(a, 2, grid_hint=(6, 6)))
    kinds = {"bj": P.BjIluPrecond, "l1bj": P.BjIluPrecond, "schur": P.SchurIluPrecond, "rap": P.RapIluPrecond,
             "rap-milu": P.RapIluPrecond}
    for name, cls in kinds.items():
        assert isinstance(P.make_preconditioner(name, a, lay), cls)
    assert P.make_preconditioner("none", a, lay) is None
    assert P.make_preconditioner("l1bj", a, lay).l1 and not P.make_preconditioner("bj", a, lay).l1
    assert P.make_preconditioner("rap-milu", a, lay).modified and not P.make_preconditioner("rap", a, lay).modified
    with pytest.raises(ValueError):
        P.make_preconditioner("jacobi", a, one_domain(P, a))
    assert set(P.PRECONDITIONER_NAMES) == {"bj", "l1bj", "schur", "rap", "rap-milu", "none"}
