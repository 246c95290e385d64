"""GPU parity of the block sweep (csrc/sweep.cu): the interface factors L_S / U_S solved by one CTA per
subdomain block -- L only, U only, L then U in one launch, and the fused forms of precond.py:242-249
(`S^-1 (r_ext - W fp)`, `y + S^-1 (E_off y)`) -- bit-exact against the CPU oracle's row-serial solves
(sparse.py:228-272) and against the separate-kernel sequence."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def orc():
    from oracle import ddilu_oracle
    return ddilu_oracle


def _oracle_solves(P, orc, f, b):
    lo, up = P.CsrMatrix.from_device(f.lower), P.CsrMatrix.from_device(f.upper)
    olo = orc.Csr(lo.n_rows, lo.n_cols, lo.row_ptr, lo.col_idx, lo.values)
    oup = orc.Csr(up.n_rows, up.n_cols, up.row_ptr, up.col_idx, up.values)
    xl = orc.tri_solve_lower(olo, b, True)
    return xl, orc.tri_solve_upper(oup, b), orc.tri_solve_upper(oup, xl)


CASES = [((20, 20, 20), 8, "schur"), ((24, 17, 9), 4, "schur"), ((40, 40), 4, "schur"), ((33, 31, 29), 2, "rap-milu"),
         ((36, 36, 36), 8, "rap"), ((48, 48, 48), 8, "schur")]


@pytest.mark.parametrize("dims,p,pc", CASES)
@pytest.mark.parametrize("max_threads,rpt,sets", [(416, 1, 3), (32, 1, 2), (256, 2, 3), (64, 2, 2)])
def test_sweep_solves_bit_exact(P, orc, dims, p, pc, max_threads, rpt, sets):
    """L, U and the fused U^-1 L^-1 against the oracle, for the thread shapes of the kernel (rows per thread,
    two or three sets); max_threads = 32 / 64 forces the loop behind the prefetched rows on the wide levels."""
    import torch
    from paper_2303_08881_b200 import device as D
    old = D.SWEEP_MAX_THREADS, D.SWEEP_ROWS_PER_THREAD, D.SWEEP_SETS
    D.SWEEP_MAX_THREADS, D.SWEEP_ROWS_PER_THREAD, D.SWEEP_SETS = max_threads, rpt, sets
    try:
        a = P.aniso3d(*dims) if len(dims) == 3 else P.aniso2d(*dims)
        layout = P.classify_and_order(a, P.partition(a, p, dims), p)
        m = P.make_preconditioner(pc, a, layout)
    finally:
        D.SWEEP_MAX_THREADS, D.SWEEP_ROWS_PER_THREAD, D.SWEEP_SETS = old
    f = m._p.schur if pc == "schur" else m._schur
    sp = f._sw
    assert sp is not None, "interface factors did not get a sweep plan"
    assert sp.n_blocks == p and sp.nct <= max_threads and sp.rpt == rpt and sp.sets == sets
    rng = np.random.default_rng(17)
    for rep in range(3):
        b = rng.standard_normal(f.n)
        bd = D.to_device_f64(b)
        ref_l, ref_u, ref_lu = _oracle_solves(P, orc, f, b)
        xl, xu, xlu = D.empty_f64(f.n), D.empty_f64(f.n), D.empty_f64(f.n)
        f.lower_solve(bd, xl)
        f.upper_solve(bd, xu)
        f.solve(bd, xlu)
        torch.cuda.synchronize()
        assert np.array_equal(xl.cpu().numpy(), ref_l), ("L", rep)
        assert np.array_equal(xu.cpu().numpy(), ref_u), ("U", rep)
        assert np.array_equal(xlu.cpu().numpy(), ref_lu), ("LU", rep)


@pytest.mark.parametrize("dims,p", [((20, 20, 20), 8), ((40, 37, 29), 4), ((40, 40), 4)])
def test_fused_products_match_separate_kernels(P, dims, p):
    """`S^-1 (r_ext - W fp)` and `y + S^-1 (E_off y)` through ddilu_sweep_rhs + ddilu_sweep_solve give the bits
    of spmv -> L solve -> U solve -> add (precond.py:242-249)."""
    import torch
    from paper_2303_08881_b200 import device as D
    from paper_2303_08881_b200.factor import solve_with_product
    a = P.aniso3d(*dims) if len(dims) == 3 else P.aniso2d(*dims)
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    m = P.make_preconditioner("schur", a, layout)
    s, f = m.system, m._p.schur
    assert f._sw is not None
    torch.manual_seed(3)
    y = torch.randn(s.n_ext + s.n_halo, dtype=torch.float64, device="cuda")
    fp = torch.randn(s.n_int, dtype=torch.float64, device="cuda")
    r = torch.randn(s.n_ext, dtype=torch.float64, device="cuda")
    t1, t2, t3 = D.empty_f64(s.n_ext), D.empty_f64(s.n_ext), D.empty_f64(s.n_ext)
    # y + S^-1 (E_off y)
    out = D.empty_f64(s.n_ext)
    solve_with_product(f, m._coupling, y, None, 0, out, add=y)
    D.spmv(m._coupling, y, t1)
    f.lower_solve(t1, t2)
    f.upper_solve(t2, t3)
    D.ewise(s.n_ext, y, t3, 0, t1)
    assert torch.equal(out, t1)
    # S^-1 (r_ext - W fp)
    solve_with_product(f, m._p.w, fp, r, 1, out)
    D.spmv(m._p.w, fp, t1, b=r, mode=1)
    f.lower_solve(t1, t2)
    f.upper_solve(t2, t3)
    assert torch.equal(out, t3)


def test_pipeline_same_with_and_without_sweep(P):
    """The preconditioner applications are bit-identical and the solves take the same iterations whether the
    interface factors use the sweep or the tiled kernels."""
    from paper_2303_08881_b200 import device as D
    dims = (24, 24, 24)
    a = P.aniso3d(*dims)
    b = P.default_rhs(a)
    res = {}
    for sweep in (True, False):
        old = D.USE_SWEEP
        D.USE_SWEEP = sweep
        try:
            layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
            for pc in ("schur", "rap", "rap-milu"):
                m = P.make_preconditioner(pc, a, layout)
                f = m._p.schur if pc == "schur" else m._schur
                assert (f._sw is not None) == sweep
                x, rep = P.fgmres(a, b, m=m.apply)
                res[(sweep, pc)] = (rep.iterations, rep.residual_history, x)
        finally:
            D.USE_SWEEP = old
    for pc in ("schur", "rap", "rap-milu"):
        it_a, h_a, x_a = res[(True, pc)]
        it_b, h_b, x_b = res[(False, pc)]
        assert it_a == it_b, pc
        assert np.array_equal(h_a, h_b), pc       # same kernels' bits in, same reductions: identical histories
        assert np.array_equal(x_a, x_b), pc


def test_sweep_refuses_unsuitable_factors(P):
    """Wide levels (a block-Jacobi factor of a whole 3D subdomain) and rows with more than 24 dependencies get no
    plan; the caller falls back to the tiled / sync-free kernels."""
    from paper_2303_08881_b200 import device as D
    dims = (24, 24, 24)
    a = P.aniso3d(*dims)
    f = P.ilu0(a).device()
    old = D.SWEEP_MAX_AVG_WIDTH
    D.SWEEP_MAX_AVG_WIDTH = 8
    try:
        assert D.build_sweep(f.lower, f.upper, *f._lev(False), *f._lev(True), [0, f.n]) is None
    finally:
        D.SWEEP_MAX_AVG_WIDTH = old
    # rows with more than 24 dependencies (27-point ILU(1): up to ~40) get no plan either
    a27 = P.convdiff27(10, 10, 10)
    f27 = P.iluk(a27, 1).device()
    assert int((f27.upper.rp[1:] - f27.upper.rp[:-1]).max().item()) - 1 > 24
    assert D.build_sweep(f27.lower, f27.upper, *f27._lev(False), *f27._lev(True), [0, f27.n]) is None


@pytest.mark.parametrize("dims,p,fill", [((24, 24, 24), 8, "ilut:0.001,20"), ((20, 18, 16), 4, "ilu0"),
                                         ((28, 28, 28), 8, "ilut:0.001,20")])
def test_sweep_long_rows_27_point(P, orc, dims, p, fill):
    """Interface factors of the 27-point problem (BASELINE config 5: ILUT(1e-3, 20), up to 20 dependencies per
    row): the long-row instances of the kernel (16 / 24 operand slots, 64-row pages, 512-thread CTAs) bit-exact
    against the oracle's serial solves, and the solve converging with the oracle's iteration count."""
    import torch
    from paper_2303_08881_b200 import device as D
    a = P.convdiff27(*dims)
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    m = P.schur_setup(a, layout, rule=P.FillRule.parse(fill))
    f = m._p.schur
    sp = f._sw
    assert sp is not None, "27-point interface factors did not get a plan"
    if fill.startswith("ilut"):
        assert sp.k in (16, 24) and sp.rpt == 1, "ILUT interface factors should take the long-row instances"
    rng = np.random.default_rng(29)
    for rep in range(2):
        b = rng.standard_normal(f.n)
        ref_l, ref_u, ref_lu = _oracle_solves(P, orc, f, b)
        bd = D.to_device_f64(b)
        xl, xu, xlu = D.empty_f64(f.n), D.empty_f64(f.n), D.empty_f64(f.n)
        f.lower_solve(bd, xl)
        f.upper_solve(bd, xu)
        f.solve(bd, xlu)
        torch.cuda.synchronize()
        assert np.array_equal(xl.cpu().numpy(), ref_l), ("L", rep)
        assert np.array_equal(xu.cpu().numpy(), ref_u), ("U", rep)
        assert np.array_equal(xlu.cpu().numpy(), ref_lu), ("LU", rep)
    x, rep_ = P.fgmres(a, P.default_rhs(a), m=m.apply)
    assert rep_.converged


@pytest.mark.timeout(300)
@pytest.mark.parametrize("budget_kb,sets", [(80, 3), (80, 2), (200, 3)])
def test_sweep_small_ring_does_not_stall(P, orc, budget_kb, sets):
    """A 4-stage ring (small shared-memory budget) with levels that straddle pages: the residency rule of
    `build_sweep` (all pages of the levels the sets work on at once must fit) either admits the factor and the
    solve finishes bit-exactly, or refuses it."""
    import torch
    from paper_2303_08881_b200 import device as D
    old = D.SWEEP_SMEM_BUDGET, D.SWEEP_SETS
    D.SWEEP_SMEM_BUDGET, D.SWEEP_SETS = budget_kb * 1024, sets
    try:
        dims = (48, 48, 48)
        a = P.aniso3d(*dims)
        layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
        m = P.make_preconditioner("schur", a, layout)
    finally:
        D.SWEEP_SMEM_BUDGET, D.SWEEP_SETS = old
    f = m._p.schur
    if f._sw is None:
        pytest.skip("refused by the residency rule")
    assert f._sw.stages == (4 if budget_kb == 80 else 8)
    b = np.random.default_rng(2).standard_normal(f.n)
    x = D.empty_f64(f.n)
    for _ in range(3):
        f.solve(D.to_device_f64(b), x)
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), _oracle_solves(P, orc, f, b)[2])


@pytest.mark.parametrize("fill", ["iluk:1", "iluk:2", "ilut:0.001,6"])
def test_sweep_with_longer_rows(P, orc, fill):
    """Interface factors of fill-in rules (4 to 8 operand slots per row: the K = 4 / 8 instances of the kernel):
    bit-exact against the oracle's serial solves, or refused when a row has more than 8 dependencies."""
    import torch
    from paper_2303_08881_b200 import device as D
    dims = (28, 26, 24)
    a = P.aniso3d(*dims)
    layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
    m = P.schur_setup(a, layout, rule=P.FillRule.parse(fill))
    f = m._p.schur
    kmax = max(int((f.lower.rp[1:] - f.lower.rp[:-1]).max().item()), int((f.upper.rp[1:] - f.upper.rp[:-1]).max().item()) - 1)
    if kmax > 24:
        assert f._sw is None
        pytest.skip(f"{kmax} dependencies per row: tiled / sync-free kernels")
    assert f._sw is not None and f._sw.k >= kmax and f._sw.k in (2, 3, 4, 8, 16, 24)
    b = np.random.default_rng(23).standard_normal(f.n)
    ref_l, ref_u, ref_lu = _oracle_solves(P, orc, f, b)
    bd = D.to_device_f64(b)
    xl, xu, xlu = D.empty_f64(f.n), D.empty_f64(f.n), D.empty_f64(f.n)
    f.lower_solve(bd, xl)
    f.upper_solve(bd, xu)
    f.solve(bd, xlu)
    torch.cuda.synchronize()
    assert np.array_equal(xl.cpu().numpy(), ref_l) and np.array_equal(xu.cpu().numpy(), ref_u)
    assert np.array_equal(xlu.cpu().numpy(), ref_lu)
    x, rep = P.fgmres(a, P.default_rhs(a), m=m.apply)
    assert rep.converged
