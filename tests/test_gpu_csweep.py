"""GPU parity of the cluster sweep (csrc/csweep.cu): the interior factors L_B / U_B solved by one thread-block
cluster per subdomain block (x in windows distributed over the CTAs' shared memory, results pushed through
distributed shared memory, one mbarrier wait per level; short-row shape for 7-point ILU(0), long-row shape for
27-point ILUT factors) -- bit-exact against the CPU oracle's row-serial solves (sparse.py:228-272) and against the
tiled kernel; factor pairs that do not qualify must be refused.  Also here: the processing order of the ILUT kernel."""

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


class _Knobs:
    """Cluster-sweep eligibility opened up for test-sized problems."""

    def __init__(self, cluster, nset, min_chunk, use=True):
        self.new = (use, cluster, nset, min_chunk, 0, 0)

    def __enter__(self):
        from paper_2303_08881_b200 import device as D
        self.old = (D.USE_CSWEEP, D.CSWEEP_CLUSTER, D.CSWEEP_NSET, D.CSWEEP_MIN_CHUNK, D.CSWEEP_MIN_AVG_WIDTH,
                    D.CSWEEP_MIN_SMS)
        (D.USE_CSWEEP, D.CSWEEP_CLUSTER, D.CSWEEP_NSET, D.CSWEEP_MIN_CHUNK, D.CSWEEP_MIN_AVG_WIDTH,
         D.CSWEEP_MIN_SMS) = self.new
        return D

    def __exit__(self, *exc):
        from paper_2303_08881_b200 import device as D
        (D.USE_CSWEEP, D.CSWEEP_CLUSTER, D.CSWEEP_NSET, D.CSWEEP_MIN_CHUNK, D.CSWEEP_MIN_AVG_WIDTH,
         D.CSWEEP_MIN_SMS) = self.old


def _oracle_solves(P, orc, f, b):
    lo, up = P.CsrMatrix.from_device(f.lower), P.CsrMatrix.from_device(f.upper)
    olo = orc.Csr(lo.n_rows, lo.n_cols, lo.row_ptr, lo.col_idx, lo.values)
    oup = orc.Csr(up.n_rows, up.n_cols, up.row_ptr, up.col_idx, up.values)
    xl = orc.tri_solve_lower(olo, b, True)
    return xl, orc.tri_solve_upper(oup, b), orc.tri_solve_upper(oup, xl)


def _interior(m, pc):
    return m._p.interior if pc == "schur" else m._interior


CASES = [((20, 20, 20), 8, "schur"), ((40, 37, 29), 4, "schur"), ((40, 40), 4, "schur"), ((33, 31, 29), 2, "rap-milu"),
         ((48, 48, 48), 8, "rap"), ((33, 33, 33), 1, "schur")]


@pytest.mark.parametrize("dims,p,pc", CASES)
@pytest.mark.parametrize("cluster,nset,min_chunk", [(16, 3, 32), (16, 4, 1), (8, 3, 8), (4, 2, 32), (2, 3, 1)])
def test_cluster_sweep_bit_exact(P, orc, dims, p, pc, cluster, nset, min_chunk):
    """L, U and U^-1 L^-1 of the interior factors against the oracle, for cluster sizes 2 .. 16, both register
    rotations and chunk rules (min_chunk 1 spreads every level over the whole cluster: most dependencies remote)."""
    import torch
    with _Knobs(cluster, nset, min_chunk) as D:
        a = P.aniso3d(*dims) if len(dims) == 3 else P.aniso2d(*dims)
        layout = P.classify_and_order(a, P.partition(a, p, dims), p)
        m = P.make_preconditioner(pc, a, layout)
    f = _interior(m, pc)
    cp = f._cs
    assert cp is not None, "interior factors did not get a cluster-sweep plan"
    # the largest cluster size <= `cluster` whose clusters can all be resident (16 fits 7 times on a B200)
    want = next(c for c in range(cluster, 0, -1) if D.csweep_active_clusters(c, cp.k, 2, 2 * max(f._lev(False)[1], f._lev(True)[1])) >= p)
    assert cp.n_blocks == p and cp.csize == want and cp.lower.depth <= nset
    rng = np.random.default_rng(23)
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


@pytest.mark.parametrize("dims,p,cluster", [((14, 13, 12), 4, 8), ((20, 20, 20), 8, 4), ((16, 16, 16), 1, 8)])
def test_cluster_sweep_long_rows_27_point(P, orc, dims, p, cluster):
    """The 20-slot instance (27-point stencil, ILUT(1e-3, 20) interior factors: up to 19 dependencies per row, deep
    narrow levels, an 8 191-double window, up to four push targets, the step table read from global memory): L, U
    and U^-1 L^-1 against the oracle."""
    import torch
    with _Knobs(cluster, 3, 8) as D:
        a = P.convdiff27(*dims)
        layout = P.classify_and_order(a, P.partition(a, p, dims), p)
        m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
    f = m._p.interior
    cp = f._cs
    assert cp is not None and cp.k == 20 and cp.csize <= 8, "27-point interior factors did not get the long-row plan"
    rng = np.random.default_rng(29)
    for rep in range(2):
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


def test_cluster_sweep_levels_wider_than_the_cta(P, orc):
    """A 48^3 block on ONE CTA: the widest levels have more than twice as many rows as the CTA has threads (they
    are cut into three steps; only the first waits, only the last signals)."""
    import torch
    dims = (48, 48, 48)
    with _Knobs(1, 3, 32) as D:
        a = P.aniso3d(*dims)
        layout = P.classify_and_order(a, P.partition(a, 1, dims), 1)
        m = P.make_preconditioner("schur", a, layout)
        threads = D.query("ddilu_csweep_threads", 3)
    f = m._p.interior
    assert f._cs is not None and f._cs.csize == 1
    widest = int(np.bincount(f._lev(False)[0][: f.n].cpu().numpy()).max())
    assert widest > 2 * threads, "the case no longer has levels wider than two steps"
    assert f._cs.lower.max_steps > f._lev(False)[1]
    b = np.random.default_rng(5).standard_normal(f.n)
    ref_l, ref_u, ref_lu = _oracle_solves(P, orc, f, b)
    xl, xu = D.empty_f64(f.n), D.empty_f64(f.n)
    f.lower_solve(D.to_device_f64(b), xl)
    f.upper_solve(D.to_device_f64(b), xu)
    torch.cuda.synchronize()
    assert np.array_equal(xl.cpu().numpy(), ref_l)
    assert np.array_equal(xu.cpu().numpy(), ref_u)


def test_cluster_sweep_refuses_unsuitable_factors(P):
    """No plan for: rows with more than 20 dependencies (27-point ILU(1)), dependencies further back than the window
    (one CTA for a 64^3 block), problems below the production thresholds; the factors then solve through the tiled /
    sync-free kernels."""
    with _Knobs(16, 3, 32) as D:
        a27 = P.convdiff27(12, 12, 12)
        lay = P.classify_and_order(a27, P.partition(a27, 8, (12, 12, 12)), 8)
        m = P.make_preconditioner("schur", a27, lay, P.FillRule.parse("iluk:1"))
        f27 = m._p.interior
        assert int((f27.upper.rp[1:] - f27.upper.rp[:-1]).max().item()) - 1 > 20
        assert f27._cs is None
    with _Knobs(1, 3, 32) as D:
        a = P.aniso3d(64, 64, 64)
        lay = P.classify_and_order(a, P.partition(a, 1, (64, 64, 64)), 1)
        m = P.make_preconditioner("schur", a, lay)
        assert m._p.interior._cs is None
    a = P.aniso3d(24, 24, 24)
    lay = P.classify_and_order(a, P.partition(a, 8, (24, 24, 24)), 8)
    m = P.make_preconditioner("schur", a, lay)
    assert m._p.interior._cs is None          # production thresholds: far too small for clusters


def test_pipeline_same_with_and_without_cluster_sweep(P):
    """Preconditioner applications are bit-identical and the solves take the same iterations whether the interior
    factors use the cluster sweep or the tiled kernel."""
    dims = (32, 32, 32)
    a = P.aniso3d(*dims)
    b = P.default_rhs(a)
    res = {}
    for use in (True, False):
        with _Knobs(16, 3, 32, use=use):
            layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
            for pc in ("schur", "rap", "rap-milu"):
                m = P.make_preconditioner(pc, a, layout)
                assert (_interior(m, pc)._cs is not None) == use
                x, rep = P.fgmres(a, b, m=m.apply)
                z = m.apply(b)
                res[(use, pc)] = (rep.iterations, np.asarray(x), np.asarray(z))
    for pc in ("schur", "rap", "rap-milu"):
        it1, x1, z1 = res[(True, pc)]
        it0, x0, z0 = res[(False, pc)]
        assert it1 == it0
        assert np.array_equal(z1, z0)
        assert np.array_equal(x1, x0)


def test_ilut_interleaved_blocks_same_factors(P):
    """The ILUT kernel takes the rows of the independent subdomain blocks round-robin (all blocks advance at once
    instead of one after the other): patterns and values of L_B, U_B, W, Z, S~ and of the factors of S~ are the bits
    of the index-order run (factor.py:482-656 is order-independent across independent blocks)."""
    import torch
    from paper_2303_08881_b200 import factor as F
    dims = (14, 13, 12)
    a = P.convdiff27(*dims)
    layout = P.classify_and_order(a, P.partition(a, 4, dims), 4)
    m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
    s = m.system
    rule = P.FillRule.parse("ilut:0.001,20")
    plain = F.d_partial_ilu(s.a_dom, s.n_int, rule, factor_schur=True)
    inter = F.d_partial_ilu(s.a_dom, s.n_int, rule, factor_schur=True, blocks=(s.int_ptr, s.ext_ptr))
    from paper_2303_08881_b200._ilut import interleaved_order
    order = interleaved_order(s.n_loc, (s.int_ptr, s.ext_ptr))
    assert order is not None and sorted(order.cpu().tolist()) == list(range(s.n_loc))
    assert order[:4].cpu().tolist() == [int(s.int_ptr[k]) for k in range(4)]      # row 0 of every block first
    pairs = [(plain.interior.lower, inter.interior.lower), (plain.interior.upper, inter.interior.upper),
             (plain.w, inter.w), (plain.z, inter.z), (plain.s_tilde, inter.s_tilde),
             (plain.schur.lower, inter.schur.lower), (plain.schur.upper, inter.schur.upper)]
    for x, y in pairs:
        assert x.nnz == y.nnz
        assert torch.equal(x.rp, y.rp) and torch.equal(x.ci[: x.nnz], y.ci[: y.nnz])
        assert torch.equal(x.val[: x.nnz], y.val[: y.nnz])
