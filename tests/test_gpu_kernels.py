"""GPU parity, kernel level: every entry of the C ABI against the CPU oracle and
the reference-generated fixtures.  Bit-exact for integer / pattern work and for
the row-serial fp64 kernels (SpMV, SpTRSV, ILU numeric); reductions (dot) are
compared to 1e-13 relative (summation order differs by design)."""

import numpy as np
import pytest

from _golden import same_csr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def orc():
    from oracle import ddilu_oracle
    return ddilu_oracle


def _csr(P):
    return lambda nr, nc, rp, ci, v: P.CsrMatrix(nr, nc, rp.copy(), ci.copy(), v.copy())


def _to_orc(orc, m):
    return orc.Csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)


def test_scan_and_sort_primitives(P):
    import torch
    from paper_2303_08881_b200 import device as D
    rng = np.random.default_rng(5)
    for n in (0, 1, 31, 2048, 2049, 100003, 1 << 21):
        a = rng.integers(0, 9, size=n).astype(np.int32)
        buf = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
        buf[:n] = torch.from_numpy(a).cuda()
        D.exclusive_scan_(buf, n)
        ref = np.concatenate([[0], np.cumsum(a)])
        assert np.array_equal(buf.cpu().numpy(), ref), n
    for n, bits in ((2, 3), (1000, 5), (70001, 11), (1 << 20, 17), (300000, 31)):
        keys = rng.integers(0, 1 << bits, size=n).astype(np.int32)
        vals = np.arange(n, dtype=np.int32)
        kd, vd = torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda()
        D.sort_pairs_(kd, vd, bits)
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(kd.cpu().numpy(), keys[order])
        assert np.array_equal(vd.cpu().numpy(), vals[order]), "sort must be stable"


def test_sparse_kernels_against_reference(P, golden_kernels):
    g = golden_kernels
    for name in g.names("kernels.names"):
        k = "k." + name
        a = g.csr(k + ".a", _csr(P))
        x = g[k + ".x"]
        y = P.spmv(a, x)
        assert np.array_equal(y, g[k + ".spmv"]), name
        ref = float(g[k + ".vdot"])
        assert abs(P.vdot(x, y) - ref) <= 1e-13 * max(1.0, abs(ref))
        same_csr(P.csr_transpose(a), g, k + ".transpose")
        same_csr(P.permute_symmetric(a, P.Permutation(g[k + ".perm_forward"])), g, k + ".permuted")
        rows = g[k + ".sub_rows"]
        same_csr(P.take_submatrix(a, rows, rows), g, k + ".take_submatrix")
        srt = np.sort(rows)
        same_csr(P.extract_block(a, srt, srt), g, k + ".extract_block")


def test_rcm_bit_exact(P, golden_kernels):
    g = golden_kernels
    for name in g.names("kernels.names"):
        k = "k." + name
        perm = P.rcm(g.csr(k + ".a", _csr(P)))
        assert np.array_equal(perm.forward, g[k + ".rcm_forward"]), name
        assert np.array_equal(perm.inverse, g[k + ".rcm_inverse"]), name


def test_partitions_bit_exact(P, golden_kernels):
    """Structured boxes, their breadth-first fallback (uneven grids) and the
    unstructured breadth-first partition (ordering.py:97-127, 148-198)."""
    import json
    g = golden_kernels
    for case in g.names("partition.cases"):
        dims, p = json.loads(case)
        a = P.poisson2d(*dims) if len(dims) == 2 else P.poisson3d(*dims)
        got = P.partition(a, p, grid_hint=tuple(dims))
        assert np.array_equal(np.asarray(got), g[f"partition.{'x'.join(map(str, dims))}.p{p}"]), case
    for name in g.names("kernels.names"):
        a = g.csr("k." + name + ".a", _csr(P))
        for p in (2, 3):
            assert np.array_equal(np.asarray(P.partition(a, p)), g[f"k.{name}.grow_owner_p{p}"]), (name, p)


def test_rcm_larger_grids(P, orc):
    for a in (P.aniso3d(17, 13, 11), P.poisson2d(64, 37), P.convdiff27(9, 10, 11)):
        fwd, inv = orc.rcm(_to_orc(orc, a))
        perm = P.rcm(a)
        assert np.array_equal(perm.forward, fwd)


def test_factorisations_against_reference(P, golden_kernels):
    g = golden_kernels
    for name in g.names("kernels.names"):
        k = "k." + name
        a = g.csr(k + ".a", _csr(P))
        n = a.n_rows
        f0 = P.ilu0(a)
        same_csr(f0.lower, g, k + ".ilu0.lower")
        same_csr(f0.upper, g, k + ".ilu0.upper")
        b = g[k + ".b"]
        assert np.array_equal(P.tri_solve_lower(f0.lower, b, unit_diag=True), g[k + ".lsolve"]), name
        assert np.array_equal(P.tri_solve_upper(f0.upper, b), g[k + ".usolve"]), name
        assert np.array_equal(f0.solve(b), g[k + ".lu_solve"]), name
        fm = P.milu0(a)
        same_csr(fm.lower, g, k + ".milu0.lower")
        same_csr(fm.upper, g, k + ".milu0.upper")
        fv = P.milu0(a, P.MiluVectors(g[k + ".milu_y"], g[k + ".milu_z"], g[k + ".milu_w"]))
        same_csr(fv.lower, g, k + ".milu0_vecs.lower")
        same_csr(fv.upper, g, k + ".milu0_vecs.upper")
        n1 = int(g[k + ".n_interior"])
        for tag, drop in (("ilu0", 0.0), ("ilu0_drop", 0.05)):       # the second exercises schur_drop_tol thinning
            pf = P.partial_ilu(a, n1, P.FillRule("ilu0"), schur_drop_tol=drop)
            kk = k + ".partial_" + tag
            same_csr(pf.interior.lower, g, kk + ".interior.lower")
            same_csr(pf.interior.upper, g, kk + ".interior.upper")
            same_csr(pf.w_block, g, kk + ".w")
            same_csr(pf.z_block, g, kk + ".z")
            same_csr(pf.s_tilde, g, kk + ".s")
            same_csr(pf.schur.lower, g, kk + ".schur.lower")
            same_csr(pf.schur.upper, g, kk + ".schur.upper")
        tl = P.extract_two_level_blocks(f0, n1)
        same_csr(tl.interior.lower, g, k + ".twolevel.interior.lower")
        same_csr(tl.interior.upper, g, k + ".twolevel.interior.upper")
        same_csr(tl.w_tilde, g, k + ".twolevel.w")
        same_csr(tl.z_tilde, g, k + ".twolevel.z")
        same_csr(tl.schur.lower, g, k + ".twolevel.schur.lower")
        same_csr(tl.schur.upper, g, k + ".twolevel.schur.upper")


def test_ilut_against_reference(P, golden_kernels):
    g = golden_kernels
    for name in g.names("kernels.names"):
        k = "k." + name
        a = g.csr(k + ".a", _csr(P))
        n = a.n_rows
        for tag, tau, mf in (("a", 1e-3, 20), ("b", 0.05, 3), ("c", 0.0, n)):
            ft = P.ilut(a, tau, mf)
            same_csr(ft.lower, g, k + f".ilut_{tag}.lower")
            same_csr(ft.upper, g, k + f".ilut_{tag}.upper")
        n1 = int(g[k + ".n_interior"])
        for tag, rule, drop in (("ilut", P.FillRule("ilut", tau=1e-2, maxfill=5), 0.0),
                                ("ilut_drop", P.FillRule("ilut", tau=1e-3, maxfill=8), 0.02)):
            pf = P.partial_ilu(a, n1, rule, schur_drop_tol=drop)
            kk = k + ".partial_" + tag
            same_csr(pf.interior.lower, g, kk + ".interior.lower")
            same_csr(pf.interior.upper, g, kk + ".interior.upper")
            same_csr(pf.w_block, g, kk + ".w")
            same_csr(pf.z_block, g, kk + ".z")
            same_csr(pf.s_tilde, g, kk + ".s")
            same_csr(pf.schur.lower, g, kk + ".schur.lower")
            same_csr(pf.schur.upper, g, kk + ".schur.upper")


def test_level_schedule_matches_oracle(P, orc):
    from paper_2303_08881_b200 import device as D
    for a in (P.aniso3d(9, 8, 7), P.convdiff27(6, 5, 7), P.poisson2d(33, 20)):
        f = P.ilu0(a)
        for t, upper in ((f.lower, False), (f.upper, True)):
            lev, ptr, rows = orc.level_schedule(_to_orc(orc, t), upper=upper)
            s = t.schedule(upper)
            assert s.n_levels == len(ptr) - 1
            assert np.array_equal(s.lev[: t.n_rows].cpu().numpy().astype(np.int64), lev)
            assert np.array_equal(s.level_ptr.cpu().numpy().astype(np.int64), ptr)
            assert np.array_equal(s.level_rows.cpu().numpy().astype(np.int64), rows)
            order = s.order.cpu().numpy()
            assert np.array_equal(order[order >= 0], rows.astype(np.int32))
            # every level starts on a warp boundary
            starts = np.cumsum(np.concatenate([[0], (np.diff(ptr) + 31) // 32 * 32]))
            assert len(order) == starts[-1]


def test_medium_kernels_bit_exact_vs_oracle(P, orc):
    """Sizes the oracle does in a second; exercises multi-CTA paths."""
    rng = np.random.default_rng(11)
    for a in (P.aniso3d(40, 37, 29), P.convdiff27(20, 19, 18, (10.0, -5.0, 2.0))):
        ao = _to_orc(orc, a)
        x = rng.standard_normal(a.n_rows)
        assert np.array_equal(P.spmv(a, x), orc.spmv(ao, x))
        f, fo = P.ilu0(a), orc.ilu0(ao)
        assert np.array_equal(f.lower.values, fo.lower.values) and np.array_equal(f.lower.col_idx, fo.lower.col_idx)
        assert np.array_equal(f.upper.values, fo.upper.values) and np.array_equal(f.upper.col_idx, fo.upper.col_idx)
        assert np.array_equal(f.solve(x), fo.solve(x))
        fm, fmo = P.milu0(a), orc.milu0(ao)
        assert np.array_equal(fm.upper.values, fmo.upper.values)
        ft, fto = P.ilut(a, 1e-3, 10), orc.ilut(ao, 1e-3, 10)
        assert np.array_equal(ft.lower.row_ptr, fto.lower.row_ptr) and np.array_equal(ft.upper.col_idx, fto.upper.col_idx)
        assert np.array_equal(ft.lower.values, fto.lower.values) and np.array_equal(ft.upper.values, fto.upper.values)
        perm = P.rcm(a)
        assert np.array_equal(perm.forward, orc.rcm(ao)[0])


def test_tri_solve_errors_and_edges(P):
    """tests/test_sparse.py:97-117-style edge cases: zero diagonal raises with the row."""
    l = P.csr_from_dense(np.array([[2.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 4.0]]), keep_zeros=False)
    with pytest.raises(ZeroDivisionError):
        P.tri_solve_lower(l, np.ones(3))
    l = P.csr_from_dense(np.array([[2.0, 0.0], [1.0, 4.0]]))
    assert np.array_equal(P.tri_solve_lower(l, np.array([2.0, 5.0])), np.array([1.0, 1.0]))
    u = P.csr_from_dense(np.array([[2.0, 1.0], [0.0, 4.0]]))
    assert np.array_equal(P.tri_solve_upper(u, np.array([3.0, 4.0])), np.array([1.0, 1.0]))
    with pytest.raises(ValueError):
        P.tri_solve_lower(l, np.ones(3))
    with pytest.raises(ValueError):
        P.spmv(l, np.ones(5))


def test_known_answers_from_reference_tests(P):
    """tests/test_factor.py:70-80, 101-109, 289-303 of the reference."""
    d = np.zeros((3, 3))
    for i in range(3):
        d[i, i] = 2.0
        if i + 1 < 3:
            d[i, i + 1] = d[i + 1, i] = -1.0
    u = P.ilu0(P.csr_from_dense(d)).upper.to_dense()
    assert u[0, 0] == 2.0 and u[1, 1] == 1.5 and abs(u[2, 2] - 4.0 / 3.0) < 1e-15
    a = P.csr_from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]), keep_zeros=True)
    assert P.ilu0(a).upper.to_dense()[0, 0] == 1e-6
    a = P.csr_from_dense(np.array([[-1e-9, 1.0], [0.0, 1.0]]))
    assert P.ilu0(a).upper.to_dense()[0, 0] == -1e-6
    pf = P.partial_ilu(P.poisson2d(2, 2), 2, P.FillRule("ilu0"))
    assert np.max(np.abs(pf.s_tilde.to_dense() - np.array([[15 / 4, -1.0], [-1.0, 56 / 15]]))) == 0.0
    assert np.max(np.abs(pf.w_block.to_dense() - np.diag([-1 / 4, -4 / 15]))) == 0.0
    assert np.max(np.abs(pf.z_block.to_dense() + np.eye(2))) == 0.0
    pf = P.partial_ilu(P.poisson2d(2, 2), 2, P.FillRule("ilut", tau=0.0, maxfill=4))
    assert np.max(np.abs(pf.s_tilde.to_dense() - np.array([[56.0, -16.0], [-16.0, 56.0]]) / 15)) < 1e-15
    # ILUT tie-break keeps the smaller column (tests/test_factor.py:222-231)
    t = P.csr_from_dense(np.array([[4.0, 0.0, 0.0], [0.0, 4.0, 0.0], [1.0, 1.0, 4.0]]))
    f = P.ilut(t, 0.0, 1)
    assert np.array_equal(f.lower.col_idx[f.lower.row_ptr[2]:f.lower.row_ptr[3]], [0])


def test_compact_row_updates_match_the_full_pass(P):
    """Coupling blocks with few non-empty rows (Z of the two-level preconditioners): the compact-row update must give
    the bits of the full `b - A x` / `A x` passes it replaces (precond.py:262, 343 of the reference)."""
    import torch
    from paper_2303_08881_b200 import device as D
    rng = np.random.default_rng(21)
    n_rows, n_cols = 5000, 300
    rows = np.sort(rng.choice(n_rows, size=400, replace=False))
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    ci, va = [], []
    for r in rows:
        k = int(rng.integers(1, 4))
        cols = np.sort(rng.choice(n_cols, size=k, replace=False))
        ci += list(cols)
        va += list(rng.standard_normal(k))
        rp[r + 1] = k
    rp = np.cumsum(rp)
    a = P.CsrMatrix(n_rows, n_cols, rp, np.array(ci, dtype=np.int64), np.array(va)).device()
    c = D.compact_rows(a)
    assert c is not None and c.csr.n_rows == len(rows)
    x = D.to_device_f64(rng.standard_normal(n_cols))
    b = rng.standard_normal(n_rows)
    b[rows[0]] = -0.0
    b[5] = -0.0 if 5 not in rows else b[5]
    full = D.empty_f64(n_rows)
    D.spmv(a, x, full, b=D.to_device_f64(b), mode=1)
    upd = D.to_device_f64(b)
    D.sub_compact(c, x, upd)
    assert np.array_equal(full.cpu().numpy().view(np.int64), upd.cpu().numpy().view(np.int64))   # bits, signs of zero included
    prod, prod_c, neg_c = D.empty_f64(n_rows), D.empty_f64(n_rows + 7), D.empty_f64(n_rows)
    D.spmv(a, x, prod)
    prod_c.fill_(3.0)
    D.spmv_compact(c, x, prod_c, n_rows)
    assert np.array_equal(prod.cpu().numpy().view(np.int64), prod_c[:n_rows].cpu().numpy().view(np.int64))
    assert float((prod_c[n_rows:] - 3.0).abs().max()) == 0.0          # nothing written behind the rows
    D.spmv_compact(c, x, neg_c, n_rows, negate=True)
    assert np.array_equal(neg_c.cpu().numpy(), -prod.cpu().numpy())   # values; the sign of exact zeros may differ
    # a matrix with most rows non-empty is left to the streaming kernel
    dense_rp = np.arange(n_rows + 1, dtype=np.int64)
    d = P.CsrMatrix(n_rows, n_cols, dense_rp, np.zeros(n_rows, dtype=np.int64), np.ones(n_rows)).device()
    assert D.compact_rows(d) is None


def test_warp_per_row_solve_bit_exact(P, orc):
    """`ddilu_sptrsv_warprow` (long rows: 27-point ILU(0) / ILUT / ILU(1) factors) against the oracle's serial solves
    and against the thread-per-row kernels, L and U, plus the zero-pivot report."""
    import torch
    from paper_2303_08881_b200 import device as D
    rng = np.random.default_rng(41)
    for a, f in ((P.convdiff27(11, 10, 9), None), (P.convdiff27(9, 9, 9), "ilut"), (P.poisson3d(12, 11, 10), "iluk")):
        fac = P.ilu0(a) if f is None else (P.ilut(a, 1e-3, 20) if f == "ilut" else P.iluk(a, 2))
        dv = fac.device()
        assert D.uses_warprow(dv.upper)
        b = rng.standard_normal(a.n_rows)
        bd = D.to_device_f64(b)
        lo, up = fac.lower, fac.upper
        ref_l = orc.tri_solve_lower(orc.Csr(lo.n_rows, lo.n_cols, lo.row_ptr, lo.col_idx, lo.values), b, True)
        ref_u = orc.tri_solve_upper(orc.Csr(up.n_rows, up.n_cols, up.row_ptr, up.col_idx, up.values), b)
        for t, sched, upper, unit, ref in ((dv.lower, dv.sched_l, False, True, ref_l), (dv.upper, dv.sched_u, True, False, ref_u)):
            out = {}
            for mode in (True, False):
                old = D.USE_WARPROW
                D.USE_WARPROW = mode
                try:
                    x = D.empty_f64(a.n_rows)
                    D.sptrsv(t, sched, bd, x, upper, unit)
                    torch.cuda.synchronize()
                    out[mode] = x.cpu().numpy()
                finally:
                    D.USE_WARPROW = old
            assert np.array_equal(out[True], ref), (f, upper)
            assert np.array_equal(out[True], out[False]), (f, upper)
    # zero pivot: reported as the failing row, like the reference (sparse.py:268-270)
    d = np.triu(rng.standard_normal((40, 40))) + 5.0 * np.eye(40)
    d[17, 17] = 0.0
    u = P.csr_from_dense(d, keep_zeros=True) if "keep_zeros" in P.csr_from_dense.__code__.co_varnames else P.csr_from_dense(d)
    with pytest.raises(ZeroDivisionError):
        P.tri_solve_upper(u, np.ones(40))
