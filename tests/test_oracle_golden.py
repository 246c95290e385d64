"""Pin the CPU oracle (oracle/) against the unmodified reference.

Fixtures in tests/golden/*.npz were written by the reference itself
(tests/golden/make_golden.py); the known answers below restate the reference's
own tests (file:line cited per test).  Everything here is bit-exact unless a
tolerance is written in the assertion.
"""

import json

import numpy as np
import pytest

from _golden import iterations, same_csr
from oracle import ddilu_oracle as orc

Csr = orc.Csr


def test_kernels_against_reference(golden_kernels):
    g = golden_kernels
    for name in g.names("kernels.names"):
        k = "k." + name
        a = g.csr(k + ".a", Csr)
        n = a.n_rows
        x = g[k + ".x"]
        y = orc.spmv(a, x)
        assert np.array_equal(y, g[k + ".spmv"])
        assert orc.vdot(x, y) == float(g[k + ".vdot"])
        same_csr(orc.csr_transpose(a), g, k + ".transpose")
        same_csr(orc.permute_symmetric(a, g[k + ".perm_forward"]), g, k + ".permuted")
        rows = g[k + ".sub_rows"]
        same_csr(orc.take_submatrix(a, rows, rows), g, k + ".take_submatrix")
        srt = np.sort(rows)
        same_csr(orc.extract_block(a, srt, srt), g, k + ".extract_block")
        rp, ci = orc.sym_adjacency(a)
        assert np.array_equal(rp, g[k + ".sym_rp"]) and np.array_equal(ci, g[k + ".sym_ci"])
        fwd, inv = orc.rcm(a)
        assert np.array_equal(fwd, g[k + ".rcm_forward"]), name
        assert np.array_equal(inv, g[k + ".rcm_inverse"]), name
        for p in (2, 3):
            assert np.array_equal(orc.partition(a, p), g[k + f".grow_owner_p{p}"])
        f0 = orc.ilu0(a)
        same_csr(f0.lower, g, k + ".ilu0.lower")
        same_csr(f0.upper, g, k + ".ilu0.upper")
        b = g[k + ".b"]
        assert np.array_equal(orc.tri_solve_lower(f0.lower, b, unit_diag=True), g[k + ".lsolve"])
        assert np.array_equal(orc.tri_solve_upper(f0.upper, b), g[k + ".usolve"])
        assert np.array_equal(f0.solve(b), g[k + ".lu_solve"])
        fm = orc.milu0(a)
        same_csr(fm.lower, g, k + ".milu0.lower")
        same_csr(fm.upper, g, k + ".milu0.upper")
        n1 = int(g[k + ".n_interior"])
        target = np.concatenate([g[k + ".milu_y"], g[k + ".milu_z"]])
        wvec = np.concatenate([g[k + ".milu_w"], np.zeros(n - n1)])
        fv = orc.milu0(a, target, wvec)
        same_csr(fv.lower, g, k + ".milu0_vecs.lower")
        same_csr(fv.upper, g, k + ".milu0_vecs.upper")
        for tag, tau, mf in (("a", 1e-3, 20), ("b", 0.05, 3), ("c", 0.0, n)):
            ft = orc.ilut(a, tau, mf)
            same_csr(ft.lower, g, k + f".ilut_{tag}.lower")
            same_csr(ft.upper, g, k + f".ilut_{tag}.upper")
        for tag, rule, drop in (("ilu0", orc.Rule("ilu0"), 0.0),
                                ("ilut", orc.Rule("ilut", 1e-2, 5), 0.0),
                                ("ilu0_drop", orc.Rule("ilu0"), 0.05),
                                ("ilut_drop", orc.Rule("ilut", 1e-3, 8), 0.02)):
            pf = orc.partial_ilu(a, n1, rule, schur_drop_tol=drop)
            kk = k + ".partial_" + tag
            same_csr(pf.interior.lower, g, kk + ".interior.lower")
            same_csr(pf.interior.upper, g, kk + ".interior.upper")
            same_csr(pf.w_block, g, kk + ".w")
            same_csr(pf.z_block, g, kk + ".z")
            same_csr(pf.s_tilde, g, kk + ".s")
            same_csr(pf.schur.lower, g, kk + ".schur.lower")
            same_csr(pf.schur.upper, g, kk + ".schur.upper")
        tl = orc.extract_two_level_blocks(f0, n1)
        same_csr(tl.interior.lower, g, k + ".twolevel.interior.lower")
        same_csr(tl.interior.upper, g, k + ".twolevel.interior.upper")
        same_csr(tl.w_tilde, g, k + ".twolevel.w")
        same_csr(tl.z_tilde, g, k + ".twolevel.z")
        same_csr(tl.schur.lower, g, k + ".twolevel.schur.lower")
        same_csr(tl.schur.upper, g, k + ".twolevel.schur.upper")


def test_structured_partitions(golden_kernels):
    g = golden_kernels
    for case in g.names("partition.cases"):
        dims, p = json.loads(case)
        a = orc.poisson2d(*dims) if len(dims) == 2 else orc.poisson3d(*dims)
        got = orc.partition(a, p, grid_hint=tuple(dims))
        assert np.array_equal(got, g[f"partition.{'x'.join(map(str, dims))}.p{p}"]), case


def test_generators_match_reference(golden_pipeline):
    g = golden_pipeline
    built = {
        "aniso2d_16": orc.aniso((16, 16), (1.0, 0.01)),
        "aniso3d_10": orc.aniso((10, 10, 10), (1.0, 1.0, 0.01)),
        "poisson3d_9x8x7": orc.poisson3d(9, 8, 7),
        "convdiff3d_8": orc.convdiff3d(8, 8, 8, (20.0, -10.0, 5.0)),
        "cd27_8": orc.convdiff27(8, 8, 8, (10.0, 10.0, 10.0)),
    }
    for name, a in built.items():
        same_csr(a, g, f"p.{name}.a")
        assert np.array_equal(orc.default_rhs(a), g[f"p.{name}.b"])


def _check_precond(g, k, pc, m):
    for d, dom in enumerate(m.domains):
        assert np.array_equal(dom.interior_nodes, g[f"{k}.dom{d}.interior_nodes"])
        assert np.array_equal(dom.exterior_nodes, g[f"{k}.dom{d}.exterior_nodes"])
    if pc in ("bj", "l1bj"):
        for d, f in enumerate(m.factors):
            same_csr(f.lower, g, f"{k}.dom{d}.factors.lower")
            same_csr(f.upper, g, f"{k}.dom{d}.factors.upper")
    elif pc == "schur":
        for d, pf in enumerate(m.partial):
            same_csr(pf.interior.lower, g, f"{k}.dom{d}.interior.lower")
            same_csr(pf.interior.upper, g, f"{k}.dom{d}.interior.upper")
            same_csr(pf.w_block, g, f"{k}.dom{d}.w")
            same_csr(pf.z_block, g, f"{k}.dom{d}.z")
            same_csr(pf.s_tilde, g, f"{k}.dom{d}.s")
            same_csr(pf.schur.lower, g, f"{k}.dom{d}.schur.lower")
            same_csr(pf.schur.upper, g, f"{k}.dom{d}.schur.upper")
        same_csr(m.coupling, g, f"{k}.coupling")
    else:
        for d, (f, blk) in enumerate(zip(m.smoother, m.blocks)):
            same_csr(f.lower, g, f"{k}.dom{d}.smoother.lower")
            same_csr(f.upper, g, f"{k}.dom{d}.smoother.upper")
            same_csr(blk.interior.lower, g, f"{k}.dom{d}.interior.lower")
            same_csr(blk.interior.upper, g, f"{k}.dom{d}.interior.upper")
            same_csr(blk.w_tilde, g, f"{k}.dom{d}.w")
            same_csr(blk.z_tilde, g, f"{k}.dom{d}.z")
            same_csr(blk.schur.lower, g, f"{k}.dom{d}.schur.lower")
            same_csr(blk.schur.upper, g, f"{k}.dom{d}.schur.upper")
        same_csr(m.a_perm, g, f"{k}.a_perm")
        assert np.array_equal(m.perm_forward, g[f"{k}.perm_forward"])


def test_pipeline_against_reference(golden_pipeline):
    """partition -> classify -> setup -> apply -> fgmres, all bit-exact."""
    g = golden_pipeline
    for tag in g.names("pipeline.cases"):
        pname, ptag, part, pc, fill = tag.split("|")
        p = int(ptag[1:])
        k = "c." + tag
        a = g.csr(f"p.{pname}.a", Csr)
        hint = tuple(int(v) for v in g[f"p.{pname}.hint"])
        owner = orc.row_block_owner(a.n_rows, p) if part == "rows" else orc.partition(a, p, hint)
        assert np.array_equal(owner, g[k + ".owner"]), tag
        layout = orc.classify_and_order(a, owner)
        assert np.array_equal(layout.interior_starts, g[k + ".interior_starts"])
        assert np.array_equal(layout.exterior_starts, g[k + ".exterior_starts"])
        assert np.array_equal(layout.perm_forward, g[k + ".global_perm_forward"])
        m = orc.make_preconditioner(pc, a, layout, orc.Rule.parse(fill), inner_iters=3)
        _check_precond(g, k, pc, m)
        r = g[f"p.{pname}.r"]
        assert np.array_equal(m.apply(r), g[k + ".apply_r"]), tag
        if (k + ".reduced_matvec") in g:
            assert np.array_equal(m.reduced_matvec(g[k + ".y"]), g[k + ".reduced_matvec"])
        if (k + ".coarse_matvec") in g:
            y = g[k + ".y"]
            assert np.array_equal(m.coarse_matvec(y), g[k + ".coarse_matvec"])
            assert np.array_equal(m.interpolate(y), g[k + ".interpolate"])
            assert np.array_equal(m.restrict(r[m.perm_inverse]), g[k + ".restrict"])
        x, rep = orc.fgmres(a, g[f"p.{pname}.b"], m=m.apply, restart=20, rtol=1e-8, max_iters=400)
        assert rep.iterations == int(g[k + ".its"]), tag
        assert rep.converged == bool(g[k + ".converged"])
        assert np.array_equal(rep.residual_history, g[k + ".history"]), tag
        assert rep.final_relres == float(g[k + ".final_relres"])
        assert np.array_equal(x, g[k + ".x"]), tag


def test_krylov_variants(golden_pipeline):
    g = golden_pipeline
    a = g.csr("p.convdiff3d_8.a", Csr)
    b = g["p.convdiff3d_8.b"]
    x, rep = orc.gmres(a, b, restart=15, rtol=1e-9, max_iters=300)
    assert rep.iterations == int(g["g.gmres_none.its"])
    assert np.array_equal(rep.residual_history, g["g.gmres_none.history"])
    assert np.array_equal(x, g["g.gmres_none.x"])
    f0 = orc.ilu0(a)
    x, rep = orc.gmres(a, b, m=f0.solve, restart=10, rtol=1e-9, max_iters=300)
    assert rep.iterations == int(g["g.gmres_ilu0.its"])
    assert np.array_equal(x, g["g.gmres_ilu0.x"])
    assert np.array_equal(orc.fixed_gmres(lambda v: orc.spmv(a, v), b, 5), g["g.fixed_gmres5"])
    assert np.array_equal(orc.fixed_gmres(lambda v: orc.spmv(a, v), b, 4, apply_m=f0.solve),
                          g["g.fixed_gmres4_m"])


# ---------------------------------------------------------------------------
# known answers restated from the reference's own tests


def _path(n):
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 2.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = -1.0
    return orc.csr_from_dense(d)


def test_tridiagonal_pivots_exact():
    """tests/test_factor.py:70-80."""
    u = orc.ilu0(_path(3)).upper.to_dense()
    assert u[0, 0] == 2.0 and u[1, 1] == 1.5 and abs(u[2, 2] - 4.0 / 3.0) < 1e-15


def test_safeguard_rules():
    """tests/test_factor.py:101-109."""
    a = orc.csr_from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]), keep_zeros=True)
    assert orc.ilu0(a).upper.to_dense()[0, 0] == 1e-6
    a = orc.csr_from_dense(np.array([[-1e-9, 1.0], [0.0, 1.0]]))
    assert orc.ilu0(a).upper.to_dense()[0, 0] == -1e-6


def test_partial_ilu_worked_example():
    """tests/test_factor.py:289-303: poisson2d(2,2), two interior nodes."""
    a = orc.poisson2d(2, 2)
    pf = orc.partial_ilu(a, 2, orc.Rule("ilu0"))
    assert np.max(np.abs(pf.s_tilde.to_dense() - np.array([[15 / 4, -1.0], [-1.0, 56 / 15]]))) == 0.0
    assert np.max(np.abs(pf.w_block.to_dense() - np.diag([-1 / 4, -4 / 15]))) == 0.0
    assert np.max(np.abs(pf.z_block.to_dense() + np.eye(2))) == 0.0
    pf = orc.partial_ilu(a, 2, orc.Rule("ilut", 0.0, 4))
    assert np.max(np.abs(pf.s_tilde.to_dense() - np.array([[56.0, -16.0], [-16.0, 56.0]]) / 15)) < 1e-15


def test_milu_identity():
    """tests/test_acceptance.py:73-87: (LU) y = A y - w, here y = 1, w = 0."""
    a = orc.aniso((7, 6, 5), (1.0, 0.3, 0.01))
    f = orc.milu0(a)
    ones = np.ones(a.n_rows)
    assert np.max(np.abs(f.lu_matvec(ones) - orc.spmv(a, ones))) < 1e-11


def test_p1_collapse_bitwise():
    """tests/test_precond.py:108-114,198-205,356-364: one domain -> all equal."""
    a = orc.aniso((6, 5, 4), (1.0, 1.0, 0.01))
    layout = orc.classify_and_order(a, orc.partition(a, 1))
    r = np.random.default_rng(1).standard_normal(a.n_rows)
    outs = [orc.make_preconditioner(pc, a, layout).apply(r) for pc in ("bj", "schur", "rap", "rap-milu")]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_level_schedule_definition():
    """Levels (absent from the reference): the 7-point box law
    of SURVEY.md 8 (full block under natural order: nx+ny+nz-2 levels)."""
    f = orc.ilu0(orc.poisson3d(5, 4, 3))
    lev, ptr, rows = orc.level_schedule(f.lower)
    assert len(ptr) - 1 == 5 + 4 + 3 - 2
    idx = np.arange(60)
    assert np.array_equal(lev, idx % 5 + (idx // 5) % 4 + idx // 20)
    assert np.array_equal(np.sort(rows), idx) and np.all(np.diff(lev[rows]) >= 0)
    levu, ptru, rowsu = orc.level_schedule(f.upper, upper=True)
    assert np.array_equal(levu, (4 - idx % 5) + (3 - (idx // 5) % 4) + (2 - idx // 20))


def test_iteration_counts_baseline_shapes():
    """tests/golden/iterations.json (reference run) at sizes the oracle does in
    seconds: exact iteration counts and final residuals."""
    for rec in iterations():
        dims = tuple(rec["dims"])
        if int(np.prod(dims)) > 40000:
            continue
        a = (orc.convdiff27(*dims, tuple(rec["param"])) if rec["kind"] == "convdiff27"
             else orc.aniso(dims, tuple(rec["param"])))
        out, rep, _ = orc.run(a, dims, rec["p"], rec["precond"], orc.Rule.parse(rec["fill"]))
        assert rep.iterations == rec["its"], rec
        assert rep.final_relres == rec["final_relres"], rec


def test_oracle_library_exports_what_the_wrapper_calls():
    """Every orc_* entry the Python half calls exists in the C half (a stale or partial build must not reach
    bench.py's reference arm)."""
    import re
    from oracle import ddilu_oracle as orc
    lib = orc.lib()
    src = open(orc.__file__).read()
    for name in sorted(set(re.findall(r"orc_[a-z0-9_]+", src))):
        assert hasattr(lib, name), name


def test_threaded_reference_arm_keeps_the_serial_results():
    """bench.py --impl reference may use host threads: SpMV rows and axpy keep every bit, the chunked dot
    agrees to rounding, and threads = 1 is the pinned serial oracle again afterwards."""
    from oracle import ddilu_oracle as orc
    a = orc.aniso((48, 48, 48), (1.0, 1.0, 0.01))
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(a.n_rows), rng.standard_normal(a.n_rows)
    ref_mv, ref_dot = orc.spmv(a, x), orc.vdot(x, y)
    try:
        assert orc.set_threads(4) == 4
        assert np.array_equal(orc.spmv(a, x), ref_mv)
        assert abs(orc.vdot(x, y) - ref_dot) <= 1e-12 * np.sqrt(a.n_rows)
    finally:
        orc.set_threads(1)
    assert orc.vdot(x, y) == ref_dot
