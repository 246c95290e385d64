"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container only (the GPU box has no /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``ddilu`` from /root/reference/pkg/src, runs the hot path on small
deterministic inputs and writes

    tests/golden/kernels.npz    sparse / ordering / factorisation kernels
    tests/golden/pipeline.npz   partition -> setup -> apply -> fgmres cases
    tests/golden/iterations.json  iteration counts on BASELINE-shaped inputs

The matrices themselves are stored too, so the fixtures are self-contained:
tests feed the stored inputs to the oracle (CPU) and to the CUDA library and
compare with the stored reference outputs.  The 27-point and anisotropic
generators do not exist in the reference; they are built here
through the reference's own ``_stencil_csr`` / ``csr_from_coo``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import ddilu  # noqa: E402
from ddilu import factor as rfac  # noqa: E402
from ddilu import ordering as rord  # noqa: E402
from ddilu import precond as rpre  # noqa: E402
from ddilu import problems as rprob  # noqa: E402
from ddilu import sparse as rsp  # noqa: E402

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


def put_factors(key, f):
    put_csr(key + ".lower", f.lower)
    put_csr(key + ".upper", f.upper)


# ---------------------------------------------------------------------------
# input generators (all deterministic)


def aniso(dims, eps):
    return rprob._stencil_csr(dims, [(-float(e), -float(e)) for e in eps], 2.0 * float(sum(eps)))


def convdiff27(nx, ny, nz, velocity):
    dims = (nx, ny, nz)
    n = nx * ny * nz
    idx = np.arange(n)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    shift = [0.5 * float(velocity[d]) / (dims[d] + 1) for d in range(3)]
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny)
                      & (z + dz >= 0) & (z + dz < nz))
                off = (dx, dy, dz)
                if off == (0, 0, 0):
                    val = 26.0
                else:
                    val = -1.0
                    if sum(abs(o) for o in off) == 1:
                        d = [abs(o) for o in off].index(1)
                        val = -1.0 + shift[d] * off[d]
                r = idx[ok]
                rows.append(r)
                cols.append(r + dx + nx * dy + nx * ny * dz)
                vals.append(np.full(len(r), val))
    return rsp.csr_from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def random_general(rng, n, extra, symmetric_pattern, dominant=True):
    rows = rng.integers(0, n, size=extra)
    cols = rng.integers(0, n, size=extra)
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    dense = np.zeros((n, n))
    dense[rows, cols] = rng.standard_normal(len(rows))
    if symmetric_pattern:
        sym = (dense != 0) | (dense.T != 0)
        hole = sym & (dense == 0)
        dense[hole] = rng.standard_normal(int(hole.sum()))
    np.fill_diagonal(dense, 0.0)
    if dominant:
        np.fill_diagonal(dense, np.sum(np.abs(dense), axis=1) + rng.uniform(1.0, 2.0, n))
    else:
        np.fill_diagonal(dense, rng.uniform(0.5, 2.0, n))
    return rsp.csr_from_dense(dense)


# ---------------------------------------------------------------------------
# kernel-level fixtures


def kernels():
    rng = np.random.default_rng(20231108)
    mats = {
        "rand_sym40": random_general(rng, 40, 90, True),
        "rand_nonsym60": random_general(rng, 60, 200, False),
        "rand_weak30": random_general(rng, 30, 120, True, dominant=False),
        "poisson2d_7x5": rprob.poisson2d(7, 5),
        "poisson3d_5x4x3": rprob.poisson3d(5, 4, 3),
        "convdiff3d_4x5x6": rprob.convdiff3d(4, 5, 6, (3.0, -2.0, 7.0)),
        "aniso3d_6": aniso((6, 6, 6), (1.0, 1.0, 0.01)),
        "cd27_5": convdiff27(5, 5, 5, (10.0, 10.0, 10.0)),
    }
    # a matrix with two components and a missing diagonal entry
    d = np.zeros((9, 9))
    for i in range(4):
        d[i, i + 1] = d[i + 1, i] = -1.0
    for i in range(5, 8):
        d[i, i + 1] = -2.0
        d[i + 1, i] = -0.5
    np.fill_diagonal(d, 3.0)
    d[6, 6] = 0.0
    mats["two_comp9"] = rsp.csr_from_dense(d)
    put("kernels.names", np.array(sorted(mats)))
    for name, a in sorted(mats.items()):
        k = "k." + name
        n = a.n_rows
        put_csr(k + ".a", a)
        x = rng.standard_normal(n)
        put(k + ".x", x)
        put(k + ".spmv", rsp.spmv(a, x))
        put(k + ".vdot", rsp.vdot(x, rsp.spmv(a, x)))
        put_csr(k + ".transpose", rsp.csr_transpose(a))
        perm = rsp.Permutation.from_order(rng.permutation(n))
        put(k + ".perm_forward", perm.forward)
        put_csr(k + ".permuted", rsp.permute_symmetric(a, perm))
        rows = rng.permutation(n)[: max(2, n // 2)]
        put(k + ".sub_rows", rows)
        put_csr(k + ".take_submatrix", rsp.take_submatrix(a, rows, rows))
        srt = np.sort(rows)
        put_csr(k + ".extract_block", rsp.extract_block(a, srt, srt))
        # orderings
        rp, ci = rord._sym_adjacency(a)
        put(k + ".sym_rp", rp)
        put(k + ".sym_ci", ci)
        r = rord.rcm(a)
        put(k + ".rcm_forward", r.forward)
        put(k + ".rcm_inverse", r.inverse)
        for p in (2, 3):
            put(k + f".grow_owner_p{p}", rord.partition(a, p))
        # factorisations
        f0 = rfac.ilu0(a)
        put_factors(k + ".ilu0", f0)
        b = rng.standard_normal(n)
        put(k + ".b", b)
        put(k + ".lsolve", rsp.tri_solve_lower(f0.lower, b, unit_diag=True))
        put(k + ".usolve", rsp.tri_solve_upper(f0.upper, b))
        put(k + ".lu_solve", f0.solve(b))
        put_factors(k + ".milu0", rfac.milu0(a))
        n1 = (2 * n) // 3
        y = rng.uniform(0.5, 1.5, n1)
        z = rng.uniform(0.5, 1.5, n - n1)
        w = 0.1 * rng.standard_normal(n1)
        put(k + ".milu_y", y)
        put(k + ".milu_z", z)
        put(k + ".milu_w", w)
        put_factors(k + ".milu0_vecs", rfac.milu0(a, rfac.MiluVectors(y, z, w)))
        for tag, tau, mf in (("a", 1e-3, 20), ("b", 0.05, 3), ("c", 0.0, n)):
            put_factors(k + f".ilut_{tag}", rfac.ilut(a, tau, mf))
        put(k + ".n_interior", n1)
        for tag, rule, drop in (("ilu0", rfac.FillRule("ilu0"), 0.0),
                                ("ilut", rfac.FillRule("ilut", tau=1e-2, maxfill=5), 0.0),
                                ("ilu0_drop", rfac.FillRule("ilu0"), 0.05),
                                ("ilut_drop", rfac.FillRule("ilut", tau=1e-3, maxfill=8), 0.02)):
            pf = rfac.partial_ilu(a, n1, rule, schur_drop_tol=drop)
            kk = k + ".partial_" + tag
            put_factors(kk + ".interior", pf.interior)
            put_csr(kk + ".w", pf.w_block)
            put_csr(kk + ".z", pf.z_block)
            put_csr(kk + ".s", pf.s_tilde)
            put_factors(kk + ".schur", pf.schur)
        tl = rfac.extract_two_level_blocks(f0, n1)
        put_factors(k + ".twolevel.interior", tl.interior)
        put_csr(k + ".twolevel.w", tl.w_tilde)
        put_csr(k + ".twolevel.z", tl.z_tilde)
        put_factors(k + ".twolevel.schur", tl.schur)
    # structured partitions (ordering.py:171-190) incl. one that falls back to BFS
    grids = [((8, 8), 4), ((6, 4, 4), 8), ((9, 7), 3), ((5, 5, 5), 2), ((12, 12, 12), 8),
             ((7, 3), 5), ((10, 1, 3), 4)]
    put("partition.cases", np.array([json.dumps([list(d), p]) for d, p in grids]))
    for dims, p in grids:
        a = (rprob.poisson2d(*dims) if len(dims) == 2 else rprob.poisson3d(*dims))
        put(f"partition.{'x'.join(map(str, dims))}.p{p}", rord.partition(a, p, grid_hint=dims))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **OUT)
    OUT.clear()


# ---------------------------------------------------------------------------
# pipeline fixtures


def put_precond(k, name, m):
    for d, dom in enumerate(m.domains):
        put(f"{k}.dom{d}.interior_nodes", dom.interior_nodes)
        put(f"{k}.dom{d}.exterior_nodes", dom.exterior_nodes)
    if name == "bj":
        for d, f in enumerate(m.factors):
            put_factors(f"{k}.dom{d}.factors", f)
    elif name == "schur":
        for d, pf in enumerate(m.partial):
            put_factors(f"{k}.dom{d}.interior", pf.interior)
            put_csr(f"{k}.dom{d}.w", pf.w_block)
            put_csr(f"{k}.dom{d}.z", pf.z_block)
            put_csr(f"{k}.dom{d}.s", pf.s_tilde)
            put_factors(f"{k}.dom{d}.schur", pf.schur)
        put_csr(f"{k}.coupling", m.coupling)
    else:
        for d, (f, blk) in enumerate(zip(m.smoother, m.blocks)):
            put_factors(f"{k}.dom{d}.smoother", f)
            put_factors(f"{k}.dom{d}.interior", blk.interior)
            put_csr(f"{k}.dom{d}.w", blk.w_tilde)
            put_csr(f"{k}.dom{d}.z", blk.z_tilde)
            put_factors(f"{k}.dom{d}.schur", blk.schur)
        put_csr(f"{k}.a_perm", m.a_perm)
        put(f"{k}.perm_forward", m.perm.forward)


def pipeline():
    rng = np.random.default_rng(777)
    problems = {
        "aniso2d_16": (aniso((16, 16), (1.0, 0.01)), (16, 16)),
        "aniso3d_10": (aniso((10, 10, 10), (1.0, 1.0, 0.01)), (10, 10, 10)),
        "poisson3d_9x8x7": (rprob.poisson3d(9, 8, 7), (9, 8, 7)),
        "convdiff3d_8": (rprob.convdiff3d(8, 8, 8, (20.0, -10.0, 5.0)), (8, 8, 8)),
        "cd27_8": (convdiff27(8, 8, 8, (10.0, 10.0, 10.0)), (8, 8, 8)),
    }
    cases = []
    for pname in ("aniso2d_16",):
        for p in (1, 4):
            for pc in ("bj", "schur", "rap", "rap-milu"):
                cases.append((pname, p, "grid", pc, "ilu0"))
    for p in (1, 2, 4, 8):
        for pc in ("bj", "schur", "rap", "rap-milu"):
            cases.append(("aniso3d_10", p, "grid", pc, "ilu0"))
    cases += [("poisson3d_9x8x7", 3, "rows", pc, "ilu0") for pc in ("bj", "schur", "rap-milu")]
    cases += [("poisson3d_9x8x7", 6, "grid", pc, "ilu0") for pc in ("schur", "rap")]
    cases += [("convdiff3d_8", 8, "grid", pc, "ilu0") for pc in ("bj", "schur", "rap", "rap-milu")]
    cases += [("cd27_8", 8, "grid", "schur", "ilut:0.001,20"), ("cd27_8", 8, "grid", "bj", "ilut:0.001,20"),
              ("cd27_8", 1, "grid", "bj", "ilut:0.001,20"), ("cd27_8", 8, "grid", "schur", "ilu0"),
              ("cd27_8", 2, "grid", "bj", "ilu0"), ("aniso3d_10", 8, "grid", "schur", "ilut:0.01,5")]
    # appended later (keeps the random draws of the cases above unchanged)
    cases += [("aniso3d_10", 8, "grid", "l1bj", "ilu0"), ("convdiff3d_8", 8, "grid", "l1bj", "ilu0"),
              ("poisson3d_9x8x7", 3, "rows", "l1bj", "ilu0")]
    put("pipeline.problems", np.array(sorted(problems)))
    for pname, (a, hint) in sorted(problems.items()):
        put_csr(f"p.{pname}.a", a)
        put(f"p.{pname}.hint", np.array(hint, dtype=np.int64))
        put(f"p.{pname}.b", rprob.default_rhs(a))
        put(f"p.{pname}.r", rng.standard_normal(a.n_rows))
    names = []
    for pname, p, part, pc, fill in cases:
        a, hint = problems[pname]
        tag = f"{pname}|p{p}|{part}|{pc}|{fill}"
        names.append(tag)
        k = "c." + tag
        owner = (rord.row_block_owner(a.n_rows, p) if part == "rows"
                 else rord.partition(a, p, grid_hint=hint))
        layout = rord.classify_and_order(a, owner)
        put(k + ".owner", owner)
        put(k + ".interior_starts", layout.interior_starts)
        put(k + ".exterior_starts", layout.exterior_starts)
        put(k + ".global_perm_forward", layout.global_perm.forward)
        rule = rfac.FillRule.parse(fill)
        m = rpre.make_preconditioner(pc, a, layout, rule, inner_iters=3)
        put_precond(k, "bj" if pc in ("bj", "l1bj") else ("schur" if pc == "schur" else "rap"), m)
        r = OUT[f"p.{pname}.r"]
        put(k + ".apply_r", m.apply(r))
        if pc == "schur" and layout.n_exterior:
            y = rng.standard_normal(layout.n_exterior)
            put(k + ".y", y)
            put(k + ".reduced_matvec", m.reduced_matvec(y))
        if pc.startswith("rap") and layout.n_exterior:
            y = rng.standard_normal(layout.n_exterior)
            put(k + ".y", y)
            put(k + ".coarse_matvec", m.coarse_matvec(y))
            put(k + ".interpolate", m.interpolate(y))
            put(k + ".restrict", m.restrict(r[m.perm.inverse]))
        b = OUT[f"p.{pname}.b"]
        x, rep = ddilu.fgmres(a, b, m=m.apply, cfg=ddilu.KrylovConfig(restart=20, rtol=1e-8, max_iters=400))
        put(k + ".its", rep.iterations)
        put(k + ".converged", rep.converged)
        put(k + ".history", rep.residual_history)
        put(k + ".final_relres", rep.final_relres)
        put(k + ".x", x)
        print(tag, rep.iterations, rep.converged, f"{rep.final_relres:.3e}")
    put("pipeline.cases", np.array(names))
    # plain gmres / fgmres without a preconditioner and fixed_gmres
    a, _ = problems["convdiff3d_8"]
    b = OUT["p.convdiff3d_8.b"]
    x, rep = ddilu.gmres(a, b, cfg=ddilu.KrylovConfig(restart=15, rtol=1e-9, max_iters=300))
    put("g.gmres_none.its", rep.iterations)
    put("g.gmres_none.history", rep.residual_history)
    put("g.gmres_none.x", x)
    f0 = rfac.ilu0(a)
    x, rep = ddilu.gmres(a, b, m=f0.solve, cfg=ddilu.KrylovConfig(restart=10, rtol=1e-9, max_iters=300))
    put("g.gmres_ilu0.its", rep.iterations)
    put("g.gmres_ilu0.history", rep.residual_history)
    put("g.gmres_ilu0.x", x)
    put("g.fixed_gmres5", ddilu.fixed_gmres(lambda v: rsp.spmv(a, v), b, 5))
    put("g.fixed_gmres4_m", ddilu.fixed_gmres(lambda v: rsp.spmv(a, v), b, 4, apply_m=f0.solve))
    np.savez_compressed(os.path.join(HERE, "pipeline.npz"), **OUT)
    OUT.clear()


# ---------------------------------------------------------------------------
# iteration counts on BASELINE-shaped inputs (restart 50, rtol 1e-8, inner 3)


def iterations():
    out = []
    specs = [
        ("aniso2d", (128, 128), (1.0, 0.01), [(1, "bj", "ilu0")]),
        ("aniso3d", (32, 32, 32), (1.0, 1.0, 0.01),
         [(1, "bj", "ilu0"), (8, "bj", "ilu0"), (8, "schur", "ilu0"), (8, "rap", "ilu0"),
          (8, "rap-milu", "ilu0"), (2, "schur", "ilu0"), (4, "rap-milu", "ilu0")]),
        ("convdiff27", (16, 16, 16), (10.0, 10.0, 10.0),
         [(1, "bj", "ilu0"), (8, "bj", "ilut:0.001,20"), (8, "schur", "ilut:0.001,20"),
          (8, "schur", "ilu0")]),
    ]
    for kind, dims, par, runs in specs:
        a = convdiff27(*dims, par) if kind == "convdiff27" else aniso(dims, par)
        b = rprob.default_rhs(a)
        for p, pc, fill in runs:
            owner = rord.partition(a, p, grid_hint=dims)
            layout = rord.classify_and_order(a, owner)
            m = rpre.make_preconditioner(pc, a, layout, rfac.FillRule.parse(fill), inner_iters=3)
            x, rep = ddilu.fgmres(a, b, m=m.apply, cfg=ddilu.KrylovConfig())
            rec = dict(kind=kind, dims=list(dims), param=list(par), p=p, precond=pc, fill=fill,
                       its=int(rep.iterations), converged=bool(rep.converged),
                       final_relres=float(rep.final_relres), n_exterior=int(layout.n_exterior))
            print(rec)
            out.append(rec)
    with open(os.path.join(HERE, "iterations.json"), "w") as fh:
        json.dump({"source": "reference ddilu 0.1.0, restart 50, rtol 1e-8, inner_iters 3, b = A*1",
                   "runs": out}, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "pipeline", "iterations"]
    for w in which:
        {"kernels": kernels, "pipeline": pipeline, "iterations": iterations}[w]()
