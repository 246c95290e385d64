"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck); logs -> profiles/r2_sanitizer_*.log.

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py [tiled|sweep|mgs|smallstep|ilut|rcm|pipeline ...]

tiled: sptrsv_tiled on interior + interface factors; csweep: the cluster sweep on interior factors (clusters of 4 and
of the largest size that fits, a 32^3 block on one CTA: levels in several steps); sweep: the block sweep (L, U, fused, with product and add);
sweep_long: its long-row instances on 27-point ILUT interface factors (+ a whole solve: device-side inner-solve
arithmetic); spgemm: sparse_matmul;
mgs: ddilu_mgs_block over ragged lengths and block shapes; ilut: ilut_kernel (27-point, fill);
rcm: cm_order_kernel on several disconnected blocks; pipeline: one schur + rap-milu FGMRES solve."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

which = sys.argv[1:] or ["tiled", "csweep", "sweep", "sweep_long", "mgs", "ilut", "rcm", "spgemm", "pipeline"]
dims = (20, 18, 17)
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 4, dims), 4)

if "tiled" in which:
    D.USE_SWEEP = False
    m = P.make_preconditioner("schur", a, layout)
    for f in (m._p.interior, m._p.schur):
        assert f._tl is not None and f._tu is not None
        r = torch.randn(f.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        f.lower_solve(r, x)
        f.upper_solve(r, x)
        torch.cuda.synchronize()
        print("tiled", f._tl.kind, f.n, float(x.abs().max()))
    D.USE_SWEEP = True

if "csweep" in which:
    old = D.CSWEEP_MIN_AVG_WIDTH, D.CSWEEP_MIN_SMS, D.CSWEEP_CLUSTER
    D.CSWEEP_MIN_AVG_WIDTH = D.CSWEEP_MIN_SMS = 0
    for cluster in (4, 16, 1):
        D.CSWEEP_CLUSTER = cluster
        aa, lay = a, layout
        if cluster == 1:
            d1 = (32, 32, 32)
            aa = P.aniso3d(*d1)
            lay = P.classify_and_order(aa, P.partition(aa, 1, d1), 1)
        m = P.make_preconditioner("schur", aa, lay)
        f = m._p.interior
        assert f._cs is not None
        r = torch.randn(f.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        f.lower_solve(r, x)
        f.upper_solve(r, x)
        f.solve(r, x)
        torch.cuda.synchronize()
        print("csweep", f.n, f._cs.csize, f._cs.lower.max_steps, f._cs.lower.depth, float(x.abs().max()))
    # the 20-slot instance: 27-point ILUT interior factors (step table in global memory, operands as one block per step)
    D.CSWEEP_CLUSTER = 8
    d27 = (14, 13, 12)
    a27 = P.convdiff27(*d27)
    lay27 = P.classify_and_order(a27, P.partition(a27, 4, d27), 4)
    m = P.make_preconditioner("schur", a27, lay27, P.FillRule.parse("ilut:0.001,20"))
    f = m._p.interior
    assert f._cs is not None and f._cs.k == 20
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(r)
    f.lower_solve(r, x)
    f.upper_solve(r, x)
    torch.cuda.synchronize()
    print("csweep long rows", f.n, f._cs.csize, f._cs.lower.max_steps, float(x.abs().max()))
    D.CSWEEP_MIN_AVG_WIDTH, D.CSWEEP_MIN_SMS, D.CSWEEP_CLUSTER = old

if "sweep" in which:
    from paper_2303_08881_b200.factor import solve_with_product
    m = P.make_preconditioner("schur", a, layout)
    f, s = m._p.schur, m.system
    assert f._sw is not None
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(r)
    f.lower_solve(r, x)
    f.upper_solve(r, x)
    f.solve(r, x)
    y = torch.randn(s.n_ext + s.n_halo, dtype=torch.float64, device="cuda")
    solve_with_product(f, m._coupling, y, None, 0, x, add=y)
    torch.cuda.synchronize()
    print("sweep", f.n, f._sw.nct, f._sw.sets, float(x.abs().max()))

if "sweep_long" in which:
    d27 = (14, 13, 12)
    a27 = P.convdiff27(*d27)
    lay27 = P.classify_and_order(a27, P.partition(a27, 4, d27), 4)
    m = P.make_preconditioner("schur", a27, lay27, P.FillRule.parse("ilut:0.001,20"))
    f = m._p.schur
    assert f._sw is not None and f._sw.k > 8
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(r)
    f.lower_solve(r, x)
    f.upper_solve(r, x)
    f.solve(r, x)
    x2, rep = P.fgmres(a27, P.default_rhs(a27), m=m.apply)
    torch.cuda.synchronize()
    print("sweep_long", f.n, f._sw.k, f._sw.nct, f._sw.sets, f._sw.stages, rep.iterations, rep.converged)

if "spgemm" in which:
    g = P.poisson3d(7, 6, 5)
    c = P.sparse_matmul(g, g)
    print("spgemm", c.nnz)

if "mgs" in which:
    red = D.Reducer()
    for n in (1, 33, 1000, 40001):
        ld = (n + 1) & ~1
        V = torch.randn((9, ld), dtype=torch.float64, device="cuda")
        w = torch.randn(ld, dtype=torch.float64, device="cuda")
        raw = torch.zeros((4, 40), dtype=torch.float64, device="cuda")
        h = torch.zeros(16, dtype=torch.float64, device="cuda")
        for kn in (1, 2, 3, 4):
            red.mgs_block(n, ld, 0, None, None, None, w, kn, V[0], raw[0])
            red.mgs_block(n, ld, kn, V[0], raw[0], h[:kn], w, min(4, 8 - kn), V[kn], raw[1])
            red.mgs_block(n, ld, min(4, 8 - kn), V[kn], raw[1], h[kn:kn + min(4, 8 - kn)], w, 0, None, h[9:10])
    torch.cuda.synchronize()
    print("mgs ok")

if "smallstep" in which:
    # the one-launch Arnoldi step of the inner GMRES (cooperative grid, two grid barriers), repeated on one workspace
    red = D.Reducer()
    for n in (1, 33, 1000, 40001, 390152):
        ld = (n + 1) & ~1
        V = torch.randn((6, ld), dtype=torch.float64, device="cuda")
        raw = torch.zeros(40, dtype=torch.float64, device="cuda")
        h = torch.zeros(16, dtype=torch.float64, device="cuda")
        for k in (1, 2, 3, 4):
            for rep in range(2):
                w = torch.randn(ld, dtype=torch.float64, device="cuda")
                red.mgs_small_step(n, ld, k, V, w, h, V[k], raw, reverse_dots=True, reverse_update=False)
    torch.cuda.synchronize()
    print("smallstep ok", float(h[0]))

if "ilut" in which:
    a27 = P.convdiff27(9, 8, 7)
    f = P.ilut(a27, 1e-3, 10)
    pf = P.partial_ilu(a27, 300, P.FillRule.parse("ilut:0.001,8"))
    print("ilut", f.lower.nnz, f.upper.nnz, pf.s_tilde.nnz)

if "rcm" in which:
    lay8 = P.classify_and_order(a, P.partition(a, 8, dims), 8)
    m = P.make_preconditioner("bj", a, lay8)
    print("rcm", [len(d.interior_nodes) for d in m.domains])
    print("rcm single", int(P.rcm(P.poisson2d(13, 11)).forward.sum()))

if "pipeline" in which:
    b = P.default_rhs(a)
    for pc in ("schur", "rap-milu"):
        m = P.make_preconditioner(pc, a, layout)
        x, rep = P.fgmres(a, b, m=m.apply)
        print("pipeline", pc, rep.iterations, rep.converged)
