"""Cluster sweep on other problem types (thresholds opened): preconditioner applications and iteration counts with and
without it must be identical -- convdiff3d 96^3 (nonsymmetric 7-point), poisson3d 80^3, aniso2d 768^2, convdiff27 48^3 ILUT."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

D.CSWEEP_MIN_AVG_WIDTH = 0
D.CSWEEP_MIN_SMS = 0
cases = [("convdiff3d", (96, 96, 96), 8, "schur", "ilu0"), ("poisson3d", (80, 80, 80), 4, "rap-milu", "ilu0"),
         ("aniso2d", (768, 768), 4, "schur", "ilu0"), ("convdiff27", (48, 48, 48), 8, "schur", "ilut:0.001,20"),
         ("aniso3d", (64, 64, 64), 8, "schur", "iluk:1")]
for kind, dims, p, pc, fill in cases:
    a = getattr(P, kind)(*dims)
    b = P.default_rhs(a)
    res = {}
    for use in (True, False):
        D.USE_CSWEEP = use
        layout = P.classify_and_order(a, P.partition(a, p, dims), p)
        m = P.make_preconditioner(pc, a, layout, P.FillRule.parse(fill))
        f = m._p.interior if pc == "schur" else m._interior
        x, rep = P.fgmres(a, b, m=m.apply)
        res[use] = (rep.iterations, np.asarray(x), np.asarray(m.apply(b)), f._cs is not None, f._cs.k if f._cs else None,
                    f._cs.csize if f._cs else None)
    same = res[True][0] == res[False][0] and np.array_equal(res[True][1], res[False][1]) and np.array_equal(res[True][2], res[False][2])
    print(kind, dims, p, pc, fill, "plan", res[True][3], "k", res[True][4], "cluster", res[True][5], "its", res[True][0], res[False][0],
          "IDENTICAL" if same else "DIFFERENT", flush=True)
    assert same and not res[False][3]
