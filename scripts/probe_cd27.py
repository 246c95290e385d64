"""convdiff27 n^3, schur + ILUT(1e-3, 20), p domains: which kernel serves the interface factors, solve timings."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n,) * 3
a = P.convdiff27(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
torch.cuda.synchronize()
t0 = time.perf_counter()
m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
torch.cuda.synchronize()
setup = time.perf_counter() - t0
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


rec = {"n": n, "p": p, "setup_s": round(setup, 3), "block_window": D.USE_BLOCK_WINDOW}
for name, f in (("interior", m._p.interior), ("interface", m._p.schur)):
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(r)
    kind = "sweep" if f._sw is not None else ("window" if f._bw is not None else ("tiled" if f._tl is not None else "syncfree"))
    rl = (f.lower.rp[1:] - f.lower.rp[:-1])
    ru = (f.upper.rp[1:] - f.upper.rp[:-1])
    rec[name] = {"rows": f.n, "kernel": kind, "levels": [f._lev(False)[1], f._lev(True)[1]],
                 "max_row": [int(rl.max().item()), int(ru.max().item())], "nnz": [f.lower.nnz, f.upper.nnz],
                 "L_us": round(timed(lambda: f.lower_solve(r, x)) * 1e6, 1),
                 "U_us": round(timed(lambda: f.upper_solve(r, x)) * 1e6, 1)}
b = P.default_rhs(a)
x, rep = P.fgmres(a, b, m=m.apply)
rec.update(its=rep.iterations, solve_s=round(rep.solve_seconds, 3), converged=rep.converged)
print(json.dumps(rec))
