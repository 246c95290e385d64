"""Long-row cluster sweep against the alternative (sync-free kernels) on the interior factors: solve seconds and
interior L / U microseconds with and without it.   python scripts/time_csweep_long.py problem n p fill"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

kind, n, p, fill = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
dims = (n,) * 3
a = getattr(P, kind)(*dims)
b = P.default_rhs(a)
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for use in (True, False, True, False):
    D.CSWEEP_LONG_ROWS = use
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = P.make_preconditioner("schur", a, layout, P.FillRule.parse(fill))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    x, rep = P.fgmres(a, b, m=m.apply)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    f = m._p.interior
    r = torch.randn(f.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(r)
    print(kind, n, p, fill, "long-row plan" if f._cs is not None else "no plan", "setup", round(t1 - t0, 3), "solve", round(t2 - t1, 3),
          "its", rep.iterations, "L/U us", round(timed(lambda: f.lower_solve(r, y)), 1), round(timed(lambda: f.upper_solve(r, y)), 1), flush=True)
    del m
