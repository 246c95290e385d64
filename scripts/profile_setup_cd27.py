"""Where the setup of the 27-point ILUT configuration goes (host wall clock, device sync per stage via cProfile)."""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 192
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n,) * 3
a = P.convdiff27(*dims)
a.device()
rule = P.FillRule.parse("ilut:0.001,20")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pr = cProfile.Profile()
    if rep == 1:
        pr.enable()
    m = P.make_preconditioner("schur", a, layout, rule)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if rep == 1:
        pr.disable()
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(22)
        print(s.getvalue()[:4500])
    print(f"rep {rep}: layout {t1 - t0:.3f} s, preconditioner {t2 - t1:.3f} s", flush=True)
    del m
