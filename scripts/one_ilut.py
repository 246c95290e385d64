"""One ILUT(1e-3, 20) factorisation of convdiff27 n^3 (p subdomains, schur) for an ncu capture of ilut_kernel."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n,) * 3
a = P.convdiff27(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
    torch.cuda.synchronize()
    print("setup", round(time.perf_counter() - t0, 3))
