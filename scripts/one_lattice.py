"""A few lattice solves of the interior factors at n^3 (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dims = (n, n, n)
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
m = P.make_preconditioner("schur", a, layout)
f = m._p.interior
r = torch.randn(f.n, dtype=torch.float64, device="cuda")
x = torch.empty_like(r)
for _ in range(3):
    f.lower_solve(r, x)
    f.upper_solve(r, x)
torch.cuda.synchronize()
