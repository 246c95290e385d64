"""A few fused interface solves (csrc/sweep.cu) for an ncu capture: python scripts/one_sweep.py [n] [p]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n, n, n)
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
m = P.make_preconditioner("schur", a, layout)
f = m._p.schur
r = torch.randn(f.n, dtype=torch.float64, device="cuda")
x = torch.empty_like(r)
for _ in range(6):
    f.solve(r, x)
torch.cuda.synchronize()
print("done", f.n, f._sw.nct, f._sw.sets)
