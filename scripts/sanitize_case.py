"""Small tiled solves for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

kern = sys.argv[1] if len(sys.argv) > 1 else "rot"
D.TILE_KERNEL = kern
dims = (20, 18, 17)
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 4, dims), 4)
m = P.make_preconditioner("schur", a, layout)
for f in (m._p.interior, m._p.schur):
    assert f._tl is not None and f._tu is not None
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(r)
    f.lower_solve(r, x)
    f.upper_solve(r, x)
    torch.cuda.synchronize()
    print(kern, f._tl.kind, f.n, float(x.abs().max()))
