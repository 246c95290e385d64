"""One schur-preconditioned FGMRES solve through the public API (for ncu captures of the kernels of the inner
GMRES: `ncu -k regex:"mgs_small_step|norm_scale_small" ... python scripts/one_schur_solve.py 256`)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dims = (n,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
m = P.make_preconditioner("schur", a, layout)
x, rep = P.fgmres(a, P.default_rhs(a), m=m.apply)
torch.cuda.synchronize()
print("its", rep.iterations, rep.converged, rep.final_relres)
