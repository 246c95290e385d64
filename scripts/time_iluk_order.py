import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import factor as F
n = 96
dims = (n,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
rule = P.FillRule.parse("iluk:2")
m = P.make_preconditioner("schur", a, layout, rule)
s = m.system
for blocks in (None, (s.int_ptr, s.ext_ptr), None, (s.int_ptr, s.ext_ptr)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p = F.d_partial_ilu(s.a_dom, s.n_int, rule, factor_schur=True, blocks=blocks)
    torch.cuda.synchronize(); print("interleaved" if blocks else "index order", round(time.perf_counter() - t0, 3), "s", p.interior.lower.nnz)
