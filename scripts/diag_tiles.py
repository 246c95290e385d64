"""Which factors tile, and how fast their solves are (diagnostics)."""
import sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dims = (n,) * 3
a = P.aniso3d(*dims)
for pc, p in (("bj", 1), ("bj", 2), ("bj", 4), ("bj", 8), ("rap", 8), ("rap-milu", 2)):
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    m = P.make_preconditioner(pc, a, layout)
    pairs = []
    if hasattr(m, "_f"):
        pairs.append(("full", m._f))
    if hasattr(m, "_smoother"):
        pairs += [("smoother", m._smoother), ("interior", m._interior), ("schur", m._schur)]
    for name, f in pairs:
        if f.n == 0:
            continue
        r = torch.randn(f.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        out = dict(pc=pc, p=p, factor=name, rows=f.n, tiled_l=f._tl is not None, tiled_u=f._tu is not None,
                   levels_l=f._lev(False)[1], levels_u=f._lev(True)[1])
        if f._tl is not None:
            out.update(tiles=f._tl.n_tiles, tile_levels=f._tl.n_tile_levels, tmax=f._tl.tmax, emax=f._tl.emax)
        for which, fn in (("L", f.lower_solve), ("U", f.upper_solve)):
            for _ in range(3):
                fn(r, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn(r, x)
            e1.record()
            torch.cuda.synchronize()
            out[which + "_us"] = round(e0.elapsed_time(e1) * 100, 1)
        print(json.dumps(out), flush=True)
    del m
