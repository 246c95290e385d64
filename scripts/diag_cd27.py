"""Do the ILUT factors of the 27-point problem tile? (diagnostics)"""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
dims = (n,) * 3
a = P.convdiff27(*dims)
for p in (8, 1):
    layout = P.classify_and_order(a, P.partition(a, p, dims), p)
    m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
    for name, f in (("interior", m._p.interior), ("schur", m._p.schur)):
        if f.n == 0:
            continue
        r = torch.randn(f.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        out = dict(p=p, factor=name, rows=f.n, nnz_l=f.lower.nnz, nnz_u=f.upper.nnz, tiled_l=f._tl is not None,
                   tiled_u=f._tu is not None, levels_l=f._lev(False)[1], levels_u=f._lev(True)[1])
        if f._tl is not None:
            out.update(kind=f._tl.kind, tiles=f._tl.n_tiles, tile_levels=f._tl.n_tile_levels, tmax=f._tl.tmax,
                       emax=f._tl.emax, kmax=f._tl.kmax)
        for which, fn in (("L", f.lower_solve), ("U", f.upper_solve)):
            for _ in range(2):
                fn(r, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn(r, x)
            e1.record()
            torch.cuda.synchronize()
            out[which + "_us"] = round(e0.elapsed_time(e1) * 200, 1)
        print(json.dumps(out), flush=True)
