"""Runs the BASELINE.json configurations once each through the public API and prints one JSON record per run."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

runs = []
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "aniso"):
    runs += [("aniso2d", (128, 128), 1, "bj", "ilu0")]
    runs += [("aniso3d", (128,) * 3, p, "bj", "ilu0") for p in (1, 2, 4, 8)]
    runs += [("aniso3d", (256,) * 3, 8, pc, "ilu0") for pc in ("bj", "schur", "rap", "rap-milu")]
    runs += [("aniso3d", (256,) * 3, p, "rap-milu", "ilu0") for p in (1, 2, 4)]
if which in ("all", "cd27"):
    runs += [("convdiff27", (48,) * 3, 8, "schur", "ilut:0.001,20"), ("convdiff27", (96,) * 3, 8, "schur", "ilut:0.001,20"),
             ("convdiff27", (96,) * 3, 8, "bj", "ilut:0.001,20")]
if which in ("all", "cd27big"):
    runs += [("convdiff27", (192,) * 3, p, "schur", "ilut:0.001,20") for p in (8, 1)]
for kind, dims, p, pc, fill in runs:
    spec = P.ProblemSpec(kind, dims)
    t0 = time.perf_counter()
    a, hint = spec.build()
    tb = time.perf_counter() - t0
    ones = torch.ones(a.n_cols, dtype=torch.float64, device="cuda")
    from paper_2303_08881_b200 import device as D
    bd = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    D.spmv(a.device(), ones, bd)
    cfg = P.RunConfig(spec, domains=p, precond=pc, fill=P.FillRule.parse(fill))
    from paper_2303_08881_b200.bench import solve_prepared
    try:
        solve_prepared(cfg, a, hint, bd)             # warm-up (allocator, lazy init)
        rec, rep, x, m = solve_prepared(cfg, a, hint, bd)
        err = float(torch.max(torch.abs(x - 1.0)).item())
        rec.update(build_s=tb, max_err_vs_ones=err, nnz=a.nnz)
    except Exception as exc:  # keep going, like the reference's sweep (bench.py:159-170)
        rec = {"problem": spec.label(), "p": p, "precond": pc, "fill": fill, "error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(rec), flush=True)
    del a
    torch.cuda.empty_cache()
