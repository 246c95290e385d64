"""Runs the five BASELINE.json configurations through the public API: one JSON record per run with setup / solve
seconds, iterations (and the oracle's count where tests/golden holds one), and the achieved GB/s of every
triangular factor pair and of the local SpMV against the measured HBM peak (algorithmic bytes of SURVEY.md 8d;
standalone launches, CUDA events, L2 flushed).

    python scripts/run_configs.py [1 2 3 4 5 ...] > profiles/r2_configs.jsonl
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200.bench import solve_prepared

which = set(sys.argv[1:]) or {"1", "2", "3", "4", "5"}
ILUT = "ilut:0.001,20"
runs = []
if "1" in which:
    runs += [(1, "aniso2d", (128, 128), 1, "bj", "ilu0")]
if "2" in which:
    runs += [(2, "aniso3d", (128,) * 3, p, "bj", "ilu0") for p in (1, 2, 4, 8)]
if "3" in which:
    runs += [(3, "aniso3d", (256,) * 3, 8, pc, "ilu0") for pc in ("schur", "rap", "bj")]
if "4" in which:
    runs += [(4, "aniso3d", (256,) * 3, p, pc, "ilu0") for p in (1, 2, 4, 8) for pc in ("rap-milu", "rap")]
if "5" in which:
    runs += [(5, "convdiff27", (192,) * 3, p, "schur", ILUT) for p in (1, 2, 4, 8)]

try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0
GOLD = {}
try:
    GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "iterations_large.json")))
except Exception:
    pass
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def factor_pairs(m):
    out = []
    if hasattr(m, "_f"):
        out.append(("block", m._f))
    if hasattr(m, "_p"):
        out += [("interior", m._p.interior), ("interface", m._p.schur)]
    if hasattr(m, "_smoother"):
        out += [("smoother", m._smoother), ("interior", m._interior), ("interface", m._schur)]
    return out


def kernel_rates(m):
    rates = {}
    for name, f in factor_pairs(m):
        n = f.n
        if n == 0:
            continue
        r = torch.randn(n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        kind = "cluster-sweep" if f._cs is not None else ("sweep" if f._sw is not None else ("tiled" if f._tl is not None else "syncfree"))
        rec = {"rows": n, "kernel": kind}
        if f._sw is not None:
            t = timed(lambda: f.solve(r, x))
            nb = sum(12 * c.nnz + 4 * (n + 1) + 16 * n for c in (f.lower, f.upper))
            rec.update(LU_us=round(t * 1e6, 1), gbs=round(nb / t / 1e9, 1), frac=round(nb / t / 1e9 / PEAK, 4))
        else:
            for tri, csr, fn in (("L", f.lower, f.lower_solve), ("U", f.upper, f.upper_solve)):
                t = timed(lambda: fn(r, x))
                nb = 12 * csr.nnz + 4 * (n + 1) + 16 * n
                rec.update({f"{tri}_us": round(t * 1e6, 1), f"{tri}_gbs": round(nb / t / 1e9, 1),
                            f"{tri}_frac": round(nb / t / 1e9 / PEAK, 4)})
        rates[name] = rec
    s = m.system
    xv = torch.randn(s.n_loc + s.n_halo, dtype=torch.float64, device="cuda")
    yv = torch.empty(s.n_loc, dtype=torch.float64, device="cuda")
    t = timed(lambda: s.spmv(xv, yv))
    nb = 12 * s.a_loc.nnz + 4 * (s.n_loc + 1) + 16 * s.n_loc
    rates["spmv"] = {"rows": s.n_loc, "nnz": s.a_loc.nnz, "us": round(t * 1e6, 1), "gbs": round(nb / t / 1e9, 1),
                     "frac": round(nb / t / 1e9 / PEAK, 4)}
    return rates


for cfg_no, kind, dims, p, pc, fill in runs:
    spec = P.ProblemSpec(kind, dims)
    t0 = time.perf_counter()
    a, hint = spec.build()
    tb = time.perf_counter() - t0
    ones = torch.ones(a.n_cols, dtype=torch.float64, device="cuda")
    bd = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    D.spmv(a.device(), ones, bd)
    cfg = P.RunConfig(spec, domains=p, precond=pc, fill=P.FillRule.parse(fill))
    try:
        solve_prepared(cfg, a, hint, bd)             # warm-up (allocator, lazy init)
        rec, rep, x, m = solve_prepared(cfg, a, hint, bd)
        rec.update(config=cfg_no, build_s=round(tb, 2), max_err_vs_ones=float(torch.max(torch.abs(x - 1.0)).item()),
                   nnz=a.nnz, ms_per_iteration=round(1e3 * rec["solve_s"] / max(1, rec["its"]), 4))
        g = GOLD.get(f"{kind}_{dims[0]}_{pc}_p{p}")
        if g is not None and g["fill"] == fill:
            rec.update(its_oracle=g["its"], its_parity=abs(rec["its"] - g["its"]) <= 1)
        rec["kernels"] = kernel_rates(m)
        del m, x
    except Exception as exc:  # keep going, like the reference's sweep (bench.py:159-170)
        rec = {"config": cfg_no, "problem": spec.label(), "p": p, "precond": pc, "fill": fill,
               "error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(rec), flush=True)
    del a
    torch.cuda.empty_cache()
