"""Block sweep (csrc/sweep.cu) vs the tiled kernel on the interface factors (aniso3d n^3, p domains): CUDA-event
timings with the L2 flushed, per-block cycle counters.  JSON lines -> gpurun_out/probe_sweep.jsonl."""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200._lib import query
from paper_2303_08881_b200.factor import solve_with_product


def timed(fn, reps=20, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--pc", default="schur")
    ap.add_argument("--out", default="gpurun_out/probe_sweep.jsonl")
    ap.add_argument("--tag", default="")
    ap.add_argument("--wsleep", type=int, default=20)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--only-sweep", action="store_true")
    ap.add_argument("--rpt", type=int, default=0)
    ap.add_argument("--sets", type=int, default=0)
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "a")

    def emit(**kw):
        kw.update(n=args.n, p=args.p, tag=args.tag, wsleep=args.wsleep, flags=args.flags, threads=args.threads)
        print(json.dumps(kw), flush=True)
        out.write(json.dumps(kw) + "\n")
        out.flush()

    dims = (args.n,) * 3
    a = P.aniso3d(*dims)
    a.device()
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    query("ddilu_sweep_set_tuning", args.wsleep, args.flags)
    if args.threads:
        D.SWEEP_MAX_THREADS = args.threads
    if args.rpt:
        D.SWEEP_ROWS_PER_THREAD = args.rpt
    if args.sets:
        D.SWEEP_SETS = args.sets
    for sweep in ((True,) if args.only_sweep else (True, False)):
        D.USE_SWEEP = sweep
        m = P.make_preconditioner(args.pc, a, layout)
        f = m._p.schur if args.pc == "schur" else m._schur
        n = f.n
        torch.manual_seed(1)
        r = torch.randn(n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        alg = sum(12 * c.nnz + 4 * (n + 1) + 16 * n for c in (f.lower, f.upper))
        rec = dict(what="interface", sweep=sweep, rows=n, nnz_l=f.lower.nnz, nnz_u=f.upper.nnz, alg_bytes=alg)
        if sweep:
            sp = f._sw
            rec.update(k=sp.k, window=sp.window, stages=sp.stages, nct=sp.nct, rpt=sp.rpt, sets=sp.sets, levels=list(sp.n_levels), blocks=sp.n_blocks,
                       smem=int(query("ddilu_sweep_smem_bytes", sp.k, sp.stages, sp.window, sp.max_lev)))
        for name, fn in (("L", lambda: f.lower_solve(r, x)), ("U", lambda: f.upper_solve(r, x)), ("LU", lambda: f.solve(r, x))):
            for fl in (True, False):
                rec[f"{name}_{'cold' if fl else 'warm'}_us"] = round(timed(fn, flush=flush if fl else None) * 1e6, 1)
        if sweep:
            D.sweep_rhs(sp, False, r)
            rec["LU_kernel_only_warm_us"] = round(timed(lambda: D.sweep_solve(sp, 3, x)) * 1e6, 1)
            rec["LU_kernel_only_cold_us"] = round(timed(lambda: D.sweep_solve(sp, 3, x), flush=flush) * 1e6, 1)
            rec["rhs_kernel_warm_us"] = round(timed(lambda: D.sweep_rhs(sp, False, r)) * 1e6, 1)
            if args.pc == "schur":
                s = m.system
                y = torch.randn(s.n_ext + s.n_halo, dtype=torch.float64, device="cuda")
                o = torch.empty(s.n_ext, dtype=torch.float64, device="cuda")
                rec["reduced_matvec_warm_us"] = round(timed(lambda: solve_with_product(f, m._coupling, y, None, 0, o, add=y)) * 1e6, 1)
                rec["reduced_matvec_cold_us"] = round(timed(lambda: solve_with_product(f, m._coupling, y, None, 0, o, add=y), flush=flush) * 1e6, 1)
            dbg = torch.zeros(sp.n_blocks * 64, dtype=torch.int64, device="cuda")
            query("ddilu_sweep_set_debug", dbg.data_ptr())
            flush.fill_(1.0)
            D.sweep_solve(sp, 3, x)
            torch.cuda.synchronize()
            query("ddilu_sweep_set_debug", None)
            d = dbg.view(-1, 16).cpu().numpy()[::4]
            rec["dbg_cycles_L_U_wait__opsL_barL_finL__opsU_barU_finU"] = [[int(v) for v in row[:11]] for row in d[:3]]
            rec["cycles_per_level_L_U"] = [round(float(d[:, 0].mean()) / sp.n_levels[0], 1), round(float(d[:, 1].mean()) / sp.n_levels[1], 1)]
        elif args.pc == "schur":
            s = m.system
            y = torch.randn(s.n_ext + s.n_halo, dtype=torch.float64, device="cuda")
            o = torch.empty(s.n_ext, dtype=torch.float64, device="cuda")
            rec["reduced_matvec_warm_us"] = round(timed(lambda: m._reduced_matvec(y, o)) * 1e6, 1)
            rec["reduced_matvec_cold_us"] = round(timed(lambda: m._reduced_matvec(y, o), flush=flush) * 1e6, 1)
        emit(**rec)
        del m


if __name__ == "__main__":
    main()
