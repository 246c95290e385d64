"""Tiled vs sync-free SpTRSV on the factors of the schur preconditioner (aniso3d n^3, p domains).
CUDA events, L2 flushed between repetitions.  Writes JSON lines to gpurun_out/probe_tiled.jsonl."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200._lib import query

PEAK = 6544.7


def timed(fn, reps=10, flush=None):
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
    ap.add_argument("--out", default="gpurun_out/probe_tiled.jsonl")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--no-sell", action="store_true")
    ap.add_argument("--grid-cap", type=int, default=0)
    ap.add_argument("--nap", type=int, default=-1)
    ap.add_argument("--tile", default="")
    ap.add_argument("--kernel", default="")
    ap.add_argument("--slab", default="")
    ap.add_argument("--wpb", type=int, default=0)
    ap.add_argument("--probe", type=int, default=0, help="timing probes of the rotating kernel (csrc/tiled.cu d_tile_probe)")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "a")

    def emit(**kw):
        kw.update(n=args.n, p=args.p, probe=args.probe)
        print(json.dumps(kw), flush=True)
        out.write(json.dumps(kw) + "\n")
        out.flush()

    query("ddilu_tiled_set_tuning", b"grid_cap", args.grid_cap)
    query("ddilu_tiled_set_tuning", b"probe", args.probe)
    if args.nap >= 0:
        query("ddilu_tiled_set_tuning", b"nap_ns", args.nap)
    if args.slab:
        from paper_2303_08881_b200.precond import LocalSystem as _LS
        _LS.SLAB = None if args.slab == "0" else tuple(int(v) for v in args.slab.split(","))
    if args.kernel:
        D.TILE_KERNEL = args.kernel
    if args.tile:
        from paper_2303_08881_b200.precond import LocalSystem
        LocalSystem.TILE_DIMS_3D = tuple(int(v) for v in args.tile.split(","))
    dims = (args.n,) * 3
    a = P.aniso3d(*dims)
    a.device()
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = P.make_preconditioner(args.pc, a, layout)
    torch.cuda.synchronize()
    emit(what="setup", pc=args.pc, setup_s=time.perf_counter() - t0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    pairs = []
    if hasattr(m, "_f"):
        pairs.append(("full", m._f))
    if hasattr(m, "_p"):
        pairs += [("interior", m._p.interior), ("schur", m._p.schur)]
    if hasattr(m, "_smoother"):
        pairs += [("smoother", m._smoother), ("interior", m._interior), ("schur", m._schur)]
    for name, f in pairs:
        n = f.n
        r = torch.randn(n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(r)
        for which, csr, ts in (("L", f.lower, f._tl), ("U", f.upper, f._tu)):
            nbytes = 12 * csr.nnz + 4 * (n + 1) + 16 * n
            rec = dict(what="sptrsv", factor=name, tri=which, rows=n, nnz=csr.nnz, alg_bytes=nbytes,
                       levels=f._lev(which == "U")[1])
            solve_t = (lambda: f.lower_solve(r, x)) if which == "L" else (lambda: f.upper_solve(r, x))
            if ts is not None:
                rec.update(tiles=ts.n_tiles, tile_levels=ts.n_tile_levels, tmax=ts.tmax, emax=ts.emax,
                           stat_max=ts.stat_max, blob_bytes=int(ts.blob.numel()),
                           kind=ts.kind,
                           smem=int(query("ddilu_tiled_smem_bytes", ts.stat_max, ts.tmax, ts.emax)),
                           smem_per_warp=int(query("ddilu_warptile_smem_per_warp", ts.stat_max, ts.tmax, ts.emax)))
                cfgs = [(128, args.wpb)]
                if args.sweep:
                    cfgs = [(128, k) for k in (0, 1, 2, 3)]
                for ct, cps in cfgs:
                    query("ddilu_tiled_set_tuning", b"ctas_per_sm", cps)
                    t = timed(solve_t, flush=flush)
                    rec[f"tiled_c{ct}_k{cps}_us"] = round(t * 1e6, 1)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(50):
                        solve_t()
                    e1.record()
                    torch.cuda.synchronize()
                    rec[f"tiled_c{ct}_k{cps}_chain_us"] = round(e0.elapsed_time(e1) * 1e3 / 50, 1)
                    rec[f"tiled_c{ct}_k{cps}_frac"] = round(nbytes / t / 1e9 / PEAK, 4)
                query("ddilu_tiled_set_tuning", b"ctas_per_sm", 0)
            if ts is not None:
                for cps in ((0, 1, 2, 3) if args.sweep else (0,)):
                    query("ddilu_tiled_set_tuning", b"ctas_per_sm", cps)
                    dbg = torch.zeros(8 * 148 * 8, dtype=torch.int64, device="cuda")
                    query("ddilu_tiled_set_debug", dbg.data_ptr())
                    solve_t()
                    torch.cuda.synchronize()
                    query("ddilu_tiled_set_debug", None)
                    d = dbg.view(-1, 8).cpu().numpy()
                    d = d[d[:, 5] > 0]
                    rec[f"dbg_k{cps}"] = dict(
                        ctas=int(len(d)), life_us=float(d[:, 0].mean() / 1965), wait_tile_us=float(d[:, 1].mean() / 1965),
                        wait_ext_us=float(d[:, 2].mean() / 1965), wait_ext_all_warps_us=float(d[:, 6].mean() / 1965), tiles_us=float(d[:, 3].mean() / 1965),
                        levels=float(d[:, 4].mean()), tiles=float(d[:, 5].mean()),
                        cyc_per_level=float(((d[:, 3] - d[:, 1]) / np.maximum(1, d[:, 4])).mean()))
                query("ddilu_tiled_set_tuning", b"ctas_per_sm", 0)
            if not args.no_sell:
                sched = f.sched_l if which == "L" else f.sched_u
                sell_t = (lambda: D.sptrsv(f.lower, sched, r, x, False, True)) if which == "L" else \
                    (lambda: D.sptrsv(f.upper, sched, r, x, True, False))
                t = timed(sell_t, flush=flush)
                rec.update(sell_us=t * 1e6, sell_frac=nbytes / t / 1e9 / PEAK)
            emit(**rec)
    if args.probe:
        return   # probe 1 reads wrong right-hand sides: timings only
    b = P.default_rhs(a)
    x, rep = P.fgmres(a, b, m=m.apply)
    emit(what="solve", pc=args.pc, its=rep.iterations, solve_s=rep.solve_seconds, relres=rep.final_relres,
         ms_per_it=rep.solve_seconds / max(1, rep.iterations) * 1e3)


if __name__ == "__main__":
    main()
