"""Lattice vs rotating-warp SpTRSV on the interior factors (aniso3d n^3, p domains): correctness against the
rotating kernel, then CUDA-event timings with the L2 flushed.  JSON lines -> gpurun_out/probe_lattice.jsonl."""

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
    ap.add_argument("--tile", default="8,8,8")
    ap.add_argument("--debug", action="store_true", help="per-warp cycle counters of the lattice kernel")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--out", default="gpurun_out/probe_lattice.jsonl")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "a")

    def emit(**kw):
        kw.update(n=args.n, p=args.p, tile=args.tile)
        print(json.dumps(kw), flush=True)
        out.write(json.dumps(kw) + "\n")
        out.flush()

    from paper_2303_08881_b200.precond import LocalSystem
    LocalSystem.TILE_DIMS_3D = tuple(int(v) for v in args.tile.split(","))
    dims = (args.n,) * 3
    a = P.aniso3d(*dims)
    a.device()
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    peak = 6544.3
    res = {}
    for lattice in (True, False):
        D.USE_LATTICE = lattice
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = P.make_preconditioner(args.pc, a, layout)
        torch.cuda.synchronize()
        emit(what="setup", lattice=lattice, setup_s=time.perf_counter() - t0)
        f = m._p.interior if hasattr(m, "_p") else (m._f if hasattr(m, "_f") else m._interior)
        n = f.n
        torch.manual_seed(1)
        r = torch.randn(n, dtype=torch.float64, device="cuda")
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
        for which, csr, ts in (("L", f.lower, f._tl), ("U", f.upper, f._tu)):
            x = torch.empty_like(r)
            solve = (lambda: f.lower_solve(r, x)) if which == "L" else (lambda: f.upper_solve(r, x))
            solve()
            torch.cuda.synchronize()
            res[(lattice, which)] = x.clone()
            nbytes = 12 * csr.nnz + 4 * (n + 1) + 16 * n
            rec = dict(what="sptrsv", lattice=lattice, kind=getattr(ts, "kind", None), tri=which, rows=n, nnz=csr.nnz,
                       alg_bytes=nbytes, tiles=getattr(ts, "n_tiles", None), tile_levels=getattr(ts, "n_tile_levels", None),
                       blob_bytes=int(ts.blob.numel()) if ts is not None else None)
            if lattice and ts is not None and ts.kind == "lattice":
                rec.update(blkmax=ts.blkmax, tmax=ts.tmax, xemax=ts.xemax,
                           smem=int(query("ddilu_lattice_smem_bytes", ts.blkmax, ts.tmax, ts.xemax)))
                for c in (int(v) for v in args.ctas.split(",")):
                    query("ddilu_lattice_set_tuning", b"ctas_per_sm", c)
                    t = timed(solve, flush=flush)
                    rec[f"c{c}_us"] = round(t * 1e6, 1)
                    rec[f"c{c}_frac"] = round(nbytes / t / 1e9 / peak, 3)
                query("ddilu_lattice_set_tuning", b"ctas_per_sm", 0)
                if args.debug:
                    dbg = torch.zeros(148 * 32 * 8, dtype=torch.int64, device="cuda")
                    query("ddilu_lattice_set_debug", dbg.data_ptr())
                    flush.fill_(1.0)
                    solve()
                    torch.cuda.synchronize()
                    query("ddilu_lattice_set_debug", None)
                    d = dbg.view(-1, 8).cpu().numpy()
                    d = d[d[:, 7] > 0]
                    names = ["life", "rhs_wait", "dep_wait", "gather", "steps", "fence", "next_block", "tiles"]
                    rec["dbg_warps"] = int(len(d))
                    rec["dbg_mean_kcycles"] = {k: round(float(d[:, i].mean()) / 1e3, 1) for i, k in enumerate(names)}
                    rec["dbg_per_tile_cycles"] = {k: round(float((d[:, i] / d[:, 7]).mean()), 0) for i, k in enumerate(names[:-1])}
            else:
                t = timed(solve, flush=flush)
                rec["us"] = round(t * 1e6, 1)
                rec["frac"] = round(nbytes / t / 1e9 / peak, 3)
            emit(**rec)
        del m
    for which in ("L", "U"):
        same = torch.equal(res[(True, which)], res[(False, which)])
        emit(what="bit_exact_vs_rot", tri=which, same=bool(same))


if __name__ == "__main__":
    main()
