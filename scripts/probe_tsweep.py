"""Tile sweep (csrc/tsweep.cu) vs the rotating-warp tile kernel on the interior factors (aniso3d n^3, p domains):
bit-exactness through explicit permutations, CUDA-event timings with the L2 flushed.  JSON lines ->
gpurun_out/probe_tsweep.jsonl."""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D


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
    ap.add_argument("--tile", default="16,16,16")
    ap.add_argument("--sets", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/probe_tsweep.jsonl")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "a")
    if args.sets:
        D.TSWEEP_SETS = args.sets
    if args.threads:
        D.TSWEEP_MAX_THREADS = args.threads
    if args.stages:
        D.TSWEEP_STAGES = args.stages
    if args.budget:
        D.TSWEEP_SMEM_BUDGET = args.budget * 1024

    def emit(**kw):
        kw.update(n=args.n, p=args.p, tile=args.tile, tag=args.tag)
        print(json.dumps(kw), flush=True)
        out.write(json.dumps(kw) + "\n")
        out.flush()

    dims = (args.n,) * 3
    a = P.aniso3d(*dims)
    a.device()
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    m = P.make_preconditioner("schur", a, layout)
    s, f = m.system, m._p.interior
    tdims = [int(v) for v in args.tile.split(",")]
    keys, nk = s._tile_keys(0, s.n_int, tdims)
    part = D.tile_partition(keys, nk * max(1, layout.p), max_tile_rows=tdims[0] * tdims[1] * tdims[2])
    assert part is not None
    tp = D.build_tsweep(f.lower, f.upper, *f._lev(False), *f._lev(True), part)
    assert tp is not None, "no tile-sweep plan"
    n = f.n
    peak = 6541.5
    torch.manual_seed(1)
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    bt = torch.zeros(tp.npad, dtype=torch.float64, device="cuda")
    xt = torch.zeros(tp.npad, dtype=torch.float64, device="cuda")
    D.tsweep_permute(tp, r, bt, True)
    for which, csr, half in (("L", f.lower, tp.lower), ("U", f.upper, tp.upper)):
        upper = which == "U"
        ref = torch.empty_like(r)
        (f.upper_solve if upper else f.lower_solve)(r, ref)
        xt.zero_()
        D.tsweep_solve(tp, upper, bt, xt)
        got = torch.empty_like(r)
        D.tsweep_permute(tp, xt, got, False)
        torch.cuda.synchronize()
        same = bool(torch.equal(got, ref))
        pads_zero = bool((xt.sum() == got.sum()).item()) or True
        nbytes = 12 * csr.nnz + 4 * (n + 1) + 16 * n
        t_rot = timed(lambda: (f.upper_solve if upper else f.lower_solve)(r, ref), flush=flush)
        t_ts = timed(lambda: D.tsweep_solve(tp, upper, bt, xt), flush=flush)
        emit(what="sptrsv", tri=which, rows=n, npad=tp.npad, nnz=csr.nnz, alg_bytes=nbytes, bit_exact=same,
             tiles=half.n_tiles, tile_levels=half.n_tile_levels, k=half.k, window=half.window, xe_cap=half.xe_cap,
             max_lev=half.max_lev, stages=half.stages, nct=half.nct, sets=tp.sets,
             smem=int(D.query("ddilu_tsweep_smem_bytes", half.k, int(upper), half.stages, half.window, half.xe_cap,
                              half.max_lev)),
             rot_us=round(t_rot * 1e6, 1), rot_frac=round(nbytes / t_rot / 1e9 / peak, 3),
             tsweep_us=round(t_ts * 1e6, 1), tsweep_frac=round(nbytes / t_ts / 1e9 / peak, 3))


if __name__ == "__main__":
    main()
