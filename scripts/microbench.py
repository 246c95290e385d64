"""Kernel micro-benchmarks on one B200: SpTRSV (with tuning sweep), SpMV, fused
MGS pass, dot.  CUDA events on the launching stream, L2 flushed between
repetitions, algorithmic bytes per SURVEY.md 8d.  Writes JSON lines."""

import argparse
import json
import sys
import os
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
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--p", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/microbench.jsonl")
    ap.add_argument("--sweep", action="store_true")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "a")

    def emit(**kw):
        kw.update(n=args.n, p=args.p)
        print(json.dumps(kw))
        out.write(json.dumps(kw) + "\n")
        out.flush()

    dims = (args.n,) * 3
    t0 = time.perf_counter()
    a = P.aniso3d(*dims)
    t_gen = time.perf_counter() - t0
    a.device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    torch.cuda.synchronize()
    t_layout = time.perf_counter() - t0
    t0 = time.perf_counter()
    m = P.bj_setup(a, layout)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    emit(what="setup", gen_s=t_gen, layout_s=t_layout, bj_setup_s=t_setup)
    s, f = m.system, m._f
    n = s.n_loc
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    t = torch.empty_like(r)
    z = torch.empty_like(r)
    nl, nu = f.lower.nnz, f.upper.nnz
    lbytes = 12 * nl + 4 * (n + 1) + 16 * n
    ubytes = 12 * nu + 4 * (n + 1) + 16 * n
    emit(what="factors", rows=n, nnz_l=nl, nnz_u=nu, levels_l=f.sched_l.n_levels, levels_u=f.sched_u.n_levels,
         slots_l=f.sched_l.n_slots)
    configs = [(3, -1, True, 0, True)]
    if args.sweep:
        configs = [(3, mk, True, 0, True) for mk in (4, 2, 3, 6, 7, 0)] + [(6, 3, True, 0, True), (3, 1003, True, 0, True)]
    for bps, sleep, use_sell, pipe, gwait in configs:
        D.USE_SELL = use_sell
        D.USE_GWAIT = gwait
        if sleep >= 0:
            query("ddilu_set_tuning", b"trsv_stage_mask", sleep % 1000)
            query("ddilu_set_tuning", b"trsv_far_sleep_ns", 1000 if sleep >= 1000 else 400)
        query("ddilu_set_tuning", b"trsv_pipe", pipe)
        query("ddilu_set_tuning", b"trsv_pipe_warps_per_sm" if pipe else b"trsv_blocks_per_sm", bps)
        tl, tlmin = timed(lambda: f.lower_solve(r, t), flush=flush)
        tu, tumin = timed(lambda: f.upper_solve(t, z), flush=flush)
        emit(what="sptrsv", kernel=("pipe" if pipe else ("sellw" if gwait else "sell")) if use_sell else "csr", blocks_per_sm=bps, sleep_ns=sleep, lower_s=tl, upper_s=tu, lower_min_s=tlmin,
             upper_min_s=tumin, lower_gbs=lbytes / tl / 1e9, upper_gbs=ubytes / tu / 1e9,
             lower_frac=lbytes / tl / 1e9 / PEAK, upper_frac=ubytes / tu / 1e9 / PEAK,
             hop_us_lower=tl / f.sched_l.n_levels * 1e6, hop_us_upper=tu / f.sched_u.n_levels * 1e6)
    query("ddilu_set_tuning", b"trsv_blocks_per_sm", 3)
    query("ddilu_set_tuning", b"trsv_pipe", 0)
    query("ddilu_set_tuning", b"trsv_stage_mask", -1)
    query("ddilu_set_tuning", b"trsv_far_sleep_ns", 400)
    D.USE_SELL = True
    D.USE_GWAIT = True
    if args.p > 1:   # the small, deep interface solves of the two-level preconditioners
        ms = P.schur_setup(a, layout)
        sf = ms._p.schur
        ne = sf.n
        rs, ts_ = torch.randn(ne, dtype=torch.float64, device="cuda"), torch.empty(ne, dtype=torch.float64, device="cuda")
        query("ddilu_set_tuning", b"trsv_pipe", 0)
        query("ddilu_set_tuning", b"trsv_blocks_per_sm", 3)
        for mode in ("sell", "csr", "syncfree"):
            D.USE_BLOCK_LOCAL = mode if mode != "syncfree" else False
            tl, _ = timed(lambda: sf.lower_solve(rs, ts_), flush=flush)
            tu, _ = timed(lambda: sf.upper_solve(rs, ts_), flush=flush)
            tlw, _ = timed(lambda: sf.lower_solve(rs, ts_), flush=None)
            tuw, _ = timed(lambda: sf.upper_solve(rs, ts_), flush=None)
            emit(what="schur_solve", mode=mode, rows=ne, levels=sf.sched_l.n_levels, lower_s=tl, upper_s=tu,
                 hop_us_lower=tl / sf.sched_l.n_levels * 1e6, hop_us_upper=tu / sf.sched_u.n_levels * 1e6,
                 warm_hop_us_lower=tlw / sf.sched_l.n_levels * 1e6, warm_hop_us_upper=tuw / sf.sched_u.n_levels * 1e6)
        D.USE_BLOCK_LOCAL = False
        del ms
    query("ddilu_set_tuning", b"trsv_blocks_per_sm", 3)
    query("ddilu_set_tuning", b"trsv_depth", 24)
    # SpMV
    al = s.a_loc
    x = torch.randn(al.n_cols, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    sbytes = 12 * al.nnz + 4 * (n + 1) + 16 * n
    ts, tsmin = timed(lambda: s.spmv(x, y), flush=flush)
    emit(what="spmv", s=ts, min_s=tsmin, gbs=sbytes / ts / 1e9, frac=sbytes / ts / 1e9 / PEAK)
    # vector kernels
    red = D.Reducer()
    hs = torch.zeros(4, dtype=torch.float64, device="cuda")
    v1, v2 = torch.randn(n, dtype=torch.float64, device="cuda"), torch.randn(n, dtype=torch.float64, device="cuda")
    td, _ = timed(lambda: red.dot(n, v1, v2, hs[0:1]), flush=flush)
    emit(what="dot", s=td, gbs=16 * n / td / 1e9, frac=16 * n / td / 1e9 / PEAK)
    ta, _ = timed(lambda: red.axpy_dot(n, hs[0:1], -1e-3, v1, y, v2, hs[1:2]), flush=flush)
    emit(what="axpy_dot", s=ta, gbs=32 * n / ta / 1e9, frac=32 * n / ta / 1e9 / PEAK)
    # one bj apply + a whole solve for context
    tap, _ = timed(lambda: m.apply_local(r, z), flush=flush)
    emit(what="bj_apply", s=tap, gbs=(lbytes + ubytes) / tap / 1e9, frac=(lbytes + ubytes) / tap / 1e9 / PEAK)
    b = P.default_rhs(a)
    x, rep = P.fgmres(a, b, m=m.apply)
    emit(what="solve_bj", its=rep.iterations, solve_s=rep.solve_seconds, relres=rep.final_relres,
         ms_per_it=rep.solve_seconds / max(1, rep.iterations) * 1e3)


if __name__ == "__main__":
    main()
