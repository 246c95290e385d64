"""Interface (Schur) factor solves: tiled kernel vs the block-local sweep with x in a shared-memory window.
CUDA events, L2 flushed between repetitions; also checks that both give the same bits."""
import argparse, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D


def timed(fn, flush, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--out", default="gpurun_out/probe_window.jsonl")
    args = ap.parse_args()
    dims = (args.n,) * 3
    a = P.aniso3d(*dims)
    layout = P.classify_and_order(a, P.partition(a, args.p, dims), args.p)
    D.USE_BLOCK_WINDOW = False
    m = P.make_preconditioner("schur", a, layout)
    f = m._p.schur
    s = m.system
    bwl = D.enable_block_window(f.lower, f.sched_l, s.ext_ptr, False, True)
    bwu = D.enable_block_window(f.upper, f.sched_u, s.ext_ptr, True, False)
    print("window plans:", None if bwl is None else bwl.wmask + 1, None if bwu is None else bwu.wmask + 1,
          "levels", f.sched_l.n_levels, f.sched_u.n_levels, "rows", f.n, flush=True)
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    r = torch.randn(f.n, dtype=torch.float64, device="cuda")
    rec = dict(n=args.n, p=args.p, rows=f.n, levels=f.sched_l.n_levels)
    for which, t, sched, bw, upper in (("L", f.lower, f.sched_l, bwl, False), ("U", f.upper, f.sched_u, bwu, True)):
        x0, x1 = torch.empty_like(r), torch.empty_like(r)
        tiled = (lambda: f.lower_solve(r, x0)) if not upper else (lambda: f.upper_solve(r, x0))
        rec[which + "_tiled_us"] = timed(tiled, flush)
        if bw is not None:
            win = lambda: D.sptrsv_block_window(t, sched, bw, r, x1, upper, not upper)
            from paper_2303_08881_b200._lib import query
            for thr in (1024, 512, 384, 256, 128):
                query("ddilu_set_tuning", b"win_threads", thr)
                rec[which + f"_window_{thr}_us"] = timed(win, flush)
                rec[which + f"_window_{thr}_warm_us"] = timed(win, torch.empty(1, dtype=torch.float64, device="cuda"))
                rec[which + f"_same_bits_{thr}"] = bool(torch.equal(x0, x1))
            query("ddilu_set_tuning", b"win_threads", 0)
            rec[which + "_window"] = bw.wmask + 1
    print(json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "a").write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
