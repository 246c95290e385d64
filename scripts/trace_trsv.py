"""Per-group timeline of the sync-free SpTRSV (diagnostics).  Prints where a level's time goes."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
bps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dims = (n1,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
m = P.bj_setup(a, layout)
f = m._f
for name, t, sched, upper, unit in (("L", f.lower, f.sched_l, False, True), ("U", f.upper, f.sched_u, True, False)):
    sell = D.get_sell(t, sched, upper, unit)
    n = t.n_rows
    ng = sched.n_slots // 32
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    stamps = torch.zeros(ng * 8, dtype=torch.int64, device="cuda")
    for rep in range(3):
        D.call("ddilu_sptrsv_sell_trace", n, sched.n_slots, bps, sched.order, sell.goff, sell.width, sell.scol,
               sell.sval, sell.sdiag, sell.gwait, b, x, stamps)
    torch.cuda.synchronize()
    st = stamps.cpu().numpy().reshape(ng, 8)
    slot_ptr = sched.slot_ptr.cpu().numpy()
    glev = np.searchsorted(slot_ptr, np.arange(ng) * 32, side="right") - 1      # level of every group
    t0, t1, t2, t3 = (st[:, k].astype(np.float64) for k in range(4))
    base = t0.min()
    L = sched.n_levels
    lvl_end = np.zeros(L)
    np.maximum.at(lvl_end, glev, t3 - base)
    lvl_first = np.full(L, 1e30)
    np.minimum.at(lvl_first, glev, t3 - base)
    d = np.diff(lvl_end)
    wait = t1 - t0
    load = t2 - t1
    fin = t3 - t2
    waited = st[:, 5] > 0
    out = {
        "factor": name, "n": n1, "p": p, "levels": int(L), "groups": int(ng), "total_us": float(lvl_end[-1] * 1e-3),
        "per_level_ns": {"mean": float(d.mean()), "median": float(np.median(d)), "p10": float(np.percentile(d, 10)),
                         "p90": float(np.percentile(d, 90))},
        "frac_groups_that_spun": float(waited.mean()),
        "spin_ns_when_spun": {"median": float(np.median(wait[waited])) if waited.any() else 0.0},
        "after_spin_to_deps_loaded_ns": {"median": float(np.median(load)), "p90": float(np.percentile(load, 90)),
                                         "mean": float(load.mean())},
        "repoll_rounds": {"mean": float(st[:, 6].mean()), "max": int(st[:, 6].max())},
        "deps_loaded_to_stored_ns": {"median": float(np.median(fin)), "p90": float(np.percentile(fin, 90))},
        "level_spread_ns (last - first store in a level)": {"median": float(np.median(lvl_end - lvl_first))},
        "timer_resolution_ns": float(np.min(np.diff(np.unique(t3)))),
    }
    print(json.dumps(out))
    np.save(f"gpurun_out/trace_{name}_{n1}_{p}.npy", st[:, :8])
