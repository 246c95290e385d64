"""Dependency-hop diagnostics: synthetic unit-lower systems through the production SpTRSV kernels."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200._lib import query


def lower_from_offsets(n, offsets, coef=-0.3):
    rows, cols = [], []
    idx = np.arange(n)
    for off in sorted(offsets, reverse=True):
        ok = idx - off >= 0
        rows.append(idx[ok]); cols.append(idx[ok] - off)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    return P.csr_from_coo(n, n, rows, cols, np.full(len(rows), coef))


def timed(fn, reps=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


cases = [
    ("single-row chain (1 lane active)", 4000, [1]),
    ("1 group/level, 1 dep (lane->lane)", 32 * 2000, [32]),
    ("1 group/level, 3 deps", 32 * 2000, [31, 32, 33]),
    ("4 groups/level, 3 deps", 128 * 2000, [127, 128, 129]),
    ("16 groups/level, 3 deps", 512 * 1000, [511, 512, 513]),
    ("172 groups/level, 3 deps", 5504 * 400, [5503, 5504, 5505]),
    ("172 groups/level, 3 far deps", 5504 * 400, [5504 - 64, 5504, 5504 + 64]),
]
for name, n, offs in cases:
    l = lower_from_offsets(n, offs)
    ld = l.device()
    sched = l.schedule(False)
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(b)
    res = {}
    D.USE_BLOCK_LOCAL = False
    for label, depth in (("syncfree", 24), ("syncfree_d0", 0)):
        query("ddilu_set_tuning", b"trsv_depth", depth)
        t = timed(lambda: D.sptrsv(ld, sched, b, out, False, True))
        res[label] = round(t / sched.n_levels * 1e6, 3)
    query("ddilu_set_tuning", b"trsv_depth", 24)
    if sched.n / sched.n_levels <= 1024:
        D.enable_block_local(sched, [0, n])
        for mode in ("sell", "csr"):
            D.USE_BLOCK_LOCAL = mode
            t = timed(lambda: D.sptrsv(ld, sched, b, out, False, True))
            res["block_" + mode] = round(t / sched.n_levels * 1e6, 3)
        sched.blocks = None
    print(json.dumps({"case": name, "n": n, "levels": sched.n_levels, "us_per_level": res}))
