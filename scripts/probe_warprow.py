"""Warp-per-row sync-free solve (ddilu_sptrsv_warprow) on the interior factors of convdiff27 n^3 + ILUT(1e-3, 20):
CTAs per SM and poll back-off (experiments build for the knobs).  JSON lines -> gpurun_out/probe_warprow.jsonl."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200._lib import query

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n,) * 3
a = P.convdiff27(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
f = m._p.interior
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
r = torch.randn(f.n, dtype=torch.float64, device="cuda")
x = torch.empty_like(r)


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


os.makedirs("gpurun_out", exist_ok=True)
out = open("gpurun_out/probe_warprow.jsonl", "a")
for bps in (0, 6, 4, 3, 2):
    for sleep in (0, 100):
        query("ddilu_set_tuning", b"wr_blocks_per_sm", bps)
        query("ddilu_set_tuning", b"trsv_sleep_ns", sleep)
        rec = {"n": n, "p": p, "ctas_per_sm": bps, "sleep_ns": sleep, "rows": f.n, "levels": [f._lev(False)[1], f._lev(True)[1]],
               "L_us": round(timed(lambda: f.lower_solve(r, x)) * 1e6, 1), "U_us": round(timed(lambda: f.upper_solve(r, x)) * 1e6, 1)}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
