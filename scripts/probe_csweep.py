"""Cluster sweep (ddilu_csweep_solve) against the tiled kernel on the interior factors of aniso3d n^3, schur / ilu0,
p subdomains: cluster size, register sets, chunk rule.  Checks bit-equality of the two kernels' results first.
JSON lines -> gpurun_out/probe_csweep.jsonl.

    python scripts/probe_csweep.py [n] [p]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D
from paper_2303_08881_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
D.USE_CSWEEP = False
m = P.make_preconditioner("schur", a, layout)
f = m._p.interior
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
torch.manual_seed(1)
r = torch.randn(f.n, dtype=torch.float64, device="cuda")
xl_ref, xu_ref = torch.empty_like(r), torch.empty_like(r)
x = torch.empty_like(r)
nnz_l, nnz_u = f.lower.nnz, f.upper.nnz
bytes_l = 12 * nnz_l + 20 * f.n          # 12 B per entry, 4 B row pointer, b and x
bytes_u = 12 * nnz_u + 20 * f.n
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
peak_gbs = float(peak.get("hbm_gbs_burst", peak.get("hbm_gbs", 6541.5))) if isinstance(peak, dict) else 6541.5


def timed(fn, reps=7):
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
out = open("gpurun_out/probe_csweep.jsonl", "a")


def emit(rec):
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()


tl, tu = timed(lambda: f.lower_solve(r, xl_ref)), timed(lambda: f.upper_solve(r, xu_ref))
emit({"n": n, "p": p, "kernel": "tiled", "rows": f.n, "levels": [f._lev(False)[1], f._lev(True)[1]],
      "L_us": round(tl * 1e6, 1), "U_us": round(tu * 1e6, 1),
      "L_frac": round(bytes_l / tl / 1e9 / peak_gbs, 3), "U_frac": round(bytes_u / tu / 1e9 / peak_gbs, 3)})

D.USE_CSWEEP = True
D.CSWEEP_MIN_AVG_WIDTH = 0
D.CSWEEP_MIN_SMS = 0
seg = m.system.int_ptr
variants = [(16, 3, 32), (16, 2, 32), (16, 4, 32), (8, 3, 32), (16, 3, 128)]
if len(sys.argv) > 3:
    variants = [tuple(int(v) for v in s.split(",")) for s in sys.argv[3:]]
for cluster, nset, min_chunk in variants:
    D.CSWEEP_CLUSTER, D.CSWEEP_NSET, D.CSWEEP_MIN_CHUNK = cluster, nset, min_chunk
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    cp = D.build_csweep(f.lower, f.upper, *f._lev(False), *f._lev(True), seg)
    t1.record()
    torch.cuda.synchronize()
    if cp is None:
        emit({"n": n, "p": p, "kernel": "csweep", "cluster": cluster, "nset": nset, "min_chunk": min_chunk, "plan": None})
        continue
    D.csweep_solve(cp, False, r, x)
    ok_l = bool(torch.equal(x, xl_ref))
    D.csweep_solve(cp, True, r, x)
    ok_u = bool(torch.equal(x, xu_ref))
    tl = timed(lambda: D.csweep_solve(cp, False, r, x))
    tu = timed(lambda: D.csweep_solve(cp, True, r, x))
    emit({"n": n, "p": p, "kernel": "csweep", "cluster": cp.csize, "nset": nset, "min_chunk": min_chunk,
          "steps": [cp.lower.max_steps, cp.upper.max_steps], "depth": [cp.lower.depth, cp.upper.depth], "consecutive": [cp.lower.contiguous, cp.upper.contiguous], "plan_ms": round(t0.elapsed_time(t1), 1),
          "bit_equal": [ok_l, ok_u], "L_us": round(tl * 1e6, 1), "U_us": round(tu * 1e6, 1),
          "L_frac": round(bytes_l / tl / 1e9 / peak_gbs, 3), "U_frac": round(bytes_u / tu / 1e9 / peak_gbs, 3)})
    if _lib.has_experiments():
        # cycle counters of the first and the last thread of every CTA (L solve): [prefetch, A, B, wait, chain, arrive + stores]
        dbg = torch.zeros(cp.n_blocks * cp.csize * 2 * 16, dtype=torch.int64, device="cuda")
        _lib.query("ddilu_csweep_set_debug", dbg.data_ptr())
        for up in (False, True):
            dbg.zero_()
            D.csweep_solve(cp, up, r, x)
            torch.cuda.synchronize()
            t = dbg.view(-1, 2, 16)[:, :, :6].double()
            nl = f._lev(up)[1]
            emit({"kernel": "csweep-cycles", "upper": up, "levels": nl,
                  "first_thread_per_level": [round(v, 1) for v in (t[:, 0].mean(0) / nl).tolist()],
                  "last_thread_per_level": [round(v, 1) for v in (t[:, 1].mean(0) / nl).tolist()]})
        _lib.query("ddilu_csweep_set_debug", None)
    del cp
