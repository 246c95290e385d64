"""Where the end-to-end step of bench.py (host CSR arrays in, host x out) spends its time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n,) * 3
a = P.aniso3d(*dims)
host = [torch.from_numpy(x).pin_memory() for x in (a.row_ptr, a.col_idx, a.values)]
ad = a.device()
ones = torch.ones(a.n_cols, dtype=torch.float64, device="cuda")
b_dev = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
D.spmv(ad, ones, b_dev)
b_host = b_dev.cpu().pin_memory()
x_host = torch.empty(a.n_rows, dtype=torch.float64).pin_memory()


def sync():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(4):
    resident = rep < 2
    t = [sync()]
    if resident:
        mat, rhs = a, b_dev
    else:
        mat = P.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
        rp, ci, v = (h.to("cuda", non_blocking=True) for h in host)
        ci32, rp32 = D.empty_i32(ci.numel()), D.empty_i32(rp.numel())
        D.call("ddilu_narrow_i64", ci.numel(), ci, ci32)
        D.call("ddilu_narrow_i64", rp.numel(), rp, rp32)
        mat._dev = D.DeviceCsr(a.n_rows, a.n_cols, rp32, ci32, v, a.nnz)
        rhs = b_host.to("cuda", non_blocking=True)
    t.append(sync())
    owner = P.partition(mat, 8, grid_hint=dims)
    layout = P.classify_and_order(mat, owner, 8)
    t.append(sync())
    m = P.make_preconditioner("schur", mat, layout)
    t.append(sync())
    x, rep_ = P.fgmres(mat, rhs, m=m.apply)
    t.append(sync())
    if not resident:
        x_host.copy_(x)
    t.append(sync())
    names = ["upload", "layout", "precond", "solve", "download"]
    print("resident" if resident else "e2e", {k: round(t[i + 1] - t[i], 4) for i, k in enumerate(names)}, "total", round(t[-1] - t[0], 4), flush=True)
