"""Where partition + classify_and_order spend their time (host wall clock, device sync per repetition)."""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n,) * 3
a = P.aniso3d(*dims)
a.device()
for rep in range(3):
    mat = P.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    mat._dev = a._dev
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    if rep == 2:
        pr.enable()
    owner = P.partition(mat, 8, dims)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    layout = P.classify_and_order(mat, owner, 8)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if rep == 2:
        pr.disable()
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25)
        print(s.getvalue()[:5000])
    print(f"rep {rep}: partition {t1 - t0:.4f} s, classify {t2 - t1:.4f} s")
