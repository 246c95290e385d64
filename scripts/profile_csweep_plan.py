"""Where the time of device.build_csweep goes (torch profiler, CUDA kernels by total time)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
D.USE_CSWEEP = False
m = P.make_preconditioner("schur", a, layout)
f, seg = m._p.interior, m.system.int_ptr
D.USE_CSWEEP = True
args = (f.lower, f.upper, *f._lev(False), *f._lev(True), seg)
D.build_csweep(*args)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
D.build_csweep(*args)
torch.cuda.synchronize()
print("plan", round((time.perf_counter() - t0) * 1e3, 1), "ms")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    D.build_csweep(*args)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22, max_name_column_width=60))
