"""Where the setup time goes (host wall clock with a device sync after every stage)."""
import os, sys, time, cProfile, pstats, io
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n,) * 3
a = P.aniso3d(*dims)
a.device()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    owner = P.partition(a, 8, dims)
    layout = P.classify_and_order(a, owner, 8)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if rep == 2:
        pr = cProfile.Profile()
        pr.enable()
    m = P.make_preconditioner("schur", a, layout)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if rep == 2:
        pr.disable()
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(28)
        print(s.getvalue()[:6000])
    print(f"rep {rep}: layout {t1 - t0:.3f} s, preconditioner {t2 - t1:.3f} s")
    del m
