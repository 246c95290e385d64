"""Launch-overhead probe: the Schur-factor solve pair and one inner-GMRES step, launched one by one vs
replayed from a CUDA graph."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n,) * 3
a = P.aniso3d(*dims)
layout = P.classify_and_order(a, P.partition(a, 8, dims), 8)
m = P.make_preconditioner("schur", a, layout)
s = m.system
y = torch.randn(s.n_ext + s.n_halo, dtype=torch.float64, device="cuda")
out = torch.empty(s.n_ext, dtype=torch.float64, device="cuda")


def body():
    for _ in range(4):
        m._reduced_matvec(y, out)     # E spmv + L_S + U_S solves + ewise


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


t_plain = timed(body)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        body()
t_graph = timed(g.replay)
print(json.dumps(dict(n=n, four_reduced_matvecs_us=t_plain, graph_us=t_graph)))
