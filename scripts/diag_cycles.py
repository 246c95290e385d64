"""Which reference cycles keep a preconditioner (and its device arrays, and the pinned owner map) alive until the
cyclic garbage collector runs: objects of the package found in gc.garbage after the last reference is dropped."""
import gc, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_08881_b200 as P
gc.disable()
dims = (32, 32, 32)
a = P.aniso3d(*dims)
a.device()
for pc in ("schur", "bj", "rap-milu"):
    owner = P.partition(a, 8, grid_hint=dims)
    layout = P.classify_and_order(a, owner, 8)
    m = P.make_preconditioner(pc, a, layout)
    x, r = P.fgmres(a, P.default_rhs(a), m=m.apply)
    del owner, layout, m, x, r
    gc.set_debug(gc.DEBUG_SAVEALL)
    n = gc.collect()
    gc.set_debug(0)
    ours = [o for o in gc.garbage if type(o).__module__.startswith("paper_2303") or type(o).__name__ in ("function", "cell", "method")]
    print(pc, "collected", n, sorted({type(o).__name__ for o in gc.garbage})[:30])
    for o in gc.garbage:
        if type(o).__name__ in ("function", "method"):
            print("   ", type(o).__name__, getattr(o, "__qualname__", o))
    gc.garbage.clear()
