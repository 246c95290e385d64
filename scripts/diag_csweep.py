"""Which rule of device.build_csweep refuses / accepts a case (DDILU_DEBUG_SWEEP prints)."""
import os
import sys

os.environ["DDILU_DEBUG_SWEEP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
D.CSWEEP_MIN_AVG_WIDTH = 0
D.CSWEEP_MIN_SMS = 0
a = P.aniso3d(n, n, n)
layout = P.classify_and_order(a, P.partition(a, p, (n, n, n)), p)
m = P.make_preconditioner("schur", a, layout)
print("plan", m._p.interior._cs is not None)
