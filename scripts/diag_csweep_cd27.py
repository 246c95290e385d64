"""Would the cluster sweep's layout fit the 27-point ILUT interior factors (config 5)?  Window reach, push targets and
level widths for a cluster of `csize` CTAs per block -- the rules of device.build_csweep without its limit of four
dependencies per row.

    python scripts/diag_csweep_cd27.py [n] [p] [csize]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08881_b200 as P
from paper_2303_08881_b200 import device as D

n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 96
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
csize = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dims = (n1,) * 3
a = P.convdiff27(*dims)
layout = P.classify_and_order(a, P.partition(a, p, dims), p)
m = P.make_preconditioner("schur", a, layout, P.FillRule.parse("ilut:0.001,20"))
f, s = m._p.interior, m.system
n, nb = f.n, len(s.int_ptr) - 1
d = D.dev()
i64 = torch.int64
seg = torch.tensor([int(v) for v in s.int_ptr], dtype=i64, device=d)
rows = torch.arange(n, dtype=i64, device=d)
blk = torch.bucketize(rows, seg[1:], right=True)
for fac, (lev, nlev), name in ((f.lower, f._lev(False), "L"), (f.upper, f._lev(True), "U")):
    lv = lev[:n].to(i64)
    key = blk * nlev + lv
    order = torch.argsort(key, stable=True)
    cnt = torch.bincount(key, minlength=nb * nlev).view(nb, nlev)
    lev_start = torch.cumsum(cnt, 1) - cnt
    pib = torch.empty(n, dtype=i64, device=d)
    pib[order] = rows - seg[blk[order]]
    ril = pib - lev_start.reshape(-1)[key]
    cs = torch.clamp((cnt + csize - 1) // csize, min=32)
    csr = cs.reshape(-1)[key]
    rk = ril // csr
    ro = ril - rk * csr
    ranks = torch.arange(csize, dtype=i64, device=d).view(1, csize, 1)
    ncl = torch.clamp(cnt.view(nb, 1, nlev) - ranks * cs.view(nb, 1, nlev), min=0)
    ncl = torch.minimum(ncl, cs.view(nb, 1, nlev).expand(nb, csize, nlev))
    ckey = (blk * csize + rk) * nlev + lv
    cta = blk * csize + rk
    rlen = (fac.rp[1:] - fac.rp[:-1]).to(i64)
    erow = torch.repeat_interleave(rows, rlen)
    ecol = fac.ci[: fac.nnz].to(i64)
    dep = ecol != erow
    remote = dep & (cta[erow] != cta[ecol])
    hkey_e = cta[erow] * n + ecol
    hu = torch.unique(hkey_e[remote])
    h_cta, h_row = hu // n, hu % n
    gkey = h_cta * nlev + lv[h_row]
    n_in = torch.bincount(gkey, minlength=nb * csize * nlev).view(nb, csize, nlev)
    gorder = torch.argsort(gkey, stable=True)
    gstart = torch.cumsum(n_in.reshape(-1), 0) - n_in.reshape(-1)
    h_idx = torch.empty_like(gkey)
    h_idx[gorder] = torch.arange(gkey.numel(), dtype=i64, device=d) - gstart[gkey[gorder]]
    n_ext = ncl + n_in
    wend = torch.cumsum(n_ext, 2)
    wstart = wend - n_ext
    wpos = wstart.reshape(-1)[ckey] + ro
    h_wpos = wstart.reshape(-1)[gkey] + ncl.reshape(-1)[gkey] + h_idx
    e_wpos = wpos[ecol].clone()
    e_wpos[remote] = h_wpos[torch.searchsorted(hu, hkey_e[remote])]
    need = torch.where(dep, wend.reshape(-1)[cta[erow] * nlev + lv[erow]] - e_wpos, torch.zeros_like(ecol))
    prow = torch.sort(h_row).values
    pidx = torch.arange(prow.numel(), dtype=i64, device=d) - torch.searchsorted(prow, prow)
    q = torch.tensor([0.5, 0.9, 0.99, 0.999], device=d)
    print(name, "rows", n, "levels", nlev, "deps/row max", int(rlen.max()) - (1 if name == "U" else 0),
          "window need max", int(need.max()), "quantiles", [int(v) for v in torch.quantile(need[dep].double()[:: max(1, need.numel() // 4000000)], q.double())],
          "halo values", hu.numel(), "push targets per row max", int(pidx.max()) + 1,
          "rows with > 3 targets", int((torch.bincount(prow) > 3).sum()),
          "widest chunk", int(ncl.max()), flush=True)
