"""Host driver of the level-of-fill factorisation (csrc/iluk.cu + the fixed-pattern numeric kernel of
csrc/factor.cu; factor.py:270-390, 704-720, 855-863)."""

from __future__ import annotations

from . import device as D
from ._lib import DdiluError, call, query

MAX_ROW_CAP = 3000  # 4 warps x 16 B x cap must fit the 200 KB shared-memory budget
MIN_ROW_CAP = 32    # first try: max(MIN_ROW_CAP, 2 (level + 1) (longest row + 1)); doubled on overflow


def d_iluk_split(a: D.DeviceCsr, n_elim: int, level: int, order=None):
    """(L pattern + prefilled values, kept pattern + prefilled values) of ILU(level); order: processing order of the
    rows for the symbolic kernel (`_ilut.interleaved_order`), the pattern does not depend on it."""
    n = a.n_rows
    lens = D.empty_i32(max(n, 1))
    call("ddilu_row_lengths", n, a.rp, lens)
    longest = int(lens[:n].max().item()) if n else 0
    row_cap = min(MAX_ROW_CAP, max(MIN_ROW_CAP, 2 * (level + 1) * (longest + 1)) if MIN_ROW_CAP >= 32 else MIN_ROW_CAP)
    done, status = D.empty_i32(max(n, 1)), D.zeros_i32(1)
    while True:
        p_cnt, k_cnt = D.zeros_i32(n + 1), D.zeros_i32(n + 1)
        slots = max(1, n * row_cap)
        p_ci, k_ci, k_lv = D.empty_i32(slots), D.empty_i32(slots), D.empty_i32(slots)
        call("ddilu_iluk_symbolic", n, a.rp, a.ci, int(n_elim), int(level), int(row_cap), p_cnt, p_ci, k_cnt, k_ci,
             k_lv, done, status, order)
        if int(status.item()) == 0:
            break
        if row_cap >= MAX_ROW_CAP:
            raise DdiluError(f"ILU({level}) working row exceeds the shared-memory capacity ({MAX_ROW_CAP} entries)")
        del p_ci, k_ci, k_lv
        row_cap = min(MAX_ROW_CAP, 2 * row_cap)
    del k_lv
    pc, kc = p_cnt[:n].clone(), k_cnt[:n].clone()
    D.exclusive_scan_(p_cnt, n)
    D.exclusive_scan_(k_cnt, n)
    pn, kn = int(p_cnt[-1].item()), int(k_cnt[-1].item())
    lo_ci, up_ci = D.empty_i32(pn), D.empty_i32(kn)
    call("ddilu_compact_cols", n, int(row_cap), pc, p_ci, p_cnt, lo_ci)
    call("ddilu_compact_cols", n, int(row_cap), kc, k_ci, k_cnt, up_ci)
    del p_ci, k_ci
    lo_v, up_v = D.empty_f64(pn), D.empty_f64(kn)
    call("ddilu_prefill", n, a.rp, a.ci, a.val, p_cnt, lo_ci, lo_v, int(n_elim), 0)
    call("ddilu_prefill", n, a.rp, a.ci, a.val, k_cnt, up_ci, up_v, int(n_elim), 1)
    return D.DeviceCsr(n, n, p_cnt, lo_ci, lo_v, pn), D.DeviceCsr(n, n, k_cnt, up_ci, up_v, kn)
