"""Host driver of the device ILUT kernel (csrc/ilut.cu; factor.py:482-656)."""

from __future__ import annotations

import ctypes

import torch

from . import device as D
from ._lib import DdiluError, call, query

MAX_ROW_CAP = 1900  # 4 warps x (24 B + 1 B) x cap must fit the 200 KB shared-memory budget


def interleaved_order(n: int, sections) -> torch.Tensor | None:
    """Processing order for a matrix whose rows are [section 0 | section 1 | ...], every section a sequence of
    independent diagonal blocks given by its pointer array (host ints, local to the section): inside a section the
    rows of all blocks are dealt round-robin (row j of block 0, row j of block 1, ...), so that the warps of the
    factorisation kernel work on every block at once instead of on one block after the other.  A row still comes
    after every row of its own block with a smaller index and after all rows of the earlier sections."""
    parts, start = [], 0
    dev = D.dev()
    for ptr in sections:
        ptr = [int(v) for v in ptr]
        m, nb = ptr[-1] - ptr[0], len(ptr) - 1
        if m <= 0:
            continue
        if nb <= 1:
            parts.append(torch.arange(start, start + m, dtype=torch.int64, device=dev))
        else:
            rows = torch.arange(m, dtype=torch.int64, device=dev)
            p = torch.tensor(ptr, dtype=torch.int64, device=dev) - ptr[0]
            blk = torch.bucketize(rows, p[1:], right=True)
            key = (rows - p[blk]) * nb + blk
            parts.append(start + torch.argsort(key))
        start += m
    if start != n or not parts:
        return None
    return torch.cat(parts).to(D.I32).contiguous()


def d_ilut_factor(a: D.DeviceCsr, n_elim: int, tau: float, maxfill: int, tau_s: float, safeguard: float,
                  order: torch.Tensor | None = None):
    from .factor import DevFactors
    n = a.n_rows
    if n == 0:
        z = D.zeros_i32(1)
        e = D.DeviceCsr(0, 0, z, D.empty_i32(0), D.empty_f64(0), 0)
        return DevFactors(e, e)
    lens = D.empty_i32(n)
    call("ddilu_row_lengths", n, a.rp, lens)
    longest = int(lens.max().item())
    row_cap = min(MAX_ROW_CAP, max(128, 4 * (longest + 1)))
    done, status = D.empty_i32(n), D.zeros_i32(1)
    while True:
        caps = (ctypes.c_int * 3)()
        query("ddilu_ilut_caps", int(maxfill), int(row_cap), ctypes.addressof(caps))
        lcap, ucap, scap = caps[0], caps[1], caps[2]
        l_cnt, u_cnt = D.zeros_i32(n + 1), D.zeros_i32(n + 1)
        l_slots = n * lcap
        u_slots = n_elim * ucap + (n - n_elim) * scap
        l_ci, l_v = D.empty_i32(max(1, l_slots)), D.empty_f64(max(1, l_slots))
        u_ci, u_v = D.empty_i32(max(1, u_slots)), D.empty_f64(max(1, u_slots))
        call("ddilu_ilut_factor", n, a.rp, a.ci, a.val, int(n_elim), float(tau), int(maxfill), float(tau_s),
             float(safeguard), int(row_cap), l_cnt, l_ci, l_v, u_cnt, u_ci, u_v, done, status, order)
        if int(status.item()) == 0:
            break
        if row_cap >= MAX_ROW_CAP:
            raise DdiluError(f"ILUT working row exceeds the shared-memory capacity ({MAX_ROW_CAP} entries)")
        row_cap = min(MAX_ROW_CAP, 2 * row_cap)
    D.exclusive_scan_(l_cnt, n)
    D.exclusive_scan_(u_cnt, n)
    # the scans overwrote the counts with offsets; recover counts as differences inside the compaction
    ln, un = int(l_cnt[-1].item()), int(u_cnt[-1].item())
    lc, uc = D.empty_i32(n), D.empty_i32(n)
    call("ddilu_row_lengths", n, l_cnt, lc)
    call("ddilu_row_lengths", n, u_cnt, uc)
    lo_ci, lo_v = D.empty_i32(ln), D.empty_f64(ln)
    up_ci, up_v = D.empty_i32(un), D.empty_f64(un)
    call("ddilu_compact_rows", n, n, lcap, lcap, lc, l_ci, l_v, l_cnt, lo_ci, lo_v)
    call("ddilu_compact_rows", n, int(n_elim), ucap, scap, uc, u_ci, u_v, u_cnt, up_ci, up_v)
    return DevFactors(D.DeviceCsr(n, n, l_cnt, lo_ci, lo_v, ln), D.DeviceCsr(n, n, u_cnt, up_ci, up_v, un))
