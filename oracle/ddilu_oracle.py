"""CPU oracle for the DD-ILU + FGMRES hot path -- TEST INFRASTRUCTURE ONLY.

numpy glue around ``ddilu_oracle.c`` restating the reference package
(``/root/reference/pkg/src/ddilu``).  Every function cites the reference lines
it follows.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module; the product (``paper_2303_08881_b200``) must never do so.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks this module
against fixtures written by the unmodified reference
(``tests/golden/make_golden.py``) and against the known answers in the
reference's own tests (cited there).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libddilu_oracle.so")


def build(force: bool = False) -> str:
    """Compile the C half with the committed Makefile (gcc, seconds)."""
    src = os.path.join(_HERE, "ddilu_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "-B", "libddilu_oracle.so"])
    return _SO


_lib = None
_I = ctypes.c_int64
_P = ctypes.c_void_p
_D = ctypes.c_double


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_vdot.restype = _D
        _lib.orc_lower_solve.restype = _I
        _lib.orc_upper_solve.restype = _I
        _lib.orc_levels.restype = _I
    return _lib


# ---------------------------------------------------------------------------
# optional threading (bench.py --impl reference only).  The reference is strictly
# serial; threads = 1 (the default) IS the pinned oracle.  With threads > 1 the
# per-domain loops of the preconditioners run side by side (independent work,
# same bits), SpMV rows and axpy are split over threads (same bits), and the dot
# product is summed in `threads` contiguous chunks (NOT the reference's
# left-to-right order: results agree to rounding, iteration counts may move by
# one).  Tests never enable it.

_threads = 1
_pool = None


def set_threads(n: int) -> int:
    """Use up to n host threads for the timed reference arm; returns the count in effect."""
    global _threads, _pool
    n = max(1, int(n))
    if _pool is not None:
        _pool.shutdown()
        _pool = None
    _threads = n
    lib().orc_set_threads(ctypes.c_int(n))
    if n > 1:
        from concurrent.futures import ThreadPoolExecutor
        _pool = ThreadPoolExecutor(max_workers=n)
    return _threads


def _pmap(fn, items):
    """[fn(x) for x in items]; independent domain work, spread over the pool when threading is on."""
    items = list(items)
    if _pool is None or len(items) < 2:
        return [fn(x) for x in items]
    # the C kernels run single-threaded inside a domain task (the domains already fill the cores)
    lib().orc_set_threads(ctypes.c_int(1))
    try:
        return list(_pool.map(fn, items))
    finally:
        lib().orc_set_threads(ctypes.c_int(_threads))


def _p(a):
    return _P(a.ctypes.data) if a is not None else _P(0)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# containers (sparse.py:40-84, 168-212)


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        out[rows, self.col_idx] = self.values
        return out


def csr_from_coo(n_rows, n_cols, rows, cols, vals):
    """sparse.py:115-147 (sorted by (row, col); duplicates are an error)."""
    rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(rows) > 1 and np.any((np.diff(rows) == 0) & (np.diff(cols) == 0)):
        raise ValueError("duplicate entry")
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    np.cumsum(rp, out=rp)
    return Csr(n_rows, n_cols, rp, cols.copy(), vals.copy())


def csr_from_dense(a, keep_zeros=False):
    """sparse.py:150-160."""
    a = np.asarray(a, dtype=np.float64)
    if keep_zeros:
        rows, cols = [x.ravel() for x in np.indices(a.shape)]
    else:
        rows, cols = np.nonzero(a)
    return csr_from_coo(a.shape[0], a.shape[1], rows, cols, a[rows, cols])


def perm_from_order(order):
    """sparse.py:206-212: returns (forward, inverse) with inverse = order."""
    order = _i64(order)
    fwd = np.empty_like(order)
    fwd[order] = np.arange(len(order), dtype=np.int64)
    return fwd, order


# ---------------------------------------------------------------------------
# kernels wrappers (sparse.py:389-528)


def spmv(a: Csr, x):
    x = _f64(x)
    out = np.empty(a.n_rows)
    lib().orc_spmv(_I(a.n_rows), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _p(x), _p(out))
    return out


def tri_solve_lower(l: Csr, b, unit_diag=False):
    b = _f64(b)
    x = np.empty_like(b)
    bad = lib().orc_lower_solve(_I(l.n_rows), _p(l.row_ptr), _p(l.col_idx), _p(l.values),
                                _p(b), _p(x), ctypes.c_int(int(unit_diag)))
    if bad >= 0:
        raise ZeroDivisionError(f"zero or missing diagonal at row {bad}")
    return x


def tri_solve_upper(u: Csr, b, unit_diag=False):
    b = _f64(b)
    x = np.empty_like(b)
    bad = lib().orc_upper_solve(_I(u.n_rows), _p(u.row_ptr), _p(u.col_idx), _p(u.values),
                                _p(b), _p(x), ctypes.c_int(int(unit_diag)))
    if bad >= 0:
        raise ZeroDivisionError(f"zero or missing diagonal at row {bad}")
    return x


def vdot(a, b):
    return float(lib().orc_vdot(_I(len(a)), _p(a), _p(b)))


def vnorm2(a):
    return float(np.sqrt(vdot(a, a)))


def axpy(alpha, v, w):
    lib().orc_axpy(_I(len(w)), _D(alpha), _p(v), _p(w))


def csr_transpose(a: Csr):
    """sparse.py:508-516."""
    rp = np.zeros(a.n_cols + 1, dtype=np.int64)
    if a.nnz:
        np.add.at(rp, a.col_idx + 1, 1)
    np.cumsum(rp, out=rp)
    ci = np.empty(a.nnz, dtype=np.int64)
    v = np.empty(a.nnz)
    lib().orc_transpose(_I(a.n_rows), _I(a.n_cols), _p(a.row_ptr), _p(a.col_idx), _p(a.values),
                        _p(rp), _p(ci), _p(v))
    return Csr(a.n_cols, a.n_rows, rp, ci, v)


def sparse_matmul(a: Csr, b: Csr):
    """sparse.py:333-370, 487-505 (`_spgemm_count`, `_spgemm_fill`): marker / accumulator loops, the first
    product of a column assigned, later ones added in traversal order, rows emitted in ascending column order
    with cancelled entries kept.  Pure-Python loops: small matrices only."""
    if a.n_cols != b.n_rows:
        raise ValueError("inner dimensions do not match")
    rp = np.zeros(a.n_rows + 1, dtype=np.int64)
    cols_out, vals_out = [], []
    marker_arr = np.full(b.n_cols, -1, dtype=np.int64)
    acc = np.zeros(b.n_cols)
    for i in range(a.n_rows):
        row_cols = []
        for ka in range(a.row_ptr[i], a.row_ptr[i + 1]):
            k = a.col_idx[ka]
            av = a.values[ka]
            for kb in range(b.row_ptr[k], b.row_ptr[k + 1]):
                j = b.col_idx[kb]
                if marker_arr[j] != i:
                    marker_arr[j] = i
                    acc[j] = av * b.values[kb]
                    row_cols.append(j)
                else:
                    acc[j] += av * b.values[kb]
        row_cols.sort()
        cols_out += row_cols
        vals_out += [acc[j] for j in row_cols]
        rp[i + 1] = len(cols_out)
    return Csr(a.n_rows, b.n_cols, rp, np.array(cols_out, dtype=np.int64), np.array(vals_out, dtype=np.float64))


def permute_symmetric(a: Csr, fwd):
    """sparse.py:431-442."""
    fwd = _i64(fwd)
    rp = np.zeros(a.n_rows + 1, dtype=np.int64)
    rp[fwd + 1] = np.diff(a.row_ptr)
    np.cumsum(rp, out=rp)
    ci = np.empty(a.nnz, dtype=np.int64)
    v = np.empty(a.nnz)
    lib().orc_permute(_I(a.n_rows), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _p(fwd),
                      _p(rp), _p(ci), _p(v))
    return Csr(a.n_rows, a.n_cols, rp, ci, v)


def _gather(a: Csr, rows, cols, resort):
    """sparse.py:445-453."""
    rows, cols = _i64(rows), _i64(cols)
    colmap = np.full(a.n_cols, -1, dtype=np.int64)
    colmap[cols] = np.arange(len(cols), dtype=np.int64)
    counts = np.empty(len(rows), dtype=np.int64)
    lib().orc_gather_rows_count(_p(a.row_ptr), _p(a.col_idx), _I(len(rows)), _p(rows),
                                _p(colmap), _p(counts))
    rp = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.empty(rp[-1], dtype=np.int64)
    v = np.empty(rp[-1])
    lib().orc_gather_rows_fill(_p(a.row_ptr), _p(a.col_idx), _p(a.values), _I(len(rows)),
                               _p(rows), _p(colmap), _p(rp), _p(ci), _p(v),
                               ctypes.c_int(int(resort)))
    return Csr(len(rows), len(cols), rp, ci, v)


def extract_block(a, rows, cols):
    """sparse.py:456-471 (sorted index sets, no re-sort)."""
    return _gather(a, rows, cols, False)


def take_submatrix(a, rows, cols):
    """sparse.py:474-484 (any order, rows re-sorted by column)."""
    return _gather(a, rows, cols, True)


# ---------------------------------------------------------------------------
# orderings (ordering.py)


def sym_adjacency(a: Csr):
    """ordering.py:72-81."""
    t = csr_transpose(a)
    n = a.n_rows
    counts = np.empty(n, dtype=np.int64)
    lib().orc_sym_merge(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(t.row_ptr), _p(t.col_idx),
                        _p(counts), _P(0), _P(0))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.empty(rp[-1], dtype=np.int64)
    lib().orc_sym_merge(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(t.row_ptr), _p(t.col_idx),
                        _P(0), _p(rp), _p(ci))
    return rp, ci


def box_factors(dims, p):
    """ordering.py:130-145."""
    factors = [1] * len(dims)
    primes, q, f = [], p, 2
    while f * f <= q:
        while q % f == 0:
            primes.append(f)
            q //= f
        f += 1
    if q > 1:
        primes.append(q)
    for f in sorted(primes, reverse=True):
        ax = max(range(len(dims)), key=lambda a: (dims[a] / factors[a], -a))
        factors[ax] *= f
    return factors


def row_block_owner(n, p):
    """ordering.py:201-216."""
    base, rem = divmod(n, p)
    sizes = np.full(p, base, dtype=np.int64)
    sizes[:rem] += 1
    return np.repeat(np.arange(p, dtype=np.int64), sizes)


def partition(a: Csr, p, grid_hint=None):
    """ordering.py:148-198."""
    n = a.n_rows
    if p == 1:
        return np.zeros(n, dtype=np.int64)
    if grid_hint is not None:
        dims = tuple(int(d) for d in grid_hint)
        factors = box_factors(dims, p)
        idx = np.arange(n)
        owner = np.zeros(n, dtype=np.int64)
        stride = dstride = 1
        for d, f in zip(dims, factors):
            starts = np.array([c[0] for c in np.array_split(np.arange(d), f)] + [d])
            coord = (idx // stride) % d
            owner += (np.searchsorted(starts, coord, side="right") - 1) * dstride
            stride *= d
            dstride *= f
        sizes = np.bincount(owner, minlength=p)
        if np.max(np.abs(sizes - n / p)) <= max(1.0, 0.1 * n / p):
            return owner
    base, rem = divmod(n, p)
    sizes = np.full(p, base, dtype=np.int64)
    sizes[:rem] += 1
    rp, ci = sym_adjacency(a)
    owner = np.full(n, -1, dtype=np.int64)
    lib().orc_grow_regions(_I(n), _p(rp), _p(ci), _I(p), _p(sizes), _p(owner))
    return owner


def classify_and_order(a: Csr, owner, p=None):
    """ordering.py:253-297 -> namespace with the DomainLayout fields."""
    n = a.n_rows
    owner = _i64(owner)
    if p is None:
        p = int(owner.max()) + 1 if n else 1
    rp, ci = sym_adjacency(a)
    ext = np.zeros(n, dtype=np.uint8)
    lib().orc_mark_exterior(_I(n), _p(rp), _p(ci), _p(owner), _p(ext))
    ext = ext.astype(bool)
    interior_of = [np.where((owner == d) & ~ext)[0].astype(np.int64) for d in range(p)]
    exterior_of = [np.where((owner == d) & ext)[0].astype(np.int64) for d in range(p)]
    istarts = np.zeros(p + 1, dtype=np.int64)
    np.cumsum([len(s) for s in interior_of], out=istarts[1:])
    estarts = np.zeros(p + 1, dtype=np.int64)
    np.cumsum([len(s) for s in exterior_of], out=estarts[1:])
    order = np.concatenate(interior_of + exterior_of) if n else np.empty(0, dtype=np.int64)
    fwd, inv = perm_from_order(order)
    return SimpleNamespace(n=n, p=p, owner=owner, interior_of=interior_of, exterior_of=exterior_of,
                           perm_forward=fwd, perm_inverse=inv, n_interior=int(istarts[-1]),
                           n_exterior=n - int(istarts[-1]), interior_starts=istarts,
                           exterior_starts=estarts)


def rcm(a: Csr):
    """ordering.py:400-416 -> (forward, inverse)."""
    n = a.n_rows
    if n == 0:
        z = np.empty(0, dtype=np.int64)
        return z, z.copy()
    rp, ci = sym_adjacency(a)
    order = np.empty(n, dtype=np.int64)
    lib().orc_cm_order(_I(n), _p(rp), _p(ci), _p(order))
    return perm_from_order(order[::-1].copy())


def level_schedule(t: Csr, upper=False):
    """Topological levels of a triangular factor (SURVEY.md 8c definition).

    Returns (lev[n], level_ptr[L+1], level_rows[n]); rows inside a level are
    in increasing index order for L and decreasing order for U (the order a
    backward sweep meets them)."""
    n = t.n_rows
    lev = np.zeros(n, dtype=np.int64)
    depth = int(lib().orc_levels(_I(n), _p(t.row_ptr), _p(t.col_idx), ctypes.c_int(int(upper)),
                                 _p(lev)))
    counts = np.bincount(lev, minlength=depth) if n else np.zeros(0, dtype=np.int64)
    ptr = np.zeros(depth + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    idx = np.arange(n, dtype=np.int64)
    if upper:
        idx = idx[::-1]
    rows = idx[np.argsort(lev[idx], kind="stable")]
    return lev, ptr, rows


# ---------------------------------------------------------------------------
# factorisations (factor.py)

DIAG_SAFEGUARD = 1e-6


@dataclass(frozen=True)
class Rule:
    """factor.py:59-105 (FillRule)."""

    kind: str = "ilu0"
    tau: float = 0.0
    maxfill: int = 0
    level: int = 0

    @staticmethod
    def parse(text):
        head, _, rest = text.partition(":")
        if head == "ilu0" and not rest:
            return Rule("ilu0")
        if head == "iluk" and rest:
            return Rule("iluk", level=int(rest))
        if head == "ilut" and rest:
            t, _, f = rest.partition(",")
            return Rule("ilut", float(t), int(f))
        raise ValueError(f"cannot parse fill rule {text!r}")

    def __str__(self):
        if self.kind == "iluk":
            return f"iluk:{self.level}"
        return f"ilut:{self.tau:g},{self.maxfill}" if self.kind == "ilut" else "ilu0"


def level0_split(a: Csr, n_elim):
    """factor.py:249-263."""
    n = a.n_rows
    pc = np.empty(n, dtype=np.int64)
    kc = np.empty(n, dtype=np.int64)
    lib().orc_split_counts(_I(n), _p(a.row_ptr), _p(a.col_idx), _I(n_elim), _p(pc), _p(kc))
    p_rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(pc, out=p_rp[1:])
    k_rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(kc, out=k_rp[1:])
    p_ci = np.empty(p_rp[-1], dtype=np.int64)
    p_v = np.empty(p_rp[-1])
    k_ci = np.empty(k_rp[-1], dtype=np.int64)
    k_v = np.empty(k_rp[-1])
    lib().orc_split_fill(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _I(n_elim),
                         _p(p_rp), _p(p_ci), _p(p_v), _p(k_rp), _p(k_ci), _p(k_v))
    return p_rp, p_ci, p_v, k_rp, k_ci, k_v


def iluk_split(a: Csr, n_elim, level):
    """factor.py:270-390: symbolic level-of-fill pattern + A's values prefilled (fill = 0)."""
    n = a.n_rows
    p_rp = np.zeros(n + 1, dtype=np.int64)
    k_rp = np.zeros(n + 1, dtype=np.int64)
    ptrs = [ctypes.c_void_p() for _ in range(2)]
    lib().orc_iluk_symbolic(_I(n), _p(a.row_ptr), _p(a.col_idx), _I(n_elim), _I(level), _p(p_rp),
                            ctypes.byref(ptrs[0]), _p(k_rp), ctypes.byref(ptrs[1]))

    def take(ptr, count):
        out = np.empty(0, dtype=np.int64) if count == 0 else \
            np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int64)), (count,)).copy()
        lib().orc_free(ptr)
        return out

    p_ci, k_ci = take(ptrs[0], int(p_rp[-1])), take(ptrs[1], int(k_rp[-1]))
    p_v, k_v = np.zeros(len(p_ci)), np.zeros(len(k_ci))
    lib().orc_prefill(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _p(p_rp), _p(p_ci), _p(p_v),
                      _I(n_elim), ctypes.c_int(0))
    lib().orc_prefill(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _p(k_rp), _p(k_ci), _p(k_v),
                      _I(n_elim), ctypes.c_int(1))
    return p_rp, p_ci, p_v, k_rp, k_ci, k_v


def _factor_on_pattern(a: Csr, n_elim, milu, target, wvec, safeguard, level=0):
    """factor.py:446-458 (level > 0: on the iluk pattern, factor.py:704-720, 855-863)."""
    n = a.n_rows
    p_rp, p_ci, p_v, k_rp, k_ci, k_v = level0_split(a, n_elim) if level <= 0 else iluk_split(a, n_elim, level)
    rownorm = np.empty(n)
    lib().orc_row_inf_norms(_I(n), _p(a.row_ptr), _p(a.values), _p(rownorm))
    if target is None:
        target = np.empty(0)
        wvec = np.empty(0)
    target, wvec = _f64(target), _f64(wvec)
    lib().orc_factor_split(_I(n), _p(p_rp), _p(p_ci), _p(p_v), _p(k_rp), _p(k_ci), _p(k_v),
                           _I(n_elim), ctypes.c_int(int(milu)), _p(target), _p(wvec),
                           _D(safeguard), _p(rownorm))
    return Csr(n, n, p_rp, p_ci, p_v), Csr(n, n, k_rp, k_ci, k_v)


@dataclass
class Factors:
    """factor.py:108-131 (IluFactors): unit L (strict), U with diagonal first."""

    lower: Csr
    upper: Csr
    kind: str = "ilu0"

    @property
    def n(self):
        return self.lower.n_rows

    def solve(self, b):
        return tri_solve_upper(self.upper, tri_solve_lower(self.lower, b, unit_diag=True))

    def lu_matvec(self, y):
        t = spmv(self.upper, y)
        return t + spmv(self.lower, t)


def ilu0(a: Csr, safeguard=DIAG_SAFEGUARD):
    """factor.py:668-677."""
    lo, up = _factor_on_pattern(a, a.n_rows, False, None, None, safeguard)
    return Factors(lo, up, "ilu0")


def milu0(a: Csr, target=None, wvec=None, safeguard=DIAG_SAFEGUARD):
    """factor.py:680-701 (target = [y | z], wvec = [w | 0]; default ones / zeros)."""
    n = a.n_rows
    target = np.ones(n) if target is None else _f64(target)
    wvec = np.zeros(n) if wvec is None else _f64(wvec)
    if np.any(target == 0.0):
        raise ValueError("milu target vector must have no zero entries")
    lo, up = _factor_on_pattern(a, n, True, target, wvec, safeguard)
    return Factors(lo, up, "milu0")


def _ilut_raw(a: Csr, n_elim, tau, maxfill, tau_s, safeguard):
    n = a.n_rows
    l_rp = np.zeros(n + 1, dtype=np.int64)
    u_rp = np.zeros(n + 1, dtype=np.int64)
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    lib().orc_ilut_factor(_I(n), _p(a.row_ptr), _p(a.col_idx), _p(a.values), _I(n_elim),
                          _D(tau), _I(maxfill), _D(tau_s), _D(safeguard), _p(l_rp),
                          ctypes.byref(ptrs[0]), ctypes.byref(ptrs[1]), _p(u_rp),
                          ctypes.byref(ptrs[2]), ctypes.byref(ptrs[3]))

    def take(ptr, count, ctype, dtype):
        if count == 0:
            out = np.empty(0, dtype=dtype)
        else:
            out = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), (count,)).copy()
        lib().orc_free(ptr)
        return out

    nl, nu = int(l_rp[-1]), int(u_rp[-1])
    l_ci = take(ptrs[0], nl, ctypes.c_int64, np.int64)
    l_v = take(ptrs[1], nl, ctypes.c_double, np.float64)
    u_ci = take(ptrs[2], nu, ctypes.c_int64, np.int64)
    u_v = take(ptrs[3], nu, ctypes.c_double, np.float64)
    return Csr(n, n, l_rp, l_ci, l_v), Csr(n, n, u_rp, u_ci, u_v)


def ilut(a: Csr, tau, maxfill, safeguard=DIAG_SAFEGUARD):
    """factor.py:723-740."""
    lo, up = _ilut_raw(a, a.n_rows, tau, maxfill, 0.0, safeguard)
    return Factors(lo, up, str(Rule("ilut", tau, maxfill)))


def iluk(a: Csr, level, safeguard=DIAG_SAFEGUARD):
    """factor.py:704-720."""
    if level < 0:
        raise ValueError("level must be nonnegative")
    if level == 0:
        return ilu0(a, safeguard)
    lo, up = _factor_on_pattern(a, a.n_rows, False, None, None, safeguard, level)
    return Factors(lo, up, f"iluk:{level}")


def factorize(a: Csr, rule: Rule, safeguard=DIAG_SAFEGUARD):
    """factor.py:743-749."""
    if rule.kind == "ilu0":
        return ilu0(a, safeguard)
    if rule.kind == "iluk":
        return iluk(a, rule.level, safeguard)
    return ilut(a, rule.tau, rule.maxfill, safeguard)


def rows_colsplit(m: Csr, r0, r1, csplit):
    """factor.py:784-803."""
    nr = r1 - r0
    lo_c = np.empty(nr, dtype=np.int64)
    z = _P(0)
    lib().orc_col_split(_p(m.row_ptr), _p(m.col_idx), _p(m.values), _I(r0), _I(r1), _I(csplit),
                        _p(lo_c), z, z, z, z, z, z)
    total = np.diff(m.row_ptr[r0:r1 + 1])
    lo_rp = np.zeros(nr + 1, dtype=np.int64)
    np.cumsum(lo_c, out=lo_rp[1:])
    hi_rp = np.zeros(nr + 1, dtype=np.int64)
    np.cumsum(total - lo_c, out=hi_rp[1:])
    lo_ci = np.empty(lo_rp[-1], dtype=np.int64)
    lo_v = np.empty(lo_rp[-1])
    hi_ci = np.empty(hi_rp[-1], dtype=np.int64)
    hi_v = np.empty(hi_rp[-1])
    lib().orc_col_split(_p(m.row_ptr), _p(m.col_idx), _p(m.values), _I(r0), _I(r1), _I(csplit),
                        z, _p(lo_rp), _p(lo_ci), _p(lo_v), _p(hi_rp), _p(hi_ci), _p(hi_v))
    return (Csr(nr, csplit, lo_rp, lo_ci, lo_v),
            Csr(nr, m.n_cols - csplit, hi_rp, hi_ci, hi_v))


def drop_small_rows(m: Csr, tol):
    """factor.py:806-822."""
    if tol <= 0.0 or m.nnz == 0:
        return m
    keep = np.ones(m.nnz, dtype=bool)
    counts = np.zeros(m.n_rows, dtype=np.int64)
    for r in range(m.n_rows):
        s0, s1 = int(m.row_ptr[r]), int(m.row_ptr[r + 1])
        vals = m.values[s0:s1]
        nrm = np.sqrt(float(np.dot(vals, vals)))
        small = (np.abs(vals) < tol * nrm) & (m.col_idx[s0:s1] != r)
        keep[s0:s1] = ~small
        counts[r] = int(np.count_nonzero(~small))
    rp = np.zeros(m.n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return Csr(m.n_rows, m.n_cols, rp, m.col_idx[keep], m.values[keep])


def partial_ilu(a: Csr, n_interior, rule: Rule, schur_drop_tol=0.0, factor_schur=True,
                safeguard=DIAG_SAFEGUARD):
    """factor.py:825-883 -> namespace(interior, w_block, z_block, s_tilde, schur, n_interior)."""
    n = a.n_rows
    if rule.kind == "ilut":
        lower, upper = _ilut_raw(a, n_interior, rule.tau, rule.maxfill, schur_drop_tol, safeguard)
        drop_tol = 0.0
    else:
        lower, upper = _factor_on_pattern(a, n_interior, False, None, None, safeguard,
                                          rule.level if rule.kind == "iluk" else 0)
        drop_tol = schur_drop_tol
    l_b, _ = rows_colsplit(lower, 0, n_interior, n_interior)
    u_b, z_blk = rows_colsplit(upper, 0, n_interior, n_interior)
    w_blk, _ = rows_colsplit(lower, n_interior, n, n_interior)
    _, s_tilde = rows_colsplit(upper, n_interior, n, n_interior)
    if drop_tol > 0.0:
        s_tilde = drop_small_rows(s_tilde, drop_tol)
    schur = factorize(s_tilde, rule, safeguard) if factor_schur else None
    return SimpleNamespace(interior=Factors(l_b, u_b, str(rule)), w_block=w_blk, z_block=z_blk,
                           s_tilde=s_tilde, schur=schur, n_interior=n_interior)


def extract_two_level_blocks(f: Factors, n_interior):
    """factor.py:886-907."""
    ints = np.arange(n_interior)
    exts = np.arange(n_interior, f.n)
    return SimpleNamespace(
        interior=Factors(extract_block(f.lower, ints, ints), extract_block(f.upper, ints, ints), f.kind),
        w_tilde=extract_block(f.lower, exts, ints),
        z_tilde=extract_block(f.upper, ints, exts),
        schur=Factors(extract_block(f.lower, exts, exts), extract_block(f.upper, exts, exts), f.kind))


# ---------------------------------------------------------------------------
# Krylov (krylov.py)


@dataclass
class Report:
    iterations: int
    converged: bool
    residual_history: np.ndarray
    final_relres: float
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0


def _back_substitute(h, g, k):
    """krylov.py:86-93."""
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        s = g[i]
        for j in range(i + 1, k):
            s -= h[i, j] * y[j]
        y[i] = s / h[i, i] if h[i, i] != 0.0 else 0.0
    return y


def _arnoldi_step(v_basis, w, h, cs, sn, g, j):
    """krylov.py:131-149: MGS against v_0..v_j, Givens update; returns hnext."""
    for i in range(j + 1):
        hij = vdot(v_basis[i], w)
        h[i, j] = hij
        axpy(-hij, v_basis[i], w)
    hnext = vnorm2(w)
    h[j + 1, j] = hnext
    for i in range(j):
        t = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
        h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
        h[i, j] = t
    denom = math.hypot(h[j, j], hnext)
    if denom == 0.0:
        cs[j], sn[j] = 1.0, 0.0
    else:
        cs[j] = h[j, j] / denom
        sn[j] = hnext / denom
    h[j, j] = cs[j] * h[j, j] + sn[j] * hnext
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]
    return hnext


def _op(a):
    return (lambda v: spmv(a, v)) if isinstance(a, Csr) else a


def restarted(a, b, m=None, x0=None, restart=50, rtol=1e-8, max_iters=20000, happy_tol=1e-14,
              flexible=True, record_history=True):
    """krylov.py:96-179 (_restarted); gmres = flexible False, fgmres = True."""
    apply_a, apply_m = _op(a), (_op(m) if m is not None else None)
    b = _f64(b)
    t0 = time.perf_counter()
    n = len(b)
    bnorm = vnorm2(b)
    scale = bnorm if bnorm > 0.0 else 1.0
    if x0 is None:
        x, r = np.zeros(n), b.copy()
    else:
        x = np.array(x0, dtype=np.float64)
        r = b - apply_a(x)
    beta = vnorm2(r)
    history = [beta / scale]
    final_rel = beta / scale
    converged = final_rel <= rtol
    its = 0
    mm = restart
    v_basis = np.empty((mm + 1, n))
    z_basis = np.empty((mm, n)) if flexible else None
    h = np.zeros((mm + 1, mm))
    cs, sn, g = np.empty(mm), np.empty(mm), np.empty(mm + 1)
    while not converged and its < max_iters:
        np.divide(r, beta, out=v_basis[0])
        g[:] = 0.0
        g[0] = beta
        k = 0
        for j in range(mm):
            z = apply_m(v_basis[j]) if apply_m is not None else v_basis[j]
            if flexible:
                z_basis[j] = z
            w = apply_a(z)
            hnext = _arnoldi_step(v_basis, w, h, cs, sn, g, j)
            its += 1
            k = j + 1
            est = abs(g[j + 1]) / scale
            history.append(est)
            if hnext < happy_tol:
                break
            np.divide(w, hnext, out=v_basis[j + 1])
            if est <= rtol or its >= max_iters:
                break
        y = _back_substitute(h, g, k)
        if flexible:
            for i in range(k):
                axpy(y[i], z_basis[i], x)
        else:
            u = np.zeros(n)
            for i in range(k):
                axpy(y[i], v_basis[i], u)
            axpy(1.0, apply_m(u) if apply_m is not None else u, x)
        r = b - apply_a(x)
        beta = vnorm2(r)
        final_rel = beta / scale
        if final_rel <= rtol:
            converged = True
    rep = Report(its, converged, np.array(history if record_history else []), final_rel)
    rep.solve_seconds = time.perf_counter() - t0
    return x, rep


def fgmres(a, b, m=None, x0=None, **kw):
    """krylov.py:200-210."""
    return restarted(a, b, m, x0, flexible=True, **kw)


def gmres(a, b, m=None, x0=None, **kw):
    """krylov.py:182-197."""
    return restarted(a, b, m, x0, flexible=False, **kw)


def fixed_gmres(apply_a, b, iters, apply_m=None, happy_tol=1e-14):
    """krylov.py:213-268."""
    n = len(b)
    if n == 0 or iters <= 0:
        return np.zeros(n)
    beta = vnorm2(b)
    if beta == 0.0:
        return np.zeros(n)
    mm = min(iters, n)
    v_basis = np.empty((mm + 1, n))
    h = np.zeros((mm + 1, mm))
    cs, sn, g = np.empty(mm), np.empty(mm), np.zeros(mm + 1)
    np.divide(b, beta, out=v_basis[0])
    g[0] = beta
    k = 0
    for j in range(mm):
        z = apply_m(v_basis[j]) if apply_m is not None else v_basis[j]
        w = apply_a(z)
        hnext = _arnoldi_step(v_basis, w, h, cs, sn, g, j)
        k = j + 1
        if hnext < happy_tol:
            break
        np.divide(w, hnext, out=v_basis[j + 1])
    y = _back_substitute(h, g, k)
    u = np.zeros(n)
    for i in range(k):
        axpy(y[i], v_basis[i], u)
    return apply_m(u) if apply_m is not None else u


# ---------------------------------------------------------------------------
# preconditioners (precond.py)


def domain_orderings(a: Csr, layout, use_rcm=True):
    """precond.py:137-147: RCM on the interior block only; exteriors keep index order."""
    def one(d):
        ints = layout.interior_of[d]
        if use_rcm and len(ints) > 1:
            _, inv = rcm(extract_block(a, ints, ints))
            ints = ints[inv]
        exts = layout.exterior_of[d]
        return SimpleNamespace(interior_nodes=ints, exterior_nodes=exts, nodes=np.concatenate([ints, exts]))
    return _pmap(one, range(layout.p))


def strip_diagonal_blocks(m: Csr, block_of):
    """precond.py:162-170."""
    keep = np.empty(m.nnz, dtype=np.uint8)
    block_of = _i64(block_of)
    lib().orc_keep_cross_block(_I(m.n_rows), _p(m.row_ptr), _p(m.col_idx), _p(block_of), _p(keep))
    keep = keep.astype(bool)
    idx = np.repeat(np.arange(m.n_rows), np.diff(m.row_ptr))
    rp = np.zeros(m.n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(idx[keep], minlength=m.n_rows), out=rp[1:])
    return Csr(m.n_rows, m.n_cols, rp, m.col_idx[keep], m.values[keep])


def add_to_diagonal(m: Csr, shifts):
    """precond.py:105-125 (diagonal present, or nothing to add where it is missing)."""
    rows = np.repeat(np.arange(m.n_rows), np.diff(m.row_ptr))
    slots = np.full(m.n_rows, -1, dtype=np.int64)
    on_diag = np.where(rows == m.col_idx)[0]
    slots[rows[on_diag]] = on_diag
    if np.any((slots < 0) & (shifts != 0.0)):
        raise NotImplementedError("oracle: l1 shift on a structurally missing diagonal")
    vals = m.values.copy()
    have = slots >= 0
    vals[slots[have]] += shifts[have]
    return Csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, vals)


class BjPrecond:
    """precond.py:177-214."""

    def __init__(self, a, layout, rule=Rule("ilu0"), use_rcm=True, l1=False):
        self.layout, self.rule = layout, rule
        self.domains = domain_orderings(a, layout, use_rcm)
        def one(d):
            dom = self.domains[d]
            local = take_submatrix(a, dom.nodes, dom.nodes)
            if l1:  # precond.py:207-212
                shifts = np.empty(len(dom.nodes))
                lib().orc_l1_row_shifts(_p(a.row_ptr), _p(a.col_idx), _p(a.values), _p(layout.owner),
                                        _I(len(dom.nodes)), _p(_i64(dom.nodes)), _I(d), _p(shifts))
                local = add_to_diagonal(local, shifts)
            return factorize(local, rule)
        self.factors = _pmap(one, range(len(self.domains)))

    def apply(self, r):
        z = np.empty_like(r)

        def one(d):
            dom = self.domains[d]
            z[dom.nodes] = self.factors[d].solve(r[dom.nodes])
        _pmap(one, range(len(self.domains)))
        return z


class SchurPrecond:
    """precond.py:221-292."""

    def __init__(self, a, layout, rule=Rule("ilu0"), inner_iters=3, schur_drop_tol=0.0, use_rcm=True):
        self.layout, self.rule, self.inner_iters = layout, rule, inner_iters
        self.domains = domain_orderings(a, layout, use_rcm)
        self.partial = _pmap(lambda d: partial_ilu(take_submatrix(a, d.nodes, d.nodes), len(d.interior_nodes), rule,
                                                   schur_drop_tol=schur_drop_tol), self.domains)
        ext_all = (np.concatenate([d.exterior_nodes for d in self.domains])
                   if layout.n_exterior else np.empty(0, dtype=np.int64))
        block_of = np.repeat(np.arange(layout.p), np.diff(layout.exterior_starts))
        self.coupling = strip_diagonal_blocks(take_submatrix(a, ext_all, ext_all), block_of)

    def _schur_solve(self, t):
        out = np.empty_like(t)
        s = self.layout.exterior_starts

        def one(d):
            out[s[d]:s[d + 1]] = self.partial[d].schur.solve(t[s[d]:s[d + 1]])
        _pmap(one, range(len(self.partial)))
        return out

    def reduced_matvec(self, y):
        return y + self._schur_solve(spmv(self.coupling, y))

    def apply(self, r):
        s = self.layout.exterior_starts
        ghat = np.empty(self.layout.n_exterior)

        def forward(d):
            dom, pf = self.domains[d], self.partial[d]
            fp = tri_solve_lower(pf.interior.lower, r[dom.interior_nodes], unit_diag=True)
            ghat[s[d]:s[d + 1]] = r[dom.exterior_nodes] - spmv(pf.w_block, fp)
            return fp
        fps = _pmap(forward, range(len(self.domains)))
        y = fixed_gmres(self.reduced_matvec, self._schur_solve(ghat), self.inner_iters)
        z = np.empty_like(r)

        def backward(d):
            dom, pf = self.domains[d], self.partial[d]
            yd = y[s[d]:s[d + 1]]
            z[dom.interior_nodes] = tri_solve_upper(pf.interior.upper, fps[d] - spmv(pf.z_block, yd))
            z[dom.exterior_nodes] = yd
        _pmap(backward, range(len(self.domains)))
        return z


class RapPrecond:
    """precond.py:304-438 (default MILU vectors: ones / zeros)."""

    def __init__(self, a, layout, modified=True, inner_iters=3, use_rcm=True):
        self.layout, self.inner_iters, self.modified = layout, inner_iters, modified
        self.domains = domain_orderings(a, layout, use_rcm)
        def one(dom):
            local = take_submatrix(a, dom.nodes, dom.nodes)
            plain = ilu0(local)
            coarse = milu0(local) if modified else plain
            return plain, extract_two_level_blocks(coarse, len(dom.interior_nodes))
        both = _pmap(one, self.domains)
        self.smoother, self.blocks = [b[0] for b in both], [b[1] for b in both]
        order = np.concatenate([d.interior_nodes for d in self.domains]
                               + [d.exterior_nodes for d in self.domains])
        self.perm_forward, self.perm_inverse = perm_from_order(order)
        self.a_perm = permute_symmetric(a, self.perm_forward)

    def _isl(self, d):
        s = self.layout.interior_starts
        return slice(s[d], s[d + 1])

    def _esl(self, d):
        s, n1 = self.layout.exterior_starts, self.layout.n_interior
        return slice(n1 + s[d], n1 + s[d + 1])

    def _csl(self, d):
        s = self.layout.exterior_starts
        return slice(s[d], s[d + 1])

    def interpolate(self, v):
        out = np.empty(self.layout.n)

        def one(d):
            blk = self.blocks[d]
            vd = v[self._csl(d)]
            out[self._isl(d)] = -tri_solve_upper(blk.interior.upper, spmv(blk.z_tilde, vd))
            out[self._esl(d)] = vd
        _pmap(one, range(len(self.blocks)))
        return out

    def restrict(self, t):
        out = np.empty(self.layout.n_exterior)

        def one(d):
            blk = self.blocks[d]
            s = tri_solve_lower(blk.interior.lower, t[self._isl(d)], unit_diag=True)
            out[self._csl(d)] = t[self._esl(d)] - spmv(blk.w_tilde, s)
        _pmap(one, range(len(self.blocks)))
        return out

    def coarse_matvec(self, v):
        return self.restrict(spmv(self.a_perm, self.interpolate(v)))

    def _coarse_precond(self, t):
        out = np.empty_like(t)

        def one(d):
            out[self._csl(d)] = self.blocks[d].schur.solve(t[self._csl(d)])
        _pmap(one, range(len(self.blocks)))
        return out

    def apply(self, r):
        b = r[self.perm_inverse]
        xhat = np.empty(self.layout.n)

        def smooth(d):
            isl, esl = self._isl(d), self._esl(d)
            sol = self.smoother[d].solve(np.concatenate([b[isl], b[esl]]))
            n1 = isl.stop - isl.start
            xhat[isl], xhat[esl] = sol[:n1], sol[n1:]
        _pmap(smooth, range(len(self.smoother)))
        res = b - spmv(self.a_perm, xhat)
        v = fixed_gmres(self.coarse_matvec, self.restrict(res), self.inner_iters,
                        apply_m=self._coarse_precond)
        x = xhat + self.interpolate(v) if len(v) else xhat
        z = np.empty_like(r)
        z[self.perm_inverse] = x
        return z


def make_preconditioner(name, a, layout, rule=Rule("ilu0"), inner_iters=3):
    """precond.py:450-474."""
    if name == "none":
        return None
    if name == "bj":
        return BjPrecond(a, layout, rule)
    if name == "l1bj":
        return BjPrecond(a, layout, rule, l1=True)
    if name == "schur":
        return SchurPrecond(a, layout, rule, inner_iters=inner_iters)
    if name == "rap":
        return RapPrecond(a, layout, modified=False, inner_iters=inner_iters)
    if name == "rap-milu":
        return RapPrecond(a, layout, modified=True, inner_iters=inner_iters)
    raise ValueError(f"unknown preconditioner {name!r}")


# ---------------------------------------------------------------------------
# problems (problems.py) + the BASELINE generators


def stencil_csr(dims, axis_coeffs, diag):
    """problems.py:29-71, without the per-row Python validation loop of
    csr_from_arrays (sparse.py:108-111): the output is sorted by construction."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n)
    strides = np.cumprod((1,) + dims[:-1])
    coord = [(idx // strides[d]) % dims[d] for d in range(len(dims))]
    below = [(-strides[d], coord[d] > 0, axis_coeffs[d][0]) for d in reversed(range(len(dims)))]
    above = [(strides[d], coord[d] < dims[d] - 1, axis_coeffs[d][1]) for d in range(len(dims))]
    counts = np.ones(n, dtype=np.int64)
    for _, mask, _ in below + above:
        counts += mask
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.empty(rp[-1], dtype=np.int64)
    vals = np.empty(rp[-1])
    pos = rp[:-1].copy()
    for off, mask, coef in below:
        r = idx[mask]
        ci[pos[r]] = r + off
        vals[pos[r]] = coef
        pos[r] += 1
    ci[pos] = idx
    vals[pos] = diag
    pos += 1
    for off, mask, coef in above:
        r = idx[mask]
        ci[pos[r]] = r + off
        vals[pos[r]] = coef
        pos[r] += 1
    return Csr(n, n, rp, ci, vals)


def poisson2d(nx, ny):
    return stencil_csr((nx, ny), [(-1.0, -1.0)] * 2, 4.0)


def poisson3d(nx, ny, nz):
    return stencil_csr((nx, ny, nz), [(-1.0, -1.0)] * 3, 6.0)


def convdiff3d(nx, ny, nz, velocity=(0.0, 0.0, 0.0)):
    """problems.py:84-100."""
    dims = (nx, ny, nz)
    coeffs = []
    for d in range(3):
        shift = 0.5 * float(velocity[d]) / (dims[d] + 1)
        coeffs.append((-1.0 - shift, -1.0 + shift))
    return stencil_csr(dims, coeffs, 6.0)


def aniso(dims, eps):
    """_stencil_csr(dims, [(-e,-e) for e in eps], 2*sum(eps))."""
    return stencil_csr(dims, [(-float(e), -float(e)) for e in eps], 2.0 * float(sum(eps)))


def convdiff27(nx, ny, nz, velocity=(10.0, 10.0, 10.0)):
    """27-point stencil, diagonal 26, all 26 neighbours -1, plus
    the centred convection shift s_d = 0.5 v_d / (n_d + 1) on the six face
    neighbours (upstream -1 - s, downstream -1 + s, as problems.py:97-99)."""
    dims = (nx, ny, nz)
    n = nx * ny * nz
    idx = np.arange(n)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    shift = [0.5 * float(velocity[d]) / (dims[d] + 1) for d in range(3)]
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny)
                      & (z + dz >= 0) & (z + dz < nz))
                off = (dx, dy, dz)
                if off == (0, 0, 0):
                    val = 26.0
                else:
                    val = -1.0
                    if sum(abs(o) for o in off) == 1:
                        d = [abs(o) for o in off].index(1)
                        val = -1.0 + shift[d] * off[d]
                r = idx[ok]
                rows.append(r)
                cols.append(r + dx + nx * dy + nx * ny * dz)
                vals.append(np.full(len(r), val))
    return csr_from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def default_rhs(a):
    """problems.py:103-105."""
    return spmv(a, np.ones(a.n_cols))


def run(a: Csr, hint, p, precond, rule=Rule("ilu0"), restart=50, rtol=1e-8, max_iters=20000,
        inner_iters=3, partition_kind="grid"):
    """bench.py:108-140 (run): returns (record, report, x) with the same
    setup / solve timing boundaries."""
    b = default_rhs(a)
    t0 = time.perf_counter()
    owner = row_block_owner(a.n_rows, p) if partition_kind == "rows" else partition(a, p, hint)
    layout = classify_and_order(a, owner)
    m = make_preconditioner(precond, a, layout, rule, inner_iters=inner_iters)
    setup_s = time.perf_counter() - t0
    x, rep = fgmres(a, b, m=m.apply if m is not None else None, restart=restart, rtol=rtol,
                    max_iters=max_iters)
    rep.setup_seconds = setup_s
    rec = dict(n=a.n_rows, p=p, precond=precond, fill=str(rule), its=rep.iterations,
               converged=rep.converged, setup_s=setup_s, solve_s=rep.solve_seconds,
               final_relres=rep.final_relres)
    return rec, rep, x
