"""Sparse containers and kernels: the reference's `ddilu.sparse` surface
(sparse.py:17-33) backed by device memory.

`CsrMatrix` and `Permutation` keep the reference's fields and invariants
(int64 / float64 host arrays, strictly increasing columns, explicit zeros
kept).  An instance can live on the host, on the device, or both: host arrays
are materialised lazily from the device copy and vice versa, so factors built
on the GPU are only copied back when somebody looks at them.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as D

__all__ = [
    "CsrMatrix", "Permutation", "csr_from_arrays", "csr_from_coo", "csr_from_dense", "csr_identity",
    "csr_transpose", "spmv", "tri_solve_lower", "tri_solve_upper", "permute_symmetric", "extract_block",
    "take_submatrix", "vdot", "vnorm2", "sparse_matmul",
]


class CsrMatrix:
    """Compressed sparse row matrix (sparse.py:40-84); immutable by convention."""

    def __init__(self, n_rows, n_cols, row_ptr=None, col_idx=None, values=None, _device: D.DeviceCsr | None = None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self._rp, self._ci, self._v = row_ptr, col_idx, values
        self._dev = _device
        self._sched = {}
        if row_ptr is None and _device is None:
            raise ValueError("CsrMatrix needs host arrays or a device matrix")

    @staticmethod
    def from_device(d: D.DeviceCsr) -> "CsrMatrix":
        return CsrMatrix(d.n_rows, d.n_cols, _device=d)

    def _pull(self):
        if self._rp is None:
            self._rp, self._ci, self._v = self._dev.to_host()

    @property
    def row_ptr(self) -> np.ndarray:
        self._pull()
        return self._rp

    @property
    def col_idx(self) -> np.ndarray:
        self._pull()
        return self._ci

    @property
    def values(self) -> np.ndarray:
        self._pull()
        return self._v

    def device(self) -> D.DeviceCsr:
        """Device copy (int32 indices); uploaded once on first use."""
        if self._dev is None:
            self._dev = D.DeviceCsr.from_host(self.n_rows, self.n_cols, self._rp, self._ci, self._v)
        return self._dev

    @property
    def nnz(self) -> int:
        return int(self._rp[-1]) if self._rp is not None else self._dev.nnz

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        out[rows, self.col_idx] = self.values
        return out

    def with_values(self, values) -> "CsrMatrix":
        values = np.asarray(values, dtype=np.float64)
        if values.shape != self.values.shape:
            raise ValueError("value array does not match pattern size")
        return CsrMatrix(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, values)

    def schedule(self, upper: bool) -> D.Schedule:
        key = bool(upper)
        if key not in self._sched:
            self._sched[key] = D.build_schedule(self.device(), upper)
        return self._sched[key]

    def __repr__(self):
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


def csr_from_arrays(n_rows, n_cols, row_ptr, col_idx, values) -> CsrMatrix:
    """Validating constructor (sparse.py:87-112); same checks, vectorised."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
    values = np.ascontiguousarray(values, dtype=np.float64)
    if n_rows < 0 or n_cols < 0:
        raise ValueError("negative dimension")
    if row_ptr.shape != (n_rows + 1,):
        raise ValueError("row_ptr has wrong length")
    if row_ptr[0] != 0 or row_ptr[-1] != len(col_idx) or len(col_idx) != len(values):
        raise ValueError("row_ptr endpoints inconsistent with entry arrays")
    if np.any(np.diff(row_ptr) < 0):
        raise ValueError("row_ptr must be nondecreasing")
    if len(col_idx) and (col_idx.min() < 0 or col_idx.max() >= n_cols):
        raise ValueError("column index out of range")
    if len(col_idx) > 1:
        bad = np.diff(col_idx) <= 0
        starts = row_ptr[1:-1]
        bad[starts[(starts > 0) & (starts < len(col_idx))] - 1] = False  # row boundaries may go down
        if np.any(bad):
            k = int(np.argmax(bad))
            row = int(np.searchsorted(row_ptr, k, side="right") - 1)
            raise ValueError(f"columns of row {row} not strictly increasing")
    return CsrMatrix(n_rows, n_cols, row_ptr, col_idx, values)


def csr_from_coo(n_rows, n_cols, rows, cols, vals) -> CsrMatrix:
    """sparse.py:115-147."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if not (len(rows) == len(cols) == len(vals)):
        raise ValueError("coordinate arrays must have equal length")
    if len(rows):
        if rows.min() < 0 or rows.max() >= n_rows:
            raise ValueError("row index out of range")
        if cols.min() < 0 or cols.max() >= n_cols:
            raise ValueError("column index out of range")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(rows) > 1:
        same = (np.diff(rows) == 0) & (np.diff(cols) == 0)
        if np.any(same):
            k = int(np.argmax(same))
            raise ValueError(f"duplicate entry at ({rows[k]}, {cols[k]})")
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return CsrMatrix(n_rows, n_cols, row_ptr, cols.copy(), vals.copy())


def csr_from_dense(a, keep_zeros: bool = False) -> CsrMatrix:
    """sparse.py:150-160."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-d array")
    if keep_zeros:
        rows, cols = np.indices(a.shape)
        rows, cols = rows.ravel(), cols.ravel()
    else:
        rows, cols = np.nonzero(a)
    return csr_from_coo(a.shape[0], a.shape[1], rows, cols, a[rows, cols])


def csr_identity(n: int) -> CsrMatrix:
    idx = np.arange(n + 1, dtype=np.int64)
    return CsrMatrix(n, n, idx, idx[:n].copy(), np.ones(n))


class Permutation:
    """forward[old] = new, inverse[new] = old (sparse.py:168-212)."""

    def __init__(self, forward, inverse=None):
        fwd = np.ascontiguousarray(forward, dtype=np.int64)
        if inverse is None:
            inv = np.empty_like(fwd)
            inv[fwd] = np.arange(len(fwd), dtype=np.int64)
        else:
            inv = np.ascontiguousarray(inverse, dtype=np.int64)
        n = len(fwd)
        if len(inv) != n:
            raise ValueError("forward and inverse must have equal length")
        if n and (fwd.min() < 0 or fwd.max() >= n or np.bincount(fwd, minlength=n).max() != 1):
            raise ValueError("forward is not a bijection")
        if np.any(inv[fwd] != np.arange(n)):
            raise ValueError("inverse does not invert forward")
        self.forward, self.inverse = fwd, inv

    @property
    def n(self) -> int:
        return len(self.forward)

    @staticmethod
    def identity(n: int) -> "Permutation":
        idx = np.arange(n, dtype=np.int64)
        return Permutation(idx, idx.copy())

    @staticmethod
    def from_order(order) -> "Permutation":
        order = np.ascontiguousarray(order, dtype=np.int64)
        fwd = np.empty_like(order)
        fwd[order] = np.arange(len(order), dtype=np.int64)
        return Permutation(fwd, order)


# ---------------------------------------------------------------------------
# operations (host arrays in, host arrays out; the arithmetic runs on the GPU)


def _vec(x, n, what="vector length does not match matrix columns"):
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (n,):
        raise ValueError(what)
    return D.to_device_f64(x)


def spmv(a: CsrMatrix, x) -> np.ndarray:
    """sparse.py:389-400: a @ x, bit-identical to the serial row sums."""
    xd = _vec(x, a.n_cols)
    out = D.empty_f64(a.n_rows)
    D.spmv(a.device(), xd, out)
    return out.cpu().numpy()


def _tri(t: CsrMatrix, b, upper: bool, unit_diag: bool) -> np.ndarray:
    b = np.asarray(b, dtype=np.float64)
    if t.n_rows != t.n_cols or b.shape != (t.n_rows,):
        raise ValueError("shape mismatch in triangular solve")
    bd = D.to_device_f64(b)
    out = D.empty_f64(max(t.n_rows, 1))[: t.n_rows]
    D.sptrsv(t.device(), t.schedule(upper), bd, out, upper, unit_diag, check=True)
    return out.cpu().numpy()


def tri_solve_lower(l: CsrMatrix, b, unit_diag: bool = False) -> np.ndarray:
    """sparse.py:403-416."""
    return _tri(l, b, False, unit_diag)


def tri_solve_upper(u: CsrMatrix, b, unit_diag: bool = False) -> np.ndarray:
    """sparse.py:419-428."""
    return _tri(u, b, True, unit_diag)


def _gather(a: CsrMatrix, rows: np.ndarray, cols: np.ndarray, resort: bool) -> CsrMatrix:
    rows_d = D.to_device_i32(rows)
    colmap = D.index_map(a.n_cols, D.to_device_i32(cols))
    out = D.gather_rows(a.device(), rows_d, len(rows), colmap, len(cols), resort=resort)
    return CsrMatrix.from_device(out)


def extract_block(a: CsrMatrix, rows, cols) -> CsrMatrix:
    """sparse.py:456-471 (strictly increasing index sets)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    for name, idx, bound in (("rows", rows, a.n_rows), ("cols", cols, a.n_cols)):
        if len(idx) and (idx.min() < 0 or idx.max() >= bound):
            raise ValueError(f"{name} out of range")
        if len(idx) > 1 and np.any(np.diff(idx) <= 0):
            raise ValueError(f"{name} must be strictly increasing")
    return _gather(a, rows, cols, resort=False)


def take_submatrix(a: CsrMatrix, rows, cols) -> CsrMatrix:
    """sparse.py:474-484 (any order; rows re-sorted by column)."""
    return _gather(a, np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64), resort=True)


def permute_symmetric(a: CsrMatrix, perm: Permutation) -> CsrMatrix:
    """sparse.py:431-442: B[p(i), p(j)] = A[i, j] = take_submatrix with rows = cols = perm.inverse."""
    if a.n_rows != a.n_cols or perm.n != a.n_rows:
        raise ValueError("permutation size does not match matrix")
    return _gather(a, perm.inverse, perm.inverse, resort=True)


def csr_transpose(a: CsrMatrix) -> CsrMatrix:
    """sparse.py:508-516: stable sort of the entries by column on the device."""
    d = a.device()
    nnz = d.nnz
    rows = D.empty_i32(max(nnz, 1))[:nnz]
    lens = D.empty_i32(max(a.n_rows, 1))
    D.call("ddilu_row_lengths", a.n_rows, d.rp, lens)
    rows = torch.repeat_interleave(torch.arange(a.n_rows, dtype=D.I32, device=D.dev()), lens[: a.n_rows].long())
    keys = d.ci.clone()
    perm = torch.arange(nnz, dtype=D.I32, device=D.dev())
    bits = max(1, int(max(a.n_cols - 1, 1)).bit_length())
    D.sort_pairs_(keys, perm, bits)
    rp = D.zeros_i32(a.n_cols + 2)
    D.call("ddilu_lower_bounds", keys, nnz, a.n_cols, rp)
    out = D.DeviceCsr(a.n_cols, a.n_rows, rp[: a.n_cols + 1], D.gather_i32(rows, perm),
                      d.val[perm.long()], nnz)
    return CsrMatrix.from_device(out)


def sparse_matmul(a: CsrMatrix, b: CsrMatrix) -> CsrMatrix:
    """sparse.py:487-505: a @ b with the exact structural pattern (entries that cancel to zero are kept).
    Count -> scan -> expand (products of a row in the reference's traversal order, stably sorted by column)
    -> scan -> sum the runs, on the device; values carry the reference's bits."""
    if a.n_cols != b.n_rows:
        raise ValueError("inner dimensions do not match")
    n = a.n_rows
    da, db = a.device(), b.device()
    off = D.zeros_i32(n + 1)
    D.call("ddilu_spgemm_bound", n, da.rp, da.ci, db.rp, off)
    D.exclusive_scan_(off, n)
    total = int(off[-1].item()) if n else 0
    s_col, s_val = D.empty_i32(max(total, 1)), D.empty_f64(max(total, 1))
    out_rp = D.zeros_i32(n + 1)
    D.call("ddilu_spgemm_expand", n, da.rp, da.ci, da.val, db.rp, db.ci, db.val, off, s_col, s_val, out_rp)
    D.exclusive_scan_(out_rp, n)
    nnz = int(out_rp[-1].item()) if n else 0
    out_ci, out_v = D.empty_i32(max(nnz, 1)), D.empty_f64(max(nnz, 1))
    D.call("ddilu_spgemm_compact", n, off, s_col, s_val, out_rp, out_ci, out_v)
    return CsrMatrix.from_device(D.DeviceCsr(n, b.n_cols, out_rp, out_ci[:nnz], out_v[:nnz], nnz))


_reducer = None


def _red():
    global _reducer
    if _reducer is None:
        _reducer = D.Reducer()
    return _reducer


def vdot(a, b) -> float:
    """sparse.py:519-523.  Device reduction: per-CTA partials added in CTA order
    (deterministic run to run; not the serial left-to-right order)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    out = D.zeros_f64(1)
    _red().dot(a.size, D.to_device_f64(a), D.to_device_f64(b), out)
    return float(out.item())


def vnorm2(a) -> float:
    """sparse.py:526-528."""
    return float(np.sqrt(vdot(a, a)))
