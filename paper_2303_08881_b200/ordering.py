"""Domain partitioning and orderings (the reference's `ddilu.ordering`,
ordering.py:25), computed on the device.

* `partition`          structured box split as one kernel (ordering.py:171-190)
* `classify_and_order` exterior marking over the symmetrised pattern + one
                       stable radix pass that yields the whole layout
                       (ordering.py:253-297)
* `rcm`                bit-exact Cuthill-McKee in one persistent launch
                       (ordering.py:304-416; csrc/rcm.cu)
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as D
from .sparse import CsrMatrix, Permutation

__all__ = ["DomainLayout", "partition", "row_block_owner", "classify_and_order", "rcm"]


def _box_factors(dims, p):
    """ordering.py:130-145: primes of p, largest first, onto the longest axis."""
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


def row_block_owner(n: int, p: int) -> np.ndarray:
    """ordering.py:201-216."""
    if p < 1:
        raise ValueError("need at least one domain")
    if p > n:
        raise ValueError(f"more domains ({p}) than nodes ({n})")
    base, rem = divmod(n, p)
    sizes = np.full(p, base, dtype=np.int64)
    sizes[:rem] += 1
    return np.repeat(np.arange(p, dtype=np.int64), sizes)


class _Owner(np.ndarray):
    """int64 owner array that remembers its device copy (avoids a re-upload)."""

    _dev = None
    _p = None          # number of domains when the map came from partition() (values 0 .. _p-1 guaranteed)
    grid_hint = None   # dims of the structured grid the owner map was cut from (tiles the solves)

    def __array_finalize__(self, obj):
        if obj is not None:
            self.grid_hint = getattr(obj, "grid_hint", None)   # views / copies may be edited: no _dev, no _p


def _wrap_owner(host: np.ndarray, dev_t: torch.Tensor | None, grid_hint=None, p: int | None = None) -> np.ndarray:
    out = host.view(_Owner)
    out._dev = dev_t
    out._p = p
    if dev_t is not None:
        # the cached device copy is only valid while the host array is untouched: hand it out read-only
        # (`owner.copy()` is writable and carries no cache); classify_and_order re-checks the flag
        out.setflags(write=False)
    out.grid_hint = tuple(int(d) for d in grid_hint) if grid_hint is not None else None
    return out


def _owner_device(owner) -> torch.Tensor:
    d = getattr(owner, "_dev", None)
    if d is not None and not owner.flags.writeable:
        return d
    return D.to_device_i32(np.asarray(owner))


def partition(a: CsrMatrix, p: int, grid_hint=None) -> np.ndarray:
    """ordering.py:148-198.  Structured boxes as one kernel; the unstructured
    breadth-first fallback (`_grow_regions`) is a strictly serial greedy sweep
    and runs as a single device thread."""
    n = a.n_rows
    if a.n_rows != a.n_cols:
        raise ValueError("partition requires a square matrix")
    if p < 1:
        raise ValueError("need at least one domain")
    if p > n:
        raise ValueError(f"more domains ({p}) than nodes ({n})")
    if p == 1:
        hint = grid_hint if grid_hint is not None and int(np.prod(grid_hint)) == n and len(grid_hint) <= 3 else None
        return _wrap_owner(np.zeros(n, dtype=np.int64), None, hint)
    hint = None
    if grid_hint is not None:
        dims = tuple(int(d) for d in grid_hint)
        if int(np.prod(dims)) != n:
            raise ValueError("grid hint does not match matrix size")
        hint = dims if len(dims) <= 3 else None
        if len(dims) <= 3:
            factors = _box_factors(dims, p)
            sizes = np.ones(1, dtype=np.int64)
            for d, f in zip(dims, factors):
                chunk = np.array([len(c) for c in np.array_split(np.arange(d), f)], dtype=np.int64)
                sizes = np.outer(chunk, sizes).ravel()
            if np.max(np.abs(sizes - n / p)) <= max(1.0, 0.1 * n / p):
                owner_d = D.box_owner(n, dims, factors)
                return _wrap_owner(D.to_host_i64(owner_d), owner_d, hint, p)
    # unstructured fallback (ordering.py:192-198): greedy breadth-first growth over the symmetrised pattern
    base, rem = divmod(n, p)
    sizes = np.full(p, base, dtype=np.int32)
    sizes[:rem] += 1
    adj = D.sym_adjacency(a.device(), sort=True)
    owner_d = D.empty_i32(n)
    work = D.empty_i32(2 * n)
    D.call("ddilu_grow_regions", n, adj.rp, adj.ci, p, torch.from_numpy(sizes).to(D.dev()), owner_d, work)
    return _wrap_owner(D.to_host_i64(owner_d), owner_d, hint, p)


class DomainLayout:
    """ordering.py:223-250; host arrays are materialised lazily from the device."""

    def __init__(self, n, p, owner, gorder_d, exterior_d, owner_d, interior_starts, exterior_starts,
                 grid_hint=None):
        self.n, self.p = int(n), int(p)
        self.grid_hint = grid_hint       # natural-order grid dims (x fastest) if the matrix is structured
        self.owner = owner
        self.interior_starts = interior_starts
        self.exterior_starts = exterior_starts
        self.n_interior = int(interior_starts[-1])
        self._gorder_d = gorder_d        # int32[n]: old index at each new position
        self._exterior_d = exterior_d    # int32[n] flags
        self._owner_d = owner_d
        self._gorder_h = None
        self._perm = None

    @property
    def n_exterior(self) -> int:
        return self.n - self.n_interior

    def _gorder(self):
        if self._gorder_h is None:
            self._gorder_h = D.to_host_i64(self._gorder_d)
        return self._gorder_h

    @property
    def interior_of(self):
        g, s = self._gorder(), self.interior_starts
        return [g[s[d]:s[d + 1]] for d in range(self.p)]

    @property
    def exterior_of(self):
        g, s, n1 = self._gorder(), self.exterior_starts, self.n_interior
        return [g[n1 + s[d]:n1 + s[d + 1]] for d in range(self.p)]

    @property
    def global_perm(self) -> Permutation:
        if self._perm is None:
            self._perm = Permutation.from_order(self._gorder())
        return self._perm

    def domain_nodes(self, d: int) -> np.ndarray:
        return np.concatenate([self.interior_of[d], self.exterior_of[d]])


def classify_and_order(a: CsrMatrix, owner, p: int | None = None, grid_hint=None) -> DomainLayout:
    """ordering.py:253-297.  grid_hint (extension): dims of the structured grid in natural
    order; an owner array made by `partition(a, p, grid_hint)` carries it already.  It only
    selects the tiled triangular solves, results do not depend on it."""
    n = a.n_rows
    if grid_hint is None:
        grid_hint = getattr(owner, "grid_hint", None)
    if grid_hint is not None:
        grid_hint = tuple(int(d) for d in grid_hint)
        if int(np.prod(grid_hint)) != n or len(grid_hint) > 3:
            grid_hint = None
    owner_h = np.asarray(owner, dtype=np.int64) if not isinstance(owner, _Owner) else owner
    if owner_h.shape != (n,):
        raise ValueError("owner array has wrong length")
    trusted = (isinstance(owner, _Owner) and getattr(owner, "_dev", None) is not None and owner._p is not None
               and not owner.flags.writeable)        # made writable again => may have been edited: re-validate, re-upload
    if p is None:
        p = owner._p if trusted else (int(owner_h.max()) + 1 if n else 1)
    if trusted:
        if owner._p > p:          # made by partition(): values are 0 .. _p-1 by construction, no host pass
            raise ValueError("owner values out of range")
    elif n and (owner_h.min() < 0 or owner_h.max() >= p):
        raise ValueError("owner values out of range")
    ad = a.device()
    owner_d = _owner_device(owner_h)
    ext = D.empty_i32(max(n, 1))
    D.call("ddilu_mark_exterior", n, ad.rp, ad.ci, owner_d, ext)
    keys, vals = D.empty_i32(max(n, 1)), D.empty_i32(max(n, 1))
    D.call("ddilu_layout_keys", n, owner_d, ext, p, keys, vals)
    D.sort_pairs_(keys[:n], vals[:n], max(1, (2 * p - 1).bit_length()))
    bounds = D.empty_i32(2 * p + 1)
    D.call("ddilu_lower_bounds", keys, n, 2 * p, bounds)
    b = D.to_host_i64(bounds)
    interior_starts = b[: p + 1].copy()
    exterior_starts = b[p:] - b[p]
    return DomainLayout(n, p, owner_h, vals[:n], ext, owner_d, interior_starts, exterior_starts, grid_hint)


def rcm(a: CsrMatrix) -> Permutation:
    """ordering.py:400-416."""
    if a.n_rows != a.n_cols:
        raise ValueError("rcm requires a square matrix")
    n = a.n_rows
    if n == 0:
        return Permutation.identity(0)
    adj = D.sym_adjacency(a.device())
    cm = D.cm_order(adj)
    seg = torch.tensor([0, n], dtype=D.I32, device=D.dev())
    return Permutation.from_order(D.to_host_i64(D.reverse_segments(cm, seg)))
