"""Incomplete LU factorisations on the device (the reference's `ddilu.factor`
surface, factor.py:36-50).

ilu0 / milu0 / partial_ilu run the level-scheduled numeric kernel of
csrc/factor.cu on the split pattern (factor.py:198-263, 397-432); ilut runs the
sync-free row kernel of csrc/ilut.cu (factor.py:482-656).  Results are device
resident; the host CSR arrays of the returned objects are materialised only
when read.  iluk (level-of-fill k > 0): symbolic phase in csrc/iluk.cu, numeric
phase = the same fixed-pattern kernel on the larger pattern.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .sparse import CsrMatrix

__all__ = [
    "FillRule", "IluFactors", "MiluVectors", "PartialIluFactors", "TwoLevelBlocks", "ilu0", "iluk", "ilut", "milu0",
    "factorize", "partial_ilu", "extract_two_level_blocks", "DIAG_SAFEGUARD",
]

DIAG_SAFEGUARD = 1e-6


@dataclass(frozen=True)
class FillRule:
    """factor.py:59-105."""

    kind: str
    level: int = 0
    tau: float = 0.0
    maxfill: int = 0

    def __post_init__(self):
        if self.kind not in ("ilu0", "iluk", "ilut"):
            raise ValueError(f"unknown fill rule {self.kind!r}")
        if self.kind == "iluk" and self.level < 0:
            raise ValueError("iluk level must be nonnegative")
        if self.kind == "ilut":
            if self.tau < 0:
                raise ValueError("ilut tau must be nonnegative")
            if self.maxfill < 1:
                raise ValueError("ilut maxfill must be at least 1")

    @staticmethod
    def parse(text: str) -> "FillRule":
        head, _, rest = text.partition(":")
        if head == "ilu0" and not rest:
            return FillRule("ilu0")
        if head == "iluk" and rest:
            return FillRule("iluk", level=int(rest))
        if head == "ilut" and rest:
            tau_s, _, fill_s = rest.partition(",")
            if not fill_s:
                raise ValueError(f"ilut needs tau and maxfill, got {text!r}")
            return FillRule("ilut", tau=float(tau_s), maxfill=int(fill_s))
        raise ValueError(f"cannot parse fill rule {text!r}")

    def __str__(self) -> str:
        if self.kind == "iluk":
            return f"iluk:{self.level}"
        if self.kind == "ilut":
            return f"ilut:{self.tau:g},{self.maxfill}"
        return "ilu0"


# ---------------------------------------------------------------------------
# device level


class DevFactors:
    """Unit-lower L (strict part stored) and U (diagonal first in each row) in
    HBM together with their level schedules."""

    def __init__(self, lower: D.DeviceCsr, upper: D.DeviceCsr, sched_l: D.Schedule | None = None):
        self.lower, self.upper = lower, upper
        self._sl, self._su = sched_l, None
        self._levs = {}            # upper? -> (lev, n_levels), shared by the tiled and the sync-free layouts
        if sched_l is not None:
            self._levs[False] = (sched_l.lev, sched_l.n_levels)
        self._tl = self._tu = None  # tiled layouts (D.TileSched) when the factor tiles
        self._bw = None             # (L, U) shared-memory-window plans of the block-local sweep
        self._sw = None             # D.SweepPlan: one CTA per diagonal block (interface factors)
        self._cs = None             # D.ClusterSweepPlan: one thread-block cluster per diagonal block (interior factors)
        self._tmp = None

    @property
    def n(self):
        return self.lower.n_rows

    def _lev(self, upper: bool):
        if upper not in self._levs:
            self._levs[upper] = D.levels(self.upper if upper else self.lower, upper)
        return self._levs[upper]

    @property
    def sched_l(self) -> D.Schedule:
        if self._sl is None:
            self._sl = D.build_schedule(self.lower, False, *self._lev(False))
        return self._sl

    @property
    def sched_u(self) -> D.Schedule:
        if self._su is None:
            self._su = D.build_schedule(self.upper, True, *self._lev(True))
        return self._su

    def prepare(self, seg_ptr=None, part: "D.TilePartition | None" = None, cluster_seg=None):
        """Build the solve layouts now (inside setup).  part: tile partition of the
        rows (structured problems) -> tiled solve, with the sync-free SELL solve as the
        fallback when the tile graph is not one-way.  seg_ptr: row ranges of independent
        diagonal blocks (one per subdomain), if known.  cluster_seg: the same for LARGE blocks
        (interior factors) -> cluster sweep when the pair qualifies; part may then be a callable
        () -> partition so that the tiles are only built when they are needed."""
        if cluster_seg is not None and D.USE_CSWEEP and self.n:
            self._cs = D.build_csweep(self.lower, self.upper, *self._lev(False), *self._lev(True), cluster_seg)
            if self._cs is not None:
                return self
        if getattr(part, "lazy", False):
            part = part()
        if seg_ptr is not None and D.USE_SWEEP and self.n:
            # small, deep, block-diagonal (the interface factors): one CTA per block walks the levels in shared
            # memory, L and U in one launch (csrc/sweep.cu); the other layouts are then built only on demand
            self._sw = D.build_sweep(self.lower, self.upper, *self._lev(False), *self._lev(True), seg_ptr)
            if self._sw is not None:
                return self
        if part is not None and D.USE_TILED and self.n:
            # part: one TilePartition for both factors, or a callable (lev, n_levels) -> TilePartition for
            # partitions that depend on the factor's own levels (wavefront-slab tiles)
            for upper in (False, True):
                fac = self.upper if upper else self.lower
                if not callable(part) and getattr(part, "geom", None) is not None and part.n == self.n:
                    # box tiles of a structured grid: the lattice solve if every tile qualifies
                    sched = D.tile_schedule(fac, part, upper)
                    ts = D.build_lattice(fac, part, upper, not upper, sched) if sched is not None else None
                    if ts is None and sched is not None:
                        ts = D.build_tiles(fac, self._lev(upper)[0], part, upper, not upper, sched)
                    if upper:
                        self._tu = ts
                    else:
                        self._tl = ts
                    continue
                lev, nlev = self._lev(upper)
                pt = part(lev, nlev) if callable(part) else part
                ts = D.build_tiles(self.upper if upper else self.lower, lev, pt, upper, not upper) \
                    if pt is not None else None
                if ts is None and callable(part) and getattr(part, "fallback", None) is not None:
                    ts = D.build_tiles(self.upper if upper else self.lower, lev, part.fallback, upper, not upper)
                if upper:
                    self._tu = ts
                else:
                    self._tl = ts
        if seg_ptr is not None and D.USE_BLOCK_WINDOW and self.n:
            bwl = D.enable_block_window(self.lower, self.sched_l, seg_ptr, False, True)
            bwu = D.enable_block_window(self.upper, self.sched_u, seg_ptr, True, False) if bwl is not None else None
            self._bw = (bwl, bwu) if bwu is not None else None
        if seg_ptr is not None and (self._tl is None or self._tu is None):
            D.enable_block_local(self.sched_l, seg_ptr) and D.enable_block_local(self.sched_u, seg_ptr)
        if self._tl is None:
            self.sched_l if D.uses_warprow(self.lower) else D.get_sell(self.lower, self.sched_l, False, True)
        if self._tu is None:
            self.sched_u if D.uses_warprow(self.upper) else D.get_sell(self.upper, self.sched_u, True, False)
        if self._tmp is None:
            self._tmp = D.empty_f64(max(self.n, 1))
        return self

    def lower_solve(self, b, out):
        if self._cs is not None:
            return D.csweep_solve(self._cs, False, b, out)
        if self._sw is not None:
            D.sweep_rhs(self._sw, False, b)
            return D.sweep_solve(self._sw, 1, out)
        if self._bw is not None:
            return D.sptrsv_block_window(self.lower, self.sched_l, self._bw[0], b, out, False, True)
        if self._tl is not None:
            return D.sptrsv_tiled(self._tl, b, out)
        return D.sptrsv(self.lower, self.sched_l, b, out, False, True)

    def upper_solve(self, b, out):
        if self._cs is not None:
            return D.csweep_solve(self._cs, True, b, out)
        if self._sw is not None:
            D.sweep_rhs(self._sw, True, b)
            return D.sweep_solve(self._sw, 2, out)
        if self._bw is not None:
            return D.sptrsv_block_window(self.upper, self.sched_u, self._bw[1], b, out, True, False)
        if self._tu is not None:
            return D.sptrsv_tiled(self._tu, b, out)
        return D.sptrsv(self.upper, self.sched_u, b, out, True, False)

    def solve(self, b, out):
        """out = U^-1 L^-1 b (factor.py:124-126)."""
        if self._sw is not None:
            D.sweep_rhs(self._sw, False, b)
            return D.sweep_solve(self._sw, 3, out)
        if self._tmp is None:
            self._tmp = D.empty_f64(max(self.n, 1))
        self.lower_solve(b, self._tmp)
        return self.upper_solve(self._tmp, out)


def solve_with_product(f: DevFactors, mat: D.DeviceCsr, y, base, mode: int, out, add=None):
    """out = (add +) U^-1 L^-1 (mat y | base - mat y | base + mat y) for mode 0 | 1 | 2: the product feeds the
    sweep's right-hand side directly and the sum is folded into its result stores (precond.py:242-249:
    `S^-1 (r_ext - W fp)`, `y + S^-1 (E_off y)`).  Needs the factor pair's sweep plan (callers keep the
    separate-kernel sequence for factors without one)."""
    if f._sw is None:
        raise RuntimeError("solve_with_product needs a sweep plan (DevFactors.prepare(seg_ptr=...))")
    D.sweep_rhs(f._sw, False, base, mat, y, mode, add=add)
    return D.sweep_solve(f._sw, 3, out, add=add is not None)


def d_level0_split(a: D.DeviceCsr, n_elim: int):
    """factor.py:249-263 on the device: (L pattern+values, U pattern+values, row inf-norms)."""
    n = a.n_rows
    p_rp, k_rp = D.zeros_i32(n + 1), D.zeros_i32(n + 1)
    rownorm = D.empty_f64(max(n, 1))
    D.call("ddilu_split_count", n, a.rp, a.ci, a.val, int(n_elim), p_rp, k_rp, rownorm)
    D.exclusive_scan_(p_rp, n)
    D.exclusive_scan_(k_rp, n)
    pn, kn = int(p_rp[-1].item()), int(k_rp[-1].item())
    p_ci, p_v, k_ci, k_v = D.empty_i32(pn), D.empty_f64(pn), D.empty_i32(kn), D.empty_f64(kn)
    D.call("ddilu_split_fill", n, a.rp, a.ci, a.val, int(n_elim), p_rp, p_ci, p_v, k_rp, k_ci, k_v)
    return D.DeviceCsr(n, n, p_rp, p_ci, p_v, pn), D.DeviceCsr(n, n, k_rp, k_ci, k_v, kn), rownorm


def d_factor_level0(a: D.DeviceCsr, n_elim: int, milu: bool = False, target: torch.Tensor | None = None,
                    wvec: torch.Tensor | None = None, safeguard: float = DIAG_SAFEGUARD, level: int = 0,
                    sections=None) -> DevFactors:
    """factor.py:446-458 `_factor_on_pattern`: split (level 0) or symbolic level-of-fill pattern
    (level > 0, factor.py:704-720, 855-863), schedule, numeric sweep."""
    n = a.n_rows
    if level > 0 and n:
        from ._iluk import d_iluk_split
        from ._ilut import interleaved_order
        lo, up = d_iluk_split(a, n_elim, level, interleaved_order(n, sections) if sections is not None else None)
        rownorm = D.empty_f64(n)                     # row inf-norms of A: by-product of the split's count pass
        D.call("ddilu_split_count", n, a.rp, a.ci, a.val, int(n_elim), D.empty_i32(n + 1), D.empty_i32(n + 1), rownorm)
    else:
        lo, up, rownorm = d_level0_split(a, n_elim)
    sched = D.build_schedule(lo, False)
    done = D.empty_i32(max(n, 1))
    D.call("ddilu_ilu0_numeric", n, sched.n_slots, sched.order, lo.rp, lo.ci, lo.val, up.rp, up.ci, up.val,
           int(n_elim), int(milu), target, wvec, float(safeguard), rownorm, done)
    return DevFactors(lo, up, sched)


def d_ilut(a: D.DeviceCsr, n_elim: int, tau: float, maxfill: int, tau_s: float,
           safeguard: float = DIAG_SAFEGUARD, sections=None) -> DevFactors:
    """sections: pointer arrays of the independent diagonal blocks, one per row section ([interiors | exteriors] or
    one section) -- the ILUT kernel then works on all blocks at once (`_ilut.interleaved_order`); the result does
    not depend on it."""
    from ._ilut import d_ilut_factor, interleaved_order
    order = interleaved_order(a.n_rows, sections) if sections is not None else None
    return d_ilut_factor(a, n_elim, tau, maxfill, tau_s, safeguard, order)


def d_factorize(a: D.DeviceCsr, rule: FillRule, safeguard: float = DIAG_SAFEGUARD, sections=None) -> DevFactors:
    if rule.kind == "ilu0" or rule.kind == "iluk":
        return d_factor_level0(a, a.n_rows, safeguard=safeguard, level=rule.level if rule.kind == "iluk" else 0,
                               sections=sections)
    return d_ilut(a, a.n_rows, rule.tau, rule.maxfill, 0.0, safeguard, sections)


class DevPartial:
    """L_B, U_B, W, Z, S~ and the factors of S~ (factor.py:165-181), device resident."""

    def __init__(self, interior: DevFactors, w: D.DeviceCsr, z: D.DeviceCsr, s_tilde: D.DeviceCsr,
                 schur: DevFactors | None, n_interior: int):
        self.interior, self.w, self.z, self.s_tilde, self.schur, self.n_interior = interior, w, z, s_tilde, schur, n_interior


def d_carve(f: DevFactors, n1: int):
    """Blocks of a factor pair cut at row/column n1 (factor.py:869-872, 886-907)."""
    n = f.n
    l_b = D.csr_block(f.lower, 0, n1, 0, n1)
    u_b = D.csr_block(f.upper, 0, n1, 0, n1)
    z = D.csr_block(f.upper, 0, n1, n1, n)
    w = D.csr_block(f.lower, n1, n, 0, n1)
    l_s = D.csr_block(f.lower, n1, n, n1, n)
    u_s = D.csr_block(f.upper, n1, n, n1, n)
    return l_b, u_b, w, z, l_s, u_s


def d_drop_small_rows(m: D.DeviceCsr, tol: float) -> D.DeviceCsr:
    """factor.py:806-822 (`schur_drop_tol` thinning, diagonal kept)."""
    if tol <= 0.0 or m.nnz == 0:
        return m
    n = m.n_rows
    rp = D.zeros_i32(n + 1)
    D.call("ddilu_drop_small_count", n, m.rp, m.ci, m.val, float(tol), rp)
    D.exclusive_scan_(rp, n)
    nnz = int(rp[-1].item())
    ci, val = D.empty_i32(nnz), D.empty_f64(nnz)
    D.call("ddilu_drop_small_fill", n, m.rp, m.ci, m.val, float(tol), rp, ci, val)
    return D.DeviceCsr(n, m.n_cols, rp, ci, val, nnz)


def d_partial_ilu(a: D.DeviceCsr, n_interior: int, rule: FillRule, schur_drop_tol: float = 0.0,
                  factor_schur: bool = True, safeguard: float = DIAG_SAFEGUARD, blocks=None) -> DevPartial:
    """factor.py:825-883.  blocks = (interior pointers, interface pointers) of the independent subdomain blocks
    when a is block-diagonal by subdomain (a scheduling hint for ILUT, see d_ilut)."""
    if rule.kind == "ilut":
        f = d_ilut(a, n_interior, rule.tau, rule.maxfill, schur_drop_tol, safeguard, sections=blocks)
        drop_tol = 0.0
    else:
        f = d_factor_level0(a, n_interior, safeguard=safeguard, level=rule.level if rule.kind == "iluk" else 0,
                            sections=blocks)
        drop_tol = schur_drop_tol
    l_b, u_b, w, z, _, s_tilde = d_carve(f, n_interior)
    s_tilde = d_drop_small_rows(s_tilde, drop_tol)
    schur = d_factorize(s_tilde, rule, safeguard, sections=blocks[1:] if blocks is not None else None) \
        if factor_schur else None
    return DevPartial(DevFactors(l_b, u_b), w, z, s_tilde, schur, n_interior)


# ---------------------------------------------------------------------------
# host-facing result types (same fields as the reference)


class IluFactors:
    """factor.py:108-131."""

    def __init__(self, lower: CsrMatrix, upper: CsrMatrix, kind: str = "ilu0", _dev: DevFactors | None = None):
        self.lower, self.upper, self.kind = lower, upper, kind
        self._dev = _dev

    @staticmethod
    def _from_device(d: DevFactors, kind: str) -> "IluFactors":
        return IluFactors(CsrMatrix.from_device(d.lower), CsrMatrix.from_device(d.upper), kind, d)

    def device(self) -> DevFactors:
        if self._dev is None:
            self._dev = DevFactors(self.lower.device(), self.upper.device())
        return self._dev

    @property
    def n(self) -> int:
        return self.lower.n_rows

    def solve(self, b) -> np.ndarray:
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (self.n,):
            raise ValueError("shape mismatch in triangular solve")
        out = D.empty_f64(max(self.n, 1))[: self.n]
        self.device().solve(D.to_device_f64(b), out)
        return out.cpu().numpy()

    def lu_matvec(self, y) -> np.ndarray:
        from .sparse import spmv
        t = spmv(self.upper, y)
        return t + spmv(self.lower, t)


@dataclass(frozen=True)
class MiluVectors:
    """factor.py:134-162."""

    y: np.ndarray
    z: np.ndarray
    w: np.ndarray

    @staticmethod
    def ones(n: int, n_exterior: int = 0) -> "MiluVectors":
        return MiluVectors(y=np.ones(n - n_exterior), z=np.ones(n_exterior), w=np.zeros(n - n_exterior))

    def full_target(self) -> np.ndarray:
        return np.concatenate([np.asarray(self.y, dtype=np.float64), np.asarray(self.z, dtype=np.float64)])

    def full_w(self, n: int) -> np.ndarray:
        w = np.asarray(self.w, dtype=np.float64)
        return np.concatenate([w, np.zeros(n - len(w))])


@dataclass(frozen=True)
class PartialIluFactors:
    """factor.py:165-181."""

    interior: IluFactors
    w_block: CsrMatrix
    z_block: CsrMatrix
    s_tilde: CsrMatrix
    schur: IluFactors | None
    n_interior: int


@dataclass(frozen=True)
class TwoLevelBlocks:
    """factor.py:184-191."""

    interior: IluFactors
    w_tilde: CsrMatrix
    z_tilde: CsrMatrix
    schur: IluFactors


def _check_square(a: CsrMatrix):
    if a.n_rows != a.n_cols:
        raise ValueError("factorization requires a square matrix")


def ilu0(a: CsrMatrix, safeguard: float = DIAG_SAFEGUARD) -> IluFactors:
    """factor.py:668-677."""
    _check_square(a)
    return IluFactors._from_device(d_factor_level0(a.device(), a.n_rows, safeguard=safeguard), "ilu0")


def milu0(a: CsrMatrix, vecs: MiluVectors | None = None, safeguard: float = DIAG_SAFEGUARD) -> IluFactors:
    """factor.py:680-701."""
    _check_square(a)
    n = a.n_rows
    if vecs is None:
        vecs = MiluVectors.ones(n)
    target = vecs.full_target()
    if len(target) != n:
        raise ValueError("milu target vector has wrong length")
    if np.any(target == 0.0):
        raise ValueError("milu target vector must have no zero entries")
    d = d_factor_level0(a.device(), n, True, D.to_device_f64(target), D.to_device_f64(vecs.full_w(n)), safeguard)
    return IluFactors._from_device(d, "milu0")


def iluk(a: CsrMatrix, level: int, safeguard: float = DIAG_SAFEGUARD) -> IluFactors:
    """factor.py:704-720."""
    _check_square(a)
    if level < 0:
        raise ValueError("level must be nonnegative")
    if level == 0:
        return ilu0(a, safeguard)
    d = d_factor_level0(a.device(), a.n_rows, safeguard=safeguard, level=level)
    return IluFactors._from_device(d, str(FillRule("iluk", level=level)))


def ilut(a: CsrMatrix, tau: float, maxfill: int, safeguard: float = DIAG_SAFEGUARD) -> IluFactors:
    """factor.py:723-740."""
    _check_square(a)
    rule = FillRule("ilut", tau=tau, maxfill=maxfill)
    return IluFactors._from_device(d_ilut(a.device(), a.n_rows, tau, maxfill, 0.0, safeguard), str(rule))


def factorize(a: CsrMatrix, rule: FillRule, safeguard: float = DIAG_SAFEGUARD) -> IluFactors:
    """factor.py:743-749."""
    _check_square(a)
    kind = "ilu0" if rule.kind == "ilu0" else str(rule)
    return IluFactors._from_device(d_factorize(a.device(), rule, safeguard), kind)


def _partial_to_host(dp: DevPartial, rule: FillRule) -> PartialIluFactors:
    schur = None
    if dp.schur is not None:
        schur = IluFactors._from_device(dp.schur, "ilu0" if rule.kind == "ilu0" else str(rule))
    return PartialIluFactors(
        interior=IluFactors._from_device(dp.interior, str(rule)),
        w_block=CsrMatrix.from_device(dp.w), z_block=CsrMatrix.from_device(dp.z),
        s_tilde=CsrMatrix.from_device(dp.s_tilde), schur=schur, n_interior=dp.n_interior)


def partial_ilu(a: CsrMatrix, n_interior: int, rule: FillRule, schur_drop_tol: float = 0.0,
                factor_schur: bool = True, safeguard: float = DIAG_SAFEGUARD) -> PartialIluFactors:
    """factor.py:825-883."""
    _check_square(a)
    if not 0 <= n_interior <= a.n_rows:
        raise ValueError("interior size out of range")
    dp = d_partial_ilu(a.device(), n_interior, rule, schur_drop_tol, factor_schur, safeguard)
    return _partial_to_host(dp, rule)


def extract_two_level_blocks(f: IluFactors, n_interior: int) -> TwoLevelBlocks:
    """factor.py:886-907."""
    l_b, u_b, w, z, l_s, u_s = d_carve(f.device(), n_interior)
    return TwoLevelBlocks(
        interior=IluFactors._from_device(DevFactors(l_b, u_b), f.kind),
        w_tilde=CsrMatrix.from_device(w), z_tilde=CsrMatrix.from_device(z),
        schur=IluFactors._from_device(DevFactors(l_s, u_s), f.kind))
