"""Domain-decomposition ILU preconditioners (the reference's `ddilu.precond`,
precond.py:64-75) with the device boundary placed where the reference loops
over domains (precond.py:189-190, 242-244, 255-266, 340-345, 371-378).

Layout in HBM.  A rank owns a contiguous block of subdomains.  Its unknowns
are numbered [interiors of its domains, RCM inside each | exteriors of its
domains] -- the reference's own ordering (precond.py:137-147, 431-435)
restricted to the rank -- followed by a halo tail holding the exterior values
of other ranks that its rows touch.  Because interiors of different domains do
not couple, the block-diagonal matrix of the rank's domains is factorised as
ONE matrix: its ILU factors are exactly the per-domain factors side by side,
and one level-scheduled sweep serves all of the rank's domains at once (more
rows per level, same depth).  The per-domain objects of the reference
(`.factors[d]`, `.partial[d]`, `.blocks[d]`, `.smoother[d]`) are views carved
from those combined factors on demand.
"""

from __future__ import annotations

import weakref

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .dist import Comm, PeerComm, domains_of_rank, get_comm
from .factor import (DevFactors, DevPartial, FillRule, IluFactors, MiluVectors, PartialIluFactors, TwoLevelBlocks,
                     d_carve, d_factor_level0, d_factorize, d_partial_ilu, solve_with_product)
from .krylov import InnerGmres, KrylovConfig, restarted_device
from .ordering import DomainLayout
from .sparse import CsrMatrix, Permutation

__all__ = [
    "BjIluPrecond", "SchurIluPrecond", "RapIluPrecond", "bj_setup", "schur_setup", "rap_setup", "schur_matvec",
    "rap_matvec", "make_preconditioner", "PRECONDITIONER_NAMES",
]

PRECONDITIONER_NAMES = ("bj", "l1bj", "schur", "rap", "rap-milu", "none")


@dataclass
class _DomainOrdering:
    """precond.py:128-134."""

    interior_nodes: np.ndarray
    exterior_nodes: np.ndarray
    nodes: np.ndarray


class LocalSystem:
    """Everything a rank holds of the partitioned matrix (see module docstring)."""

    def __init__(self, a: CsrMatrix, layout: DomainLayout, use_rcm: bool = True, comm: Comm | None = None):
        self.comm = comm if comm is not None else get_comm()
        self.a, self.layout = a, layout
        n, p = layout.n, layout.p
        ad = a.device()
        self.doms = domains_of_rank(p, self.comm)
        d0, d1 = self.doms.start, self.doms.stop
        ist, est, n1g = layout.interior_starts, layout.exterior_starts, layout.n_interior
        g = layout._gorder_d
        ints = g[int(ist[d0]):int(ist[d1])]
        exts = g[n1g + int(est[d0]):n1g + int(est[d1])]
        self.n_int, self.n_ext = ints.numel(), exts.numel()
        self.n_loc = self.n_int + self.n_ext
        self.int_ptr = (ist[d0:d1 + 1] - ist[d0]).astype(np.int64)   # local interior starts per domain
        self.ext_ptr = (est[d0:d1 + 1] - est[d0]).astype(np.int64)
        self.n_ext_global = layout.n_exterior
        # --- RCM of the interior blocks (precond.py:141-144), all local domains in one launch
        if use_rcm and self.n_int > 1:
            cmap = D.index_map(n, ints)
            pat = D.gather_rows(ad, ints, self.n_int, cmap, self.n_int, filt=4, resort=True, with_values=False)
            adj = D.sym_adjacency(pat)
            seg = torch.from_numpy(self.int_ptr.astype(np.int32)).to(D.dev())
            cm = D.cm_order(adj, seg)      # interiors of different domains never couple: ordered concurrently
            ints = D.gather_i32(ints, D.reverse_segments(cm, seg))
        self.nodes = torch.cat([ints, exts]).contiguous()          # global index of each local row
        colmap = D.index_map(n, self.nodes)
        # --- halo plan
        self.n_halo = 0
        self.halo_nodes = None
        self.send_idx = None
        self.send_counts = [0] * self.comm.size
        self.recv_counts = [0] * self.comm.size
        if self.comm.active:
            colmap = self._plan_halo(ad, layout, colmap)
        # --- local rows of A: columns = [local | halo]
        self.a_loc = D.gather_rows(ad, self.nodes, self.n_loc, colmap, self.n_loc + self.n_halo, resort=True)
        self._a_dom = None
        self._colmap = colmap
        self._sendbuf = D.empty_f64(max(1, sum(self.send_counts)))
        self._xbuf = None
        self._tile_parts = {}
        self._ext_tdims = None

    # ------------------------------------------------------------------ tiles
    TILE_TARGET_ROWS = 512
    TILE_DIMS_3D = (8, 8, 8)      # interior box tile (x, y, z nodes); 512 rows, 22 wavefront levels on a 7-point grid

    def _tile_keys(self, r0: int, r1: int, tdims):
        lay = self.layout
        owner = lay._owner_d if lay.p > 1 else None
        return D.box_tile_keys(self.nodes[r0:r1], r1 - r0, lay.grid_hint, tdims, owner)

    def _int_tdims(self):
        nd = len(self.layout.grid_hint)
        if nd == 3:
            return list(self.TILE_DIMS_3D)
        return [32, 16] if nd == 2 else [self.TILE_TARGET_ROWS]

    SLAB = None           # (fx, fy, levels): wavefront-slab tiles for interior factors instead of boxes -- a
                          # measured alternative (fewer levels per tile, but every level then
                          # waits for a neighbour tile's previous level; 450 vs 418 us), off by default

    def tile_part_interior(self):
        """Tile partition of the interior rows for a factor pair: a callable (lev, n_levels) -> partition
        that cuts WAVEFRONT SLABS (footprint box x a range of the factor's own levels: every level of a
        tile holds the whole footprint, so a 512-row tile has 8 levels instead of the 22 of an 8^3 box),
        with the plain box partition as fallback.  3D grids only; otherwise the box partition."""
        box = self.tile_part("int")
        lay = self.layout
        if box is None or len(lay.grid_hint) != 3 or not self.SLAB:
            return box
        owner = lay._owner_d if lay.p > 1 else None
        nodes, n_int, dims, p = self.nodes, self.n_int, lay.grid_hint, max(1, lay.p)
        f0, f1, delta = self.SLAB

        def slab(lev, n_levels):
            keys, rng = D.slab_tile_keys(nodes[:n_int], n_int, dims, (f0, f1), lev, n_levels, delta, owner, p)
            return D.tile_partition(keys, rng)

        slab.fallback = box
        return slab

    def lazy_tile_part_interior(self):
        """tile_part_interior, built on first use (the cluster sweep does not need tiles)."""
        def make():
            return self.tile_part_interior()
        make.lazy = True
        return make

    def _ext_partition(self, max_rows: int, int_keys, int_range: int):
        """Box tiles of the interface rows with at most max_rows rows each (edge 32, 16, ... until it
        fits); with int_keys the interior rows (keys below int_range) are partitioned along."""
        lay = self.layout
        nd, p = len(lay.grid_hint), max(1, lay.p)
        e = 32 if nd == 3 else D.TILE_MAX_ROWS
        while e >= 2:
            keys, nk = self._tile_keys(self.n_int, self.n_loc, [e] * nd)
            if isinstance(int_keys, torch.Tensor):
                keys, rng = torch.cat([int_keys, keys + int_range]), int_range + nk * p
            else:
                rng = nk * p
            part = D.tile_partition(keys, rng)
            if part is not None:
                sizes = part.tile_ptr[1:] - part.tile_ptr[:-1]
                ext_tiles = part.tile_of[self.n_int if isinstance(int_keys, torch.Tensor) else 0:].long().unique()
                if int(sizes[ext_tiles].max().item()) <= max_rows:
                    return part, [e] * nd
            e //= 2
        return None, None

    def tile_part(self, which: str):
        """Tile partition of the local rows for the tiled triangular solves: box tiles of
        the structured grid (`layout.grid_hint`), None for unstructured matrices.
        which: 'int' (interior rows), 'ext' (interface rows), 'all' (both, interior first)."""
        lay = self.layout
        if not D.USE_TILED or lay.grid_hint is None:
            return None
        if which in self._tile_parts:
            return self._tile_parts[which]
        nd = len(lay.grid_hint)
        p = max(1, lay.p)
        part = None
        if which == "int" and self.n_int:
            keys, nk = self._tile_keys(0, self.n_int, self._int_tdims())
            part = D.tile_partition(keys, nk * p)
            if part is not None:     # box tiles of the grid: candidates for the lattice solve
                part.geom = (self.nodes[: self.n_int], tuple(lay.grid_hint), tuple(self._int_tdims()))
        elif which == "ext" and self.n_ext:
            part, self._ext_tdims = self._ext_partition(D.TILE_MAX_ROWS, 0, 0)
        elif which == "all":
            if self.n_ext == 0:
                part = self.tile_part("int")
            elif self.tile_part("int") is not None:
                # interface rows of a full-block factor also depend on interior rows (W): keep their tiles at
                # <= 512 rows so that tile + boundary dependencies fit the shared-memory budget
                ki, nki = self._tile_keys(0, self.n_int, self._int_tdims())
                part, _ = self._ext_partition(self.TILE_TARGET_ROWS, ki, nki * p)
        self._tile_parts[which] = part
        return part

    # ------------------------------------------------------------------ halo
    def _plan_halo(self, ad, layout, colmap):
        n, comm = layout.n, self.comm
        per = layout.p // comm.size
        n1g, est = layout.n_interior, layout.exterior_starts
        flags = D.zeros_i32(n)
        D.call("ddilu_mark_foreign_cols", self.n_loc, self.nodes, ad.rp, ad.ci, colmap, flags)
        gext = layout._gorder_d[n1g:]                      # all exteriors in layout order
        need = flags[gext.long()] > 0
        halo_nodes = gext[need].contiguous()
        self.halo_nodes = halo_nodes
        self.n_halo = halo_nodes.numel()
        pos = torch.nonzero(need).flatten().cpu().numpy()   # positions in the exterior section
        rank_bounds = np.array([est[r * per] for r in range(comm.size)] + [est[-1]])
        self.recv_counts = np.diff(np.searchsorted(pos, rank_bounds)).astype(int).tolist()
        # what each peer needs from me: my exterior columns touched by its rows
        extmap = D.index_map(n, self.nodes[self.n_int:])
        sflags = D.zeros_i32(max(1, comm.size * self.n_ext))
        D.call("ddilu_mark_sends", n, ad.rp, ad.ci, layout._owner_d, per, comm.rank, extmap, self.n_ext, sflags)
        sf = sflags[: comm.size * self.n_ext].view(comm.size, self.n_ext) > 0
        self.send_counts = sf.sum(dim=1).cpu().numpy().astype(int).tolist()
        self.send_idx = torch.nonzero(sf)[:, 1].to(D.I32).contiguous()
        if hasattr(comm, "reserve"):            # peer-memory transport: mailbox room for the largest message (collective)
            comm.reserve(max(max(self.send_counts), max(self.recv_counts), 1))
        return D.index_map(n, halo_nodes, offset=self.n_loc, base=colmap)

    def exchange_halo(self, src_ext: torch.Tensor, halo_out: torch.Tensor, async_op: bool = False):
        """halo_out[:n_halo] <- exterior values of the other ranks; src_ext is
        this rank's exterior section (n_ext entries).  Returns a work handle when
        the exchange was started asynchronously (caller must .wait())."""
        if not self.comm.active:
            return None
        ns = sum(self.send_counts)
        if isinstance(self.comm, PeerComm):      # peer memory: the pack is part of the sending kernel
            return self.comm.all_to_all(halo_out[: self.n_halo], src_ext, self.recv_counts, self.send_counts,
                                        async_op=async_op, idx=self.send_idx)
        D.gather(ns, self.send_idx, src_ext, self._sendbuf)
        return self.comm.all_to_all(halo_out[: self.n_halo], self._sendbuf[:ns], self.recv_counts, self.send_counts,
                                    async_op=async_op)

    # ----------------------------------------------------------------- matvec
    def spmv(self, x: torch.Tensor, out: torch.Tensor, b: torch.Tensor | None = None, mode: int = 0):
        """out[:n_loc] = A_loc [x | halo(x)]; x needs n_loc + n_halo entries.
        Interior rows never touch the halo, so they run while it is in flight."""
        if x.numel() < self.n_loc + self.n_halo:
            if self._xbuf is None:
                self._xbuf = D.empty_f64(self.n_loc + self.n_halo)
            self._xbuf[: self.n_loc].copy_(x[: self.n_loc])
            x = self._xbuf
        if self.comm.active:
            # start the halo exchange, run the interior rows while it is in flight, then the interface rows
            work = self.exchange_halo(x[self.n_int:self.n_loc], x[self.n_loc:], async_op=True)
            D.spmv(self.a_loc, x, out, b, mode, 0, self.n_int)
            if work is not None:
                work.wait()
            D.spmv(self.a_loc, x, out, b, mode, self.n_int, self.n_loc)
        else:
            D.spmv(self.a_loc, x, out, b, mode)
        return out

    @property
    def a_dom(self) -> D.DeviceCsr:
        """Block-diagonal part: entries whose row and column share a subdomain."""
        if self._a_dom is None:
            if self.layout.p == 1:
                self._a_dom = self.a_loc
            else:
                # halo columns belong to other domains, so the same-domain filter drops them too
                self._a_dom = D.gather_rows(self.a.device(), self.nodes, self.n_loc, self._colmap, self.n_loc,
                                            dom=self.layout._owner_d, filt=1, resort=True)
        return self._a_dom

    def coupling(self) -> D.DeviceCsr:
        """E_off: exterior rows x [local exteriors | halo], same-domain entries
        removed (precond.py:287-291)."""
        n = self.layout.n
        exts = self.nodes[self.n_int:]
        cmap = D.index_map(n, exts)
        if self.n_halo:
            cmap = D.index_map(n, self.halo_nodes, offset=self.n_ext, base=cmap)
        return D.gather_rows(self.a.device(), exts, self.n_ext, cmap, self.n_ext + self.n_halo,
                             dom=self.layout._owner_d, filt=2, resort=True)

    # ------------------------------------------------------- host-side helpers
    def local_domain(self, k: int):
        """(interior range, exterior range) of the k-th local domain in local numbering."""
        return ((int(self.int_ptr[k]), int(self.int_ptr[k + 1])),
                (self.n_int + int(self.ext_ptr[k]), self.n_int + int(self.ext_ptr[k + 1])))

    def domain_orderings(self):
        nodes = D.to_host_i64(self.nodes)
        out = []
        for k in range(len(self.doms)):
            (i0, i1), (e0, e1) = self.local_domain(k)
            ints, exts = nodes[i0:i1], nodes[e0:e1]
            out.append(_DomainOrdering(ints, exts, np.concatenate([ints, exts])))
        return out

    def domain_view(self, m: D.DeviceCsr, k: int, rows: str, cols: str) -> CsrMatrix:
        """Sub-block of a combined local matrix for local domain k; rows / cols
        in {'int', 'ext', 'all'} select the sections in the reference's per-domain order."""
        (i0, i1), (e0, e1) = self.local_domain(k)

        def idx(kind, shift):
            parts = []
            if kind in ("int", "all"):
                parts.append(torch.arange(i0, i1, dtype=D.I32, device=D.dev()))
            if kind in ("ext", "all"):
                parts.append(torch.arange(e0 - shift, e1 - shift, dtype=D.I32, device=D.dev()))
            return torch.cat(parts)

        # matrices carved at n_int have exterior indices starting at 0
        rshift = self.n_int if (rows == "ext" and m.n_rows == self.n_ext) else 0
        cshift = self.n_int if (cols == "ext" and m.n_cols in (self.n_ext, self.n_ext + self.n_halo)) else 0
        r, c = idx(rows, rshift), idx(cols, cshift)
        cmap = D.index_map(m.n_cols, c)
        return CsrMatrix.from_device(D.gather_rows(m, r, r.numel(), cmap, c.numel(), resort=False))


# ---------------------------------------------------------------------------


class _DDPrecond:
    """Shared host/device plumbing of the three preconditioner families."""

    def __init__(self, a: CsrMatrix, layout: DomainLayout, use_rcm: bool):
        self.layout = layout
        self.system = LocalSystem(a, layout, use_rcm)
        self._a = a
        self._domains = None
        self._graph = None
        s = self.system
        self._r = D.empty_f64(max(1, s.n_loc))
        self._z = D.empty_f64(max(1, s.n_loc + s.n_halo))

    # host views ----------------------------------------------------------
    @property
    def domains(self):
        if self._domains is None:
            self._domains = self.system.domain_orderings()
        return self._domains

    # operators -----------------------------------------------------------
    def apply_local(self, r: torch.Tensor, z: torch.Tensor):
        raise NotImplementedError

    # applications without host reads ------------------------------------
    def _inner_solvers(self):
        inner = getattr(self, "_inner", None)
        return [inner] if inner is not None else []

    def cycle_failed(self) -> bool:
        """Did a device-side inner solve since the last call meet an early exit of the reference (one host read)?"""
        failed = False
        for inner in self._inner_solvers():
            if not inner.safe and int(inner.flag.item()):
                inner.flag.zero_()
                failed = True
        return failed

    def set_safe(self, on: bool):
        for inner in self._inner_solvers():
            inner.safe = on            # (the graphed application checks it and runs the plain method while set)

    def graphed_apply(self):
        """apply_local replayed from a CUDA graph when the problem is small enough to be launch-bound (one
        rank, no profiling hooks); the plain method otherwise."""
        if self._graph is None:
            self._graph = _GraphedApply(self)
        return self._graph

    def apply(self, r):
        """z = M^-1 r in the ORIGINAL ordering (precond.py:187, 251, 368).  numpy in ->
        numpy out; a CUDA tensor in -> a CUDA tensor out."""
        s = self.system
        on_device = isinstance(r, torch.Tensor)
        rd = r if on_device else D.to_device_f64(np.asarray(r, dtype=np.float64))
        D.gather(s.n_loc, s.nodes, rd, self._r)
        self.apply_local(self._r, self._z)
        if self.cycle_failed():                    # early exit of an inner solve: the reference's own control flow
            self.set_safe(True)
            self.apply_local(self._r, self._z)
            self.set_safe(False)
        z = torch.zeros(self.layout.n, dtype=D.F64, device=D.dev()) if s.comm.active \
            else torch.empty(self.layout.n, dtype=D.F64, device=D.dev())
        D.scatter(s.n_loc, s.nodes, self._z, z)
        s.comm.allreduce_sum_(z)
        return z if on_device else z.cpu().numpy()

    def _device_apply_for(self, fn):
        if getattr(fn, "__name__", "") != "apply":
            return None

        def dev_apply(x, out):
            out[: self.layout.n].copy_(self.apply(x[: self.layout.n]))
        return dev_apply

    # fast solve path -------------------------------------------------------
    def accepts_operator(self, a) -> bool:
        return a is self._a

    def _solve_local(self, b: np.ndarray, x0, cfg: KrylovConfig, flexible: bool):
        """(F)GMRES in the rank-local permuted numbering: no gather/scatter per
        iteration, halo exchange inside the matvec, allreduced dots."""
        s = self.system
        n = self.layout.n
        on_device = isinstance(b, torch.Tensor)
        bd = b if on_device else D.to_device_f64(b)
        b_loc = D.empty_f64(max(1, s.n_loc))
        D.gather(s.n_loc, s.nodes, bd, b_loc)
        x0_loc = None
        if x0 is not None:
            x0_loc = D.empty_f64(max(1, s.n_loc))
            x0d = x0 if isinstance(x0, torch.Tensor) else D.to_device_f64(np.asarray(x0, dtype=np.float64))
            D.gather(s.n_loc, s.nodes, x0d, x0_loc)
        guard = self if self._inner_solvers() else None
        try:
            x_loc, report = restarted_device(s.n_loc, s.spmv, self.graphed_apply(), b_loc, x0_loc, cfg, flexible,
                                             s.comm, pad=s.n_halo, guard=guard)
        finally:
            if guard is not None:
                self.set_safe(False)
        x = torch.zeros(n, dtype=D.F64, device=D.dev()) if s.comm.active else D.empty_f64(n)
        D.scatter(s.n_loc, s.nodes, x_loc, x)
        s.comm.allreduce_sum_(x)
        return (x if on_device else x.cpu().numpy()), report


# Off by default: measured on B200, the stream already runs ahead of the GPU down to 128^3 (the solve is bound by
# kernel latencies, not by launches: 0.174 s either way), and a fresh capture per preconditioner costs 20-50 ms;
# it pays for many solves with ONE preconditioner on small problems (64^3: 0.060 -> 0.052 s per solve).
GRAPH_APPLY = os.environ.get("DDILU_GRAPHS", "0") == "1"
GRAPH_MAX_ROWS = 6_000_000      # above this a step is GPU-bound (98 % busy at 16.8 M rows): replaying buys nothing
GRAPH_WARMUP = 2                # eager applications before the capture (lazy workspaces, kernel attributes)


class _GraphedApply:
    """`apply_local(r, z)` captured once into a CUDA graph on fixed buffers and replayed: an application of a
    two-level preconditioner is 30-60 small launches, which at <= 128^3 rows per GPU cost more host time than
    GPU time.  Needs an application without host reads (device-side inner-solve arithmetic, krylov.DEVICE_COEF)
    and a single rank; anything else, and any capture failure, falls back to the plain method."""

    def __init__(self, owner):
        s = owner.system
        # weak: the preconditioner owns this object (`_graph`); a strong reference back would be a cycle that keeps the
        # preconditioner, its device arrays (GBs) and the pinned owner map alive until the cyclic collector runs --
        # measured as +55 ms on most setups of a setup+solve loop (fresh pinned / device allocations every step)
        self._owner = weakref.ref(owner)
        self.n = s.n_loc
        self.enabled = (GRAPH_APPLY and not s.comm.active and 0 < s.n_loc <= GRAPH_MAX_ROWS
                        and all(not i.safe for i in owner._inner_solvers()))
        self.calls = 0
        self.graph = None
        self.r = self.z = None

    def __call__(self, r, z):
        from . import _lib
        from . import krylov
        owner = self._owner()
        if (not self.enabled or _lib.profile is not None or not krylov.DEVICE_COEF
                or any(i.safe for i in owner._inner_solvers())):
            return owner.apply_local(r, z)
        n = self.n
        if self.graph is None:
            self.calls += 1
            if self.calls <= GRAPH_WARMUP:
                return owner.apply_local(r, z)
            s = owner.system
            self.r = D.empty_f64(n)
            self.z = D.empty_f64(n + s.n_halo)
            self.r.copy_(r[:n])
            try:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    owner.apply_local(self.r, self.z)
                self.graph = g
            except Exception:
                self.enabled = False
                try:
                    torch.cuda.synchronize()
                except Exception:
                    pass
                return owner.apply_local(r, z)
        else:
            self.r.copy_(r[:n])
        self.graph.replay()
        z[:n].copy_(self.z[:n])
        return z


class BjIluPrecond(_DDPrecond):
    """precond.py:177-191: one ILU solve per domain (all local domains in one sweep)."""

    def __init__(self, a, layout, rule: FillRule, l1: bool, use_rcm: bool = True):
        super().__init__(a, layout, use_rcm)
        self.rule, self.l1 = rule, l1
        mat = self.system.a_dom
        if l1:
            # precond.py:207-212: add each row's off-domain absolute sum to the diagonal before factorising
            s = self.system
            ad = a.device()
            shifts = D.empty_f64(max(1, s.n_loc))
            D.call("ddilu_l1_row_shifts", s.n_loc, s.nodes, ad.rp, ad.ci, ad.val, layout._owner_d, shifts)
            vals = mat.val.clone()
            missing = D.zeros_i32(1)
            D.call("ddilu_add_to_diagonal", s.n_loc, mat.rp, mat.ci, vals, shifts, missing)
            if int(missing.item()):
                raise NotImplementedError("l1bj on a matrix with structurally missing diagonal entries")
            mat = D.DeviceCsr(mat.n_rows, mat.n_cols, mat.rp, mat.ci, vals, mat.nnz)
        self._f = d_factorize(mat, rule, sections=(self.system.int_ptr, self.system.ext_ptr)).prepare(
            part=self.system.tile_part("all"))
        self._factors = None

    @property
    def factors(self):
        if self._factors is None:
            kind = "ilu0" if self.rule.kind == "ilu0" else str(self.rule)
            s = self.system
            self._factors = [IluFactors(s.domain_view(self._f.lower, k, "all", "all"),
                                        s.domain_view(self._f.upper, k, "all", "all"), kind)
                             for k in range(len(s.doms))]
        return self._factors

    def apply_local(self, r, z):
        self._f.solve(r, z)


COMPACT_Z = True   # schur apply: update only the rows of Z that have entries (the full pass streamed 20 n bytes)


class SchurIluPrecond(_DDPrecond):
    """precond.py:221-267."""

    def __init__(self, a, layout, rule: FillRule, inner_iters: int, schur_drop_tol: float = 0.0,
                 use_rcm: bool = True):
        super().__init__(a, layout, use_rcm)
        s = self.system
        self.rule, self.inner_iters = rule, inner_iters
        self._p = d_partial_ilu(s.a_dom, s.n_int, rule, schur_drop_tol=schur_drop_tol, factor_schur=True,
                                blocks=(s.int_ptr, s.ext_ptr))
        self._p.interior.prepare(part=s.lazy_tile_part_interior(), cluster_seg=s.int_ptr)
        self._p.schur.prepare(seg_ptr=s.ext_ptr, part=s.tile_part("ext"))   # interface factors: one block per subdomain
        self._coupling = s.coupling()
        ne, nh = s.n_ext, s.n_halo
        self._inner = InnerGmres(ne, inner_iters, s.comm, pad=nh, n_global=s.n_ext_global)
        self._fp = D.empty_f64(max(1, s.n_int))
        self._t1 = D.empty_f64(max(1, s.n_int))
        self._g = D.empty_f64(max(1, ne))
        self._c = D.empty_f64(max(1, ne))
        self._sv = D.empty_f64(max(1, ne))
        self._rhs = D.empty_f64(max(1, ne))
        self._y = D.empty_f64(max(1, ne + nh))
        self._ybuf = D.empty_f64(max(1, ne + nh))
        self._partial = None
        self._coupling_host = None
        self._zc = D.compact_rows(self._p.z) if COMPACT_Z else None   # Z has entries next to the interface only

    # host views
    @property
    def partial(self):
        if self._partial is None:
            s, p = self.system, self._p
            kind_s = "ilu0" if self.rule.kind == "ilu0" else str(self.rule)
            out = []
            for k in range(len(s.doms)):
                (i0, i1), (e0, e1) = s.local_domain(k)
                out.append(PartialIluFactors(
                    interior=IluFactors(s.domain_view(p.interior.lower, k, "int", "int"),
                                        s.domain_view(p.interior.upper, k, "int", "int"), str(self.rule)),
                    w_block=s.domain_view(p.w, k, "ext", "int"),
                    z_block=s.domain_view(p.z, k, "int", "ext"),
                    s_tilde=s.domain_view(p.s_tilde, k, "ext", "ext"),
                    schur=IluFactors(s.domain_view(p.schur.lower, k, "ext", "ext"),
                                     s.domain_view(p.schur.upper, k, "ext", "ext"), kind_s),
                    n_interior=i1 - i0))
            self._partial = out
        return self._partial

    @property
    def coupling(self) -> CsrMatrix:
        if self._coupling_host is None:
            self._coupling_host = CsrMatrix.from_device(self._coupling)
        return self._coupling_host

    # device operators
    def _schur_solve(self, t, out):
        self._p.schur.solve(t, out)

    def _reduced_matvec(self, y, out):
        """out = y + S~^-1 (E_off y)  (precond.py:247-249); y carries the halo tail."""
        s = self.system
        if y.numel() < s.n_ext + s.n_halo:
            self._ybuf[: s.n_ext].copy_(y[: s.n_ext])
            y = self._ybuf
        s.exchange_halo(y[: s.n_ext], y[s.n_ext:])
        if self._p.schur._sw is not None:
            # E_off y feeds the sweep's right-hand side, `y +` rides on its result stores: two launches
            solve_with_product(self._p.schur, self._coupling, y, None, 0, out, add=y)
            return
        D.spmv(self._coupling, y, self._c)
        self._schur_solve(self._c, self._sv)
        D.ewise(s.n_ext, y, self._sv, 0, out)

    def reduced_matvec(self, y) -> np.ndarray:
        s = self.system
        yd = D.empty_f64(max(1, s.n_ext + s.n_halo))
        yd[: s.n_ext].copy_(torch.from_numpy(np.asarray(y, dtype=np.float64))[self._ext_slice()])
        out = D.empty_f64(max(1, s.n_ext))
        self._reduced_matvec(yd, out)
        return self._ext_global(out)

    def _ext_slice(self):
        est = self.layout.exterior_starts
        return slice(int(est[self.system.doms.start]), int(est[self.system.doms.stop]))

    def _ext_global(self, loc):
        full = torch.zeros(self.layout.n_exterior, dtype=D.F64, device=D.dev())
        full[self._ext_slice()] = loc[: self.system.n_ext]
        self.system.comm.allreduce_sum_(full)
        return full.cpu().numpy()

    def apply_local(self, r, z):
        s, p = self.system, self._p
        ni, ne = s.n_int, s.n_ext
        p.interior.lower_solve(r[:ni], self._fp)                      # fp = L_B^-1 r_int
        if p.schur._sw is not None:
            solve_with_product(p.schur, p.w, self._fp, r[ni:], 1, self._rhs)   # S~^-1 (r_ext - W fp)
        else:
            D.spmv(p.w, self._fp, self._g, b=r[ni:], mode=1)          # ghat = r_ext - W fp
            self._schur_solve(self._g, self._rhs)                     # S~^-1 ghat
        self._inner.solve(self._reduced_matvec, self._rhs, self._y, n_global=s.n_ext_global)
        if self._zc is not None:
            D.sub_compact(self._zc, self._y, self._fp)                # fp - Z y on the rows that have entries, in place
            p.interior.upper_solve(self._fp, z[:ni])
        else:
            D.spmv(p.z, self._y, self._t1, b=self._fp, mode=1)        # fp - Z y
            p.interior.upper_solve(self._t1, z[:ni])
        if ne:
            z[ni:ni + ne].copy_(self._y[:ne])


class RapIluPrecond(_DDPrecond):
    """precond.py:304-385: block-Jacobi smoothing + interface coarse correction."""

    def __init__(self, a, layout, modified: bool, vecs: MiluVectors | None, inner_iters: int, use_rcm: bool = True):
        super().__init__(a, layout, use_rcm)
        s = self.system
        self.inner_iters, self.modified = inner_iters, modified
        plain = d_factor_level0(s.a_dom, s.n_loc).prepare(part=s.tile_part("all"))
        self._smoother = plain
        if modified:
            if vecs is None:
                target = torch.ones(max(1, s.n_loc), dtype=D.F64, device=D.dev())
                wvec = torch.zeros(max(1, s.n_loc), dtype=D.F64, device=D.dev())
            else:
                target, wvec = self._local_vecs(vecs)
            coarse = d_factor_level0(s.a_dom, s.n_loc, True, target, wvec)
        else:
            coarse = plain
        l_b, u_b, w, z, l_s, u_s = d_carve(coarse, s.n_int)
        self._interior = DevFactors(l_b, u_b).prepare(part=s.lazy_tile_part_interior(), cluster_seg=s.int_ptr)
        self._w, self._zt = w, z
        self._ztc = D.compact_rows(z) if COMPACT_Z else None
        self._schur = DevFactors(l_s, u_s).prepare(seg_ptr=s.ext_ptr, part=s.tile_part("ext"))
        self._coarse_kind = coarse
        ni, ne, nh = s.n_int, s.n_ext, s.n_halo
        self._inner = InnerGmres(ne, inner_iters, s.comm, n_global=s.n_ext_global)
        self._xhat = D.empty_f64(max(1, s.n_loc + nh))
        self._pv = D.empty_f64(max(1, s.n_loc + nh))
        self._res = D.empty_f64(max(1, s.n_loc))
        self._av = D.empty_f64(max(1, s.n_loc))
        self._ti = D.empty_f64(max(1, ni))
        self._ti2 = D.empty_f64(max(1, ni))
        self._rr = D.empty_f64(max(1, ne))
        self._v = D.empty_f64(max(1, ne))
        self._blocks = self._smoother_host = self._a_perm = self._perm = None

    def _local_vecs(self, vecs: MiluVectors):
        """precond.py:415-426: user vectors are given in the layout's ordering."""
        s, lay = self.system, self.layout
        gpos = np.empty(lay.n, dtype=np.int64)
        gpos[lay._gorder()] = np.arange(lay.n)
        nodes = D.to_host_i64(s.nodes)
        pos = gpos[nodes]                                  # position of each local row in the layout order
        yfull = np.concatenate([np.asarray(vecs.y, dtype=np.float64), np.asarray(vecs.z, dtype=np.float64)])
        wfull = np.concatenate([np.asarray(vecs.w, dtype=np.float64), np.zeros(lay.n_exterior)])
        return D.to_device_f64(yfull[pos]), D.to_device_f64(wfull[pos])

    # host views
    @property
    def smoother(self):
        if self._smoother_host is None:
            s = self.system
            self._smoother_host = [IluFactors(s.domain_view(self._smoother.lower, k, "all", "all"),
                                              s.domain_view(self._smoother.upper, k, "all", "all"), "ilu0")
                                   for k in range(len(s.doms))]
        return self._smoother_host

    @property
    def blocks(self):
        if self._blocks is None:
            s = self.system
            kind = "milu0" if self.modified else "ilu0"
            self._blocks = [TwoLevelBlocks(
                interior=IluFactors(s.domain_view(self._interior.lower, k, "int", "int"),
                                    s.domain_view(self._interior.upper, k, "int", "int"), kind),
                w_tilde=s.domain_view(self._w, k, "ext", "int"),
                z_tilde=s.domain_view(self._zt, k, "int", "ext"),
                schur=IluFactors(s.domain_view(self._schur.lower, k, "ext", "ext"),
                                 s.domain_view(self._schur.upper, k, "ext", "ext"), kind))
                for k in range(len(s.doms))]
        return self._blocks

    @property
    def a_perm(self) -> CsrMatrix:
        if self._a_perm is None:
            self._a_perm = CsrMatrix.from_device(self.system.a_loc)
        return self._a_perm

    @property
    def perm(self) -> Permutation:
        if self._perm is None:
            self._perm = Permutation.from_order(D.to_host_i64(self.system.nodes))
        return self._perm

    # device operators (all in the local [interior | exterior] numbering)
    def _interpolate(self, v, out):
        """out = [-U_B^-1 (Z v); v]  (precond.py:337-346)."""
        s = self.system
        ni, ne = s.n_int, s.n_ext
        if self._ztc is not None:
            # Z has entries next to the interface only; U_B^-1 (-(Z v)) = -(U_B^-1 (Z v)) bit for bit
            D.spmv_compact(self._ztc, v, self._ti, ni, negate=True)
            self._interior.upper_solve(self._ti, out)
        else:
            D.spmv(self._zt, v, self._ti)
            self._interior.upper_solve(self._ti, self._ti2)
            D.ewise(ni, self._ti2, None, 2, out)
        if ne:
            out[ni:ni + ne].copy_(v[:ne])

    def _restrict(self, t, out):
        """out = t_ext - W (L_B^-1 t_int)  (precond.py:348-355)."""
        ni = self.system.n_int
        self._interior.lower_solve(t[:ni], self._ti)
        D.spmv(self._w, self._ti, out, b=t[ni:], mode=1)

    def _coarse_matvec(self, v, out):
        """R (A (P v))  (precond.py:357-359)."""
        self._interpolate(v, self._pv)
        self.system.spmv(self._pv, self._av)
        self._restrict(self._av, out)

    def _coarse_precond(self, t, out):
        self._schur.solve(t, out)

    def apply_local(self, r, z):
        s = self.system
        n, ne = s.n_loc, s.n_ext
        self._smoother.solve(r, self._xhat)                           # xhat = (L_A U_A)^-1 b
        s.spmv(self._xhat, self._res, b=r, mode=1)                    # res = b - A xhat
        self._restrict(self._res, self._rr)
        self._inner.solve(self._coarse_matvec, self._rr, self._v, apply_m=self._coarse_precond,
                          n_global=s.n_ext_global)
        if s.n_ext_global:
            self._interpolate(self._v, self._pv)
            D.ewise(n, self._xhat, self._pv, 0, z)
        else:
            z[:n].copy_(self._xhat[:n])

    # host-facing pieces of the reference API
    def _ext_slice(self):
        est = self.layout.exterior_starts
        return slice(int(est[self.system.doms.start]), int(est[self.system.doms.stop]))

    def _ext_in(self, v):
        vd = D.empty_f64(max(1, self.system.n_ext))
        vd[: self.system.n_ext].copy_(torch.from_numpy(np.asarray(v, dtype=np.float64))[self._ext_slice()])
        return vd

    def _ext_out(self, loc):
        full = torch.zeros(self.layout.n_exterior, dtype=D.F64, device=D.dev())
        full[self._ext_slice()] = loc[: self.system.n_ext]
        self.system.comm.allreduce_sum_(full)
        return full.cpu().numpy()

    def coarse_matvec(self, v) -> np.ndarray:
        out = D.empty_f64(max(1, self.system.n_ext))
        self._coarse_matvec(self._ext_in(v), out)
        return self._ext_out(out)

    def interpolate(self, v) -> np.ndarray:
        """Result in the reference's permuted ordering [all interiors | all exteriors] (single rank)."""
        if self.system.comm.active:
            raise NotImplementedError("interpolate() as a host call is single-rank only")
        out = D.empty_f64(max(1, self.system.n_loc))
        self._interpolate(self._ext_in(v), out)
        return out[: self.system.n_loc].cpu().numpy()

    def restrict(self, t) -> np.ndarray:
        if self.system.comm.active:
            raise NotImplementedError("restrict() as a host call is single-rank only")
        out = D.empty_f64(max(1, self.system.n_ext))
        self._restrict(D.to_device_f64(np.asarray(t, dtype=np.float64)), out)
        return out[: self.system.n_ext].cpu().numpy()


# ---------------------------------------------------------------------------
# setup entry points (same names / arguments as the reference)


def bj_setup(a: CsrMatrix, layout: DomainLayout, rule: FillRule = FillRule("ilu0"), l1: bool = False,
             use_rcm: bool = True) -> BjIluPrecond:
    """precond.py:194-214."""
    return BjIluPrecond(a, layout, rule, l1, use_rcm)


def schur_setup(a: CsrMatrix, layout: DomainLayout, rule: FillRule = FillRule("ilu0"), inner_iters: int = 3,
                schur_drop_tol: float = 0.0, use_rcm: bool = True) -> SchurIluPrecond:
    """precond.py:270-292."""
    return SchurIluPrecond(a, layout, rule, inner_iters, schur_drop_tol, use_rcm)


def rap_setup(a: CsrMatrix, layout: DomainLayout, modified: bool = True, vecs: MiluVectors | None = None,
              inner_iters: int = 3, use_rcm: bool = True) -> RapIluPrecond:
    """precond.py:388-438."""
    return RapIluPrecond(a, layout, modified, vecs, inner_iters, use_rcm)


def schur_matvec(m: SchurIluPrecond, y) -> np.ndarray:
    """precond.py:295-297."""
    return m.reduced_matvec(y)


def rap_matvec(m: RapIluPrecond, v) -> np.ndarray:
    """precond.py:441-443."""
    return m.coarse_matvec(v)


def make_preconditioner(name: str, a: CsrMatrix, layout: DomainLayout, rule: FillRule = FillRule("ilu0"),
                        inner_iters: int = 3):
    """precond.py:450-474."""
    if name == "none":
        return None
    if name == "bj":
        return bj_setup(a, layout, rule)
    if name == "l1bj":
        return bj_setup(a, layout, rule, l1=True)
    if name == "schur":
        return schur_setup(a, layout, rule, inner_iters=inner_iters)
    if name == "rap":
        return rap_setup(a, layout, modified=False, inner_iters=inner_iters)
    if name == "rap-milu":
        return rap_setup(a, layout, modified=True, inner_iters=inner_iters)
    raise ValueError(f"unknown preconditioner {name!r}")
