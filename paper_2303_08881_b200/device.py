"""Device-side building blocks: CSR matrices in HBM and thin wrappers that
launch the library's kernels on them.  torch is used for allocation, streams
and host<->device copies only.

HBM layout: row_ptr int32[n+1], col_idx int32[nnz] (strictly increasing per
row), values float64[nnz]; vectors float64.  int32 halves the index traffic of
the reference's int64 arrays (sparse.py:95-96); nnz < 2^31 is enforced here.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, query

I32 = torch.int32
F64 = torch.float64
INT_MAX = 2**31 - 1


def dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def empty_i32(n):
    return torch.empty(int(n), dtype=I32, device=dev())


def zeros_i32(n):
    return torch.zeros(int(n), dtype=I32, device=dev())


def empty_f64(n):
    return torch.empty(int(n), dtype=F64, device=dev())


def zeros_f64(n):
    return torch.zeros(int(n), dtype=F64, device=dev())


def to_device_i32(a) -> torch.Tensor:
    """Host int array (any int dtype) -> device int32 (values must fit)."""
    a = np.ascontiguousarray(a)
    if a.size and (int(a.max()) > INT_MAX or int(a.min()) < -INT_MAX - 1):
        raise ValueError("index does not fit the device int32 layout")
    if a.dtype == np.int64 and a.size > (1 << 16):
        # narrow on the device: one pinned int64 copy, no host pass
        wide = torch.from_numpy(a).to(dev(), non_blocking=False)
        out = empty_i32(a.size)
        call("ddilu_narrow_i64", a.size, wide, out)
        return out
    return torch.from_numpy(a.astype(np.int32, copy=False)).to(dev())


def to_device_f64(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev())


def to_host_i64(t: torch.Tensor) -> np.ndarray:
    """Device int32 -> host int64 (the reference's index dtype).  Large arrays are widened on the device and
    land in pinned memory (one 25 GB/s copy instead of a pageable copy plus a host-side astype: 5 ms instead
    of 55 ms for the 16.8 M-entry owner map); the returned array owns that pinned block."""
    n = t.numel()
    if n < (1 << 20) or not t.is_cuda:
        return t.cpu().numpy().astype(np.int64)
    wide = torch.empty(n, dtype=torch.int64, device=t.device)
    call("ddilu_widen_i32", n, t.contiguous(), wide)
    host = torch.empty(n, dtype=torch.int64, pin_memory=True)
    host.copy_(wide)
    return host.numpy()


def exclusive_scan_(buf: torch.Tensor, n: int) -> torch.Tensor:
    """In-place exclusive scan of buf[0:n]; buf has n+1 entries, buf[n] = total."""
    tmp = empty_i32(query("ddilu_scan_tmp_elems", n))
    call("ddilu_exclusive_scan_i32", buf, buf, n, tmp)
    return buf


def sort_pairs_(keys: torch.Tensor, vals: torch.Tensor, bits: int):
    n = keys.numel()
    if n <= 1:
        return
    ka, va = torch.empty_like(keys), torch.empty_like(vals)
    tmp = empty_i32(query("ddilu_sort_tmp_elems", n))
    call("ddilu_sort_pairs_i32", keys, vals, ka, va, n, int(bits), tmp)


@dataclass
class DeviceCsr:
    n_rows: int
    n_cols: int
    rp: torch.Tensor
    ci: torch.Tensor
    val: torch.Tensor | None
    _nnz: int = -1

    @property
    def nnz(self) -> int:
        if self._nnz < 0:
            self._nnz = int(self.rp[-1].item()) if self.n_rows else 0
        return self._nnz

    @staticmethod
    def from_host(n_rows, n_cols, row_ptr, col_idx, values) -> "DeviceCsr":
        nnz = int(row_ptr[-1]) if len(row_ptr) else 0
        if nnz > INT_MAX or max(n_rows, n_cols) > INT_MAX:
            raise ValueError("matrix too large for the int32 device layout")
        return DeviceCsr(int(n_rows), int(n_cols), to_device_i32(row_ptr), to_device_i32(col_idx),
                         to_device_f64(values), nnz)

    def to_host(self):
        vals = self.val.cpu().numpy() if self.val is not None else np.zeros(self.nnz)
        return to_host_i64(self.rp), to_host_i64(self.ci), vals


# ---------------------------------------------------------------------------
# kernels


def spmv(a: DeviceCsr, x: torch.Tensor, out: torch.Tensor, b: torch.Tensor | None = None, mode: int = 0,
         r0: int = 0, r1: int | None = None):
    """out[r0:r1] = A x | b - A x | b + A x  (rows r0..r1)."""
    r1 = a.n_rows if r1 is None else r1
    avg = a.nnz / a.n_rows if a.n_rows else 0.0     # row-length hint: rows per CTA / stage size
    call("ddilu_spmv_csr_f64_tuned", int(r0), int(r1), a.rp, a.ci, a.val, x, b, out, int(mode), float(avg))
    return out


@dataclass
class CompactRows:
    """The non-empty rows of a very sparse coupling block (Z: interior x exterior has entries in the rows next to
    the interface only): `vec[rows] -= A[rows, :] x` touches those rows instead of streaming all of them."""

    rows: torch.Tensor      # int32 indices of the non-empty rows
    csr: DeviceCsr          # the same entries (col_idx / values shared) with a compacted row_ptr
    t_in: torch.Tensor
    t_out: torch.Tensor
    zeros: torch.Tensor = None


def compact_rows(a: DeviceCsr, max_fraction: float = 0.25) -> "CompactRows | None":
    if a.n_rows == 0 or a.nnz == 0:
        return None
    cnt = a.rp[1:] - a.rp[:-1]
    rows = torch.nonzero(cnt > 0).reshape(-1)
    k = int(rows.numel())
    if k == 0 or k > max_fraction * a.n_rows:
        return None
    rp = zeros_i32(k + 1)
    rp[1:] = torch.cumsum(cnt[rows], 0).to(I32)      # empty rows hold no entries: col_idx / values stay as they are
    return CompactRows(rows.to(I32).contiguous(), DeviceCsr(k, a.n_cols, rp, a.ci, a.val, a.nnz), empty_f64(k), empty_f64(k))


def sub_compact(c: CompactRows, x: torch.Tensor, vec: torch.Tensor):
    """vec[rows] = vec[rows] - A[rows, :] x, the same row arithmetic as `spmv(..., b=vec, mode=1)`; the other rows of
    `b - A x` equal b bit for bit (b - 0.0)."""
    k = c.csr.n_rows
    gather(k, c.rows, vec, c.t_in)
    spmv(c.csr, x, c.t_out, b=c.t_in, mode=1)
    scatter(k, c.rows, c.t_out, vec)


def spmv_compact(c: CompactRows, x: torch.Tensor, out: torch.Tensor, n_rows: int, negate: bool = False):
    """out[:n_rows] = A x for a matrix whose non-empty rows are `c.rows` (the empty rows give +0.0, as the row loop does)."""
    k = c.csr.n_rows
    out[:n_rows].zero_()
    if negate:   # 0 - A x: negation commutes with every later operation bit for bit (only the sign of exact zeros differs)
        if c.zeros is None:
            c.zeros = torch.zeros(k, dtype=F64, device=dev())
        spmv(c.csr, x, c.t_out, b=c.zeros, mode=1)
    else:
        spmv(c.csr, x, c.t_out)
    scatter(k, c.rows, c.t_out, out)


@dataclass
class Schedule:
    """Level schedule of a triangular factor (SURVEY.md 8c definition)."""

    n: int
    n_levels: int
    n_slots: int
    order: torch.Tensor        # padded schedule, -1 = empty slot
    level_ptr: torch.Tensor    # n_levels + 1
    level_rows: torch.Tensor   # rows sorted by (level, index); index descending for U
    lev: torch.Tensor
    slot_ptr: torch.Tensor = None   # n_levels + 1 padded level starts
    sell: dict = None          # unit_diag -> Sell (schedule-ordered sliced-ELL copy of the factor)
    blocks: "BlockLocal" = None  # set for small, deep, block-diagonal factors


@dataclass
class BlockLocal:
    n_blocks: int
    start: torch.Tensor        # [n_blocks * n_levels] first position of block d / level l in level_rows
    cnt: torch.Tensor
    sstart: torch.Tensor       # the same as schedule slots (levels padded to 32)


@dataclass
class Sell:
    goff: torch.Tensor | None  # n_groups + 1 offsets into scol / sval; None = uniform width
    width: int                 # entries per lane in the uniform layout
    scol: torch.Tensor
    sval: torch.Tensor
    sdiag: torch.Tensor | None
    bad_row: int               # first row with a zero / missing diagonal, or INT_MAX
    gwait: torch.Tensor | None = None   # per group: the dependency that is latest in the schedule
    gfar1: torch.Tensor | None = None   # the same indicator one level further back (gwait of gwait's group)
    gfar2: torch.Tensor | None = None   # two levels further back


def levels(t: DeviceCsr, upper: bool):
    """(lev int32[n], n_levels): lev[i] = 1 + max lev[j] over the dependencies of row i."""
    n = t.n_rows
    lev = empty_i32(max(n, 1))
    mx = zeros_i32(1)
    call("ddilu_levels", n, t.rp, t.ci, int(upper), lev, mx)
    return lev, (int(mx.item()) + 1 if n else 0)


def build_schedule(t: DeviceCsr, upper: bool, lev=None, n_levels: int = 0) -> Schedule:
    n = t.n_rows
    if lev is None:
        lev, n_levels = levels(t, upper)
    if n == 0:
        z = zeros_i32(1)
        return Schedule(0, 0, 0, z, z, z, z)
    keys, rows = empty_i32(n), empty_i32(n)
    ka, ra = empty_i32(n), empty_i32(n)
    tmp = empty_i32(query("ddilu_sort_tmp_elems", n))
    level_ptr, slot_ptr = empty_i32(n_levels + 1), empty_i32(n_levels + 1)
    order = empty_i32(n + 32 * n_levels)
    call("ddilu_schedule_build", n, lev, n_levels, int(upper), keys, rows, ka, ra, tmp, level_ptr, slot_ptr, order)
    n_slots = int(slot_ptr[-1].item())
    return Schedule(n, n_levels, n_slots, order[:n_slots], level_ptr, rows, lev, slot_ptr)


class TriSolveError(ZeroDivisionError):
    pass


# ---------------------------------------------------------------------------
# tiled triangular solve (csrc/tiled.cu)

USE_TILED = True
TILE_KERNEL = "rot"       # "rot": CTA-per-tile kernel with rotating compute warps (production; the others need an experiments build);
                          # "warp": warp-per-tile kernels (independent warps; lean records when rows have <= 3
                          # dependencies) -- measured alternative, same throughput per SM
TILE_MAX_ROWS = 1024
TILE_SMEM_LIMIT = 112 * 1024      # per CTA: at least two CTAs per SM
TILE_RELAX_BATCH = 8
TILE_RELAX_MAX_BATCHES = 64


@dataclass
class TilePartition:
    """Rows of a factor clustered into tiles (shared by the L and U solve of a factor pair)."""

    n: int
    n_tiles: int
    tile_of: torch.Tensor     # int32[n]
    tpos: torch.Tensor        # int32[n] position of the row in trows
    tile_ptr: torch.Tensor    # int32[n_tiles + 1]
    trows: torch.Tensor       # int32[n] rows grouped by tile, ascending inside a tile
    max_rows: int
    geom: tuple = None        # (grid node of every row, grid dims, tile dims) when the tiles are grid boxes


@dataclass
class TileSched:
    """Static blocks of a tiled factor in tile-schedule order."""

    n: int
    n_tiles: int
    n_tile_levels: int
    blk_off16: torch.Tensor   # int32[n_tiles + 1], 16-byte units into blob
    blob: torch.Tensor        # uint8
    stat_max: int
    tmax: int
    emax: int
    kmax: int
    has_diag: bool
    bad_row: int
    kind: str = "rot"        # which solve kernel the item lists were cut for


def box_tile_keys(nodes: torch.Tensor | None, n: int, dims, tdims, owner: torch.Tensor | None):
    """(keys int32[n], keys per owner): key = box of the grid node (+ owner * boxes)."""
    nd = len(dims)
    arr = ctypes.c_int * nd
    d, t = arr(*[int(v) for v in dims]), arr(*[int(v) for v in tdims])
    nk = ctypes.c_longlong(0)
    keys = empty_i32(max(1, n))
    call("ddilu_tile_box_keys", int(n), nodes, nd, ctypes.addressof(d), ctypes.addressof(t), owner, keys,
         ctypes.addressof(nk))
    return keys[:n], int(nk.value)


def slab_tile_keys(nodes: torch.Tensor | None, n: int, dims, tdims2, lev: torch.Tensor, n_levels: int, delta: int,
                   owner: torch.Tensor | None, n_owners: int):
    """(keys int32[n], key range): key = (owner, footprint box in the first two grid coordinates,
    lev // delta) -- wavefront-slab tiles of a factor whose levels are `lev`."""
    nd = len(dims)
    arr = ctypes.c_int * nd
    arr2 = ctypes.c_int * 2
    d, t = arr(*[int(v) for v in dims]), arr2(int(tdims2[0]), int(tdims2[1]))
    nk = ctypes.c_longlong(0)
    keys = empty_i32(max(1, n))
    call("ddilu_tile_slab_keys", int(n), nodes, nd, ctypes.addressof(d), ctypes.addressof(t), lev, int(n_levels),
         int(delta), owner, int(n_owners), keys, ctypes.addressof(nk))
    return keys[:n], int(nk.value)


def tile_partition(keys: torch.Tensor, key_range: int, max_tile_rows: int | None = None) -> TilePartition | None:
    """Compact the keys into tile ids; None if a tile would exceed max_tile_rows (default TILE_MAX_ROWS)."""
    n = keys.numel()
    if n == 0:
        return None
    keys = keys.clone()
    rows = torch.arange(n, dtype=I32, device=dev())
    sort_pairs_(keys, rows, max(1, int(key_range - 1).bit_length()))
    flags = empty_i32(n + 1)
    call("ddilu_tile_heads", n, keys, flags)
    exclusive_scan_(flags, n)
    n_tiles = int(flags[-1].item())
    tile_of, tpos, tile_ptr = empty_i32(n), empty_i32(n), empty_i32(n_tiles + 1)
    call("ddilu_tile_assign", n, keys, flags, rows, tile_of, tpos, tile_ptr)
    max_rows = int((tile_ptr[1:] - tile_ptr[:-1]).max().item())
    if max_rows > (TILE_MAX_ROWS if max_tile_rows is None else max_tile_rows):
        return None
    return TilePartition(n, n_tiles, tile_of, tpos, tile_ptr, rows, max_rows)


def tile_schedule(t: DeviceCsr, part: TilePartition, upper: bool):
    """(tsched, n_tile_levels): the tiles in a topological order of the tile graph (cross-tile dependencies of
    the factor, relaxed to tile levels on the device); None when the graph is cyclic or too deep."""
    n = t.n_rows
    cnt = zeros_i32(n + 1)
    call("ddilu_tile_edges_count", n, t.rp, t.ci, int(upper), part.tile_of, cnt)
    exclusive_scan_(cnt, n)
    n_edges = int(cnt[-1].item())
    edges = empty_i32(max(2, 2 * n_edges))
    call("ddilu_tile_edges_fill", n, t.rp, t.ci, int(upper), part.tile_of, cnt, edges)
    nt = part.n_tiles
    tlev = zeros_i32(nt)
    flags = zeros_i32(2)
    converged = n_edges == 0
    for _ in range(TILE_RELAX_MAX_BATCHES):
        if converged:
            break
        call("ddilu_tile_relax", n_edges, edges, nt, tlev, flags, TILE_RELAX_BATCH)
        f = flags.cpu().numpy()
        if f[1]:
            return None
        converged = not f[0]
    if not converged:
        return None
    del edges
    n_tile_levels = int(tlev.max().item()) + 1
    tsched = torch.arange(nt, dtype=I32, device=dev())
    sort_pairs_(tlev, tsched, max(1, int(n_tile_levels - 1).bit_length()))
    return tsched, n_tile_levels


@dataclass
class LatticeSched:
    """Layout of the lattice solve (csrc/lattice.cu): per tile a 32-entry table and a block of boundary columns
    + row records in (step, slot, lane) order; tiles in schedule order."""

    n: int
    n_tiles: int
    n_tile_levels: int
    tab: torch.Tensor         # int32[n_tiles * 32 * 4]
    blob: torch.Tensor        # uint8
    flags: torch.Tensor       # int32[n_tiles] per-tile completion flags of the running solve
    n_slots: int              # 1: <= 32 lines per tile, 2: <= 64
    has_diag: bool
    bad_row: int
    blkmax: int = 0           # largest tile block (bytes), row count, boundary-value count: size the shared memory
    tmax: int = 0
    xemax: int = 0
    kind: str = "lattice"


USE_LATTICE = os.environ.get("DDILU_LATTICE", "0") == "1"   # measured 2-4x slower than the rotating kernel


def build_lattice(t: DeviceCsr, part: TilePartition, upper: bool, unit_diag: bool, sched=None) -> "LatticeSched | None":
    """Lattice layout of a triangular factor whose tiles are boxes of a structured grid (part.geom = (grid node
    of every row, grid dims, tile dims)); None when some tile is not a lattice with one-way axes, a row has more
    than 3 dependencies, or the tile graph is cyclic -- the caller then uses the general tiled solve."""
    geom = getattr(part, "geom", None)
    n = t.n_rows
    if not USE_LATTICE or not _lib.has_experiments() or geom is None or n == 0 or part.n != n:
        return None
    nodes, dims, tdims = geom
    d3 = [int(v) for v in dims] + [1] * (3 - len(dims))
    t3 = [int(v) for v in tdims] + [1] * (3 - len(tdims))
    if t3[1] * t3[2] > 64 or t3[0] + t3[1] + t3[2] - 2 > 32 or t3[0] * t3[1] * t3[2] > 1024:
        return None
    sched = sched if sched is not None else tile_schedule(t, part, upper)
    if sched is None:
        return None
    tsched, n_tile_levels = sched
    nt = part.n_tiles
    pos = empty_i32(nt)
    pos[tsched.long()] = torch.arange(nt, dtype=I32, device=dev())
    arr = ctypes.c_int * 3
    dd, tt = arr(*d3), arr(*t3)
    has_diag = not unit_diag
    blk = zeros_i32(nt + 1)
    stats = torch.tensor([0, 0, 0, INT_MAX, 0, 0, 0], dtype=I32, device=dev())
    args = (nt, tsched, pos, part.tile_ptr, part.trows, part.tile_of, t.rp, t.ci, t.val, nodes,
            ctypes.addressof(dd), ctypes.addressof(tt), int(upper), int(has_diag))
    call("ddilu_lattice_build", 0, *args, None, blk, stats, None)
    st = [int(v) for v in stats.cpu().numpy()]
    if st[0] or st[1] > query("ddilu_lattice_max_ext"):
        return None
    exclusive_scan_(blk, nt)
    total16 = int(blk[-1].item())
    blob = torch.empty(max(16, 16 * total16), dtype=torch.uint8, device=dev())
    tab = torch.empty(nt * 32 * 4, dtype=I32, device=dev())
    call("ddilu_lattice_build", 1, *args, tab, blk, stats, blob)
    st = [int(v) for v in stats.cpu().numpy()]
    if st[0]:
        return None
    blkmax, tmax, xemax = (st[5] + 15) & ~15, st[6], st[1]
    if query("ddilu_lattice_smem_bytes", blkmax, tmax, xemax) > 226 * 1024:
        return None
    return LatticeSched(n, nt, n_tile_levels, tab, blob, zeros_i32(nt), 2 if t3[1] * t3[2] > 32 else 1, has_diag, st[3],
                        blkmax, tmax, xemax)


def sptrsv_lattice(ls: LatticeSched, b: torch.Tensor, out: torch.Tensor, check: bool = False):
    if check and ls.bad_row != INT_MAX:
        raise TriSolveError(f"zero or missing diagonal at row {ls.bad_row}")
    call("ddilu_sptrsv_lattice", ls.n_tiles, ls.tab, ls.blob, ls.flags, ls.n_slots, int(ls.has_diag), ls.blkmax,
         ls.tmax, ls.xemax, b, out)
    return out


def build_tiles(t: DeviceCsr, lev: torch.Tensor, part: TilePartition, upper: bool, unit_diag: bool,
                sched=None) -> TileSched | None:
    """Tile schedule + static blocks of a triangular factor; None when the tile
    graph is cyclic / too deep or a tile does not fit the shared-memory budget
    (the caller then uses the sync-free solve)."""
    n = t.n_rows
    if part is None or n == 0 or part.n != n:
        return None
    sched = sched if sched is not None else tile_schedule(t, part, upper)
    if sched is None:
        return None
    tsched, n_tile_levels = sched
    nt = part.n_tiles
    has_diag = not unit_diag
    args = (nt, tsched, part.tile_ptr, part.trows, part.tile_of, part.tpos, t.rp, t.ci, t.val, lev, int(upper),
            int(has_diag))
    ITEM_WARPS = {"lean": 0, "warp": 1, "rot": 4}

    def count(kind):
        blk = zeros_i32(nt + 1)
        stats = torch.tensor([0, 0, 0, INT_MAX, 0], dtype=I32, device=dev())
        call("ddilu_tile_build", 0, *args, ITEM_WARPS[kind], blk, stats, None)
        return blk, stats, [int(v) for v in stats.cpu().numpy()]

    # kernel choice: lean records (rows with <= 3 dependencies) > warp-per-tile > CTA-per-tile, by what fits
    kind = "lean" if TILE_KERNEL == "warp" else TILE_KERNEL
    blk, stats, (tmax, emax, stat_max, _, kmax) = count(kind)
    if tmax + emax + 34 >= 0xFFFF:
        return None
    if kind == "lean" and (kmax > 3 or query("ddilu_warptile_smem_per_warp", stat_max, tmax + 32, emax) > 226 * 1024):
        kind = "warp"
        blk, stats, (tmax, emax, stat_max, _, kmax) = count(kind)
    if kind == "warp" and (TILE_KERNEL != "warp" or
                           query("ddilu_warptile_smem_per_warp", stat_max, tmax, emax) > 113 * 1024):
        kind = "rot"        # fewer than two warps per SM would fit: the CTA-per-tile kernel shares one ring
        blk, stats, (tmax, emax, stat_max, _, kmax) = count(kind)
    if kind == "rot" and query("ddilu_tiled_smem_bytes", stat_max, tmax, emax) > TILE_SMEM_LIMIT:
        return None
    exclusive_scan_(blk, nt)
    total16 = int(blk[-1].item())
    blob = torch.empty(max(16, 16 * total16), dtype=torch.uint8, device=dev())
    call("ddilu_tile_build", 1, *args, ITEM_WARPS[kind], blk, stats, blob)
    bad = int(stats[3].item())
    return TileSched(n, nt, n_tile_levels, blk, blob, stat_max, tmax, emax, kmax, has_diag, bad, kind)


def sptrsv_tiled(ts, b: torch.Tensor, out: torch.Tensor, check: bool = False):
    if ts.kind == "lattice":
        return sptrsv_lattice(ts, b, out, check)
    if check and ts.bad_row != INT_MAX:
        raise TriSolveError(f"zero or missing diagonal at row {ts.bad_row}")
    entry = {"lean": "ddilu_sptrsv_lean", "warp": "ddilu_sptrsv_warptile", "rot": "ddilu_sptrsv_tiled"}[ts.kind]
    call(entry, ts.n, ts.n_tiles, ts.blk_off16, ts.blob, ts.stat_max, ts.tmax, ts.emax, ts.kmax, int(ts.has_diag),
         b, out)
    return out


USE_SELL = True   # False: CSR thread-per-row kernel (kept for comparison runs)
USE_WARPROW = os.environ.get("DDILU_WARPROW", "1") == "1"   # warp-per-row sync-free solve for long rows
WARPROW_MIN_AVG_ROW = 8.0     # stored entries per row from which a warp per row pays
UNIFORM_SELL = True
USE_GWAIT = True
USE_BLOCK_WINDOW = os.environ.get("DDILU_BLOCK_WINDOW", "0") == "1"   # interface factors: CTA-per-block sweep, x window in shared memory
USE_BLOCK_LOCAL = False   # "sell" | "csr": CTA-per-block sweeps (measured slower: 0.77 us/level floor)


def build_sell(t: DeviceCsr, sched: Schedule, upper: bool, unit_diag: bool) -> Sell:
    n_groups = sched.n_slots // 32
    gw = zeros_i32(n_groups + 1)
    sdiag = None if unit_diag else empty_f64(max(1, sched.n_slots))
    bad = torch.full((1,), INT_MAX, dtype=I32, device=dev())
    gwait = empty_i32(max(1, n_groups)) if USE_GWAIT else None
    pos = empty_i32(max(1, t.n_rows)) if USE_GWAIT else None
    call("ddilu_sell_width", sched.n_slots, sched.order, t.rp, t.ci, t.val, int(upper), int(unit_diag), gw, sdiag,
         bad, pos, gwait)
    gfar1 = gfar2 = None
    if USE_GWAIT and n_groups:
        gfar1, gfar2 = empty_i32(n_groups), empty_i32(n_groups)
        call("ddilu_compose_wait", n_groups, gwait, pos, gwait, gfar1)
        call("ddilu_compose_wait", n_groups, gwait, pos, gfar1, gfar2)
    wmax = int(gw[:n_groups].max().item()) // 32 if n_groups else 0
    exclusive_scan_(gw, n_groups)
    total = int(gw[-1].item())
    uniform = wmax * 32 * n_groups
    if UNIFORM_SELL and uniform <= 1.25 * total + 1024:
        # short, regular rows (stencils): pad every group to the widest one and drop the descriptor array
        scol, sval = empty_i32(max(1, uniform)), empty_f64(max(1, uniform))
        call("ddilu_sell_fill", sched.n_slots, sched.order, t.rp, t.ci, t.val, int(upper), None, wmax, scol, sval)
        return Sell(None, wmax, scol, sval, sdiag, int(bad.item()), gwait, gfar1, gfar2)
    scol, sval = empty_i32(max(1, total)), empty_f64(max(1, total))
    call("ddilu_sell_fill", sched.n_slots, sched.order, t.rp, t.ci, t.val, int(upper), gw, 0, scol, sval)
    return Sell(gw, 0, scol, sval, sdiag, int(bad.item()), gwait, gfar1, gfar2)


BLOCK_LOCAL_MAX_WIDTH = 1024   # average rows per level per block up to which the CTA-per-block sweep is used


BLOCK_WINDOW_MAX = 16384   # doubles of shared memory per block (128 KB)


@dataclass
class BlockWindow:
    """Plan of the block-local sweep with x in a shared-memory window (`ddilu_sptrsv_blockwin_sell`)."""

    lbase: torch.Tensor        # [n_blocks * n_levels] block-local position of the first row of (block, level)
    scol_loc: torch.Tensor     # sell.scol with block-local positions instead of row ids
    sdinv: torch.Tensor | None  # RN(1 / pivot), 0 where the kernel must divide
    wmask: int


def enable_block_window(t: DeviceCsr, sched: Schedule, seg_ptr, upper: bool, unit_diag: bool) -> "BlockWindow | None":
    """Block-diagonal factor with narrow levels (interface factors: one block per subdomain): number the rows of a
    block in schedule order and check that every dependency lies less than a shared-memory window behind the end
    of the level that reads it.  Returns None when the factor does not qualify."""
    if sched.n == 0 or not enable_block_local(sched, seg_ptr):
        return None
    sell = get_sell(t, sched, upper, unit_diag)
    bl, L, n = sched.blocks, sched.n_levels, sched.n
    nb = bl.n_blocks
    cnt = bl.cnt.view(nb, L).to(torch.int64)
    base = torch.cumsum(cnt, 1) - cnt                       # block-local position of the first row of a level
    flat_cnt = cnt.reshape(-1)
    seg = torch.repeat_interleave(torch.arange(nb * L, device=dev()), flat_cnt)     # (block, level) of element e
    first = torch.cumsum(flat_cnt, 0) - flat_cnt
    within = torch.arange(int(flat_cnt.sum().item()), device=dev()) - first[seg]
    q = bl.start.to(torch.int64)[seg] + within                                       # position in level_rows
    rows = sched.level_rows.to(torch.int64)[q]
    lp = torch.empty(n, dtype=torch.int64, device=dev())
    lend = torch.empty(n, dtype=torch.int64, device=dev())
    lp[rows] = base.reshape(-1)[seg] + within
    lend[rows] = (base + cnt).reshape(-1)[seg]
    G = sched.n_slots // 32
    if sell.goff is None:
        n_ent = G * sell.width * 32
        e = torch.arange(n_ent, device=dev())
        grp = e // (32 * sell.width)
    else:
        n_ent = int(sell.goff[G].item())
        e = torch.arange(n_ent, device=dev())
        grp = torch.searchsorted(sell.goff[: G + 1].to(torch.int64), e, right=True) - 1
    dep = sell.scol[:n_ent].to(torch.int64)
    valid = dep >= 0
    qd = lp[dep.clamp(min=0)]
    slot_rows = sched.order.to(torch.int64)[grp * 32 + (e & 31)]      # entries of a group are lane-minor
    row_end = lend[slot_rows.clamp(min=0)]
    need = torch.where(valid & (slot_rows >= 0), row_end - qd, torch.zeros_like(qd))
    max_need = int(need.max().item()) if need.numel() else 1
    w = 1
    while w < max(max_need, 32):
        w <<= 1
    if os.environ.get("DDILU_DEBUG_WINDOW"):
        print("block window: need", max_need, "window", w, "blocks", nb, "levels", L, flush=True)
    if w > BLOCK_WINDOW_MAX:
        return None
    scol_loc = torch.full((max(1, sell.scol.numel()),), -1, dtype=I32, device=dev())
    scol_loc[:n_ent] = torch.where(valid, qd, torch.full_like(qd, -1)).to(I32)
    sdinv = None
    if sell.sdiag is not None:
        d = sell.sdiag
        a = d.abs()
        ok = (a >= 2.0 ** -400) & (a < 2.0 ** 401)          # the exponent window of exact_div (csrc/common.cuh)
        sdinv = torch.where(ok, 1.0 / d, torch.zeros_like(d)).contiguous()
    return BlockWindow(base.to(I32).reshape(-1).contiguous(), scol_loc, sdinv, w - 1)


def sptrsv_block_window(t: DeviceCsr, sched: Schedule, bw: BlockWindow, b: torch.Tensor, out: torch.Tensor, upper: bool,
                        unit_diag: bool):
    bl = sched.blocks
    sell = get_sell(t, sched, upper, unit_diag)
    call("ddilu_sptrsv_blockwin_sell", bl.n_blocks, sched.n_levels, bl.sstart, bl.cnt, bw.lbase, sched.order,
         sell.goff, sell.width, bw.scol_loc, sell.sval, sell.sdiag, bw.sdinv, bw.wmask, b, out)
    return out


# ---------------------------------------------------------------------------
# block sweep (csrc/sweep.cu): interface factors, one CTA per subdomain block

USE_SWEEP = os.environ.get("DDILU_SWEEP", "1") == "1"
SWEEP_MAX_AVG_WIDTH = 512      # average rows per level of a block up to which one CTA per block is the right shape
SWEEP_SMEM_BUDGET = 200 * 1024
SWEEP_SMEM_BUDGET_LONG = 224 * 1024     # long rows: large windows (27-point interfaces reach 16 k positions back)
SWEEP_MAX_LEVELS = 6144        # level table of a block in shared memory (L + U)
SWEEP_MAX_THREADS = 416        # compute threads per set (wider levels loop)
SWEEP_ROWS_PER_THREAD = 1      # rows of a level per thread (1, 2); measured at 256^3 / 128^3: 1 row, 3 sets is the fastest shape
SWEEP_SETS = 3                 # compute sets taking the levels in turn (2, 3)
SWEEP_SETS_LONG = 2            # the same for long rows (k > 8): two sets leave more threads per set in a 512-thread CTA


@dataclass
class SweepPlan:
    """Layout of `ddilu_sweep_solve` for a block-diagonal factor pair: rows of a block in schedule order
    (level-major), operands in 256-row pages, positions padded to whole pages per block."""

    n: int
    n_blocks: int
    k: int                     # operand slots per row
    window: int                # shared-memory window (doubles, power of two)
    stages: int                # ring depth (power of two)
    sets: int                  # compute sets taking the levels in turn
    nct: int                   # compute threads per set
    rpt: int                   # rows of a level per thread
    max_lev: int
    npad: int                  # padded position space (n_pages * 256)
    blocks: torch.Tensor       # int32[n_blocks * 8]
    levtab: torch.Tensor
    pages_l: torch.Tensor
    pages_u: torch.Tensor
    rowof_l: torch.Tensor      # int32[npad]: row at a position of the L schedule, -1 = padding
    rowof_u: torch.Tensor
    rhs: torch.Tensor          # f64[npad] right-hand side in schedule order
    tmp: torch.Tensor          # f64[npad] U-phase right-hand side written by the L phase
    addbuf: torch.Tensor       # f64[npad] vector added to the results, in U schedule order
    bad_row: int
    n_levels: tuple = (0, 0)


def build_sweep(lower: DeviceCsr, upper: DeviceCsr, lev_l: torch.Tensor, nlev_l: int, lev_u: torch.Tensor,
                nlev_u: int, seg_ptr) -> "SweepPlan | None":
    """Plan of the block sweep for the factor pair (L strictly lower, U with its diagonal) whose independent
    diagonal blocks are the row ranges seg_ptr (host ints); None when the pair does not qualify (a dependency
    leaves its block, rows with more than 8 dependencies, levels too wide or too many, window too large)."""
    n = lower.n_rows
    nb = len(seg_ptr) - 1
    if not USE_SWEEP or n == 0 or nb < 1 or nlev_l == 0 or nlev_u == 0:
        return None
    d = dev()
    i64 = torch.int64
    # dependency counts -> operand slots per row (long rows: 64-row pages, one row per thread, 512-thread CTAs)
    kl = int((lower.rp[1:] - lower.rp[:-1]).max().item())
    ku = int((upper.rp[1:] - upper.rp[:-1]).max().item()) - 1
    kmax = max(kl, ku, 1)
    k = next((c for c in (2, 3, 4, 8, 16, 24) if kmax <= c), None)
    if k is None:
        return None
    P = query("ddilu_sweep_page_rows", k)
    seg = torch.tensor([int(v) for v in seg_ptr], dtype=i64, device=d)
    if int(seg[-1].item()) != n or int(seg[0].item()) != 0:
        return None
    rows = torch.arange(n, dtype=i64, device=d)
    blk = torch.bucketize(rows, seg[1:], right=True)
    sizes = seg[1:] - seg[:-1]
    n_pages_b = (sizes + P - 1) // P
    page0 = torch.cumsum(n_pages_b, 0) - n_pages_b
    n_pages = int(n_pages_b.sum().item())
    npad = n_pages * P
    plans = []
    for fac, lev, nlev, up in ((lower, lev_l, nlev_l, False), (upper, lev_u, nlev_u, True)):
        key = blk * nlev + lev[:n].to(i64)
        order = torch.argsort(key, stable=True)
        cnt = torch.bincount(key, minlength=nb * nlev).view(nb, nlev)
        lpos = torch.empty(n, dtype=i64, device=d)
        lpos[order] = rows - seg[blk[order]]
        gpos = page0[blk] * P + lpos
        lev_end = torch.cumsum(cnt, 1)
        # dependencies: same block, and not further back than the window behind the end of the reader's level
        nnz = fac.nnz
        rlen = (fac.rp[1:] - fac.rp[:-1]).to(i64)
        erow = torch.repeat_interleave(rows, rlen)
        ecol = fac.ci[:nnz].to(i64)
        dep = ecol != erow
        if bool((blk[ecol] != blk[erow]).any().item()):
            return None
        row_end = lev_end.reshape(-1)[key]
        need = torch.where(dep, row_end[erow] - lpos[ecol], torch.zeros_like(ecol))
        max_need = int(need.max().item()) if nnz else 1
        nz = cnt > 0
        plans.append((fac, up, lpos, gpos, lev_end[nz], nz.sum(1), int(cnt.max().item()), max_need))
    window = 32
    while window < max(p[7] for p in plans):
        window <<= 1
    width_max = max(p[6] for p in plans)
    nlev_b = plans[0][5] + plans[1][5]
    max_lev = int(nlev_b.max().item())
    avg_width = float(n) / max(1, int(plans[0][5].sum().item()))
    if os.environ.get("DDILU_DEBUG_SWEEP"):
        print(f"sweep plan: k {k} (max deps {kmax}), page rows {P}, window {window}, widest level {width_max}, "
              f"levels per block {max_lev}, average width {avg_width:.1f}", flush=True)
    if window > 16384 or max_lev > SWEEP_MAX_LEVELS or avg_width > SWEEP_MAX_AVG_WIDTH:
        return None
    rpt, sets = SWEEP_ROWS_PER_THREAD, SWEEP_SETS
    helpers = query("ddilu_sweep_helper_threads")
    cta_max = 1024
    if k > 8:
        rpt, sets, cta_max = 1, SWEEP_SETS_LONG, 512
    nct = min(SWEEP_MAX_THREADS, ((cta_max - helpers) // sets) & ~31, max(32, ((width_max + rpt - 1) // rpt + 31) & ~31))
    stages = 0
    budget = SWEEP_SMEM_BUDGET_LONG if k > 8 else SWEEP_SMEM_BUDGET
    for st in (16, 8, 4):
        if query("ddilu_sweep_smem_bytes", k, st, window, max_lev) <= budget:
            stages = st
            break
    # ring residency.  Short rows (blocking operand prefetch): the sets work on up to `sets` consecutive levels at
    # once and a page is freed only when the progress counter (start of the level being executed) has passed it, so
    # all pages of those levels must fit.  Long rows (64-row pages): the prefetch never waits for a page -- rows
    # whose page has not landed are fetched behind the level barrier -- so only the pages of ONE level, plus the
    # page it shares with its predecessor, must fit.
    if stages < 4 or (width_max > (stages - 1) * P if k > 8 else sets * width_max > (stages - 2) * P):
        return None
    # level tables: per block its L levels then its U levels
    lev_off = torch.cumsum(nlev_b, 0) - nlev_b
    lt_l, lt_u = plans[0][4], plans[1][4]
    nl, nu = plans[0][5], plans[1][5]
    levtab = torch.empty(int(nlev_b.sum().item()), dtype=i64, device=d)
    off_l = torch.repeat_interleave(lev_off, nl) + (torch.arange(lt_l.numel(), device=d) -
                                                    torch.repeat_interleave(torch.cumsum(nl, 0) - nl, nl))
    off_u = torch.repeat_interleave(lev_off + nl, nu) + (torch.arange(lt_u.numel(), device=d) -
                                                         torch.repeat_interleave(torch.cumsum(nu, 0) - nu, nu))
    levtab[off_l] = lt_l
    levtab[off_u] = lt_u
    blocks = torch.zeros((nb, 8), dtype=i64, device=d)
    blocks[:, 0], blocks[:, 1], blocks[:, 2], blocks[:, 3], blocks[:, 4] = sizes, page0, nl, nu, lev_off
    bad = torch.full((1,), INT_MAX, dtype=I32, device=d)
    gpos_u32 = plans[1][3].to(I32).contiguous()
    pages, rowof = [], []
    for fac, up, lpos, gpos, _, _, _, _ in plans:
        pg = torch.zeros(n_pages * query("ddilu_sweep_page_bytes", k, int(up)), dtype=torch.uint8, device=d)
        call("ddilu_sweep_fill", n, fac.rp, fac.ci, fac.val, int(up), k, gpos.to(I32).contiguous(),
             lpos.to(I32).contiguous(), None if up else gpos_u32, window, pg, bad)
        ro = torch.full((npad,), -1, dtype=I32, device=d)
        ro[gpos] = rows.to(I32)
        pages.append(pg)
        rowof.append(ro)
    return SweepPlan(n, nb, k, window, stages, sets, nct, rpt, max_lev, npad, blocks.to(I32).contiguous().view(-1),
                     levtab.to(I32).contiguous(), pages[0], pages[1], rowof[0], rowof[1], zeros_f64(npad),
                     zeros_f64(npad), zeros_f64(npad), int(bad.item()), (int(nl.max().item()), int(nu.max().item())))


def sweep_rhs(sp: SweepPlan, upper: bool, b: torch.Tensor | None, mat: "DeviceCsr | None" = None,
              y: torch.Tensor | None = None, mode: int = 0, add: torch.Tensor | None = None):
    """sp.rhs <- right-hand side in the schedule order of L (or U): b gathered, or (mode 0) mat y,
    (mode 1) b - mat y, (mode 2) b + mat y; with `add` also sp.addbuf <- add in U schedule order."""
    ro = sp.rowof_u if upper else sp.rowof_l
    extra = (sp.rowof_u, add, sp.addbuf) if add is not None else (None, None, None)
    if mat is None:
        call("ddilu_sweep_rhs", sp.npad, ro, None, None, None, None, b, 0, sp.rhs, *extra)
    else:
        call("ddilu_sweep_rhs", sp.npad, ro, mat.rp, mat.ci, mat.val, y, b, mode, sp.rhs, *extra)


def sweep_solve(sp: SweepPlan, phases: int, out: torch.Tensor, add: bool = False, check: bool = False):
    """out[row] = x (+ add[row], staged by sweep_rhs) with x = L^-1 rhs (phases 1), U^-1 rhs (2) or
    U^-1 L^-1 rhs (3), rhs = sp.rhs."""
    if check and (phases & 2) and sp.bad_row != INT_MAX:
        raise TriSolveError(f"zero or missing diagonal at row {sp.bad_row}")
    call("ddilu_sweep_solve", sp.n_blocks, sp.blocks, sp.levtab, sp.pages_l, sp.pages_u, sp.k, sp.window, sp.stages,
         sp.sets, sp.nct, sp.rpt, sp.max_lev, phases, sp.rhs, sp.tmp, out, sp.addbuf if add else None)
    return out


# ---------------------------------------------------------------------------
# cluster sweep (csrc/csweep.cu): block-diagonal factors with LARGE deep blocks (the interior factors L_B / U_B) --
# a thread-block cluster per block, x in a window distributed over the CTAs' shared memory

USE_CSWEEP = os.environ.get("DDILU_CSWEEP", "1") == "1"
CSWEEP_CLUSTER = int(os.environ.get("DDILU_CSWEEP_CLUSTER", "16"))   # CTAs per block at most (the largest size whose clusters can all be resident is taken)
CSWEEP_NSET = int(os.environ.get("DDILU_CSWEEP_DEPTH", "4"))         # stages of the operand ring at most (as many as fit)
CSWEEP_MIN_CHUNK = int(os.environ.get("DDILU_CSWEEP_MIN_CHUNK", "32"))   # rows of a level a CTA takes at least (narrow levels stay on few CTAs)
CSWEEP_MIN_AVG_WIDTH = 2000    # average rows per level of a block from which a cluster pays (measured: 128^3 / p = 8, 1 340 rows per level, is a tie with the tiled kernel; 192^3, 3 000 rows, 1.3x faster)
CSWEEP_MIN_SMS = 60            # blocks x cluster size: SMs the launch must fill to have the bandwidth of the GPU
CSWEEP_LONG_ROWS = os.environ.get("DDILU_CSWEEP_LONG", "1") == "1"    # 20-slot instance for 27-point / ILUT factors
_csweep_active = {}


def csweep_active_clusters(csize: int, k: int, depth: int, max_steps: int) -> int:
    key = (csize, k, depth, max_steps)
    if key not in _csweep_active:
        _csweep_active[key] = query("ddilu_csweep_active_clusters", csize, k, depth, max_steps)
    return _csweep_active[key]


@dataclass
class ClusterSweepHalf:
    """One factor (L or U) in the layout of `ddilu_csweep_solve`."""

    ctas: torch.Tensor         # int32[n_blocks * csize * 4]
    steps: torch.Tensor        # int32[total steps * 8]
    coef: torch.Tensor
    code: torch.Tensor         # 16-bit halves of the packed words: dependency slots, push targets
    rowid: torch.Tensor
    piv: torch.Tensor | None
    blob: torch.Tensor | None  # long rows: the operands step by step in one buffer (instead of coef / code / rowid / piv)
    np: int
    max_steps: int
    depth: int                 # stages of the operand ring
    contiguous: bool           # every level chunk is a range of consecutive rows (no row-id loads)


@dataclass
class ClusterSweepPlan:
    n: int
    n_blocks: int
    csize: int
    k: int
    nset: int
    lower: ClusterSweepHalf
    upper: ClusterSweepHalf
    bad_row: int


def build_csweep(lower: DeviceCsr, upper: DeviceCsr, lev_l: torch.Tensor, nlev_l: int, lev_u: torch.Tensor,
                 nlev_u: int, seg_ptr) -> "ClusterSweepPlan | None":
    """Plan of the cluster sweep for the factor pair (L strictly lower, U with its diagonal) whose independent
    diagonal blocks are the row ranges seg_ptr (host ints); None when the pair does not qualify (a dependency
    leaves its block, more than 20 dependencies per row, short-row blocks too few / too narrow for clusters, a
    dependency further back than the window, a result needed by too many other CTAs, clusters cannot be resident).
    Up to 4 dependencies per row: the short-row shape of the kernel (7-point ILU(0)); 5 .. 20: the long-row shape
    (27-point / ILUT / ILU(k) factors)."""
    n = lower.n_rows
    nb = len(seg_ptr) - 1
    if not USE_CSWEEP or n == 0 or nb < 1 or nlev_l == 0 or nlev_u == 0:
        return None
    d = dev()
    i64 = torch.int64
    debug = bool(os.environ.get("DDILU_DEBUG_SWEEP"))
    kl = int((lower.rp[1:] - lower.rp[:-1]).max().item())
    ku = int((upper.rp[1:] - upper.rp[:-1]).max().item()) - 1
    kmax = max(kl, ku, 1)
    k = next((c for c in ((3, 4, 20) if CSWEEP_LONG_ROWS else (3, 4)) if kmax <= c), None)
    if k is None:
        return None
    # short rows (7-point ILU(0)): the tiled kernel is the better one for narrow levels; long rows (27-point / ILUT):
    # the alternative is the sync-free warp-per-row solve at ~1.3 us per level, a cluster wins at any width
    if k <= 4 and n / (nb * max(nlev_l, nlev_u)) < CSWEEP_MIN_AVG_WIDTH:
        return None
    W = query("ddilu_csweep_window", k)
    nset = CSWEEP_NSET
    lev_cap = 2 * max(nlev_l, nlev_u)           # steps of a CTA: its levels, the wide ones in several pieces
    if query("ddilu_csweep_smem_bytes", k, 1, 2, lev_cap) > 227 * 1024:
        return None
    cmax = min(16, CSWEEP_CLUSTER, 1 << query("ddilu_csweep_rank_bits", k))
    csize = next((c for c in range(cmax, 0, -1) if csweep_active_clusters(c, k, 2, lev_cap) >= nb), 0)
    if debug:
        print(f"cluster sweep: {nb} blocks -> clusters of {csize}", flush=True)
    if not csize or (k <= 4 and nb * csize < CSWEEP_MIN_SMS):
        return None
    seg = torch.tensor([int(v) for v in seg_ptr], dtype=i64, device=d)
    if int(seg[-1].item()) != n or int(seg[0].item()) != 0:
        return None
    rows = torch.arange(n, dtype=i64, device=d)
    blk = torch.bucketize(rows, seg[1:], right=True)
    halves = []
    bad = torch.full((1,), INT_MAX, dtype=I32, device=d)
    for fac, lev, nlev, up in ((lower, lev_l, nlev_l, False), (upper, lev_u, nlev_u, True)):
        lv = lev[:n].to(i64)
        key = blk * nlev + lv
        order = torch.argsort(key, stable=True)
        cnt = torch.bincount(key, minlength=nb * nlev).view(nb, nlev)
        lev_start = torch.cumsum(cnt, 1) - cnt
        pib = torch.empty(n, dtype=i64, device=d)              # position in the block's level-major order
        pib[order] = rows - seg[blk[order]]
        ril = pib - lev_start.reshape(-1)[key]                 # rank of the row inside its level (rows of a level by index)
        cs = torch.clamp((cnt + csize - 1) // csize, min=CSWEEP_MIN_CHUNK)        # chunk rows per (block, level)
        csr = cs.reshape(-1)[key]
        rk = ril // csr                                        # CTA of the row
        ro = ril - rk * csr
        ranks = torch.arange(csize, dtype=i64, device=d).view(1, csize, 1)
        ncl = torch.clamp(cnt.view(nb, 1, nlev) - ranks * cs.view(nb, 1, nlev), min=0)
        ncl = torch.minimum(ncl, cs.view(nb, 1, nlev).expand(nb, csize, nlev))    # rows of CTA (b, r) in level l
        npad = (ncl + 3) // 4 * 4                              # every chunk starts at a multiple of 4 positions (16-byte runs)
        lstart = torch.cumsum(npad, 2) - npad
        lend = lstart + ncl
        ckey = (blk * csize + rk) * nlev + lv
        lpos = lstart.reshape(-1)[ckey] + ro
        rows_cta = (lstart + npad)[:, :, -1].reshape(-1)
        padded = (rows_cta + 31) // 32 * 32
        base = torch.cumsum(padded, 0) - padded
        npos = int(padded.sum().item())
        gpos = base[blk * csize + rk] + lpos
        cta = blk * csize + rk                                 # CTA of every row
        nnz = fac.nnz
        rlen = (fac.rp[1:] - fac.rp[:-1]).to(i64)
        erow = torch.repeat_interleave(rows, rlen)
        ecol = fac.ci[:nnz].to(i64)
        cta_r, cta_c = cta[erow], cta[ecol]                    # CTA of the reader / of the dependency, per entry
        if bool((cta_r // csize != cta_c // csize).any().item()):      # a dependency leaves its block
            return None
        dep = ecol != erow
        # halo: (consumer CTA, producer row) pairs whose CTAs differ; a CTA numbers the values it holds level by
        # level -- own rows of the level, then the level's halo values (in row order)
        remote = dep & (cta_r != cta_c)
        hkey_e = cta_r * n + ecol
        hu = torch.unique(hkey_e[remote])                      # sorted by (consumer CTA, producer row)
        h_cta, h_row = hu // n, hu % n
        h_lev = lv[h_row]
        gkey = h_cta * nlev + h_lev
        n_in = torch.bincount(gkey, minlength=nb * csize * nlev).view(nb, csize, nlev)
        gorder = torch.argsort(gkey, stable=True)
        gstart = (torch.cumsum(n_in.reshape(-1), 0) - n_in.reshape(-1))
        h_idx = torch.empty_like(gkey)
        h_idx[gorder] = torch.arange(gkey.numel(), dtype=i64, device=d) - gstart[gkey[gorder]]
        n_ext = ncl + n_in
        wend = torch.cumsum(n_ext, 2)                          # window positions: end of every level per CTA
        wstart = wend - n_ext
        wpos = wstart.reshape(-1)[ckey] + ro                   # own rows
        h_wpos = wstart.reshape(-1)[gkey] + ncl.reshape(-1)[gkey] + h_idx
        # window slot of every dependency in the READER's CTA, and how far back it lies
        e_wpos = wpos[ecol]
        if hu.numel():
            hit = torch.searchsorted(hu, hkey_e[remote])
            e_wpos = e_wpos.clone()
            e_wpos[remote] = h_wpos[hit]
        need = torch.where(dep, wend.reshape(-1)[cta_r * nlev + lv[erow]] - e_wpos, torch.zeros_like(ecol))
        max_need = int(need.max().item()) if nnz else 1
        # push targets of every row: the other CTAs that hold its value, (slot << 4 | rank)
        NP = query("ddilu_csweep_max_push", k)
        RB = query("ddilu_csweep_rank_bits", k)
        porder = torch.argsort(h_row, stable=True)
        prow = h_row[porder]
        pidx = torch.arange(prow.numel(), dtype=i64, device=d) - torch.searchsorted(prow, prow)
        max_push = int(pidx.max().item()) + 1 if prow.numel() else 0
        nz = cnt > 0
        nlev_b = torch.where(nz.any(1), nlev - torch.flip(nz, [1]).to(i64).argmax(1), torch.zeros(nb, dtype=i64, device=d))
        max_lev = int(nlev_b.max().item())
        width_cta = int(ncl.max().item())
        # chunks that are ranges of consecutive rows need no row ids
        # (`order` lists the rows by block, level, index, and a chunk is a run of it: first and last row by lookup)
        nclf = ncl.reshape(-1)
        blk_first = (seg[:-1].view(nb, 1) + lev_start).view(nb, 1, nlev)          # run of a (block, level) in `order`
        run0 = (blk_first + ranks * cs.view(nb, 1, nlev)).expand(nb, csize, nlev).reshape(-1)
        some = nclf > 0
        row_lo = torch.where(some, order[torch.where(some, run0, torch.zeros_like(run0))], torch.full_like(run0, n))
        row_hi = torch.where(some, order[torch.where(some, run0 + nclf - 1, torch.zeros_like(run0))], torch.full_like(run0, -1))
        consecutive = (nclf == 0) | (row_hi - row_lo + 1 == nclf)
        contiguous = bool(consecutive.all().item())
        row0 = torch.where((nclf > 0) & consecutive, row_lo, torch.full_like(row_lo, -1))
        NT = query("ddilu_csweep_threads", k)
        # steps: a CTA's chunk of a level, cut into pieces of at most one row per thread; the first piece waits for
        # the previous level, the last one signals
        nsub = torch.clamp((nclf + NT - 1) // NT, min=1)
        # levels behind the block's last one do not exist for the kernel
        live = (torch.arange(nlev, dtype=i64, device=d).view(1, 1, nlev) < nlev_b.view(nb, 1, 1)).expand(nb, csize, nlev).reshape(-1)
        nsub = torch.where(live, nsub, torch.zeros_like(nsub))
        steps_cta = nsub.view(nb * csize, nlev).sum(1)
        max_steps = int(steps_cta.max().item())
        depth = next((dd for dd in range(nset, 1, -1) if query("ddilu_csweep_smem_bytes", k, int(up), dd, max_steps) <= 227 * 1024), 0)
        if debug:
            print(f"cluster sweep plan ({'U' if up else 'L'}): k {k}, cluster {csize}, furthest dependency {max_need} "
                  f"(window {W}), widest level per CTA {width_cta} ({NT} threads, <= {max_steps} steps, ring depth {depth}), "
                  f"levels per block {max_lev}, positions {npos} for {n} rows, halo values {hu.numel()}, "
                  f"push targets per row <= {max_push}, consecutive chunks: {contiguous}", flush=True)
        if max_need > W or max_push > NP or not depth:
            return None
        tot = int(nsub.sum().item())
        src = torch.repeat_interleave(torch.arange(nsub.numel(), dtype=i64, device=d), nsub)    # (CTA, level) of a step
        first = torch.cumsum(nsub, 0) - nsub
        e = torch.arange(tot, dtype=i64, device=d) - first[src]                                  # piece index
        s_start = lstart.reshape(-1)[src] + e * NT
        s_end = torch.minimum(lend.reshape(-1)[src], s_start + NT)
        s_slot = (wstart.reshape(-1)[src] + e * NT) % W
        s_row0 = torch.where(row0[src] >= 0, row0[src] + e * NT, row0[src])
        is_first, is_last = e == 0, e == nsub[src] - 1
        s_tx = torch.where(is_first, 8 * n_in.reshape(-1)[src], torch.zeros_like(e))
        s_flags = is_first.to(i64) + 2 * is_last.to(i64)
        zero = torch.zeros_like(e)
        steps = torch.stack([s_start, s_end, s_slot, s_row0, s_tx, s_flags, zero, zero], 1)
        # who signals whom at the end of a level: a CTA its own mbarrier and those of the CTAs it exchanges values
        # with, in BOTH directions -- the producer must know that its consumer is done reading before it overwrites
        # the consumer's window slots, and a coupled pair must stay within one level of each other (two mbarrier
        # phases are in flight at most)
        ncta = nb * csize
        pairs = h_cta * ncta + cta[h_row]                                           # (consumer, producer)
        pairs = torch.unique(torch.cat([pairs, cta[h_row] * ncta + h_cta]))
        pa, pb = pairs // ncta, pairs % ncta
        sigmask = torch.ones(ncta, dtype=i64, device=d) << (torch.arange(ncta, dtype=i64, device=d) % csize)
        sigmask = sigmask.scatter_reduce(0, pa, torch.ones_like(pb) << (pb % csize), "sum")        # pairs are unique: sum = or
        signallers = 1 + torch.bincount(pb, minlength=ncta)
        ctas = torch.zeros((ncta, 4), dtype=i64, device=d)
        ctas[:, 0], ctas[:, 1] = base, sigmask | (signallers << 16)
        ctas[:, 2] = torch.cumsum(steps_cta, 0) - steps_cta
        ctas[:, 3] = steps_cta
        pcode = (((h_wpos[porder] % W) << RB) | (h_cta[porder] % csize)).to(torch.int32).to(torch.int16) \
            if prow.numel() else None
        half = k + pidx                                                              # half index of a push target
        if k > 4:
            # long rows: the operands step by step in one blob (one bulk copy per step in the kernel)
            REC = query("ddilu_csweep_long_record_bytes", k, int(up))
            r4s = (s_end - s_start + 3) // 4 * 4
            bbytes = r4s * REC
            boff = torch.cumsum(bbytes, 0) - bbytes
            steps[:, 6] = boff // 16
            st_row = first[ckey] + ro // NT                                          # step of every row
            off = ro % NT
            blob = torch.zeros(max(16, int(bbytes.sum().item())), dtype=torch.uint8, device=d)
            call("ddilu_csweep_fill_long", n, fac.rp, fac.ci, fac.val, int(up), k, boff[st_row].contiguous(),
                 r4s[st_row].to(I32).contiguous(), off.to(I32).contiguous(), (e_wpos % W).to(I32).contiguous(), blob, bad)
            if pcode is not None:
                pr4, pst = r4s[st_row[prow]], st_row[prow]
                at = boff[pst] + (8 * k + (16 if up else 0)) * pr4 + 4 * ((half // 2) * pr4 + off[prow]) + 2 * (half % 2)
                blob.view(torch.int16)[at // 2] = pcode
            coef = code = rowid = piv = None
        else:
            blob = None
            NWD = query("ddilu_csweep_code_words", k)
            coef = torch.zeros(k * npos, dtype=F64, device=d)
            code = torch.full((NWD * npos * 2,), -1, dtype=torch.int16, device=d)      # halves; 0xffff: no push target
            if pcode is not None:
                code[2 * ((half // 2) * npos + gpos[prow]) + half % 2] = pcode
            rowid = torch.zeros(npos, dtype=I32, device=d)
            piv = torch.ones(2 * npos, dtype=F64, device=d) if up else None
            call("ddilu_csweep_fill", n, fac.rp, fac.ci, fac.val, int(up), k, gpos.to(I32).contiguous(),
                 (e_wpos % W).to(I32).contiguous(), npos, coef, code, rowid, piv, bad)
        halves.append(ClusterSweepHalf(ctas.to(I32).contiguous().view(-1), steps.to(I32).contiguous().view(-1),
                                       coef, code, rowid, piv, blob, npos, max_steps, depth, contiguous))
    return ClusterSweepPlan(n, nb, csize, k, nset, halves[0], halves[1], int(bad.item()))


def csweep_solve(cp: ClusterSweepPlan, upper: bool, b: torch.Tensor, out: torch.Tensor, check: bool = False):
    """out = L^-1 b (upper False) or U^-1 b (upper True) on the cluster-sweep layout (vectors by row)."""
    if check and upper and cp.bad_row != INT_MAX:
        raise TriSolveError(f"zero or missing diagonal at row {cp.bad_row}")
    h = cp.upper if upper else cp.lower
    call("ddilu_csweep_solve", cp.n_blocks, cp.csize, h.ctas, h.steps, h.coef, h.code, h.rowid, h.piv, h.blob, h.np, cp.k,
         int(upper), h.max_steps, h.depth, b, out)
    return out


# ---------------------------------------------------------------------------
# tile sweep (csrc/experiments/tsweep.cu): interior factors with vectors in tile order.  EXPERIMENT (needs a
# DDILU_EXPERIMENTS=1 build; scripts/probe_tsweep.py): bit-exact, 0.62-0.66 of the HBM roofline when the tiles
# are made independent, but 0.30 / 0.42 (L / U) with the real tile dependencies -- 16^3 tiles leave ~190 tiles
# per tile level for ~300 resident CTAs and every tile level costs a whole tile time; not integrated.

USE_TSWEEP = os.environ.get("DDILU_TSWEEP", "1") == "1"
TSWEEP_TILE_3D = (16, 16, 16)
TSWEEP_SETS = 3
TSWEEP_MAX_THREADS = 192       # compute threads per set
TSWEEP_STAGES = 4
TSWEEP_SMEM_BUDGET = 110 * 1024     # two CTAs per SM


@dataclass
class TileSweepHalf:
    """One factor (L or U) of a tile-sweep plan."""

    n_tiles: int
    tiles: torch.Tensor        # int32[n_tiles * 16], schedule order
    levtab: torch.Tensor
    extpos: torch.Tensor
    prods: torch.Tensor
    pages: torch.Tensor
    flags: torch.Tensor
    k: int
    window: int
    xe_cap: int
    max_lev: int
    stages: int
    nct: int
    n_tile_levels: int


@dataclass
class TileSweepPlan:
    """Tile-order layout of an interior factor pair: vpos[row] = position of a row in the tile-ordered vectors
    (tiles padded to whole pages), npad = length of those vectors."""

    n: int
    npad: int
    vpos: torch.Tensor         # int32[n]
    lower: TileSweepHalf
    upper: TileSweepHalf
    bad_row: int
    sets: int


def build_tsweep(lower: DeviceCsr, upper: DeviceCsr, lev_l: torch.Tensor, nlev_l: int, lev_u: torch.Tensor,
                 nlev_u: int, part: TilePartition) -> "TileSweepPlan | None":
    """Tile-sweep plan of the factor pair on the tile partition `part` (large box tiles); None when the pair does
    not qualify: cyclic tile graph, U not walking the reverse of L's order inside a tile, more than 8
    dependencies per row, window / boundary buffers too large."""
    n = lower.n_rows
    if not USE_TSWEEP or not _lib.has_experiments() or part is None or n == 0 or part.n != n:
        return None
    P = 256
    d = dev()
    i64 = torch.int64
    nt = part.n_tiles
    tile = part.tile_of.to(i64)
    rows = torch.arange(n, dtype=i64, device=d)
    tptr = part.tile_ptr.to(i64)
    sizes = tptr[1:] - tptr[:-1]
    n_pages_t = (sizes + P - 1) // P
    page0_t = torch.cumsum(n_pages_t, 0) - n_pages_t
    tpad = n_pages_t * P
    n_pages = int(n_pages_t.sum().item())
    ll, lu = lev_l[:n].to(i64), lev_u[:n].to(i64)
    order = torch.argsort(tile * nlev_l + ll, stable=True)
    lpos = torch.empty(n, dtype=i64, device=d)
    lpos[order] = rows - tptr[tile[order]]
    # U must walk the reverse order: along L's order the U level never increases inside a tile
    to, uo = tile[order], lu[order]
    same = to[1:] == to[:-1]
    if bool(((uo[1:] > uo[:-1]) & same).any().item()):
        return None
    upos = tpad[tile] - 1 - lpos
    vpos = page0_t[tile] * P + lpos
    kl = int((lower.rp[1:] - lower.rp[:-1]).max().item())
    ku = int((upper.rp[1:] - upper.rp[:-1]).max().item()) - 1
    kmax = max(kl, ku, 1)
    k = next((c for c in (2, 3, 4, 8) if kmax <= c), None)
    if k is None:
        return None
    bad = torch.full((1,), INT_MAX, dtype=I32, device=d)
    halves = []
    for fac, lev, nlev, up, pos in ((lower, ll, nlev_l, False, lpos), (upper, lu, nlev_u, True, upos)):
        sched = tile_schedule(fac, part, up)
        if sched is None:
            return None
        tsched, n_tile_levels = sched
        tsched = tsched.to(i64)
        ord_of_tile = torch.empty(nt, dtype=i64, device=d)
        ord_of_tile[tsched] = torch.arange(nt, dtype=i64, device=d)
        front = (tpad - sizes) if up else torch.zeros_like(sizes)
        key = tile * nlev + lev
        cnt = torch.bincount(key, minlength=nt * nlev).view(nt, nlev)
        nz = cnt > 0
        nlev_t = nz.sum(1)
        lev_end = torch.cumsum(cnt, 1) + front[:, None]        # end position of (tile, level) in the own space
        max_lev = int(nlev_t.max().item())
        width_max = int(cnt.max().item())
        # entries
        nnz = fac.nnz
        rlen = (fac.rp[1:] - fac.rp[:-1]).to(i64)
        erow = torch.repeat_interleave(rows, rlen)
        ecol = fac.ci[:nnz].to(i64)
        dep = ecol != erow
        cross = dep & (tile[ecol] != tile[erow])
        inner = dep & ~cross
        row_end = lev_end.reshape(-1)[key]
        need = torch.where(inner, row_end[erow] - pos[ecol], torch.zeros_like(ecol))
        max_need = int(need.max().item()) if nnz else 1
        window = 32
        while window < max_need:
            window <<= 1
        # boundary dependencies: one slot per cross-tile entry, numbered inside the reader's tile
        cidx = torch.nonzero(cross).flatten()
        ct = tile[erow[cidx]]
        o2 = torch.argsort(ct, stable=True)
        cidx, ct = cidx[o2], ct[o2]
        n_ext_t = torch.bincount(ct, minlength=nt)
        ext_first = torch.cumsum(n_ext_t, 0) - n_ext_t
        eidx = torch.arange(cidx.numel(), dtype=i64, device=d) - ext_first[ct]
        xe_cap = int(n_ext_t.max().item()) if cidx.numel() else 0
        xe_cap = (xe_cap + 1) & ~1
        if window > 8192 or window + 2 + xe_cap > 65535:
            return None
        ecode = torch.full((max(nnz, 1),), -1, dtype=I32, device=d)
        ecode[cidx] = (window + 1 + eidx).to(I32)
        # the boundary lists are stored tile by tile in SCHEDULE order
        sizes_s = n_ext_t[tsched]
        ext_off_s = torch.cumsum(sizes_s, 0) - sizes_s
        ext_off_t = torch.empty(nt, dtype=i64, device=d)
        ext_off_t[tsched] = ext_off_s
        extpos = torch.empty(max(cidx.numel(), 1), dtype=I32, device=d)
        extpos[(ext_off_t[ct] + eidx)] = vpos[ecol[cidx]].to(I32)
        # producer tiles
        pk = torch.unique(ct * nt + tile[ecol[cidx]])
        pt, pj = pk // nt, pk % nt
        n_prod_t = torch.bincount(pt, minlength=nt)
        prod_first = torch.cumsum(n_prod_t, 0) - n_prod_t
        pidx = torch.arange(pk.numel(), dtype=i64, device=d) - prod_first[pt]
        psz_s = n_prod_t[tsched]
        prod_off_s = torch.cumsum(psz_s, 0) - psz_s
        prod_off_t = torch.empty(nt, dtype=i64, device=d)
        prod_off_t[tsched] = prod_off_s
        prods = torch.empty(max(pk.numel(), 1), dtype=I32, device=d)
        prods[(prod_off_t[pt] + pidx)] = ord_of_tile[pj].to(I32)
        # level tables tile by tile in schedule order
        lsz_s = nlev_t[tsched]
        lev_off_s = torch.cumsum(lsz_s, 0) - lsz_s
        lev_off_t = torch.empty(nt, dtype=i64, device=d)
        lev_off_t[tsched] = lev_off_s
        tl = torch.repeat_interleave(torch.arange(nt, dtype=i64, device=d), nlev_t)      # tile of each table entry
        within = torch.arange(tl.numel(), dtype=i64, device=d) - (torch.cumsum(nlev_t, 0) - nlev_t)[tl]
        levtab = torch.empty(max(tl.numel(), 1), dtype=I32, device=d)
        levtab[lev_off_t[tl] + within] = lev_end[nz].to(I32)
        hdr = torch.zeros((nt, 16), dtype=i64, device=d)
        for col, v in enumerate((sizes, page0_t, nlev_t, lev_off_t, n_ext_t, ext_off_t, n_prod_t, prod_off_t, front)):
            hdr[:, col] = v
        if os.environ.get("DDILU_TSWEEP_NODEPS") == "1":    # timing experiment only (wrong results): no producer waits
            hdr[:, 6] = 0
        hdr = hdr[tsched].to(I32).contiguous().view(-1)
        nct = min(TSWEEP_MAX_THREADS, max(32, (width_max + 31) & ~31))
        stages = TSWEEP_STAGES
        if query("ddilu_tsweep_smem_bytes", k, int(up), stages, window, xe_cap, max_lev) > TSWEEP_SMEM_BUDGET:
            stages = 2
            if query("ddilu_tsweep_smem_bytes", k, int(up), stages, window, xe_cap, max_lev) > 220 * 1024:
                return None
        pages = torch.zeros(n_pages * query("ddilu_tsweep_page_bytes", k, int(up)), dtype=torch.uint8, device=d)
        gpos = (page0_t[tile] * P + pos).to(I32).contiguous()
        call("ddilu_tsweep_fill", n, fac.rp, fac.ci, fac.val, int(up), k, gpos, pos.to(I32).contiguous(), ecode,
             window, pages, bad)
        halves.append(TileSweepHalf(nt, hdr, levtab, extpos, prods, pages, zeros_i32(nt), k, window, xe_cap, max_lev,
                                    stages, nct, n_tile_levels))
    return TileSweepPlan(n, n_pages * P, vpos.to(I32).contiguous(), halves[0], halves[1], int(bad.item()), TSWEEP_SETS)


def tsweep_solve(tp: TileSweepPlan, upper: bool, b_tile: torch.Tensor, x_tile: torch.Tensor, check: bool = False):
    """x = L^-1 b (or U^-1 b) with both vectors in tile order (tp.npad entries, pads 0)."""
    if check and upper and tp.bad_row != INT_MAX:
        raise TriSolveError(f"zero or missing diagonal at row {tp.bad_row}")
    h = tp.upper if upper else tp.lower
    call("ddilu_tsweep_solve", h.n_tiles, h.tiles, h.levtab, h.extpos, h.prods, h.pages, h.flags, h.k, int(upper),
         h.window, h.xe_cap, h.max_lev, h.stages, tp.sets, h.nct, b_tile, x_tile)
    return x_tile


def tsweep_permute(tp: TileSweepPlan, src: torch.Tensor, dst: torch.Tensor, to_tile: bool):
    """Row order -> tile order (dst must be zero at the pads) or back."""
    call("ddilu_tsweep_permute", tp.n, tp.vpos, src, dst, int(to_tile))
    return dst


def enable_block_local(sched: Schedule, seg_ptr) -> bool:
    """Use the CTA-per-block sweep for this factor if its independent row blocks
    (seg_ptr, host ints) have narrow levels; returns whether it was enabled.  (Experiments build only:
    measured slower than the tiled kernel and than the TMA-fed block sweep of csrc/sweep.cu.)"""
    nb = len(seg_ptr) - 1
    if sched.n == 0 or nb < 1 or sched.n_levels == 0 or not _lib.has_experiments():
        return False
    if sched.n / (nb * sched.n_levels) > BLOCK_LOCAL_MAX_WIDTH:
        return False
    seg = torch.tensor([int(v) for v in seg_ptr], dtype=I32, device=dev())
    start, cnt = empty_i32(nb * sched.n_levels), empty_i32(nb * sched.n_levels)
    call("ddilu_blocklocal_table", sched.n, nb, seg, sched.n_levels, sched.lev, sched.level_rows, start, cnt)
    L = sched.n_levels
    sstart = (start.view(nb, L) - sched.level_ptr[:L].view(1, L) + sched.slot_ptr[:L].view(1, L)).contiguous().view(-1)
    sched.blocks = BlockLocal(nb, start, cnt, sstart)
    return True


def uses_warprow(t: DeviceCsr) -> bool:
    """Whether `sptrsv` serves this factor with the warp-per-row kernel (long rows) instead of the SELL layout."""
    return bool(USE_WARPROW and t.n_rows and t.nnz >= WARPROW_MIN_AVG_ROW * t.n_rows)


def get_sell(t: DeviceCsr, sched: Schedule, upper: bool, unit_diag: bool) -> Sell:
    if sched.sell is None:
        sched.sell = {}
    key = bool(unit_diag)
    if key not in sched.sell:
        sched.sell[key] = build_sell(t, sched, upper, unit_diag)
    return sched.sell[key]


_err_flag = None


def _err():
    global _err_flag
    if _err_flag is None or _err_flag.device != dev():
        _err_flag = torch.full((1,), INT_MAX, dtype=I32, device=dev())
    return _err_flag


def sptrsv(t: DeviceCsr, sched: Schedule, b: torch.Tensor, out: torch.Tensor, upper: bool, unit_diag: bool,
           check: bool = False):
    """out = T^-1 b with the sync-free kernel; `check` reads the error flag back
    (a host sync) and raises like the reference does (sparse.py:414-415)."""
    if t.n_rows == 0:
        return out
    if sched.blocks is not None and USE_BLOCK_LOCAL == "sell":
        bl = sched.blocks
        sell = get_sell(t, sched, upper, unit_diag)
        if check and sell.bad_row != INT_MAX:
            raise TriSolveError(f"zero or missing diagonal at row {sell.bad_row}")
        call("ddilu_sptrsv_blocklocal_sell", bl.n_blocks, sched.n_levels, bl.sstart, bl.cnt, sched.order, sell.goff,
             sell.width, sell.scol, sell.sval, sell.sdiag, b, out)
        return out
    if sched.blocks is not None and USE_BLOCK_LOCAL == "csr":
        bl = sched.blocks
        call("ddilu_sptrsv_blocklocal", bl.n_blocks, sched.n_levels, bl.start, bl.cnt, sched.level_rows, t.rp, t.ci,
             t.val, b, out, int(upper), int(unit_diag), _err())
        if check:
            bad = int(_err().item())
            if bad != INT_MAX:
                _err().fill_(INT_MAX)
                raise TriSolveError(f"zero or missing diagonal at row {bad}")
        return out
    if uses_warprow(t):
        # long rows (ILUT / ILU(k) / 27-point factors): a warp per row
        call("ddilu_sptrsv_warprow", t.n_rows, sched.n_slots, sched.order, t.rp, t.ci, t.val, b, out, int(upper),
             int(unit_diag), _err())
        if check:
            bad = int(_err().item())
            if bad != INT_MAX:
                _err().fill_(INT_MAX)
                raise TriSolveError(f"zero or missing diagonal at row {bad}")
        return out
    if USE_SELL:
        sell = get_sell(t, sched, upper, unit_diag)
        if check and sell.bad_row != INT_MAX:
            raise TriSolveError(f"zero or missing diagonal at row {sell.bad_row}")
        call("ddilu_sptrsv_sell", t.n_rows, sched.n_slots, sched.n_levels, sched.order, sell.goff, sell.width,
             sell.scol, sell.sval, sell.sdiag, sell.gwait if USE_GWAIT else None,
             sell.gfar1 if USE_GWAIT else None, sell.gfar2 if USE_GWAIT else None,
             float(sell.scol.numel() / max(1, sched.n_slots)), b, out)
        return out
    call("ddilu_sptrsv", t.n_rows, sched.n_slots, sched.order, t.rp, t.ci, t.val, b, out, int(upper),
         int(unit_diag), _err())
    if check:
        bad = int(_err().item())
        if bad != INT_MAX:
            _err().fill_(INT_MAX)
            raise TriSolveError(f"zero or missing diagonal at row {bad}")
    return out


def csr_block(a: DeviceCsr, r0: int, r1: int, c0: int, c1: int) -> DeviceCsr:
    """Rows [r0, r1) x columns [c0, c1) with columns shifted to start at 0
    (factor.py:784-803 `_csr_rows_colsplit`, sparse.py:456-471 on ranges)."""
    nr = r1 - r0
    rp = zeros_i32(nr + 1)
    call("ddilu_csr_block_count", a.rp, a.ci, r0, r1, c0, c1, rp)
    exclusive_scan_(rp, nr)
    nnz = int(rp[-1].item())
    ci, val = empty_i32(nnz), empty_f64(nnz)
    call("ddilu_csr_block_fill", a.rp, a.ci, a.val, r0, r1, c0, c1, rp, ci, val)
    return DeviceCsr(nr, c1 - c0, rp, ci, val, nnz)


def gather_rows(a: DeviceCsr, rows: torch.Tensor | None, n_sel: int, colmap: torch.Tensor, n_cols_out: int,
                dom: torch.Tensor | None = None, filt: int = 0, resort: bool = True,
                with_values: bool = True) -> DeviceCsr:
    """Row gather with column remap (sparse.py:445-453 `_gather`)."""
    rp = zeros_i32(n_sel + 1)
    call("ddilu_gather_rows_count", n_sel, rows, a.rp, a.ci, colmap, dom, filt, rp)
    exclusive_scan_(rp, n_sel)
    nnz = int(rp[-1].item())
    ci = empty_i32(nnz)
    val = empty_f64(nnz) if with_values else None
    call("ddilu_gather_rows_fill", n_sel, rows, a.rp, a.ci, a.val if with_values else None, colmap, dom, filt, rp,
         ci, val, int(resort))
    return DeviceCsr(n_sel, n_cols_out, rp, ci, val, nnz)


def index_map(n_total: int, nodes: torch.Tensor, offset: int = 0, base: torch.Tensor | None = None) -> torch.Tensor:
    """map[nodes[k]] = offset + k, -1 elsewhere (sparse.py:469-470 colmap)."""
    m = base if base is not None else torch.full((int(n_total),), -1, dtype=I32, device=dev())
    call("ddilu_build_map", nodes.numel(), nodes, int(offset), m)
    return m


def sym_adjacency(pattern: DeviceCsr, sort: bool = False) -> DeviceCsr:
    """Symmetrised pattern without the diagonal (ordering.py:72-81); neighbour
    order inside a row is unspecified unless `sort` (RCM only uses sets and degrees)."""
    n = pattern.n_rows
    rp = zeros_i32(n + 1)
    call("ddilu_sym_adj_count", n, pattern.rp, pattern.ci, rp)
    exclusive_scan_(rp, n)
    nnz = int(rp[-1].item())
    ci = empty_i32(nnz)
    cursor = empty_i32(max(n, 1))
    call("ddilu_sym_adj_fill", n, pattern.rp, pattern.ci, rp, cursor, ci)
    if sort:
        call("ddilu_sort_rows_i32", n, rp, ci)
    return DeviceCsr(n, n, rp, ci, None, nnz)


def cm_order(adj: DeviceCsr, seg_ptr: torch.Tensor | None = None) -> torch.Tensor:
    """Cuthill-McKee order (not reversed) of a symmetric adjacency.  seg_ptr (int32 device,
    optional): node ranges that are not connected to each other (one per subdomain); they are
    ordered concurrently, with the same result."""
    n = adj.n_rows
    order = empty_i32(max(n, 1))
    work = empty_i32(query("ddilu_cm_work_elems", n))
    n_seg = seg_ptr.numel() - 1 if seg_ptr is not None else 1
    if seg_ptr is not None and 1 < n_seg <= 64:
        call("ddilu_cm_order_segments", n, adj.rp, adj.ci, n_seg, seg_ptr, order, work)
    else:
        call("ddilu_cm_order", n, adj.rp, adj.ci, order, work)
    return order[:n]


def reverse_segments(cm: torch.Tensor, seg_ptr: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(cm)
    call("ddilu_reverse_segments", cm.numel(), cm, seg_ptr.numel() - 1, seg_ptr, out)
    return out


def gather_i32(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """src[idx] for int32 tensors (index plumbing; torch indexing kernel)."""
    return src[idx.long()]


# ---------------------------------------------------------------------------
# vector kernels


class Reducer:
    """Workspace of the deterministic two-stage reductions (one per stream of use)."""

    def __init__(self):
        nbytes = query("ddilu_reduce_ws_bytes")
        self.ws = torch.zeros(nbytes // 8 + 1, dtype=F64, device=dev())
        self.mgs_ws = None

    def dot(self, n, x, y, out, reverse=False):
        call("ddilu_dot_dir", int(n), x, y, out, self.ws, int(reverse))

    def axpy_dot(self, n, alpha_dev, alpha_host, v, w, u, out, reverse=False):
        call("ddilu_axpy_dot_dir", int(n), alpha_dev, float(alpha_host), v, w, u, out, self.ws, int(reverse))

    def mgs_block(self, n, ld, kp, vprev, raw_prev, hout, w, kn, vnext, out, reverse=False):
        """One pass of the blocked modified Gram-Schmidt (`ddilu_mgs_block`)."""
        if self.mgs_ws is None:
            self.mgs_ws = torch.zeros(query("ddilu_mgs_ws_bytes") // 8 + 1, dtype=F64, device=dev())
        if _lib.profile is not None:
            _lib.profile_tag = (int(n), int(kp), int(kn))
        call("ddilu_mgs_block", int(n), int(ld), int(kp), vprev, raw_prev, hout, w, int(kn), vnext, out, self.mgs_ws,
             int(reverse))
        _lib.profile_tag = None


    def mgs_small_step(self, n, ld, k, v, w, hout, vout, raw, reverse_dots=False, reverse_update=False):
        """One Arnoldi step on a short vector in one cooperative launch (`ddilu_mgs_small_step`)."""
        if self.mgs_ws is None:
            self.mgs_ws = torch.zeros(query("ddilu_mgs_ws_bytes") // 8 + 1, dtype=F64, device=dev())
        call("ddilu_mgs_small_step", int(n), int(ld), int(k), v, w, hout, vout, raw, self.mgs_ws, int(reverse_dots),
             int(reverse_update))


    def norm_scale_small(self, n, x, out, y):
        """out = <x, x>, y = x / sqrt(out) in one cooperative launch (`ddilu_norm_scale_small`)."""
        if self.mgs_ws is None:
            self.mgs_ws = torch.zeros(query("ddilu_mgs_ws_bytes") // 8 + 1, dtype=F64, device=dev())
        call("ddilu_norm_scale_small", int(n), x, out, y, self.mgs_ws, self.ws)


def axpy(n, alpha, v, w, alpha_dev=None):
    call("ddilu_axpy_dot", int(n), alpha_dev, float(alpha), v, w, None, None, None)


def scale(n, x, y, alpha_dev=None, alpha_host=1.0, take_sqrt=False, multiply=False):
    call("ddilu_scale", int(n), x, alpha_dev, float(alpha_host), int(take_sqrt), int(multiply), y)


def multi_axpy(n, k, basis, ld, coef, x, overwrite=False):
    call("ddilu_multi_axpy", int(n), int(k), basis, int(ld), coef, x, int(overwrite))


def ewise(n, a, b, op, z):
    call("ddilu_ewise", int(n), a, b, int(op), z)


def gather(n, idx, src, dst):
    call("ddilu_gather", int(n), idx, src, dst)


def scatter(n, idx, src, dst):
    call("ddilu_scatter", int(n), idx, src, dst)


def box_owner(n, dims, factors) -> torch.Tensor:
    nd = len(dims)
    arr = ctypes.c_int * nd
    owner = empty_i32(n)
    d, f = arr(*[int(v) for v in dims]), arr(*[int(v) for v in factors])
    call("ddilu_box_owner", int(n), nd, ctypes.addressof(d), ctypes.addressof(f), owner)
    return owner
