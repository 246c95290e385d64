"""Restarted GMRES / FGMRES and the fixed-iteration inner GMRES, device
resident (the reference's `ddilu.krylov`, krylov.py:27).

The control flow is the reference's, line for line (krylov.py:96-179, 213-268):
modified Gram-Schmidt Arnoldi, Givens rotations with `math.hypot`, the
estimate-based in-cycle break, convergence declared only on the recomputed true
residual.  What changed is where the work runs:

* vectors (V, Z, w, x, r) never leave HBM,
* the MGS loop runs in blocks of 4 basis vectors (`ddilu_mgs_block`: one pass
  subtracts the previous block and accumulates the next block's dots and Gram
  entries, from which the SAME coefficients h_i = <v_i, w_i> follow; 20n bytes
  per basis vector instead of the reference's 40n), the coefficients stay on
  the device between the passes,
* the host sees one small copy per Arnoldi step (the new Hessenberg column),
  which it needs for the rotation / stopping logic,
* with several ranks every block of dots is followed by one small allreduce.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import device as D
from .dist import Comm, get_comm
from .sparse import CsrMatrix

__all__ = ["KrylovConfig", "SolveReport", "gmres", "fgmres", "fixed_gmres", "release_workspace"]


@dataclass(frozen=True)
class KrylovConfig:
    """krylov.py:32-52."""

    restart: int = 50
    rtol: float = 1e-8
    max_iters: int = 20000
    happy_tol: float = 1e-14
    record_history: bool = True

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart length must be positive")
        if not self.rtol > 0:
            raise ValueError("rtol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")


@dataclass
class SolveReport:
    """krylov.py:55-71."""

    iterations: int
    converged: bool
    residual_history: np.ndarray
    final_relres: float
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0


def _back_substitute(h: np.ndarray, g: np.ndarray, k: int) -> np.ndarray:
    """krylov.py:86-93."""
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        s = g[i]
        for j in range(i + 1, k):
            s -= h[i, j] * y[j]
        y[i] = s / h[i, i] if h[i, i] != 0.0 else 0.0
    return y


def _givens(h, cs, sn, g, j, hnext):
    """krylov.py:137-149: apply the previous rotations to column j, form the new one."""
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


class Arnoldi:
    """Device workspace of one (F)GMRES instance: bases, w, Hessenberg column."""

    def __init__(self, n: int, m: int, comm: Comm, flexible: bool, pad: int = 0):
        self.n, self.m, self.comm = int(n), int(m), comm
        self.ld = (self.n + int(pad) + 1) & ~1  # even leading dimension keeps rows 16-byte aligned
        self.V = torch.empty((m + 1, self.ld), dtype=D.F64, device=D.dev())
        self.Z = torch.empty((m, self.ld), dtype=D.F64, device=D.dev()) if flexible else None
        self.w = torch.empty(self.ld, dtype=D.F64, device=D.dev())
        self.hdev = torch.zeros(m + 2, dtype=D.F64, device=D.dev())
        self.coef = torch.zeros(m + 1, dtype=D.F64, device=D.dev())
        self.red = D.Reducer()
        self.raw = None

    def norm2(self, x) -> float:
        """sqrt(<x, x>) summed over ranks (sparse.py:526-528)."""
        s = self.hdev[self.m + 1:self.m + 2]
        self.red.dot(self.n, x, x, s)
        self.comm.allreduce_sum_(s)
        return math.sqrt(float(s.item()))

    def mgs(self, j: int, h: torch.Tensor | None = None):
        """Orthogonalise self.w against V[0..j] (krylov.py:131-136).  Returns the
        host copy of [h_0j .. h_jj, |w|^2]; with a device buffer `h` (>= j + 2 entries) the column
        stays on the device and nothing is read back (no host synchronisation)."""
        n, V, w, red, comm = self.n, self.V, self.w, self.red, self.comm
        to_host = h is None
        if to_host:
            h = self.hdev
        if MGS_BLOCK > 1:
            self._mgs_blocked(j, h)
            return h[: j + 2].cpu().numpy() if to_host else None
        # consecutive passes walk the vectors in alternating directions (the SpMV that produced w ran forward):
        # a pass starts with the tail of w and of the shared basis vector that the previous pass left in L2
        # (126 MB against 3 x 134 MB per pass at 256^3)
        alt = ALTERNATE_MGS
        red.dot(n, V[0], w, h[0:1], reverse=alt)
        comm.allreduce_sum_(h[0:1])
        for i in range(j):
            red.axpy_dot(n, h[i:i + 1], -1.0, V[i], w, V[i + 1], h[i + 1:i + 2], reverse=alt and (i & 1) == 1)
            comm.allreduce_sum_(h[i + 1:i + 2])
        red.axpy_dot(n, h[j:j + 1], -1.0, V[j], w, w, h[j + 1:j + 2], reverse=alt and (j & 1) == 1)
        comm.allreduce_sum_(h[j + 1:j + 2])
        return h[: j + 2].cpu().numpy() if to_host else None

    def _mgs_blocked(self, j: int, h: torch.Tensor):
        """The same orthogonalisation in blocks of MGS_BLOCK basis vectors (`ddilu_mgs_block`): pass b subtracts
        block b-1 from w in the MGS order and accumulates <v_i, w> and the block's Gram entries <v_i, v_l> of
        block b, from which the consuming pass recovers the MGS coefficients h_i = <v_i, w_i>.  Moves
        (16/k + 16) n bytes per basis vector instead of 32 n and needs one allreduce per block."""
        n, V, w, red, comm = self.n, self.V, self.w, self.red, self.comm
        kmax = min(MGS_BLOCK, D.query("ddilu_mgs_max_block"))
        nv = j + 1
        npass = (nv + kmax - 1) // kmax
        if self.raw is None or self.raw.shape[0] < npass:
            self.raw = torch.zeros(((self.m + kmax) // kmax + 1, 40), dtype=D.F64, device=D.dev())
        raw = self.raw
        alt = ALTERNATE_MGS
        ps, pk = 0, 0
        for b in range(npass):
            s = b * kmax
            k = min(kmax, nv - s)
            red.mgs_block(n, self.ld, pk, V[ps] if pk else None, raw[b - 1] if pk else None, h[ps:ps + pk] if pk else None,
                          w, k, V[s], raw[b], reverse=alt and (b & 1) == 0)
            comm.allreduce_sum_(raw[b, : k + k * (k - 1) // 2])
            ps, pk = s, k
        red.mgs_block(n, self.ld, pk, V[ps], raw[npass - 1], h[ps:ps + pk], w, 0, None, h[j + 1:j + 2],
                      reverse=alt and (npass & 1) == 0)
        comm.allreduce_sum_(h[j + 1:j + 2])

    def small_step_ok(self, j: int) -> bool:
        """One-launch Arnoldi step (`ddilu_mgs_small_step`): single rank, all of V[0..j] in one block of the
        blocked Gram-Schmidt, a vector short enough to stay in L2 between the phases."""
        return (SMALL_STEP and MGS_BLOCK > 1 and not self.comm.active and 0 < self.n <= SMALL_STEP_MAX_N
                and j + 1 <= min(MGS_BLOCK, D.query("ddilu_mgs_small_max"), D.query("ddilu_mgs_max_block")))

    def mgs_normalise_small(self, j: int, h: torch.Tensor):
        """`mgs(j, h)` + `normalise_into(j, h)` in one launch: same passes, same directions, same bits."""
        if self.raw is None:
            self.raw = torch.zeros(((self.m + MGS_BLOCK) // MGS_BLOCK + 1, 40), dtype=D.F64, device=D.dev())
        alt = ALTERNATE_MGS
        self.red.mgs_small_step(self.n, self.ld, j + 1, self.V, self.w, h, self.V[j + 1], self.raw[0],
                                reverse_dots=alt, reverse_update=False)

    def normalise_into(self, j: int, h: torch.Tensor | None = None):
        """V[j+1] = w / hnext with hnext = sqrt(h[j+1]) read on the device (krylov.py:156)."""
        h = self.hdev if h is None else h
        D.scale(self.n, self.w, self.V[j + 1], alpha_dev=h[j + 1:j + 2], take_sqrt=True)

    def combine(self, basis, y: np.ndarray, x, overwrite: bool):
        """x (+)= sum_i y_i basis[i] (krylov.py:160-166, 264-267)."""
        k = len(y)
        self.coef[:k].copy_(torch.from_numpy(np.ascontiguousarray(y)))
        D.multi_axpy(self.n, k, basis, self.ld, self.coef, x, overwrite)


DevOp = Callable[[torch.Tensor, torch.Tensor], None]  # op(x, out): out[:n] = Op x[:n]

KEEP_WORKSPACE = os.environ.get("DDILU_KEEP_WORKSPACE", "0") == "1"   # measured: holding the 13.5 GB across steps makes the NEXT setup 0.23 s slower (its temporaries no longer fit the allocator's cached blocks); opt-in for repeated solves with one preconditioner
_ws_cache: dict = {}


def _workspace(n: int, m: int, comm: Comm, flexible: bool, pad: int) -> Arnoldi:
    """The Arnoldi workspace of a solve (bases V, Z: (2 m + 1) n doubles, 13.5 GB at 256^3).  The most recent one is
    kept and reused by the next solve of the same shape when KEEP_WORKSPACE is on (off by default, see above).
    `release_workspace()` frees it."""
    key = (int(n), int(m), bool(flexible), int(pad), comm.rank, comm.size, str(D.dev()))
    ws = _ws_cache.get("ws") if KEEP_WORKSPACE and _ws_cache.get("key") == key else None
    if ws is None:
        _ws_cache.clear()
        ws = Arnoldi(n, m, comm, flexible, pad)
        if KEEP_WORKSPACE:
            _ws_cache.update(key=key, ws=ws)
    ws.comm = comm
    return ws


def release_workspace() -> None:
    """Free the cached Arnoldi workspace of the last solve."""
    _ws_cache.clear()

DEVICE_COEF = os.environ.get("DDILU_DEVICE_COEF", "1") == "1"   # inner GMRES: rotations / back substitution on the device (no host read per application)
L2_PERSIST_W = False  # pin the Arnoldi work vector in the persisting part of L2 during a solve (measured: slower)
MGS_BLOCK = int(os.environ.get("DDILU_MGS_BLOCK", "4"))  # basis vectors per pass of the blocked Gram-Schmidt (1: the vector-by-vector launches)
SMALL_STEP = os.environ.get("DDILU_SMALL_STEP", "1") == "1"   # inner GMRES: dots + update + normalisation of a step in one cooperative launch
SMALL_STEP_MAX_N = 4 << 20                                     # ... for vectors that stay in L2 between the phases
ALTERNATE_MGS = True  # consecutive MGS steps traverse the vectors in alternating directions (L2 reuse)


def restarted_device(n: int, apply_a: DevOp, apply_m: DevOp | None, b: torch.Tensor, x0: torch.Tensor | None,
                     cfg: KrylovConfig, flexible: bool, comm: Comm, pad: int = 0, guard=None):
    """krylov.py:96-179 on device vectors of local length n.  Vectors handed to
    `apply_a` have `pad` extra trailing entries (halo landing zone).  Returns
    (x[:n] device tensor, SolveReport).  guard: the preconditioner object when its applications run without
    host reads (device-side inner-solve arithmetic, CUDA-graph replay); guard.cycle_failed() is asked once per
    restart cycle whether an application hit one of the reference's early exits, and the cycle is then redone
    on the host-read path (guard.set_safe)."""
    m = cfg.restart
    ws = _workspace(n, m, comm, flexible, pad)
    V, Z, w = ws.V, ws.Z, ws.w
    if L2_PERSIST_W and n * 8 > (32 << 20):
        # w is read and written by every MGS step, the basis streams through once: keep w in persisting L2
        D.call("ddilu_l2_persist_window", w, w.numel() * 8)
    bnorm = ws.norm2(b)
    scale = bnorm if bnorm > 0.0 else 1.0
    x = torch.zeros(ws.ld, dtype=D.F64, device=D.dev())
    r = torch.empty(ws.ld, dtype=D.F64, device=D.dev())
    if x0 is None:
        r[:n].copy_(b[:n])
    else:
        x[:n].copy_(x0[:n])
        apply_a(x, w)
        D.ewise(n, b, w, 1, r)
    u = torch.empty(ws.ld, dtype=D.F64, device=D.dev()) if not flexible else None
    beta = ws.norm2(r)
    history = [beta / scale]
    final_rel = beta / scale
    converged = final_rel <= cfg.rtol
    its = 0
    h = np.zeros((m + 1, m))
    cs, sn, g = np.empty(m), np.empty(m), np.empty(m + 1)
    while not converged and its < cfg.max_iters:
        D.scale(n, r, V[0], alpha_host=beta)
        g[:] = 0.0
        g[0] = beta
        k = 0
        for j in range(m):
            if apply_m is not None:
                z = Z[j] if flexible else u
                apply_m(V[j], z)
            else:
                z = V[j]
                if flexible:
                    Z[j][:n].copy_(z[:n])
            apply_a(z, w)
            col = ws.mgs(j)
            h[: j + 1, j] = col[: j + 1]
            hnext = math.sqrt(col[j + 1]) if col[j + 1] > 0.0 else 0.0
            h[j + 1, j] = hnext
            _givens(h, cs, sn, g, j, hnext)
            its += 1
            k = j + 1
            est = abs(g[j + 1]) / scale
            history.append(est)
            if hnext < cfg.happy_tol:
                break
            ws.normalise_into(j)
            if est <= cfg.rtol or its >= cfg.max_iters:
                break
        if guard is not None and guard.cycle_failed():
            # an inner solve of this cycle left the reference's loop early (zero right-hand side, happy
            # breakdown): x and r are untouched so far -- redo the cycle with a host read per application
            guard.set_safe(True)
            its -= k
            del history[len(history) - k:]
            continue
        y = _back_substitute(h, g, k)
        if flexible:
            ws.combine(Z, y, x, overwrite=False)
        else:
            ws.combine(V, y, w, overwrite=True)
            if apply_m is not None:
                apply_m(w, u)
                if guard is not None and guard.cycle_failed():
                    guard.set_safe(True)
                    apply_m(w, u)
                D.axpy(n, 1.0, u, x)
            else:
                D.axpy(n, 1.0, w, x)
        apply_a(x, w)
        D.ewise(n, b, w, 1, r)
        beta = ws.norm2(r)
        final_rel = beta / scale
        if final_rel <= cfg.rtol:
            converged = True
    if L2_PERSIST_W and n * 8 > (32 << 20):
        D.call("ddilu_l2_persist_window", None, 0)
    report = SolveReport(iterations=its, converged=converged,
                         residual_history=np.array(history if cfg.record_history else []),
                         final_relres=final_rel)
    return x[:n], report


class InnerGmres:
    """krylov.py:213-268 `fixed_gmres` with a persistent device workspace (the
    two-level preconditioners call it once per outer iteration)."""

    def __init__(self, n: int, iters: int, comm: Comm, pad: int = 0, happy_tol: float = 1e-14,
                 n_global: int | None = None):
        self.n, self.iters, self.comm, self.happy_tol = int(n), int(iters), comm, happy_tol
        # the step count follows the GLOBAL system size (krylov.py:232: m = min(iters, n)); a rank with few
        # (or no) interface unknowns still runs every step, so its workspace is sized from the global count
        ng = self.n if n_global is None else int(n_global)
        self.m = max(1, min(self.iters, max(ng, 1)))
        self.ws = Arnoldi(self.n, self.m, comm, flexible=False, pad=pad)
        self.z = torch.empty(self.ws.ld, dtype=D.F64, device=D.dev())
        self.u = torch.empty(self.ws.ld, dtype=D.F64, device=D.dev())
        self.hcols = None   # device Hessenberg columns of one solve: row j = [h_0j .. h_jj, |w|^2], last row = <b, b>
        self.flag = D.zeros_i32(1)   # sticky: a device-side solve met an early exit of the reference
        self.safe = False            # True: host read per solve (the reference's control flow, step by step if needed)

    def solve(self, apply_a: DevOp, b: torch.Tensor, out: torch.Tensor, apply_m: DevOp | None = None,
              n_global: int | None = None):
        """The m Arnoldi steps are queued WITHOUT reading anything back: the Hessenberg columns stay in
        a device buffer, the basis is normalised with device scalars, and ONE copy at the end feeds the
        reference's host arithmetic (Givens rotations, back substitution: identical operations, identical
        bits).  The reference's early exits (beta == 0, happy breakdown: krylov.py:228-231, 252-253) are
        detected in that copy; the breakdown case is then redone step by step, exactly as the reference
        would have run it."""
        n, ws = self.n, self.ws
        ng = n if n_global is None else n_global
        if ng == 0 or self.iters <= 0:
            out[:n].zero_()
            return out
        m = min(self.iters, ng, self.m)
        if self.hcols is None:
            self.hcols = torch.zeros((self.m + 1, self.m + 2), dtype=D.F64, device=D.dev())
        H = self.hcols
        V, w = ws.V, ws.w
        bb = H[self.m, 0:1]                      # <b, b>
        if ws.small_step_ok(0):
            ws.red.norm_scale_small(n, b, bb, V[0])       # the two launches below in one
        else:
            ws.red.dot(n, b, b, bb)
            self.comm.allreduce_sum_(bb)
            D.scale(n, b, V[0], alpha_dev=bb, take_sqrt=True)
        for j in range(m):
            if apply_m is not None:
                apply_m(V[j], self.z)
                apply_a(self.z, w)
            else:
                apply_a(V[j], w)
            if ws.small_step_ok(j):
                ws.mgs_normalise_small(j, H[j])
            else:
                ws.mgs(j, H[j])
                ws.normalise_into(j, H[j])
        if DEVICE_COEF and not self.safe and m <= D.query("ddilu_gmres_small_max"):
            # rotations + back substitution on the device: nothing is read back; an early exit of the
            # reference raises self.flag and the caller redoes the application with safe = True
            D.call("ddilu_gmres_small_solve", m, H, H.stride(0), bb, float(self.happy_tol), ws.coef, self.flag)
            if apply_m is not None:
                D.multi_axpy(n, m, V, ws.ld, ws.coef, self.u, True)
                apply_m(self.u, out)
            else:
                D.multi_axpy(n, m, V, ws.ld, ws.coef, out, True)
            return out
        host = H.cpu().numpy()                   # the one synchronisation of the inner solve
        beta = math.sqrt(float(host[self.m, 0]))
        if beta == 0.0:
            out[:n].zero_()
            return out
        h = np.zeros((m + 1, m))
        cs, sn, g = np.empty(m), np.empty(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        for j in range(m):
            col = host[j]
            h[: j + 1, j] = col[: j + 1]
            hnext = math.sqrt(col[j + 1]) if col[j + 1] > 0.0 else 0.0
            h[j + 1, j] = hnext
            _givens(h, cs, sn, g, j, hnext)
            k = j + 1
            if hnext < self.happy_tol:
                if j + 1 < m:   # the queued steps after a breakdown divided by ~0: redo it the reference's way
                    return self._solve_stepwise(apply_a, b, out, apply_m, m)
                break
        y = _back_substitute(h, g, k)
        if apply_m is not None:
            ws.combine(V, y, self.u, overwrite=True)
            apply_m(self.u, out)
        else:
            ws.combine(V, y, out, overwrite=True)
        return out

    def _solve_stepwise(self, apply_a: DevOp, b: torch.Tensor, out: torch.Tensor, apply_m: DevOp | None, m: int):
        """krylov.py:213-268 with a host read per Arnoldi step (used after a happy breakdown)."""
        n, ws = self.n, self.ws
        beta = ws.norm2(b)
        if beta == 0.0:
            out[:n].zero_()
            return out
        V, w = ws.V, ws.w
        h = np.zeros((m + 1, m))
        cs, sn, g = np.empty(m), np.empty(m), np.zeros(m + 1)
        D.scale(n, b, V[0], alpha_host=beta)
        g[0] = beta
        k = 0
        for j in range(m):
            if apply_m is not None:
                apply_m(V[j], self.z)
                apply_a(self.z, w)
            else:
                apply_a(V[j], w)
            col = ws.mgs(j)
            h[: j + 1, j] = col[: j + 1]
            hnext = math.sqrt(col[j + 1]) if col[j + 1] > 0.0 else 0.0
            h[j + 1, j] = hnext
            _givens(h, cs, sn, g, j, hnext)
            k = j + 1
            if hnext < self.happy_tol:
                break
            ws.normalise_into(j)
        y = _back_substitute(h, g, k)
        if apply_m is not None:
            ws.combine(V, y, self.u, overwrite=True)
            apply_m(self.u, out)
        else:
            ws.combine(V, y, out, overwrite=True)
        return out


# ---------------------------------------------------------------------------
# public entry points


def _device_operator(op, n: int) -> DevOp:
    """CsrMatrix -> device SpMV; any other callable is the caller's own host
    operator (numpy in, numpy out) and is invoked as such."""
    if isinstance(op, CsrMatrix):
        ad = op.device()

        def matvec(x, out):
            D.spmv(ad, x, out)
        return matvec
    dev_apply = getattr(op, "_device_apply", None)
    if dev_apply is None and hasattr(op, "__self__"):
        dev_apply = getattr(op.__self__, "_device_apply_for", lambda f: None)(op)
    if dev_apply is not None:
        return dev_apply

    def host_op(x, out):
        res = np.asarray(op(x[:n].cpu().numpy()), dtype=np.float64)
        out[:n].copy_(torch.from_numpy(res))
    return host_op


def _solve(a, b, m, x0, cfg: KrylovConfig | None, flexible: bool):
    cfg = cfg or KrylovConfig()
    on_device = isinstance(b, torch.Tensor)   # device-resident fast path: CUDA tensor in -> CUDA tensor out
    if not on_device:
        b = np.asarray(b, dtype=np.float64)
    t0 = time.perf_counter()
    owner = getattr(m, "__self__", None)
    fast = getattr(owner, "_solve_local", None)
    if fast is not None and getattr(m, "__name__", "") == "apply" and owner.accepts_operator(a):
        x, report = fast(b, x0, cfg, flexible)  # permuted, rank-local, halo-exchanging path
    else:
        n = len(b)
        apply_a = _device_operator(a, n)
        apply_m = _device_operator(m, n) if m is not None else None
        bd = b if on_device else D.to_device_f64(b)
        x0d = None
        if x0 is not None:
            x0d = x0 if isinstance(x0, torch.Tensor) else D.to_device_f64(np.asarray(x0, dtype=np.float64))
        xd, report = restarted_device(n, apply_a, apply_m, bd, x0d, cfg, flexible, Comm())
        x = xd.clone() if on_device else xd.cpu().numpy()
    torch.cuda.synchronize()
    report.solve_seconds = time.perf_counter() - t0
    return x, report


def gmres(a, b, m=None, x0=None, cfg: KrylovConfig | None = None):
    """krylov.py:182-197."""
    return _solve(a, b, m, x0, cfg, flexible=False)


def fgmres(a, b, m=None, x0=None, cfg: KrylovConfig | None = None):
    """krylov.py:200-210."""
    return _solve(a, b, m, x0, cfg, flexible=True)


def fixed_gmres(apply_a, b, iters: int, apply_m=None, happy_tol: float = 1e-14) -> np.ndarray:
    """krylov.py:213-268 for host operators (numpy in / numpy out)."""
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    if n == 0 or iters <= 0:
        return np.zeros(n)
    inner = InnerGmres(n, iters, Comm(), happy_tol=happy_tol)
    out = D.empty_f64(n)
    op_a = _device_operator(apply_a, n)
    op_m = _device_operator(apply_m, n) if apply_m is not None else None
    bd = D.to_device_f64(b)
    inner.solve(op_a, bd, out, op_m)
    if not inner.safe and int(inner.flag.item()):
        # the device-side arithmetic met one of the reference's early exits (zero right-hand side, happy
        # breakdown): redo the solve with the reference's own control flow
        inner.flag.zero_()
        inner.safe = True
        inner.solve(op_a, bd, out, op_m)
    return out.cpu().numpy()
