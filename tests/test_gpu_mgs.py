"""Blocked modified Gram-Schmidt (`ddilu_mgs_block`) against the reference's
vector-by-vector loop (krylov.py:131-136).

The oracle is the loop itself in numpy fp64 on the same vectors:
`h_i = <v_i, w>; w -= h_i v_i` for i = 0..j, then |w|^2.  The blocked kernel
recovers the same coefficients from one pass per block of 4 vectors
(h_i = <v_i, w_0> - sum_{l<i} h_l <v_i, v_l>); they differ from the loop only
by the rounding of the reductions.  Tolerances: coefficients to 1e-12 of
|w_0|, the updated w to 1e-12 of |w_0| per entry, and -- the property that
matters to GMRES -- the orthogonality of the result against the basis must not
be worse than the loop's.  The basis is deliberately NOT orthonormal in the
second case (Gram entries of order 0.1), where a classical Gram-Schmidt would
be visibly wrong and the block recurrence must still follow MGS."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mgs_loop(V, w):
    w = w.copy()
    h = np.zeros(V.shape[0] + 1)
    for i in range(V.shape[0]):
        h[i] = float(np.dot(V[i], w))
        w -= h[i] * V[i]
    h[-1] = float(np.dot(w, w))
    return h, w


@pytest.mark.parametrize("n", [1, 7, 1000, 100003, (1 << 20) + 5])
@pytest.mark.parametrize("nv", [1, 2, 3, 4, 5, 8, 11])
@pytest.mark.parametrize("orthonormal", [True, False])
def test_blocked_mgs_matches_the_loop(n, nv, orthonormal):
    import torch
    from paper_2303_08881_b200 import krylov as K
    from paper_2303_08881_b200.dist import Comm
    rng = np.random.default_rng(1000 * nv + n % 997 + int(orthonormal))
    ws = K.Arnoldi(n, max(nv, 2), Comm(), flexible=False, pad=3)
    Vh = rng.standard_normal((nv, n))
    if orthonormal and n >= nv:
        Vh = np.linalg.qr(Vh.T)[0].T.copy()
    else:
        Vh /= np.linalg.norm(Vh, axis=1)[:, None]
        if n > 1:
            Vh[1:] += 0.1 * Vh[:-1]          # neighbouring basis vectors overlap
    wh = rng.standard_normal(n) * 3.0
    ws.V.zero_()
    ws.V[:nv, :n] = torch.from_numpy(Vh).cuda()
    results = {}
    for block in (1, 4, 7, 8):
        K.MGS_BLOCK = block
        try:
            ws.w.zero_()
            ws.w[:n] = torch.from_numpy(wh).cuda()
            col = ws.mgs(nv - 1)
            results[block] = (col.copy(), ws.w[:n].cpu().numpy())
        finally:
            K.MGS_BLOCK = 4
    h_ref, w_ref = _mgs_loop(Vh, wh)
    scale = np.linalg.norm(wh)
    for block, (col, wd) in results.items():
        assert col.shape == (nv + 1,)
        assert np.max(np.abs(col[:nv] - h_ref[:nv])) <= 1e-12 * scale, block
        assert abs(col[nv] - h_ref[nv]) <= 1e-11 * scale * scale, block
        assert np.max(np.abs(wd - w_ref)) <= 1e-12 * scale, block
    # the pad / untouched tail of w stays zero
    assert float(ws.w[n:].abs().max()) == 0.0 if ws.w.numel() > n else True
    if orthonormal and n >= nv:
        # orthogonality of the result against the basis: not worse than the one-vector-at-a-time loop
        def loss(wd):
            return np.max(np.abs(Vh @ wd)) / max(np.linalg.norm(wd), 1e-300)
        for block in (4, 7, 8):
            assert loss(results[block][1]) <= max(4.0 * loss(results[1][1]), 1e-14), block


def test_blocked_mgs_column_stays_on_device():
    """With a device buffer nothing is read back and the column lands in it (inner GMRES path)."""
    import torch
    from paper_2303_08881_b200 import krylov as K
    from paper_2303_08881_b200.dist import Comm
    n, nv = 5000, 6
    rng = np.random.default_rng(3)
    ws = K.Arnoldi(n, nv, Comm(), flexible=False)
    Vh = np.linalg.qr(rng.standard_normal((n, nv)))[0].T.copy()
    wh = rng.standard_normal(n)
    ws.V.zero_()
    ws.V[:nv, :n] = torch.from_numpy(Vh).cuda()
    ws.w.zero_()
    ws.w[:n] = torch.from_numpy(wh).cuda()
    buf = torch.full((nv + 3,), -7.0, dtype=torch.float64, device="cuda")
    assert ws.mgs(nv - 1, buf) is None
    h_ref, _ = _mgs_loop(Vh, wh)
    got = buf.cpu().numpy()
    assert np.allclose(got[: nv + 1], h_ref, rtol=0, atol=1e-12 * np.linalg.norm(wh))
    assert np.all(got[nv + 1:] == -7.0)


@pytest.mark.parametrize("n", [1, 7, 1000, 100003, 390152, (1 << 20) + 5])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_small_step_is_the_three_launches_bit_for_bit(n, k):
    """`ddilu_mgs_small_step` (one cooperative launch per Arnoldi step of the inner GMRES, krylov.py:236-256)
    against `mgs` + `normalise_into`: coefficients, <w, w>, the updated w and the new basis vector identical to
    the last bit, repeatedly on the same workspace (the grid-barrier counters must come back to zero)."""
    import torch
    from paper_2303_08881_b200 import krylov as K
    from paper_2303_08881_b200.dist import Comm
    rng = np.random.default_rng(77 * k + n % 991)
    ws = K.Arnoldi(n, 5, Comm(), flexible=False, pad=3)
    assert ws.small_step_ok(k - 1)
    Vh = rng.standard_normal((k, n))
    Vh /= np.linalg.norm(Vh, axis=1)[:, None]
    if n > 1:
        Vh[1:] += 0.05 * Vh[:-1]
    ws.V.zero_()
    ws.V[:k, :n] = torch.from_numpy(Vh).cuda()
    for rep in range(3):
        wh = rng.standard_normal(n) * (rep + 1.5)
        h_a = torch.zeros(8, dtype=torch.float64, device="cuda")
        ws.w.zero_()
        ws.w[:n] = torch.from_numpy(wh).cuda()
        ws.mgs(k - 1, h_a)
        ws.normalise_into(k - 1, h_a)
        ref = (h_a.cpu().numpy().copy(), ws.w[:n].cpu().numpy().copy(), ws.V[k, :n].cpu().numpy().copy())
        h_b = torch.zeros(8, dtype=torch.float64, device="cuda")
        ws.w.zero_()
        ws.w[:n] = torch.from_numpy(wh).cuda()
        ws.V[k].zero_()
        ws.mgs_normalise_small(k - 1, h_b)
        torch.cuda.synchronize()
        got = (h_b.cpu().numpy(), ws.w[:n].cpu().numpy(), ws.V[k, :n].cpu().numpy())
        for a, b in zip(ref, got):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("n", [1, 7, 1000, 100003, 390152, (1 << 20) + 5])
def test_norm_scale_small_is_dot_plus_scale_bit_for_bit(n):
    """`ddilu_norm_scale_small` (krylov.py:226-232: beta = ||b||, v_0 = b / beta in one cooperative launch)
    against `ddilu_dot` + `ddilu_scale`, interleaved with the one-launch Arnoldi step on the same workspace."""
    import torch
    from paper_2303_08881_b200 import device as D
    from paper_2303_08881_b200 import krylov as K
    from paper_2303_08881_b200.dist import Comm
    rng = np.random.default_rng(n % 983)
    ws = K.Arnoldi(n, 3, Comm(), flexible=False, pad=1)
    for rep in range(3):
        x = torch.from_numpy(rng.standard_normal(n) * (rep + 0.5)).cuda()
        s_a = torch.zeros(1, dtype=torch.float64, device="cuda")
        y_a = torch.zeros(n, dtype=torch.float64, device="cuda")
        ws.red.dot(n, x, x, s_a)
        D.scale(n, x, y_a, alpha_dev=s_a, take_sqrt=True)
        s_b = torch.zeros(1, dtype=torch.float64, device="cuda")
        ws.red.norm_scale_small(n, x, s_b, ws.V[0])
        h = torch.zeros(8, dtype=torch.float64, device="cuda")
        ws.w[:n].copy_(x * 0.3 + 1.0)
        ws.mgs_normalise_small(0, h)                 # shares the barrier counters
        torch.cuda.synchronize()
        assert np.array_equal(s_a.cpu().numpy().view(np.uint64), s_b.cpu().numpy().view(np.uint64))
        assert np.array_equal(y_a.cpu().numpy().view(np.uint64), ws.V[0, :n].cpu().numpy().view(np.uint64))
