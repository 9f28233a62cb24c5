"""GPU parity of the matched-filter adjoint (K5, rfr_filter_backward) and the masked heatmap loss
(K7, rfr_heatmap_loss) against the oracle's O7 / O8 on identical seeded inputs (NEXT-1 / NEXT-3).

  K5  rel-L2 <= 1e-4 on the complex gradient rows (the north_star signal tolerance: the output is a
      signal-shaped sum of the same class as the forward)
  K7  loss rel <= 1e-5, dL/dP rel-L2 <= 1e-6, mask and history bit-exact
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import AntennaSet

pytestmark = pytest.mark.gpu

TOL_SIG = 1e-4


def rfr():
    from paper_2605_29097_b200 import rfr as m
    m.load()
    return m


def dev():
    return torch.device("cuda:0")


def t32(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float32)).to(dev())


def f32c(z):
    z = np.asarray(z)
    return torch.as_tensor(np.stack([z.real, z.imag], -1).astype(np.float32)).to(dev())


def c64(t):
    a = t.detach().cpu().numpy().astype(np.float64)
    return a[..., 0] + 1j * a[..., 1]


def rel(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (n if n > 0 else 1.0)


def seeded_filter_state(n_q, seed):
    """Seeded M (complex64), P = |M| (float32) and dL/dP (float32) for the adjoint."""
    rng = np.random.default_rng(seed)
    M = (rng.standard_normal(n_q) + 1j * rng.standard_normal(n_q)).astype(np.complex64)
    P = np.abs(M).astype(np.float32)
    gP = rng.standard_normal(n_q).astype(np.float32)
    return M, P, gP


def gpu_filter_backward(gP, M, P, A, grid, qx, qy, qz, eps, pass_power=True):
    m = rfr()
    DA = m.DeviceAntennas.from_host(A, dev())
    n_q = len(qx)
    ws = m.workspace(0, A.n, grid.n_freq, n_q, dev())
    out = torch.full((A.n, grid.n_freq, 2), float("nan"), device=dev())
    m.rfr_filter_backward(t32(gP), f32c(M), DA, grid, t32(qx), t32(qy), t32(qz), out, ws,
                          power=t32(P) if pass_power else None, eps=eps)
    torch.cuda.synchronize()
    return c64(out)


def test_filter_backward_full_c1():
    p = synth.make("c1")
    b = p.bundles[0]
    S = b.samples
    sig = oracle.forward(S, p.sharpness, b.antennas, p.grid).astype(np.complex64)
    M, P = oracle.filter(sig.astype(np.complex128), b.antennas, p.grid, S.x, S.y, S.z)
    M32, P32 = M.astype(np.complex64), P.astype(np.float32)
    gP = (P32 * np.random.default_rng(1).uniform(-1, 1, P.shape)).astype(np.float32)
    got = gpu_filter_backward(gP, M32, P32, b.antennas, p.grid, S.x, S.y, S.z, eps=1e-30)
    ref = oracle.filter_backward(gP, M32, P32, b.antennas, p.grid, S.x, S.y, S.z, eps=1e-30)
    assert np.all(np.isfinite(got))
    assert rel(got, ref) <= TOL_SIG


@pytest.mark.parametrize("name,rows", [("c3", 4), ("c5", 2)])
def test_filter_backward_sampled_rows_full_size(name, rows):
    """Queries = every sample of the config (the bench's filter queries); oracle on sampled rows."""
    p = synth.make(name)
    b = p.bundles[0]
    S = b.samples
    M, P, gP = seeded_filter_state(S.n, 11)
    got = gpu_filter_backward(gP, M, P, b.antennas, p.grid, S.x, S.y, S.z, eps=1e-20)
    sel = np.sort(np.random.default_rng(12).choice(b.antennas.n, rows, replace=False))
    ref = oracle.filter_backward(gP, M, P, b.antennas, p.grid, S.x, S.y, S.z, eps=1e-20, rows=sel)
    assert np.all(np.isfinite(got))
    assert rel(got[sel], ref) <= TOL_SIG


def _tiny(n_freq, n_ant=5, n_q=23, seed=0, bistatic=False):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    P = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)]
    R = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)] if bistatic else None
    A = AntennaSet(f32(P[:, 0]), f32(P[:, 1]), f32(P[:, 2]),
                   *([f32(R[:, 0]), f32(R[:, 1]), f32(R[:, 2])] if bistatic else [None] * 3))
    q = [f32(rng.uniform(-0.02, 0.02, n_q)), f32(rng.uniform(-0.02, 0.02, n_q)),
         f32(rng.uniform(0.18, 0.24, n_q))]
    return A, q, synth.uniform_grid(n_freq)


@pytest.mark.parametrize("n_freq", [1, 7, 16, 37, 100, 256, 512])
@pytest.mark.parametrize("bistatic", [False, True])
def test_filter_backward_ragged_and_bistatic(n_freq, bistatic):
    A, q, grid = _tiny(n_freq, bistatic=bistatic)
    M, P, gP = seeded_filter_state(len(q[0]), n_freq)
    for pass_power in (True, False):
        got = gpu_filter_backward(gP, M, P, A, grid, *q, eps=1e-20, pass_power=pass_power)
        ref = oracle.filter_backward(gP, M, P, A, grid, *q, eps=1e-20)
        assert rel(got, ref) <= TOL_SIG, (n_freq, bistatic, pass_power)


@pytest.mark.parametrize("bistatic", [False, True])
def test_filter_backward_tiled_path(bistatic):
    """Tiled K5: several chunks per tile (3001 queries), a ragged antenna block (131 = 128 + 3);
    the call must have taken the tiled path -- the r2 engine (DESIGN 5e) when monostatic, the r1
    tiled Chebyshev kernels (DESIGN 6b) when bistatic."""
    m = rfr()
    A, q, grid = _tiny(128, n_ant=131, n_q=3001, seed=5, bistatic=bistatic)
    M, P, gP = seeded_filter_state(len(q[0]), 21)
    DA = m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(0, A.n, grid.n_freq, len(q[0]), dev())
    out = torch.full((A.n, grid.n_freq, 2), float("nan"), device=dev())
    m.rfr_filter_backward(t32(gP), f32c(M), DA, grid, *[t32(v) for v in q], out, ws,
                          power=t32(P), eps=1e-20)
    torch.cuda.synchronize()
    if bistatic:
        st = m.cheb_state(ws)
        assert st["sel"] == 1 and st["P_tiled_filter"] > 0, st
    else:
        st = m.rfr_plan_state(ws)
        assert st["applied"] == 1 and st["P"] > 0 and st["n_points"] == len(q[0]), st
    ref = oracle.filter_backward(gP, M, P, A, grid, *q, eps=1e-20)
    assert rel(c64(out), ref) <= TOL_SIG


def test_filter_backward_eps_guard_and_empty():
    m = rfr()
    A, q, grid = _tiny(16)
    n_q = len(q[0])
    M = np.zeros(n_q, np.complex64)
    P = np.zeros(n_q, np.float32)
    got = gpu_filter_backward(np.ones(n_q, np.float32), M, P, A, grid, *q, eps=1e-12)
    assert np.all(got == 0)
    # no queries: the gradient is zero
    DA = m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(0, A.n, grid.n_freq, 0, dev())
    out = torch.full((A.n, grid.n_freq, 2), float("nan"), device=dev())
    e = torch.empty(0, device=dev())
    m.rfr_filter_backward(e, torch.empty(0, 2, device=dev()), DA, grid, e, e, e, out, ws)
    torch.cuda.synchronize()
    assert torch.all(out == 0)


def test_filter_backward_is_adjoint_of_gpu_filter_through_oracle_pin():
    """End-to-end pairing on the GPU: Re<F(s), c> == Re<s, F^H(c)> with F = rfr_filter (K4) and
    F^H = rfr_filter_backward (K5), both in fp32, to 1e-4 relative."""
    m = rfr()
    A, q, grid = _tiny(64, n_ant=16, n_q=200, seed=4)
    rng = np.random.default_rng(5)
    s = (rng.standard_normal((A.n, 64)) + 1j * rng.standard_normal((A.n, 64))).astype(np.complex64)
    c = (rng.standard_normal(200) + 1j * rng.standard_normal(200)).astype(np.complex64)
    DA = m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(0, A.n, 64, 200, dev())
    Pq = torch.empty(200, device=dev())
    Mq = torch.empty(200, 2, device=dev())
    qt = [t32(v) for v in q]
    m.rfr_filter(f32c(s), DA, grid, *qt, Pq, ws, mf=Mq)
    FH = torch.empty(A.n, 64, 2, device=dev())
    m.rfr_filter_backward(t32(np.abs(c)), f32c(c), DA, grid, *qt, FH, ws, eps=0.0)
    torch.cuda.synchronize()
    lhs = np.real(np.vdot(c.astype(np.complex128), c64(Mq)))
    rhs = np.real(np.vdot(c64(FH), s.astype(np.complex128)))
    assert abs(lhs - rhs) <= 1e-4 * np.linalg.norm(c) * np.linalg.norm(c64(Mq))


# ------------------------------------------------------------------------------------ K7
def _heat_inputs(n, n_cells, seed):
    rng = np.random.default_rng(seed)
    P = rng.uniform(0, 1, n).astype(np.float32)
    Pgt = rng.uniform(0, 1, n).astype(np.float32)
    cell = rng.integers(0, n_cells, n).astype(np.int32)
    H = rng.uniform(0, 1, n_cells).astype(np.float32)
    return P, Pgt, cell, H


@pytest.mark.parametrize("n", [1, 1000, 262147])
def test_heatmap_loss_masked(n):
    m = rfr()
    P, Pgt, cell, H = _heat_inputs(n, 97, n)
    thr, ratio = 0.4, 0.3
    # keep the decision away from fp32/fp64 rounding of ratio * H (the two sides agree exactly)
    marg = np.abs(P - np.float32(ratio) * H[cell]) > 1e-5
    P = np.where(marg, P, P + 2e-5).astype(np.float32)
    ws = m.workspace(1, 1, 1, 0, dev())
    gP = torch.empty(n, device=dev())
    L = torch.empty(1, device=dev())
    mk = torch.empty(n, dtype=torch.uint8, device=dev())
    Ht = t32(H)
    m.rfr_heatmap_loss(t32(P), t32(Pgt), gP, L, ws, cell=torch.as_tensor(cell).to(dev()),
                       history=Ht, thr_hi=thr, ratio=ratio, mask=mk)
    torch.cuda.synchronize()
    L_ref, g_ref, mask_ref, H_ref = oracle.heatmap_loss(P, Pgt, cell, H, thr, ratio)
    assert np.array_equal(mk.cpu().numpy().astype(bool), mask_ref)
    assert abs(L.item() - L_ref) <= 1e-5 * max(L_ref, 1e-30)
    assert rel(gP.cpu().numpy(), g_ref) <= 1e-6
    assert np.array_equal(Ht.cpu().numpy(), H_ref.astype(np.float32))


def test_heatmap_loss_unmasked():
    m = rfr()
    P, Pgt, _, _ = _heat_inputs(5000, 1, 3)
    ws = m.workspace(1, 1, 1, 0, dev())
    gP = torch.empty(5000, device=dev())
    L = torch.empty(1, device=dev())
    m.rfr_heatmap_loss(t32(P), t32(Pgt), gP, L, ws)
    torch.cuda.synchronize()
    L_ref, g_ref, _, _ = oracle.heatmap_loss(P, Pgt)
    assert abs(L.item() - L_ref) <= 1e-5 * L_ref
    assert rel(gP.cpu().numpy(), g_ref) <= 1e-6
