"""GPU parity: librfr (fp32, sm_100a) against the fp64 oracle on the same seeded inputs.

Every stage gets identical inputs on both sides (no oracle input ever comes from the CUDA path):
  forward   samples -> signal                         rel-L2 <= 1e-4 (north_star)
  filter    oracle / seeded signal -> |M|              rel-L2 <= 1e-4
  loss      seeded (signal, target) -> (L, G)          rel <= 1e-5
  backward  oracle / seeded G -> per-sample gradients  rel-L2 <= 1e-3 per field (north_star)
Small configs (c0, c1) are compared in full; large ones (c2-c5) run at full size in the bench's
launch configuration and are compared on sampled antenna rows / rays / queries, which the oracle
computes exactly (each output element is an independent full sum).
"""
import functools

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import AntennaSet, FreqGrid, SampleSet

pytestmark = pytest.mark.gpu

TOL_SIG = 1e-4
TOL_GRAD = 1e-3
FIELDS = ("sdf", "refl", "nx", "ny", "nz", "power")


def rfr():
    from paper_2605_29097_b200 import rfr as m
    m.load()
    return m


@functools.lru_cache(maxsize=None)
def problem(name):
    return synth.make(name)


def dev():
    return torch.device("cuda:0")


def c64(t):
    a = t.detach().cpu().numpy().astype(np.float64)
    return a[..., 0] + 1j * a[..., 1]


def f32c(z):
    z = np.asarray(z)
    return torch.as_tensor(np.stack([z.real, z.imag], -1).astype(np.float32)).to(dev())


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    n = np.linalg.norm(np.asarray(b))
    return d / n if n > 0 else d


def gpu_forward(S, A, grid, s, flags=0, ws=None):
    m = rfr()
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(A, dev())
    if ws is None:
        ws = m.workspace(S.n, A.n, grid.n_freq, 0, dev())
    out = torch.full((A.n, grid.n_freq, 2), float("nan"), device=dev())
    m.rfr_forward(DS, s, DA, grid, out, ws, flags)
    torch.cuda.synchronize()
    return out, ws


def gpu_backward(G, S, A, grid, s, flags=0):
    m = rfr()
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(S.n, A.n, grid.n_freq, 0, dev())
    out = m.Grads.empty(S.n, dev())
    for k in m.Grads.NAMES:
        getattr(out, k).fill_(float("nan"))
    m.rfr_backward(f32c(G), DS, s, DA, grid, out, ws, flags)
    torch.cuda.synchronize()
    return {k: getattr(out, k).cpu().numpy().astype(np.float64) for k in m.Grads.NAMES}, ws


def gpu_filter(sig, A, grid, qx, qy, qz):
    m = rfr()
    DA = m.DeviceAntennas.from_host(A, dev())
    q = [torch.as_tensor(np.ascontiguousarray(v, np.float32)).to(dev()) for v in (qx, qy, qz)]
    ws = m.workspace(0, A.n, grid.n_freq, len(qx), dev())
    P = torch.full((len(qx),), float("nan"), device=dev())
    M = torch.full((len(qx), 2), float("nan"), device=dev())
    m.rfr_filter(f32c(sig), DA, grid, *q, P, ws, mf=M)
    torch.cuda.synchronize()
    return P.cpu().numpy().astype(np.float64), c64(M)


def check_grads(g_gpu, g_ref, idx=None, tol=TOL_GRAD, what=""):
    for k in FIELDS:
        a = g_gpu[k] if idx is None else g_gpu[k][idx]
        b = g_ref[k]
        assert np.all(np.isfinite(a)), (what, k)
        if np.linalg.norm(b) == 0:
            assert np.linalg.norm(a) <= 1e-30 + 1e-6 * max(np.linalg.norm(g_ref[f]) for f in FIELDS)
            continue
        e = rel(a, b)
        assert e <= tol, f"{what} grad {k}: rel-L2 {e:.3e}"


# ----------------------------------------------------------------------------------- forward
@pytest.mark.parametrize("name", ["c0a", "c0b", "c1"])
def test_forward_full(name):
    p = problem(name)
    b = p.bundles[0]
    out, _ = gpu_forward(b.samples, b.antennas, p.grid, p.sharpness)
    ref = oracle.forward(b.samples, p.sharpness, b.antennas, p.grid)
    assert np.all(np.isfinite(c64(out)))
    assert rel(c64(out), ref) <= TOL_SIG


@pytest.mark.parametrize("name,rows", [("c2", 24), ("c3", 8), ("c4", 4), ("c5", 2)])
def test_forward_sampled_rows_full_size(name, rows):
    """Full-size run in the bench's launch configuration; oracle on sampled antenna rows."""
    p = problem(name)
    rng = np.random.default_rng(99)
    for k, b in enumerate(p.bundles[:2]):
        out, _ = gpu_forward(b.samples, b.antennas, p.grid, p.sharpness)
        sel = np.sort(rng.choice(b.antennas.n, rows, replace=False))
        ref = oracle.forward(b.samples, p.sharpness, b.antennas, p.grid, rows=sel)
        got = c64(out)
        assert np.all(np.isfinite(got))
        assert rel(got[sel], ref) <= TOL_SIG, (name, k)


# ----------------------------------------------------------------------------------- filter
def test_filter_full_c1():
    p = problem("c1")
    b = p.bundles[0]
    sig = oracle.forward(b.samples, p.sharpness, b.antennas, p.grid).astype(np.complex64)
    P, M = gpu_filter(sig, b.antennas, p.grid, b.samples.x, b.samples.y, b.samples.z)
    Mr, Pr = oracle.filter(sig.astype(np.complex128), b.antennas, p.grid, b.samples.x, b.samples.y,
                           b.samples.z)
    assert rel(P, Pr) <= TOL_SIG and rel(M, Mr) <= TOL_SIG


@pytest.mark.parametrize("name,nq", [("c3", 192), ("c5", 192)])
def test_filter_sampled_queries_full_size(name, nq):
    p = problem(name)
    b = p.bundles[0]
    sig = p.random_grad()                      # seeded complex signal [n_ant][n_freq]
    S = b.samples
    P, M = gpu_filter(sig, b.antennas, p.grid, S.x, S.y, S.z)
    sel = np.sort(np.random.default_rng(5).choice(S.n, nq, replace=False))
    Mr, Pr = oracle.filter(sig.astype(np.complex128), b.antennas, p.grid, S.x[sel], S.y[sel],
                           S.z[sel])
    assert rel(P[sel], Pr) <= TOL_SIG and rel(M[sel], Mr) <= TOL_SIG


# ----------------------------------------------------------------------------------- loss
def test_loss_residual():
    m = rfr()
    rng = np.random.default_rng(8)
    n = 64 * 65 + 3
    s = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    y = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    ws = m.workspace(1, 1, 1, 0, dev())
    G = torch.empty(n, 2, device=dev())
    L = torch.empty(1, device=dev())
    m.rfr_loss(f32c(s), f32c(y), G, L, ws)
    torch.cuda.synchronize()
    L_ref, G_ref = oracle.loss(s.astype(np.complex128), y.astype(np.complex128))
    assert abs(L.item() - L_ref) <= 1e-5 * L_ref
    assert rel(c64(G), G_ref) <= 1e-7


# ----------------------------------------------------------------------------------- backward
@pytest.mark.parametrize("name", ["c0a", "c0b", "c1"])
def test_backward_full(name):
    p = problem(name)
    b = p.bundles[0]
    F = oracle.forward(b.samples, p.sharpness, b.antennas, p.grid)
    y = F + np.sqrt(np.mean(np.abs(F) ** 2) / 10 ** (p.snr_db / 10)) * p.noise_unit()
    y = y + 0.3 * F if name.startswith("c0") else y     # a non-trivial residual on the tiny cases
    _, G = oracle.loss(F, y)
    G32 = G.astype(np.complex64)
    g_gpu, _ = gpu_backward(G32, b.samples, b.antennas, p.grid, p.sharpness)
    g_ref = oracle.backward(G32.astype(np.complex128), b.samples, p.sharpness, b.antennas, p.grid)
    check_grads(g_gpu, g_ref, what=name)
    assert abs(g_gpu["sharpness"][0] - g_ref["sharpness"]) <= TOL_GRAD * max(
        abs(g_ref["sharpness"]), 1e-30), (g_gpu["sharpness"], g_ref["sharpness"])


@pytest.mark.parametrize("name,n_rays", [("c2", 12), ("c3", 6), ("c4", 3)])
def test_backward_sampled_rays_full_size(name, n_rays):
    p = problem(name)
    b = p.bundles[0]
    G = p.random_grad()
    g_gpu, _ = gpu_backward(G, b.samples, b.antennas, p.grid, p.sharpness)
    S = b.samples
    # favour rays that cross a surface (non-zero alpha) so every field is exercised
    f = S.sdf.reshape(S.n_rays, S.n_per_ray)
    crossing = np.nonzero((f.min(1) < 0) & (f.max(1) > 0))[0]
    rng = np.random.default_rng(6)
    pool = crossing if len(crossing) >= n_rays else np.arange(S.n_rays)
    rays = np.sort(rng.choice(pool, n_rays, replace=False))
    idx = (rays[:, None] * S.n_per_ray + np.arange(S.n_per_ray)[None, :]).ravel()
    g_ref = oracle.backward(G.astype(np.complex128), S, p.sharpness, b.antennas, p.grid, rays=rays)
    check_grads(g_gpu, g_ref, idx=idx, what=name)


# ----------------------------------------------------------------------------------- edge cases
def _tiny(n_freq=37, n_rays=3, n_per_ray=5, n_ant=5, seed=0, bistatic=False, phi=False):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    xy = rng.uniform(-0.02, 0.02, (n_rays, 2))
    z = np.sort(rng.uniform(0.18, 0.24, (n_rays, n_per_ray)), axis=1)
    X = np.concatenate([np.repeat(xy[:, None, :], n_per_ray, 1), z[..., None]], -1).reshape(-1, 3)
    nrm = rng.normal(size=(X.shape[0], 3))
    nrm[:, 2] = -np.abs(nrm[:, 2]) - 1.0
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    S = SampleSet(f32(X[:, 0]), f32(X[:, 1]), f32(X[:, 2]),
                  f32(np.sort(rng.uniform(-4e-3, 4e-3, (n_rays, n_per_ray)), 1)[:, ::-1].ravel()),
                  f32(rng.uniform(0.3, 1, X.shape[0])), f32(nrm[:, 0]), f32(nrm[:, 1]),
                  f32(nrm[:, 2]), f32(rng.uniform(0.5, 1, X.shape[0])), n_rays, n_per_ray,
                  f32(rng.uniform(0.95, 1.0, X.shape[0])) if phi else None)
    P = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)]
    R = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)] if bistatic else None
    A = AntennaSet(f32(P[:, 0]), f32(P[:, 1]), f32(P[:, 2]),
                   *(([f32(R[:, 0]), f32(R[:, 1]), f32(R[:, 2])]) if bistatic else [None] * 3),
                   f32(rng.uniform(0.95, 1.0, n_ant)) if phi else None,
                   f32(rng.uniform(0.95, 1.0, n_ant)) if (phi and bistatic) else None)
    return S, A, synth.uniform_grid(n_freq), 500.0


@pytest.mark.parametrize("n_freq", [1, 7, 8, 15, 16, 31, 37, 64, 100, 129, 512])
@pytest.mark.parametrize("variant", ["mono", "bistatic", "phi", "bistatic_phi", "nogain"])
def test_edge_ragged_bins_and_variants(n_freq, variant):
    S, A, grid, s = _tiny(n_freq=n_freq, bistatic="bistatic" in variant, phi="phi" in variant)
    flags = 1 if variant == "nogain" else 0
    out, _ = gpu_forward(S, A, grid, s, flags)
    ref = oracle.forward(S, s, A, grid, flags=flags)
    assert rel(c64(out), ref) <= TOL_SIG, variant
    G = (np.random.default_rng(2).standard_normal((A.n, n_freq, 2)) @ [1, 1j]).astype(np.complex64)
    g_gpu, _ = gpu_backward(G, S, A, grid, s, flags)
    g_ref = oracle.backward(G.astype(np.complex128), S, s, A, grid, flags=flags)
    check_grads(g_gpu, g_ref, what=variant)
    P, M = gpu_filter(G, A, grid, S.x, S.y, S.z)
    Mr, Pr = oracle.filter(G.astype(np.complex128), A, grid, S.x, S.y, S.z)
    assert rel(M, Mr) <= TOL_SIG


def test_edge_empty_inputs():
    m = rfr()
    S, A, grid, s = _tiny(n_rays=2)
    # no antennas: forward is a no-op, backward gives zero gradients
    A0 = A.slice(0, 0)
    g, _ = gpu_backward(np.zeros((0, grid.n_freq), np.complex64), S, A0, grid, s)
    for k in FIELDS:
        assert np.all(g[k] == 0)
    assert g["sharpness"][0] == 0
    # no rays: forward writes zeros
    S0 = S.subset_rays(np.arange(0))
    out, _ = gpu_forward(S0, A, grid, s)
    assert np.all(c64(out) == 0)
    # no queries
    DA = m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(0, A.n, grid.n_freq, 0, dev())
    e = torch.empty(0, device=dev())
    m.rfr_filter(torch.zeros(A.n, grid.n_freq, 2, device=dev()), DA, grid, e, e, e, e, ws)


def test_edge_one_sample_per_ray_and_many_rays():
    S, A, grid, s = _tiny(n_rays=1000, n_per_ray=1, n_ant=3, n_freq=40)
    out, _ = gpu_forward(S, A, grid, s)
    assert np.all(c64(out) == 0)          # alpha_last = 0 on every one-sample ray (Q8)
    S, A, grid, s = _tiny(n_rays=700, n_per_ray=2, n_ant=3, n_freq=40)
    out, _ = gpu_forward(S, A, grid, s)
    assert rel(c64(out), oracle.forward(S, s, A, grid)) <= TOL_SIG


@pytest.mark.parametrize("n_per_ray", [31, 32, 33, 64, 70])
def test_edge_long_rays_blend_scans(n_per_ray):
    """K1 / K1' run one warp per ray in chunks of 32 samples (transmittance by a product scan, the
    reverse recurrence Q_l = gT_{l+1} + (1 - alpha_{l+1}) Q_{l+1} by a suffix scan, both carried
    across chunks): rays shorter than, equal to and longer than a chunk, with a ragged last chunk,
    on dense alpha (s f ~ +-2: every sample blends), against O1 / O6 (App. A.5)."""
    S, A, grid, s = _tiny(n_rays=9, n_per_ray=n_per_ray, n_ant=6, n_freq=24, seed=n_per_ray)
    out, _ = gpu_forward(S, A, grid, s)
    assert rel(c64(out), oracle.forward(S, s, A, grid)) <= TOL_SIG
    G = (np.random.default_rng(5).standard_normal((A.n, grid.n_freq, 2)) @ [1, 1j]).astype(np.complex64)
    g_gpu, _ = gpu_backward(G, S, A, grid, s)
    g_ref = oracle.backward(G.astype(np.complex128), S, s, A, grid)
    check_grads(g_gpu, g_ref, what=f"n_per_ray={n_per_ray}")


def test_domain_and_finite_flags():
    m = rfr()
    S, A, grid, s = _tiny()
    x = S.x.copy(); y = S.y.copy(); z = S.z.copy()
    x[0], y[0], z[0] = A.tx_x[0], A.tx_y[0], A.tx_z[0] + np.float32(0.0005)
    S2 = S.replace(x=x, y=y, z=z)
    out, ws = gpu_forward(S2, A, grid, s)
    assert m.rfr_poll_flags(ws) & m.RFR_FLAG_DOMAIN
    assert rel(c64(out), oracle.forward(S2, s, A, grid)) <= TOL_SIG
    refl = S.refl.copy(); refl[3] = np.nan
    _, ws = gpu_forward(S.replace(refl=refl), A, grid, s, flags=m.RFR_CHECK_FINITE)
    assert m.rfr_poll_flags(ws) & m.RFR_FLAG_NUMERIC
    _, ws = gpu_forward(S, A, grid, s, flags=m.RFR_CHECK_FINITE)
    assert m.rfr_poll_flags(ws) == 0


def test_determinism_bitwise():
    p = problem("c2")
    b = p.bundles[0]
    o1, _ = gpu_forward(b.samples, b.antennas, p.grid, p.sharpness)
    o2, _ = gpu_forward(b.samples, b.antennas, p.grid, p.sharpness)
    assert torch.equal(o1, o2)
    G = p.random_grad()
    g1, _ = gpu_backward(G, b.samples, b.antennas, p.grid, p.sharpness)
    g2, _ = gpu_backward(G, b.samples, b.antennas, p.grid, p.sharpness)
    for k in g1:
        assert np.array_equal(g1[k], g2[k])


def test_sharded_backward_and_filter_equal_unsharded():
    """T7: the multi-GPU algorithm on one GPU -- per-shard partials (antenna slices = pointer
    offsets), summed in rank order as the all-reduce would, then the finish kernel."""
    m = rfr()
    p = problem("c1")
    b = p.bundles[0]
    G = p.random_grad()
    DS, DA = m.DeviceSamples.from_host(b.samples, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    Gt = f32c(G)
    n, na = b.samples.n, b.antennas.n
    ws = m.workspace(n, na, p.grid.n_freq, n, dev())
    world = 4
    parts = []
    for r in range(world):
        lo, hi = m.shard_range(na, r, world)
        pr = torch.empty(5, n, device=dev())
        m.rfr_backward_partial(Gt[lo:hi], DS, p.sharpness, DA.slice(lo, hi), p.grid, pr, ws)
        parts.append(pr)
    total = parts[0].clone()
    for pr in parts[1:]:
        total += pr
    out = m.Grads.empty(n, dev())
    m.rfr_backward_finish(total, DS, p.sharpness, out, ws)
    torch.cuda.synchronize()
    g_ref = oracle.backward(G.astype(np.complex128), b.samples, p.sharpness, b.antennas, p.grid)
    check_grads({k: getattr(out, k).cpu().numpy().astype(np.float64) for k in m.Grads.NAMES}, g_ref)
    # filter: partial M per shard, summed, then |M|
    Ms = []
    for r in range(world):
        lo, hi = m.shard_range(na, r, world)
        M = torch.empty(n, 2, device=dev())
        m.rfr_filter_partial(Gt[lo:hi], DA.slice(lo, hi), p.grid, DS.x, DS.y, DS.z, M, ws)
        Ms.append(M)
    Mt = sum(Ms[1:], Ms[0].clone())
    P = torch.empty(n, device=dev())
    m.rfr_filter_power(Mt, P)
    torch.cuda.synchronize()
    _, Pr = oracle.filter(G.astype(np.complex128), b.antennas, p.grid, b.samples.x, b.samples.y,
                          b.samples.z)
    assert rel(P.cpu().numpy(), Pr) <= TOL_SIG


def test_reuse_blend_matches_recompute():
    m = rfr()
    p = problem("c1")
    b = p.bundles[0]
    DS, DA = m.DeviceSamples.from_host(b.samples, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    ws = m.workspace(b.samples.n, b.antennas.n, p.grid.n_freq, 0, dev())
    sig = torch.empty(b.antennas.n, p.grid.n_freq, 2, device=dev())
    m.rfr_forward(DS, p.sharpness, DA, p.grid, sig, ws)
    G = f32c(p.random_grad())
    o1, o2 = m.Grads.empty(b.samples.n, dev()), m.Grads.empty(b.samples.n, dev())
    m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o1, ws, flags=m.RFR_REUSE_BLEND)
    m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o2, ws)
    torch.cuda.synchronize()
    for k in m.Grads.NAMES:
        assert torch.equal(getattr(o1, k), getattr(o2, k))


def test_abi_argument_errors():
    m = rfr()
    S, A, grid, s = _tiny()
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(S.n, A.n, grid.n_freq, 0, dev())
    sig = torch.empty(A.n, grid.n_freq, 2, device=dev())
    with pytest.raises(m.RfrError, match="invalid argument"):
        m.rfr_forward(DS, -1.0, DA, grid, sig, ws)
    with pytest.raises(m.RfrError, match="invalid argument"):
        m.rfr_forward(DS, s, DA, FreqGrid(77e9, 0.0, grid.n_freq), sig, ws)
    with pytest.raises(m.RfrError, match="workspace too small"):
        m.rfr_forward(DS, s, DA, grid, sig, ws.truncated(64))
    with pytest.raises(m.RfrError):
        m.rfr_forward(DS, s, DA, grid, sig.cpu(), ws)     # no CPU fallback
    # more samples than the workspace was planned for
    small = m.workspace(S.n - 1, A.n, grid.n_freq, 0, dev())
    with pytest.raises(m.RfrError, match="workspace too small"):
        m.rfr_forward(DS, s, DA, grid, sig, small)


def test_workspace_regions_are_stable_across_call_types():
    """K1 records cached by rfr_forward survive a filter, a filter adjoint and a loss call on the
    same workspace (the layout depends only on the planning dims), so RFR_REUSE_BLEND afterwards
    gives bitwise the gradients of a fresh K1."""
    m = rfr()
    p = problem("c1")
    b = p.bundles[0]
    DS, DA = m.DeviceSamples.from_host(b.samples, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    n, na, nf = b.samples.n, b.antennas.n, p.grid.n_freq
    ws = m.workspace(n, na, nf, n, dev())
    sig = torch.empty(na, nf, 2, device=dev())
    m.rfr_forward(DS, p.sharpness, DA, p.grid, sig, ws)
    P, M = torch.empty(n, device=dev()), torch.empty(n, 2, device=dev())
    m.rfr_filter(sig, DA, p.grid, DS.x, DS.y, DS.z, P, ws, mf=M)
    G = torch.empty_like(sig)
    m.rfr_filter_backward(P, M, DA, p.grid, DS.x, DS.y, DS.z, G, ws, power=P, eps=1e-30)
    L = torch.empty(1, device=dev())
    m.rfr_loss(sig, sig, torch.empty_like(sig), L, ws)
    o1, o2 = m.Grads.empty(n, dev()), m.Grads.empty(n, dev())
    m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o1, ws, flags=m.RFR_REUSE_BLEND)
    m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o2, ws)
    torch.cuda.synchronize()
    for k in m.Grads.NAMES:
        assert torch.equal(getattr(o1, k), getattr(o2, k)), k


def test_comm_path_one_rank_is_identity():
    """librfr's NCCL communicator (rfr_comm_*) on one rank: rfr_backward / rfr_filter with the comm
    issue the all-reduce and return bitwise the same results as without it."""
    m = rfr()
    p = problem("c1")
    b = p.bundles[0]
    DS, DA = m.DeviceSamples.from_host(b.samples, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    n = b.samples.n
    ws = m.workspace(n, b.antennas.n, p.grid.n_freq, n, dev())
    G = f32c(p.random_grad())
    comm = m.Comm.create()
    try:
        o1, o2 = m.Grads.empty(n, dev()), m.Grads.empty(n, dev())
        m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o1, ws)
        m.rfr_backward(G, DS, p.sharpness, DA, p.grid, o2, ws, comm=comm)
        P1, P2 = torch.empty(n, device=dev()), torch.empty(n, device=dev())
        m.rfr_filter(G, DA, p.grid, DS.x, DS.y, DS.z, P1, ws)
        m.rfr_filter(G, DA, p.grid, DS.x, DS.y, DS.z, P2, ws, comm=comm)
        torch.cuda.synchronize()
        for k in m.Grads.NAMES:
            assert torch.equal(getattr(o1, k), getattr(o2, k)), k
        assert torch.equal(P1, P2)
    finally:
        comm.close()
