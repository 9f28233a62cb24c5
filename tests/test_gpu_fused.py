"""GPU parity of rfr_backward_filter (K3 + K4 in one tensor-core sweep, queries = samples) against
the fp64 oracle, plus its agreement with the separate rfr_backward / rfr_filter calls.

Same inputs on both sides; tolerances as the separate calls (north_star): signals / M rel-L2 <= 1e-4,
gradients rel-L2 <= 1e-3 per field.  Bin counts 128 / 256 / 512 take the tensor-core kernel; a
ragged count (37) takes the SIMT fallback (two sweeps)."""
import functools

import numpy as np
import pytest
import torch

import oracle
import synth

from test_gpu_parity import (FIELDS, TOL_GRAD, TOL_SIG, _tiny, c64, check_grads, dev, f32c, rel,
                             rfr)

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def problem(name):
    return synth.make(name)


def gpu_fused(G, sig, S, A, grid, s, flags=0, n_q=None):
    m = rfr()
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(S.n, A.n, grid.n_freq, S.n if n_q is None else n_q, dev())
    out = m.Grads.empty(S.n, dev())
    for k in m.Grads.NAMES:
        getattr(out, k).fill_(float("nan"))
    P = torch.full((S.n,), float("nan"), device=dev())
    M = torch.full((S.n, 2), float("nan"), device=dev())
    m.rfr_backward_filter(f32c(G), f32c(sig), DS, s, DA, grid, out, P, ws, mf=M, flags=flags)
    torch.cuda.synchronize()
    g = {k: getattr(out, k).cpu().numpy().astype(np.float64) for k in m.Grads.NAMES}
    return g, P.cpu().numpy().astype(np.float64), c64(M)


def _check_all(g, P, M, G, sig, S, A, grid, s, rays=None, qsel=None, what=""):
    g_ref = oracle.backward(G.astype(np.complex128), S, s, A, grid, rays=rays)
    idx = None
    if rays is not None:
        idx = (np.asarray(rays)[:, None] * S.n_per_ray + np.arange(S.n_per_ray)[None, :]).ravel()
    check_grads(g, g_ref, idx=idx, what=what)
    if idx is None:
        assert abs(g["sharpness"][0] - g_ref["sharpness"]) <= TOL_GRAD * max(
            abs(g_ref["sharpness"]), 1e-30)
    q = np.arange(S.n) if qsel is None else qsel
    Mr, Pr = oracle.filter(sig.astype(np.complex128), A, grid, S.x[q], S.y[q], S.z[q])
    assert rel(P[q], Pr) <= TOL_SIG and rel(M[q], Mr) <= TOL_SIG, what


@pytest.mark.parametrize("name", ["c0b", "c1"])
def test_fused_full(name):
    p = problem(name)
    b = p.bundles[0]
    G = p.random_grad()
    sig = oracle.forward(b.samples, p.sharpness, b.antennas, p.grid).astype(np.complex64)
    g, P, M = gpu_fused(G, sig, b.samples, b.antennas, p.grid, p.sharpness)
    _check_all(g, P, M, G, sig, b.samples, b.antennas, p.grid, p.sharpness, what=name)


@pytest.mark.parametrize("name,n_rays", [("c2", 8), ("c3", 4), ("c4", 2)])
def test_fused_sampled_full_size(name, n_rays):
    """Full-size run (bench launch configuration, split-K over antennas), sampled rays."""
    p = problem(name)
    b = p.bundles[0]
    S = b.samples
    G = p.random_grad()
    sig = (0.5 * p.random_grad() + 0.25 * np.conj(G)).astype(np.complex64)   # a second seeded row set
    g, P, M = gpu_fused(G, sig, S, b.antennas, p.grid, p.sharpness)
    f = S.sdf.reshape(S.n_rays, S.n_per_ray)
    crossing = np.nonzero((f.min(1) < 0) & (f.max(1) > 0))[0]
    rng = np.random.default_rng(11)
    pool = crossing if len(crossing) >= n_rays else np.arange(S.n_rays)
    rays = np.sort(rng.choice(pool, n_rays, replace=False))
    qsel = np.sort(rng.choice(S.n, 96, replace=False))
    _check_all(g, P, M, G, sig, S, b.antennas, p.grid, p.sharpness, rays=rays, qsel=qsel, what=name)


@pytest.mark.parametrize("n_freq", [128, 256, 512, 37])
@pytest.mark.parametrize("variant", ["mono", "bistatic", "phi"])
def test_fused_tiny_variants(n_freq, variant):
    """Ragged sample / antenna counts (several 128-sample tiles + a tail), bistatic and Eq. 7 variants."""
    S, A, grid, s = _tiny(n_freq=n_freq, n_rays=70, n_per_ray=4, n_ant=7, seed=3,
                          bistatic=variant == "bistatic", phi=variant == "phi")
    rng = np.random.default_rng(4)
    G = (rng.standard_normal((A.n, n_freq)) + 1j * rng.standard_normal((A.n, n_freq))).astype(np.complex64)
    sig = (rng.standard_normal((A.n, n_freq)) + 1j * rng.standard_normal((A.n, n_freq))).astype(np.complex64)
    g, P, M = gpu_fused(G, sig, S, A, grid, s)
    _check_all(g, P, M, G, sig, S, A, grid, s, what=f"{variant}/{n_freq}")


def test_fused_matches_separate_calls():
    """Same outputs as rfr_backward + rfr_filter(queries = samples) on c2: the gradients come from
    the same kernel family (rounding-level); the standalone filter runs the tensor-core sweep while
    the fused call takes the Chebyshev-moment path, so M / |M| agree to the parity tolerance."""
    m = rfr()
    p = problem("c2")
    b = p.bundles[0]
    S = b.samples
    G = p.random_grad()
    sig = (0.7 * p.random_grad()[::-1]).astype(np.complex64)
    g, P, M = gpu_fused(G, sig, S, b.antennas, p.grid, p.sharpness)
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    ws = m.workspace(S.n, b.antennas.n, p.grid.n_freq, S.n, dev())
    out = m.Grads.empty(S.n, dev())
    m.rfr_backward(f32c(G), DS, p.sharpness, DA, p.grid, out, ws)
    P2 = torch.empty(S.n, device=dev())
    M2 = torch.empty(S.n, 2, device=dev())
    m.rfr_filter(f32c(sig), DA, p.grid, DS.x, DS.y, DS.z, P2, ws, mf=M2)
    torch.cuda.synchronize()
    for k in FIELDS:
        a = getattr(out, k).cpu().numpy().astype(np.float64)
        assert rel(g[k], a) <= 1e-5, k
    assert rel(M, c64(M2)) <= TOL_SIG and rel(P, P2.cpu().numpy()) <= TOL_SIG


def test_fused_empty_and_errors():
    m = rfr()
    S, A, grid, s = _tiny(n_freq=128, n_rays=2, n_per_ray=3, n_ant=3)
    # workspace planned without queries: the fused call needs n_query >= n_samples
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(A, dev())
    ws = m.workspace(S.n, A.n, grid.n_freq, 0, dev())
    out = m.Grads.empty(S.n, dev())
    P = torch.empty(S.n, device=dev())
    G = torch.zeros(A.n, grid.n_freq, 2, device=dev())
    with pytest.raises(m.RfrError):
        m.rfr_backward_filter(G, G, DS, s, DA, grid, out, P, ws)
    # no antennas: zero gradients, zero filter
    A0 = A.slice(0, 0)
    DA0 = m.DeviceAntennas.from_host(A0, dev())
    ws = m.workspace(S.n, 1, grid.n_freq, S.n, dev())
    m.rfr_backward_filter(G, G, DS, s, DA0, grid, out, P, ws)
    torch.cuda.synchronize()
    assert torch.all(P == 0)
    for k in FIELDS:
        assert torch.all(getattr(out, k) == 0), k


def test_fused_sharded_equals_oracle_and_comm_identity():
    """Multi-GPU algorithm on one GPU: per-shard fused partials (antenna slices = pointer offsets)
    summed in rank order as the all-reduce would, then K1' and |M|; and the NCCL path of
    rfr_backward_filter on one rank is bitwise the same as without it."""
    m = rfr()
    p = problem("c1")
    b = p.bundles[0]
    G = p.random_grad()
    sig = (0.5 * p.random_grad()[::-1]).astype(np.complex64)
    DS, DA = m.DeviceSamples.from_host(b.samples, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    Gt, St = f32c(G), f32c(sig)
    n, na = b.samples.n, b.antennas.n
    ws = m.workspace(n, na, p.grid.n_freq, n, dev())
    world = 4
    part_tot = torch.zeros(5, n, device=dev())
    m_tot = torch.zeros(n, 2, device=dev())
    for r in range(world):
        lo, hi = m.shard_range(na, r, world)
        pr, mr = torch.empty(5, n, device=dev()), torch.empty(n, 2, device=dev())
        m.rfr_backward_filter_partial(Gt[lo:hi], St[lo:hi], DS, p.sharpness, DA.slice(lo, hi),
                                      p.grid, pr, mr, ws)
        part_tot += pr
        m_tot += mr
    out = m.Grads.empty(n, dev())
    m.rfr_backward_finish(part_tot, DS, p.sharpness, out, ws)
    P = torch.empty(n, device=dev())
    m.rfr_filter_power(m_tot, P)
    torch.cuda.synchronize()
    g = {k: getattr(out, k).cpu().numpy().astype(np.float64) for k in m.Grads.NAMES}
    _check_all(g, P.cpu().numpy().astype(np.float64), c64(m_tot), G, sig, b.samples, b.antennas,
               p.grid, p.sharpness, what="sharded")
    comm = m.Comm.create()
    try:
        o1, o2 = m.Grads.empty(n, dev()), m.Grads.empty(n, dev())
        P1, P2 = torch.empty(n, device=dev()), torch.empty(n, device=dev())
        m.rfr_backward_filter(Gt, St, DS, p.sharpness, DA, p.grid, o1, P1, ws)
        m.rfr_backward_filter(Gt, St, DS, p.sharpness, DA, p.grid, o2, P2, ws, comm=comm)
        torch.cuda.synchronize()
        for k in m.Grads.NAMES:
            assert torch.equal(getattr(o1, k), getattr(o2, k)), k
        assert torch.equal(P1, P2)
    finally:
        comm.close()


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_chebyshev_path_matches_direct_kernels(name):
    """The three implementations of the path on the same full-size inputs: the r2 tiled engine
    (default: Horner sweeps over per-(antenna, tile) coefficients, DESIGN 5e), the r1 Chebyshev
    kernels (RFR_R1) and the direct kernels (RFR_DIRECT: K2 recurrence, tensor-core adjoint).
    Forward signal, fused matched filter and gradients agree far inside the parity tolerances, and
    each call reports the path it took."""
    m = rfr()
    p = problem(name)
    b = p.bundles[0]
    S = b.samples
    DS, DA = m.DeviceSamples.from_host(S, dev()), m.DeviceAntennas.from_host(b.antennas, dev())
    ws = m.workspace(S.n, b.antennas.n, p.grid.n_freq, S.n, dev())
    res = {}
    for key, fl in (("r2", 0), ("r1", m.RFR_R1), ("direct", m.RFR_DIRECT)):
        sig = torch.empty(b.antennas.n, p.grid.n_freq, 2, device=dev())
        m.rfr_forward(DS, p.sharpness, DA, p.grid, sig, ws, flags=fl)
        G = f32c(p.random_grad())
        out = m.Grads.empty(S.n, dev())
        P = torch.empty(S.n, device=dev())
        M = torch.empty(S.n, 2, device=dev())
        m.rfr_backward_filter(G, sig, DS, p.sharpness, DA, p.grid, out, P, ws, mf=M,
                              flags=fl | m.RFR_REUSE_BLEND)
        st = m.cheb_state(ws) if key != "r2" else m.rfr_plan_state(ws)
        torch.cuda.synchronize()
        res[key] = (c64(sig), c64(M), {k: getattr(out, k).cpu().numpy().astype(np.float64)
                                       for k in FIELDS}, st)
    assert res["r2"][3]["applied"] == 1 and 8 <= res["r2"][3]["P"] <= 16, res["r2"][3]
    assert res["r1"][3]["sel"] == 1 and res["direct"][3]["sel"] == 0
    for a_, b_ in (("r2", "direct"), ("r1", "direct"), ("r2", "r1")):
        assert rel(res[a_][0], res[b_][0]) <= 1e-5, (a_, b_)
        assert rel(res[a_][1], res[b_][1]) <= 1e-5, (a_, b_)
        for k in FIELDS:
            assert rel(res[a_][2][k], res[b_][2][k]) <= 1e-4, (a_, b_, k)


def test_fused_and_filter_determinism_bitwise():
    """The fused sweep (tiled filter: ordered tile sort, fixed-order moment sums; compacted
    backward) and the standalone filter give bitwise identical results when repeated."""
    m = rfr()
    p = problem("c2")
    b = p.bundles[0]
    S = b.samples
    G = p.random_grad()
    sig = (0.5 * p.random_grad()[::-1]).astype(np.complex64)
    r1 = gpu_fused(G, sig, S, b.antennas, p.grid, p.sharpness)
    r2 = gpu_fused(G, sig, S, b.antennas, p.grid, p.sharpness)
    for k in FIELDS:
        assert np.array_equal(r1[0][k], r2[0][k]), k
    assert np.array_equal(r1[1], r2[1]) and np.array_equal(r1[2], r2[2])
    DA = m.DeviceAntennas.from_host(b.antennas, dev())
    q = [torch.as_tensor(np.ascontiguousarray(v, np.float32)).to(dev()) for v in (S.x, S.y, S.z)]
    ws = m.workspace(0, b.antennas.n, p.grid.n_freq, S.n, dev())
    out = []
    for _ in range(2):
        P = torch.empty(S.n, device=dev())
        m.rfr_filter(f32c(sig), DA, p.grid, *q, P, ws)
        torch.cuda.synchronize()
        out.append(P.cpu().numpy())
    assert np.array_equal(out[0], out[1])
