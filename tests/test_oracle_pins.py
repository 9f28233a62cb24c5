"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test checks the oracle against something other than itself: closed forms, the paper's worked
values (tests/golden), invariants, dense numerical integration of the paper's integral definitions,
central finite differences, Euler/adjoint identities and brute-force geometry.  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate
from scipy.special import expit

import oracle
import synth
from synth import AntennaSet, FreqGrid, SampleSet

C = 299792458.0
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64), dtype=np.float32)


def mk_samples(pos, sdf, refl=None, n=None, power=None, n_per_ray=None, phi=None):
    pos = np.asarray(pos, np.float64).reshape(-1, 3)
    k = pos.shape[0]
    refl = np.ones(k) if refl is None else refl
    power = np.ones(k) if power is None else power
    n = np.tile([0.0, 0.0, -1.0], (k, 1)) if n is None else np.asarray(n, np.float64).reshape(-1, 3)
    npr = k if n_per_ray is None else n_per_ray
    return SampleSet(f32(pos[:, 0]), f32(pos[:, 1]), f32(pos[:, 2]), f32(sdf), f32(refl),
                     f32(n[:, 0]), f32(n[:, 1]), f32(n[:, 2]), f32(power), k // npr, npr,
                     None if phi is None else f32(phi))


def mk_ants(pos, rx=None, phi_tx=None, phi_rx=None):
    pos = np.asarray(pos, np.float64).reshape(-1, 3)
    r = [None] * 3 if rx is None else [f32(np.asarray(rx).reshape(-1, 3)[:, c]) for c in range(3)]
    return AntennaSet(f32(pos[:, 0]), f32(pos[:, 1]), f32(pos[:, 2]), *r,
                      None if phi_tx is None else f32(phi_tx), None if phi_rx is None else f32(phi_rx))


def single_reflector(u=0.25, normal=(0.0, 0.0, -1.0), s=1e5):
    """A 2-sample ray: sample 0 at depth u just outside a surface (f=+1 cm), sample 1 inside
    (f=-1 cm).  With s*1cm = 1000 the NeuS alpha_0 = 1 - e^-1000 = 1 exactly, T_0 = 1, and the last
    sample has alpha = 0, so the signal is a single term."""
    S = mk_samples([[0, 0, u], [0, 0, u + 0.01]], [0.01, -0.01],
                   n=[normal, normal], n_per_ray=2)
    return S, s


# ------------------------------------------------------------------------------------------ P1
def test_p1_single_reflector_closed_form():
    g = json.load(open(os.path.join(GOLD, "p1_single_reflector.json")))
    S, s = single_reflector(g["u_m"])
    A = mk_ants([[0, 0, 0]])
    grid = FreqGrid(77e9, 62.5e6, 64)
    sig = oracle.forward(S, s, A, grid)[0]
    # paper's worked value (hand arithmetic in the golden file)
    assert abs(sig[0] - complex(g["s0_re"], g["s0_im"])) < 1e-12
    assert abs(abs(sig[0]) - g["amplitude"]) < 1e-14
    # closed form for every bin: (1/pi^2) exp(-j 2 pi f_m 2u/c)   (Eq. 1, 2, 4)
    f = grid.f0 + grid.df * np.arange(grid.n_freq)
    expect = np.exp(-2j * np.pi * f * 2 * 0.25 / C) / np.pi ** 2
    np.testing.assert_allclose(sig, expect, rtol=0, atol=1e-13)


def test_p2_spec_worked_values():
    g = json.load(open(os.path.join(GOLD, "p1_single_reflector.json")))["spec_worked_values"]
    A = mk_ants([[0, 0, 0]])
    # tau(0.3 m) = 0.6 / c
    S, s = single_reflector(0.3)
    amp, tau = oracle.pair(S, 0, s, A, 0)
    assert abs(tau - 2 * float(np.float32(0.3)) / C) < 1e-24      # fp32 input widened exactly
    assert abs(tau / g["tau_at_0p3_m"] - 1) < 1e-7
    # decay at u = 0.5 m and u = 1/(4 pi) with every other factor 1
    S, s = single_reflector(0.5)
    amp, _ = oracle.pair(S, 0, s, A, 0)
    assert abs(amp - g["decay_at_0p5_m"]) < 1e-15
    u = float(np.float32(1 / (4 * np.pi)))
    S, s = single_reflector(u)
    amp, _ = oracle.pair(S, 0, s, A, 0)
    assert abs(amp - 1.0 / (4 * np.pi * u) ** 2) < 1e-12 and abs(amp - 1.0) < 1e-6
    # tau = 3/(2 f0) -> exp(-j 3 pi) = -1 at bin 0 (SPEC L53 half-cycle, shifted past u_min)
    d = 3 * C / (4 * 77e9)
    S, s = single_reflector(d)
    sig = oracle.forward(S, s, A, FreqGrid(77e9, 1e6, 1))[0, 0]
    d32 = float(np.float32(d))
    amp = 1 / (4 * np.pi * d32) ** 2
    assert abs(sig / amp - np.exp(-2j * np.pi * 77e9 * 2 * d32 / C)) < 1e-12
    assert abs(sig / amp + 1) < 1e-6
    # bandwidth and range resolution from the paper's chirp
    B = 70.15e12 * 64 / 1.25e6
    assert abs(B - g["bandwidth_hz"]) < 1 and abs(C / (2 * B) - g["range_resolution_m"]) < 1e-12


def test_p2_path_loss_inverse_square():
    A = mk_ants([[0, 0, 0]])
    S1, s1 = single_reflector(0.2)
    S2, s2 = single_reflector(0.4)
    a1, _ = oracle.pair(S1, 0, s1, A, 0)
    a2, _ = oracle.pair(S2, 0, s2, A, 0)
    assert abs(a1 / a2 - 4.0) < 1e-12


@pytest.mark.parametrize("theta_deg", [0.0, 10.0, 30.0, 44.0, 46.0, 60.0, 90.0, 150.0])
def test_p1_directive_gain_tilted_normal(theta_deg):
    """Specular law: with the normal tilted by theta from the ray, the mirror direction w_o makes
    angle 2 theta with the return ray, so (w_o . w_r) = cos(2 theta), clamped at 0 (Q4)."""
    th = math.radians(theta_deg)
    nrm = (math.sin(th), 0.0, -math.cos(th))
    S, s = single_reflector(0.25, normal=nrm)
    amp, _ = oracle.pair(S, 0, s, mk_ants([[0, 0, 0]]), 0)
    n32 = np.array([np.float32(nrm[0]), 0.0, np.float32(nrm[2])], np.float64)
    cos_t = -n32[2] / np.linalg.norm(n32) * np.linalg.norm(n32)   # n . w with w = +z
    g_exact = max(2 * (n32[2] ** 2) - 1, 0.0)                     # cos 2theta = 2cos^2 - 1
    assert abs(amp - g_exact / np.pi ** 2) < 1e-12
    assert abs(g_exact - max(math.cos(2 * th), 0.0)) < 1e-6
    del cos_t


def test_no_gain_flag_drops_directive_factor():
    S, s = single_reflector(0.25, normal=(1.0, 0.0, 0.0))       # grazing: gain 0
    A = mk_ants([[0, 0, 0]])
    amp0, _ = oracle.pair(S, 0, s, A, 0)
    amp1, _ = oracle.pair(S, 0, s, A, 0, flags=oracle.FLAG_NO_GAIN)
    assert amp0 == 0.0 and abs(amp1 - 1 / np.pi ** 2) < 1e-14


# ------------------------------------------------------------------------------------------ P3 / P4
def _c1_small():
    p = synth.make("c1")
    b = p.bundles[0]
    return p, b.samples.subset_rays(np.arange(0, 256, 7)), b.antennas.take([0, 9, 27, 63])


def test_p3_superposition_over_disjoint_rays():
    p, S, A = _c1_small()
    n = S.n_rays
    sa = oracle.forward(S.subset_rays(np.arange(0, n // 2)), p.sharpness, A, p.grid)
    sb = oracle.forward(S.subset_rays(np.arange(n // 2, n)), p.sharpness, A, p.grid)
    st = oracle.forward(S, p.sharpness, A, p.grid)
    assert np.linalg.norm(st - sa - sb) <= 1e-13 * np.linalg.norm(st)


def test_p3_linearity_in_reflectivity_and_power():
    p, S, A = _c1_small()
    base = oracle.forward(S, p.sharpness, A, p.grid)
    dbl = oracle.forward(S.replace(refl=f32(S.refl * 2)), p.sharpness, A, p.grid)
    assert np.linalg.norm(dbl - 2 * base) <= 1e-14 * np.linalg.norm(base)
    rng = np.random.default_rng(5)
    p1 = f32(rng.uniform(0, 1, S.n))
    p2 = f32(rng.uniform(0, 1, S.n))
    s12 = oracle.forward(S.replace(power=f32(p1.astype(np.float64) + p2)), p.sharpness, A, p.grid)
    s1 = oracle.forward(S.replace(power=p1), p.sharpness, A, p.grid)
    s2 = oracle.forward(S.replace(power=p2), p.sharpness, A, p.grid)
    assert np.linalg.norm(s12 - s1 - s2) <= 1e-7 * np.linalg.norm(s12)   # p1+p2 rounded to fp32


def test_p4_tx_rx_swap_symmetry_and_monostatic_limit():
    p, S, _ = _c1_small()
    rng = np.random.default_rng(3)
    tx = np.c_[rng.uniform(-0.05, 0.05, (5, 2)), np.zeros(5)]
    rx = np.c_[rng.uniform(-0.05, 0.05, (5, 2)), np.zeros(5)]
    a = oracle.forward(S, p.sharpness, mk_ants(tx, rx=rx), p.grid)
    b = oracle.forward(S, p.sharpness, mk_ants(rx, rx=tx), p.grid)
    assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(a)
    m = oracle.forward(S, p.sharpness, mk_ants(tx), p.grid)
    mb = oracle.forward(S, p.sharpness, mk_ants(tx, rx=tx), p.grid)
    assert np.linalg.norm(m - mb) <= 1e-15 * np.linalg.norm(m)


# ------------------------------------------------------------------------------------------ P5
def _phi(s, f):
    return expit(s * np.asarray(f, np.float64))


def test_p5_blend_invariants_on_configs():
    for name in ("c1", "c2"):
        p = synth.make(name)
        S = p.bundles[0].samples
        al, om, T = oracle.blend(S.sdf, S.n_rays, S.n_per_ray, p.sharpness)
        al, T = al.reshape(S.n_rays, -1), T.reshape(S.n_rays, -1)
        assert np.all(al >= 0) and np.all(al <= 1)
        assert np.all(T[:, 0] == 1.0)
        assert np.all(np.diff(T, axis=1) <= 0)
        assert np.all((T * al).sum(1) <= 1 + 1e-12)
        assert np.all(al[:, -1] == 0)


def test_p5_transmittance_telescopes_on_monotone_rays():
    """For f decreasing along a ray, prod_{l<k} Phi_{l+1}/Phi_l = Phi_k/Phi_0 (telescoping), and
    sum_k T_k alpha_k = 1 - Phi_{N-1}/Phi_0.  Evaluated here with direct logistic values."""
    rng = np.random.default_rng(11)
    s = 300.0
    f = np.sort(rng.uniform(-0.01, 0.02, (6, 12)), axis=1)[:, ::-1].copy()
    al, om, T = oracle.blend(f32(f).ravel(), 6, 12, s)
    ff = f32(f).astype(np.float64)
    Phi = _phi(s, ff)
    np.testing.assert_allclose(T.reshape(6, 12), Phi / Phi[:, :1], rtol=1e-12, atol=0)
    np.testing.assert_allclose((T * al).reshape(6, 12).sum(1), 1 - Phi[:, -1] / Phi[:, 0], rtol=1e-12)
    # alpha_k = max((Phi_k - Phi_{k+1}) / Phi_k, 0) evaluated directly
    a_direct = np.maximum((Phi[:, :-1] - Phi[:, 1:]) / Phi[:, :-1], 0)
    np.testing.assert_allclose(al.reshape(6, 12)[:, :-1], a_direct, rtol=1e-10, atol=1e-15)


def test_p5_alpha_equals_integral_of_opaque_density():
    """alpha_i = 1 - exp(-int_{u_i}^{u_{i+1}} rho du), rho = max(-(dPhi_s/du)/Phi_s, 0)
    (PAPER L805-818), by adaptive quadrature along a ray through a sphere, on intervals where f is
    monotone (the NeuS discretisation is exact there)."""
    s = 400.0
    c, r = np.array([0.0, 0.0, 0.25]), 0.03
    x0 = np.array([0.007, -0.004, 0.0])

    def f_of(u):
        return np.linalg.norm(x0 + np.array([0, 0, u]) - c) - r

    def rho(u, h=1e-7):
        dphi = (_phi(s, f_of(u + h)) - _phi(s, f_of(u - h))) / (2 * h)
        return max(-dphi / _phi(s, f_of(u)), 0.0)

    us = np.linspace(0.20, 0.245, 10)                      # before the sphere centre: f decreasing
    pos = np.c_[np.full(10, x0[0]), np.full(10, x0[1]), us]
    fs = np.array([f_of(u) for u in us])
    al, _, _ = oracle.blend(f32(fs), 1, 10, s)
    for k in range(9):
        u_a = float(np.float32(us[k]))
        u_b = float(np.float32(us[k + 1]))
        # the oracle sees fp32 SDF values; integrate between the points where f equals them
        integ, _ = integrate.quad(rho, u_a, u_b, epsabs=1e-12, epsrel=1e-10, limit=200)
        ref = 1 - math.exp(-integ)
        fa, fb = float(np.float32(fs[k])), float(np.float32(fs[k + 1]))
        shift = (math.log(_phi(s, fs[k])) - math.log(_phi(s, fa))) - \
                (math.log(_phi(s, fs[k + 1])) - math.log(_phi(s, fb)))
        assert abs(al[k] - ref) < 1e-6 + abs(shift), (k, al[k], ref)
    del pos


def test_p5_step_limit_and_two_slab_squaring():
    # large s: alpha -> 1 on the interval that crosses the surface
    al, _, T = oracle.blend(f32([0.01, 0.005, -0.005, -0.01]), 1, 4, 1e5)
    assert al[1] == 1.0 and T[2] < 1e-200 and al[0] < 1e-200
    # two identical slabs along a ray square the single-slab transmittance (round trip)
    s = 2000.0                        # free space between the slabs saturates Phi to 1
    z = np.linspace(0, 0.1, 401)      # slab centres on the same grid phase
    slab = lambda zz, zc: np.abs(zz - zc) - 0.001
    f1 = slab(z, 0.03)
    f2 = np.minimum(slab(z, 0.03), slab(z, 0.07))
    _, _, T1 = oracle.blend(f32(f1), 1, 401, s)
    _, _, T2 = oracle.blend(f32(f2), 1, 401, s)
    assert 0.01 < T1[-1] < 0.5 and abs(T2[-1] - T1[-1] ** 2) < 1e-6 * T1[-1] ** 2


def test_p6_lensless_transmittance_correction_sign():
    """Eq. 7 against brute force: T along the real antenna->point ray by dense integration of rho,
    versus T along the primary ray corrected by the origin Phi terms.  The derivation (PAPER
    L856-877) gives T' = T + Phi(o_p) - Phi(o_r); the printed Eq. 7 (L339) has the opposite sign.
    Reading Q11: the ABI computes T - Phi_apr + Phi_ant; callers pass negated Phi arrays for the
    derived form.  This test records which form matches the brute force."""
    s = 30.0
    c, r = np.array([0.0, 0.0, 0.25]), 0.03
    sdf = lambda X: np.linalg.norm(X - c, axis=-1) - r
    Phi = lambda X: _phi(s, sdf(X))

    def T_along(o, x, n=4000):
        """exp(-int rho) from o to x: rho = max(-(d Phi/du)/Phi, 0) -> sum of positive log drops."""
        u = np.linspace(0, 1, n)
        lp = np.log(Phi(o[None, :] + u[:, None] * (x - o)[None, :]))
        return math.exp(np.minimum(np.diff(lp), 0).sum())

    x = np.array([0.01, 0.0, 0.205])          # a point in front of the sphere
    o_p = np.array([0.01, 0.0, 0.0])          # primary-ray origin on the aperture (w_p = +z)
    errs_printed, errs_derived = [], []
    for ax in (-0.08, -0.04, 0.04, 0.08):     # antennas up to ~22 deg off axis
        o_r = np.array([ax, 0.03, 0.0])
        Tp, Tr = T_along(o_p, x), T_along(o_r, x)
        printed = Tp - Phi(o_p) + Phi(o_r)
        derived = Tp + Phi(o_p) - Phi(o_r)
        errs_printed.append(abs(printed - Tr))
        errs_derived.append(abs(derived - Tr))
    assert max(errs_derived) < 5e-3
    assert max(errs_printed) > max(errs_derived)
    # and the oracle applies T_j - Phi_apr_j + Phi_ant_i, clamped (printed form, Q11/Q12)
    S, s2 = single_reflector(0.25)
    S = S.replace(phi_origin=f32([0.9, 0.9]))
    A0 = mk_ants([[0, 0, 0]])
    A1 = mk_ants([[0, 0, 0]], phi_tx=[0.8])
    a0, _ = oracle.pair(S, 0, s2, A0, 0)       # T = clamp(1 - 0.9 + 1) = 1
    a1, _ = oracle.pair(S, 0, s2, A1, 0)       # T = 1 - 0.9 + 0.8 = 0.9
    t = 1.0 - float(np.float32(0.9)) + float(np.float32(0.8))
    assert abs(a1 / a0 - t * t) < 1e-12


# ------------------------------------------------------------------------------------------ P7 / P8
def _fd_problem():
    p = synth.make("c0b")
    b = p.bundles[0]
    rng = np.random.default_rng(17)
    y = (rng.standard_normal((4, 8)) + 1j * rng.standard_normal((4, 8))) * 1e-3
    return p, b.samples, b.antennas, y


def _loss64(S, s, A, grid, y, fields):
    """L = 1/2 ||F(fields) - y||^2 with fp64 fields substituted (no fp32 rounding)."""
    keep = {}
    for k, v in fields.items():
        keep[k] = v
    F = oracle.forward(_S64(S, keep), s, A, grid)
    return 0.5 * np.sum(np.abs(F - y) ** 2)


class _S64(SampleSet):
    """SampleSet whose arrays are float64 (the oracle widens float32; float64 passes through)."""

    def __init__(self, S, override):
        kw = {f: np.asarray(override.get(f, getattr(S, f)), np.float64) for f in S.FIELDS}
        super().__init__(**kw, n_rays=S.n_rays, n_per_ray=S.n_per_ray, phi_origin=S.phi_origin)


def test_p7_backward_matches_central_finite_differences():
    p, S, A, y = _fd_problem()
    s = p.sharpness
    base = {f: getattr(S, f).astype(np.float64) for f in S.FIELDS}
    F = oracle.forward(S, s, A, p.grid)
    _, G = oracle.loss(F, y)
    g = oracle.backward(G, S, s, A, p.grid)
    worst = 0.0
    for field in ("sdf", "refl", "nx", "ny", "nz", "power"):
        for j in range(S.n):
            v = base[field][j]
            h = 1e-6 * max(abs(v), 1e-3)
            up = dict(base)
            up[field] = base[field].copy()
            up[field][j] = v + h
            dn = dict(base)
            dn[field] = base[field].copy()
            dn[field][j] = v - h
            fd = (_loss64(S, s, A, p.grid, y, up) - _loss64(S, s, A, p.grid, y, dn)) / (2 * h)
            an = g[field][j]
            scale = max(abs(fd), abs(an), 1e-12 * 1e3)
            err = abs(fd - an) / scale
            worst = max(worst, err)
            assert err < 1e-5, (field, j, fd, an)
    # sharpness
    h = 1e-6 * s
    Lp = 0.5 * np.sum(np.abs(oracle.forward(S, s + h, A, p.grid) - y) ** 2)
    Lm = 0.5 * np.sum(np.abs(oracle.forward(S, s - h, A, p.grid) - y) ** 2)
    fd = (Lp - Lm) / (2 * h)
    assert abs(fd - g["sharpness"]) <= 1e-5 * max(abs(fd), 1e-12)


def _bistatic_phi_fd_problem():
    """c0b's samples seen by a BISTATIC 2x2 array (rx offset from tx in all three axes) with
    distinct Eq. 7 origin terms Phi_apr (per sample), Phi_tx, Phi_rx (per antenna): the branch of
    O6 the monostatic, Phi-free c0b never reaches -- the S2 cross terms T_r chi_t + T_t chi_r, the
    chi gating at both clamps (reading Q25b) and the bistatic dg/dn (Eq. 7 P:L335-341,
    origin terms detached P:L351-352)."""
    p = synth.make("c0b")
    b = p.bundles[0]
    tx = b.antennas
    rx = np.stack([tx.tx_x + 0.015, tx.tx_y - 0.007, tx.tx_z + 0.003], -1)
    # Phi_apr: 0.70 at sample 1 lifts T_raw above 1 there (T_1 < 1 depends on the sdf); 0.995 at
    # sample 6 (T_6 = 0.24) pushes T_raw below 0 for the antennas with Phi_ant < 0.75
    phi_apr = f32([0.98, 0.70, 0.93, 0.60, 0.96, 0.72, 0.995, 0.62])
    A = mk_ants(np.stack([tx.tx_x, tx.tx_y, tx.tx_z], -1), rx=rx,
                phi_tx=[0.97, 0.81, 0.95, 0.66], phi_rx=[0.75, 0.99, 0.84, 0.91])
    rng = np.random.default_rng(29)
    # normals tilted 5-30 deg off the array axis (either sign): gains mostly > 0, so the bistatic
    # dg/dn is exercised (c0b's isotropic normals clamp most gains to 0)
    th, ph = np.radians(rng.uniform(5, 30, 8)), rng.uniform(0, 2 * np.pi, 8)
    sgn = np.where(rng.random(8) < 0.5, -1.0, 1.0)
    nrm = sgn[:, None] * np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), -np.cos(th)], -1)
    S = b.samples.replace(phi_origin=phi_apr, nx=f32(nrm[:, 0]), ny=f32(nrm[:, 1]), nz=f32(nrm[:, 2]))
    y = (rng.standard_normal((4, 8)) + 1j * rng.standard_normal((4, 8))) * 1e-3
    return p, S, A, y


def test_p7_bistatic_phi_backward_matches_central_finite_differences():
    """P7 on the bistatic / Eq. 7-corrected branch of O6.  The case is built so that every piece
    of that branch is exercised away from its kinks (checked below before the FD comparison):
    pairs with the upper T clamp active on a T_j < 1 that depends on the SDF, pairs with the
    lower clamp active, pairs where exactly one of T_t, T_r is clamped (so a T_t <-> T_r swap of
    the S2 cross terms changes the result), and positive and clamped gains."""
    p, S, A, y = _bistatic_phi_fd_problem()
    s = p.sharpness
    _, _, T = oracle.blend(S.sdf, S.n_rays, S.n_per_ray, s)
    papr = S.phi_origin.astype(np.float64)
    Tt = T[:, None] + (A.phi_tx.astype(np.float64)[None, :] - papr[:, None])
    Tr = T[:, None] + (A.phi_rx.astype(np.float64)[None, :] - papr[:, None])
    first = (np.arange(S.n) % S.n_per_ray) == 0          # T_j = 1 there, independent of sdf
    for raw in (Tt, Tr):                                  # away from both kinks
        assert np.min(np.abs(raw)) > 1e-3 and np.min(np.abs(raw - 1.0)) > 1e-3
    upper_dep = ((Tt > 1) | (Tr > 1)) & ~first[:, None]
    assert np.any(upper_dep), "upper clamp must act on a T_j that depends on the sdf"
    assert np.any((Tt < 0) | (Tr < 0)), "lower clamp must act somewhere"
    one_clamped = ((Tt > 0) & (Tt < 1)) != ((Tr > 0) & (Tr < 1))
    assert np.any(one_clamped & ~first[:, None] & (T[:, None] < 1))
    base = {f: getattr(S, f).astype(np.float64) for f in S.FIELDS}
    F = oracle.forward(S, s, A, p.grid)
    _, G = oracle.loss(F, y)
    g = oracle.backward(G, S, s, A, p.grid)
    checked = 0
    for field in ("sdf", "refl", "nx", "ny", "nz", "power"):
        for j in range(S.n):
            v = base[field][j]
            h = 1e-6 * max(abs(v), 1e-3)
            up = dict(base)
            up[field] = base[field].copy()
            up[field][j] = v + h
            dn = dict(base)
            dn[field] = base[field].copy()
            dn[field][j] = v - h
            fd = (_loss64(S, s, A, p.grid, y, up) - _loss64(S, s, A, p.grid, y, dn)) / (2 * h)
            an = g[field][j]
            scale = max(abs(fd), abs(an), 1e-12 * 1e3)
            assert abs(fd - an) / scale < 1e-5, (field, j, fd, an)
            checked += abs(an) > 1e-12
    assert checked >= 30                                   # most probes carry a real gradient
    h = 1e-6 * s
    Lp = 0.5 * np.sum(np.abs(oracle.forward(S, s + h, A, p.grid) - y) ** 2)
    Lm = 0.5 * np.sum(np.abs(oracle.forward(S, s - h, A, p.grid) - y) ** 2)
    fd = (Lp - Lm) / (2 * h)
    assert abs(fd - g["sharpness"]) <= 1e-5 * max(abs(fd), 1e-12)


def test_p7_bistatic_phi_fd_detects_swapped_cross_terms():
    """Sensitivity of the pin above: the sdf gradient built from S2 with T_t <-> T_r swapped in the
    cross terms (T_t chi_t + T_r chi_r) differs from the oracle's by far more than the FD
    tolerance on this case, so the FD test would catch that mistake."""
    p, S, A, y = _bistatic_phi_fd_problem()
    s = p.sharpness
    F = oracle.forward(S, s, A, p.grid)
    _, G = oracle.loss(F, y)
    part = oracle.backward_partials(G, S, s, A, p.grid)
    # rebuild S2 with the swapped pairing from per-antenna partials of single-antenna sets
    _, _, T = oracle.blend(S.sdf, S.n_rays, S.n_per_ray, s)
    papr = S.phi_origin.astype(np.float64)
    S2_swapped = np.zeros(S.n)
    for i in range(A.n):
        Ai = A.take([i])
        pi_ = oracle.backward_partials(G[i:i + 1], S, s, Ai, p.grid)
        tt = T + (float(A.phi_tx[i]) - papr)
        tr = T + (float(A.phi_rx[i]) - papr)
        Tt, Tr = np.clip(tt, 0, 1), np.clip(tr, 0, 1)
        ct = (tt > 0) & ((tt < 1) | (float(A.phi_tx[i]) - papr <= 0))
        cr = (tr > 0) & ((tr < 1) | (float(A.phi_rx[i]) - papr <= 0))
        # pi_[:,1] = R g gamma (Tr ct + Tt cr); R g gamma = pi_[:,0] / (Tt Tr) where Tt Tr > 0
        ok = (Tt * Tr) > 0
        rgg = np.where(ok, pi_[:, 0] / np.where(ok, Tt * Tr, 1.0), 0.0)
        S2_swapped += rgg * (Tt * ct + Tr * cr)
        assert np.allclose(np.where(ok, rgg * (Tr * ct + Tt * cr), pi_[:, 1]), pi_[:, 1],
                           rtol=1e-9, atol=1e-30)
    part_sw = part.copy()
    part_sw[:, 1] = S2_swapped
    g = oracle.backward_finish(part, S, s)
    g_sw = oracle.backward_finish(part_sw, S, s)
    rel = np.linalg.norm(g_sw["sdf"] - g["sdf"]) / np.linalg.norm(g["sdf"])
    assert rel > 1e-3


def test_p8_euler_identity_for_linear_loss():
    """F is homogeneous of degree 1 in power p and in reflectivity a, so for the linear loss
    L = Re<F, G> the backward must satisfy sum_j p_j dL/dp_j = L = sum_j a_j dL/da_j."""
    p = synth.make("c1")
    b = p.bundles[0]
    S = b.samples.subset_rays(np.arange(0, 256, 5))
    A = b.antennas.take([0, 7, 36, 63])
    rng = np.random.default_rng(23)
    G = rng.standard_normal((4, p.grid.n_freq)) + 1j * rng.standard_normal((4, p.grid.n_freq))
    F = oracle.forward(S, p.sharpness, A, p.grid)
    L = np.sum(F.real * G.real + F.imag * G.imag)
    g = oracle.backward(G, S, p.sharpness, A, p.grid)
    assert abs(np.dot(S.power.astype(np.float64), g["power"]) - L) <= 1e-10 * abs(L)
    assert abs(np.dot(S.refl.astype(np.float64), g["refl"]) - L) <= 1e-10 * abs(L)


def test_backward_partials_sum_over_antenna_shards():
    """Antenna sharding (north_star multi-GPU): per-sample partials are additive over antennas."""
    p = synth.make("c1")
    b = p.bundles[0]
    S = b.samples.subset_rays(np.arange(0, 256, 9))
    rng = np.random.default_rng(2)
    G = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    full = oracle.backward_partials(G, S, p.sharpness, b.antennas, p.grid)
    parts = sum(oracle.backward_partials(G[lo:lo + 16], S, p.sharpness, b.antennas.slice(lo, lo + 16),
                                         p.grid) for lo in range(0, 64, 16))
    assert np.linalg.norm(full - parts) <= 1e-12 * np.linalg.norm(full)


def test_q25b_uncorrected_clamp_is_identity_including_t_equal_one():
    """Without the Eq. 7 correction A_ij = w g gamma T_j^2, so dA/dT_j = 2 w g gamma T_j: the
    partials obey S2_j T_j = 2 S1_j for every T_j > 0 -- including the samples where T_j = 1
    exactly (first samples, and samples behind intervals whose alpha rounds away), where the
    [0, 1] clamp is the identity on the feasible side (reading Q25b)."""
    p = synth.make("c1")
    b = p.bundles[0]
    S = b.samples.subset_rays(np.arange(0, 256, 5))
    rng = np.random.default_rng(21)
    G = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    part = oracle.backward_partials(G, S, p.sharpness, b.antennas, p.grid)
    _, _, T = oracle.blend(S.sdf, S.n_rays, S.n_per_ray, p.sharpness)
    on = T > 0
    assert np.any(T == 1.0) and np.any((T > 0) & (T < 1))
    lhs, rhs = part[on, 1] * T[on], 2.0 * part[on, 0]
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    one = T == 1.0
    assert np.allclose(part[one, 1], 2.0 * part[one, 0], rtol=1e-12, atol=0)


# ------------------------------------------------------------------------------------------ P9
def test_p9_filter_autocorrelation_is_n_freq():
    grid = FreqGrid(77e9, 62.5e6, 64)
    A = mk_ants([[0.01, -0.02, 0.0]])
    q = np.array([0.03, 0.01, 0.27])
    d = np.linalg.norm(f32(q).astype(np.float64) - f32([0.01, -0.02, 0.0]).astype(np.float64))
    f = grid.f0 + grid.df * np.arange(64)
    sig = np.exp(-2j * np.pi * f * 2 * d / C)[None, :]
    M, P = oracle.filter(sig, A, grid, f32([q[0]]), f32([q[1]]), f32([q[2]]))
    assert abs(P[0] - 64.0) < 1e-9 and abs(M[0] - 64.0) < 1e-9
    _, P0 = oracle.filter(np.zeros((1, 64)), A, grid, f32([q[0]]), f32([q[1]]), f32([q[2]]))
    assert P0[0] == 0.0


def test_p9_filter_of_traced_point_is_real_and_peaks_at_target():
    """Signs (Q2): the filter conjugates the tracing phase, so at the reflector M = N_f sum_i A_i is
    real and positive; along depth the peak is within one range resolution c/2B of the target."""
    grid = synth.uniform_grid(64)
    ants = synth.plane_antennas(8, 8, 0.10)
    u = 0.25
    S, s = single_reflector(u)
    sig = oracle.forward(S, s, ants, grid)
    amps = np.array([oracle.pair(S, 0, s, ants, i)[0] for i in range(64)])
    M, P = oracle.filter(sig, ants, grid, f32([0.0]), f32([0.0]), f32([u]))
    assert abs(M[0].imag) < 1e-9 * abs(M[0]) and abs(M[0].real - 64 * amps.sum()) < 1e-9 * M[0].real
    zq = np.linspace(0.15, 0.35, 401)
    _, Pz = oracle.filter(sig, ants, grid, f32(np.zeros(401)), f32(np.zeros(401)), f32(zq))
    assert abs(zq[np.argmax(Pz)] - u) <= C / (2 * 4e9)


def test_p9_filter_shift_covariance():
    p = synth.make("c0a")
    b = p.bundles[0]
    rng = np.random.default_rng(4)
    sig = rng.standard_normal((4, 8)) + 1j * rng.standard_normal((4, 8))
    q = np.c_[rng.uniform(-0.02, 0.02, (16, 2)), rng.uniform(0.15, 0.25, 16)]
    shift = np.array([0.125, -0.0625, 0.25])     # exactly representable shifts
    A = b.antennas
    A2 = AntennaSet(A.tx_x.astype(np.float64) + shift[0], A.tx_y.astype(np.float64) + shift[1],
                    A.tx_z.astype(np.float64) + shift[2])          # exact in fp64
    q32 = f32(q).astype(np.float64)
    _, P1 = oracle.filter(sig, A, p.grid, f32(q32[:, 0]), f32(q32[:, 1]), f32(q32[:, 2]))
    _, P2 = oracle.filter(sig, A2, p.grid, q32[:, 0] + shift[0], q32[:, 1] + shift[1], q32[:, 2] + shift[2])
    assert np.max(np.abs(P1 - P2) / P1) < 1e-9


# ------------------------------------------------------------------------------------------ misc
def test_loss_and_residual():
    rng = np.random.default_rng(1)
    s = rng.standard_normal((3, 5)) + 1j * rng.standard_normal((3, 5))
    y = rng.standard_normal((3, 5)) + 1j * rng.standard_normal((3, 5))
    L, G = oracle.loss(s, y)
    np.testing.assert_array_equal(G, s - y)
    assert abs(L - 0.5 * np.sum(np.abs(s - y) ** 2)) < 1e-13


def test_domain_guard_zeroes_close_pairs():
    S = mk_samples([[0, 0, 0.0005], [0, 0, 0.01]], [0.01, -0.01], n_per_ray=2)
    A = mk_ants([[0, 0, 0]])
    amp, _ = oracle.pair(S, 0, 1e5, A, 0)
    assert amp == 0.0
    sig = oracle.forward(S, 1e5, A, FreqGrid(77e9, 1e9, 4))
    assert np.all(sig == 0)
