"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the renderer's arithmetic (no alpha / transmittance / gain / path loss /
phase): it only builds analytic scenes, samples positions, evaluates the scene SDF and its analytic
gradient, draws reflectivities, and draws unit complex noise.  Recipes follow SURVEY.md section 8(d)
and the readings in DESIGN.md ("Input recipe").  The paper's own data is a private radar capture
("we collected our own dataset"), so these configs stand in for it with the paper's
physical parameters: 77 GHz start, ~4 GHz sweep (L892), lambda/2 pitch (L889), 15-50 cm standoff.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

C_LIGHT = 299792458.0
F0 = 77e9
BANDWIDTH = 4e9
SHARPNESS = 2e4                          # 1/m (BASELINE configs[0]: "s = 200/cm"; reading Q21)
HALF_WAVELENGTH_79GHZ = C_LIGHT / 79e9 / 2.0   # 1.89742 mm (reading Q23)


@dataclasses.dataclass
class SampleSet:
    """SoA float32 per-sample fields, ray-major and depth-sorted along the primary direction."""
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    sdf: np.ndarray
    refl: np.ndarray
    nx: np.ndarray
    ny: np.ndarray
    nz: np.ndarray
    power: np.ndarray
    n_rays: int
    n_per_ray: int
    phi_origin: Optional[np.ndarray] = None

    FIELDS = ("x", "y", "z", "sdf", "refl", "nx", "ny", "nz", "power")

    @property
    def n(self) -> int:
        return self.n_rays * self.n_per_ray

    def subset_rays(self, rays: np.ndarray) -> "SampleSet":
        idx = (np.asarray(rays, np.int64)[:, None] * self.n_per_ray
               + np.arange(self.n_per_ray)[None, :]).ravel()
        kw = {f: getattr(self, f)[idx] for f in self.FIELDS}
        po = None if self.phi_origin is None else self.phi_origin[idx]
        return SampleSet(**kw, n_rays=len(rays), n_per_ray=self.n_per_ray, phi_origin=po)

    def replace(self, **kw) -> "SampleSet":
        return dataclasses.replace(self, **kw)


@dataclasses.dataclass
class AntennaSet:
    tx_x: np.ndarray
    tx_y: np.ndarray
    tx_z: np.ndarray
    rx_x: Optional[np.ndarray] = None     # None => monostatic (rx == tx)
    rx_y: Optional[np.ndarray] = None
    rx_z: Optional[np.ndarray] = None
    phi_tx: Optional[np.ndarray] = None   # None => Phi_s = 1 at the real-ray origins
    phi_rx: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return int(self.tx_x.shape[0])

    def slice(self, lo: int, hi: int) -> "AntennaSet":
        def s(a):
            return None if a is None else a[lo:hi]
        return AntennaSet(*(s(getattr(self, f.name)) for f in dataclasses.fields(self)))

    def take(self, idx) -> "AntennaSet":
        idx = np.asarray(idx, np.int64)

        def s(a):
            return None if a is None else a[idx]
        return AntennaSet(*(s(getattr(self, f.name)) for f in dataclasses.fields(self)))


@dataclasses.dataclass
class FreqGrid:
    f0: float
    df: float
    n_freq: int


@dataclasses.dataclass
class Bundle:
    """One primary-ray bundle and the antennas that see it (one forward/backward call)."""
    samples: SampleSet
    antennas: AntennaSet


@dataclasses.dataclass
class Problem:
    name: str
    bundles: List[Bundle]
    grid: FreqGrid
    sharpness: float
    snr_db: float
    seed: int
    passes: Tuple[str, ...]

    @property
    def n_contrib(self) -> int:
        """points x antennas x bins per pass, summed over bundles (BASELINE metric unit)."""
        return sum(b.samples.n * b.antennas.n for b in self.bundles) * self.grid.n_freq

    def noise_unit(self, k: int = 0) -> np.ndarray:
        """Unit-power circular complex Gaussian noise [n_ant][n_freq] for bundle k (reading Q18)."""
        b = self.bundles[k]
        rng = np.random.default_rng((self.seed, 7919, k))
        re = rng.standard_normal((b.antennas.n, self.grid.n_freq))
        im = rng.standard_normal((b.antennas.n, self.grid.n_freq))
        return (re + 1j * im) / np.sqrt(2.0)

    def random_grad(self, k: int = 0) -> np.ndarray:
        """Seeded complex upstream gradient G [n_ant][n_freq] (complex64) for backward parity
        cases whose forward is too large for the oracle: the backward is linear in G."""
        b = self.bundles[k]
        rng = np.random.default_rng((self.seed, 104729, k))
        g = rng.standard_normal((b.antennas.n, self.grid.n_freq, 2)).astype(np.float32)
        return (g[..., 0] + 1j * g[..., 1]).astype(np.complex64)


def uniform_grid(n_freq: int) -> FreqGrid:
    """f_m = 77 GHz + m * 4 GHz / N_f (reading Q1: the FMCW sample convention)."""
    return FreqGrid(F0, BANDWIDTH / n_freq, n_freq)


# ----------------------------------------------------------------------------- analytic scenes
@dataclasses.dataclass
class Prim:
    kind: str            # "sphere" | "box" | "hollow_box"
    center: np.ndarray   # (3,)
    size: np.ndarray     # sphere: (radius,), box: half extents (3,), hollow: (outer half, wall)
    refl: Optional[float] = None


def _prim_sdf_grad(p: Prim, X: np.ndarray):
    """SDF (inside-negative, reading Q7) and its analytic gradient for points X [..., 3] (fp64)."""
    d = X - p.center
    if p.kind == "sphere":
        r = np.linalg.norm(d, axis=-1)
        sdf = r - p.size[0]
        with np.errstate(invalid="ignore", divide="ignore"):
            g = d / np.maximum(r, 1e-30)[..., None]
        return sdf, g
    if p.kind == "box":
        return _box_sdf_grad(d, p.size)
    if p.kind == "hollow_box":                      # max(box_outer, -box_inner)
        s1, g1 = _box_sdf_grad(d, np.full(3, p.size[0]))
        s2, g2 = _box_sdf_grad(d, np.full(3, p.size[0] - p.size[1]))
        use1 = s1 >= -s2
        return np.where(use1, s1, -s2), np.where(use1[..., None], g1, -g2)
    raise ValueError(p.kind)


def _box_sdf_grad(d: np.ndarray, h: np.ndarray):
    q = np.abs(d) - h
    qo = np.maximum(q, 0.0)
    out_len = np.linalg.norm(qo, axis=-1)
    qmax = q.max(axis=-1)
    sdf = out_len + np.minimum(qmax, 0.0)
    sgn = np.where(d >= 0, 1.0, -1.0)
    with np.errstate(invalid="ignore", divide="ignore"):
        g_out = sgn * qo / np.maximum(out_len, 1e-30)[..., None]
    axis = np.argmax(q, axis=-1)
    g_in = np.zeros_like(d)
    np.put_along_axis(g_in, axis[..., None], np.take_along_axis(sgn, axis[..., None], -1), -1)
    g = np.where((qmax > 0)[..., None], g_out, g_in)
    return sdf, g


def scene_eval(prims: List[Prim], X: np.ndarray, chunk: int = 1 << 20):
    """Union (min) SDF, normalised gradient of the active primitive, and active index."""
    X = np.asarray(X, np.float64)
    flat = X.reshape(-1, 3)
    sdf = np.empty(flat.shape[0])
    nrm = np.empty_like(flat)
    act = np.empty(flat.shape[0], np.int64)
    for lo in range(0, flat.shape[0], chunk):
        Y = flat[lo:lo + chunk]
        best = np.full(Y.shape[0], np.inf)
        bg = np.zeros_like(Y)
        bi = np.zeros(Y.shape[0], np.int64)
        for k, p in enumerate(prims):
            s, g = _prim_sdf_grad(p, Y)
            take = s < best
            best = np.where(take, s, best)
            bg = np.where(take[:, None], g, bg)
            bi = np.where(take, k, bi)
        n = np.linalg.norm(bg, axis=-1, keepdims=True)
        bg = np.where(n > 0, bg / np.maximum(n, 1e-30), np.array([0.0, 0.0, 1.0]))
        sdf[lo:lo + chunk], nrm[lo:lo + chunk], act[lo:lo + chunk] = best, bg, bi
    return (sdf.reshape(X.shape[:-1]), nrm.reshape(X.shape), act.reshape(X.shape[:-1]))


def _random_prims(rng, n: int, lo: np.ndarray, hi: np.ndarray, size_range=(0.01, 0.06),
                  no_overlap=False, kinds=None) -> List[Prim]:
    prims: List[Prim] = []
    tries = 0
    while len(prims) < n:
        tries += 1
        if tries > 100000:
            raise RuntimeError("could not place primitives")
        kind = kinds[len(prims)] if kinds else ("sphere" if rng.random() < 0.5 else "box")
        if isinstance(size_range, dict):
            sr = size_range[kind]
        else:
            sr = size_range
        if kind == "sphere":
            diam = rng.uniform(*sr) if sr[0] != sr[1] else sr[0]
            half = np.full(3, diam / 2)
            size = np.array([diam / 2])
        else:                                     # full edge length per axis (reading Q22)
            edges = rng.uniform(sr[0], sr[1], 3)
            half = edges / 2
            size = half
        c = rng.uniform(lo + half, hi - half)
        if no_overlap and any(np.all(np.abs(c - q.center) < half + _half(q)) for q in prims):
            continue
        prims.append(Prim(kind, c, size))
    return prims


def _half(p: Prim) -> np.ndarray:
    return np.full(3, p.size[0]) if p.kind == "sphere" else p.size


# ----------------------------------------------------------------------------- geometry helpers
def plane_antennas(n_u: int, n_v: int, pitch_or_extent: float, center=(0.0, 0.0, 0.0),
                   R: Optional[np.ndarray] = None, by_extent: bool = True) -> AntennaSet:
    """Row-major grid in the plane spanned by R[:,0], R[:,1]; edge-to-edge linspace (reading Q23)."""
    if by_extent:
        u = np.linspace(-pitch_or_extent / 2, pitch_or_extent / 2, n_u)
        v = np.linspace(-pitch_or_extent / 2, pitch_or_extent / 2, n_v)
    else:
        u = (np.arange(n_u) - (n_u - 1) / 2) * pitch_or_extent
        v = (np.arange(n_v) - (n_v - 1) / 2) * pitch_or_extent
    U, V = np.meshgrid(u, v, indexing="ij")
    P = np.stack([U.ravel(), V.ravel(), np.zeros(U.size)], -1)
    if R is not None:
        P = P @ R.T
    P = P + np.asarray(center)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return AntennaSet(f(P[:, 0]), f(P[:, 1]), f(P[:, 2]))


def _rot_y(theta: float) -> np.ndarray:
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def _pack(X: np.ndarray, prims: List[Prim], refl: np.ndarray, n_rays: int, n_per_ray: int,
          power: Optional[np.ndarray] = None) -> SampleSet:
    sdf, nrm, _ = scene_eval(prims, X)
    f = lambda a: np.ascontiguousarray(a.reshape(-1), dtype=np.float32)
    n = X.reshape(-1, 3).shape[0]
    pw = np.ones(n) if power is None else power
    return SampleSet(f(X[..., 0]), f(X[..., 1]), f(X[..., 2]), f(sdf), f(refl), f(nrm[..., 0]),
                     f(nrm[..., 1]), f(nrm[..., 2]), f(pw), n_rays, n_per_ray)


def scene_sdf(prims: List[Prim], X: np.ndarray) -> np.ndarray:
    """Union (min) SDF only (no gradient), fp64."""
    best = None
    for p in prims:
        d = X - p.center
        if p.kind == "sphere":
            v = np.linalg.norm(d, axis=-1) - p.size[0]
        elif p.kind == "box":
            q = np.abs(d) - p.size
            v = np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(-1), 0.0)
        else:
            v, _ = _prim_sdf_grad(p, X)
        best = v if best is None else np.minimum(best, v)
    return best


def _first_crossing(prims, starts: np.ndarray, direction: np.ndarray, u0: float, u1: float,
                    tol: float = 1e-7, max_iter: int = 2000):
    """First outside->inside zero crossing of the union SDF along x = start + u*dir after u0, by
    sphere tracing (the union of exact primitive SDFs never over-estimates the distance).  Rays
    that start inside first march out.  Returns u (nan where the ray misses before u1)."""
    n = starts.shape[0]
    u = np.full(n, u0, dtype=np.float64)
    found = np.full(n, np.nan)
    live = np.ones(n, bool)
    # leave any object the ray starts in
    for _ in range(max_iter):
        idx = np.nonzero(live)[0]
        if idx.size == 0:
            break
        s = scene_sdf(prims, starts[idx] + u[idx, None] * direction)
        inside = s < 0
        if not inside.any():
            break
        u[idx[inside]] += np.maximum(-s[inside], 1e-5)
        live[idx[inside & (u[idx] > u1)]] = False
    for _ in range(max_iter):
        idx = np.nonzero(live)[0]
        if idx.size == 0:
            break
        s = scene_sdf(prims, starts[idx] + u[idx, None] * direction)
        hit = s < tol
        found[idx[hit]] = u[idx[hit]]
        live[idx[hit]] = False
        go = ~hit
        u[idx[go]] += s[go]
        live[idx[go & (u[idx] > u1)]] = False
    return found


def _mixed_depths(rng, crossing: np.ndarray, u0: float, u1: float, n_per_ray: int,
                  band: float = 5e-3) -> np.ndarray:
    """Reading Q19: half stratified over [u0,u1], half uniform within +-band of the first zero
    crossing (rays that miss get stratified depths instead); sorted along the ray."""
    n_rays = crossing.shape[0]
    half = n_per_ray // 2
    cells = (u1 - u0) / half
    strat = u0 + (np.arange(half)[None, :] + rng.random((n_rays, half))) * cells
    near = crossing[:, None] + rng.uniform(-band, band, (n_rays, n_per_ray - half))
    near = np.clip(near, u0, u1)
    miss = np.isnan(crossing)
    cells2 = (u1 - u0) / (n_per_ray - half)
    strat2 = u0 + (np.arange(n_per_ray - half)[None, :] + rng.random((n_rays, n_per_ray - half))) * cells2
    near[miss] = strat2[miss]
    return np.sort(np.concatenate([strat, near], axis=1), axis=1)


# ----------------------------------------------------------------------------- configurations
def make_c0(variant: str = "a") -> Problem:
    """Test-only tiny case: 2x2 antennas on 2 cm, 8 bins, 2 rays x 4 depths."""
    ants = plane_antennas(2, 2, 0.02)
    zs = np.array([0.185, 0.195, 0.205, 0.215])
    xs = np.array([-0.004, 0.004])
    X = np.zeros((2, 4, 3))
    X[:, :, 0] = xs[:, None]
    X[:, :, 2] = zs[None, :]
    prims = [Prim("sphere", np.array([0.0, 0.0, 0.20]), np.array([0.01]))]
    if variant == "a":
        S = _pack(X, prims, np.ones(8), 2, 4)
        return Problem("c0a", [Bundle(S, ants)], uniform_grid(8), SHARPNESS, 20.0, 100,
                       ("fwd", "filter", "bwd"))
    rng = np.random.default_rng(101)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    n = rng.normal(size=(8, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    S = SampleSet(f32(X[..., 0].ravel()), f32(X[..., 1].ravel()), f32(X[..., 2].ravel()),
                  f32(rng.uniform(-5e-3, 5e-3, 8)), f32(rng.uniform(0.5, 1.0, 8)),
                  f32(n[:, 0]), f32(n[:, 1]), f32(n[:, 2]), f32(rng.uniform(0.5, 1.0, 8)), 2, 4)
    return Problem("c0b", [Bundle(S, ants)], uniform_grid(8), 500.0, 20.0, 101,
                   ("fwd", "filter", "bwd"))


def make_c1() -> Problem:
    """BASELINE configs[0] (seed 0): 8x8 antennas on 10 cm, 64 bins, 16^3 grid in z=20-30 cm,
    sphere r=3 cm, refl U(0.5,1), power 1, 20 dB target noise."""
    seed = 0
    rng = np.random.default_rng(seed)
    ants = plane_antennas(8, 8, 0.10)
    c = -0.05 + (np.arange(16) + 0.5) * 0.00625
    zc = 0.20 + (np.arange(16) + 0.5) * 0.00625
    Xg, Yg = np.meshgrid(c, c, indexing="ij")
    X = np.zeros((256, 16, 3))
    X[:, :, 0] = Xg.ravel()[:, None]
    X[:, :, 1] = Yg.ravel()[:, None]
    X[:, :, 2] = zc[None, :]
    prims = [Prim("sphere", np.array([0.0, 0.0, 0.25]), np.array([0.03]))]
    S = _pack(X, prims, rng.uniform(0.5, 1.0, 4096), 256, 16)
    return Problem("c1", [Bundle(S, ants)], uniform_grid(64), SHARPNESS, 20.0, seed,
                   ("fwd", "filter", "bwd"))


def make_c2() -> Problem:
    """BASELINE configs[1] (seed 1): 32x32 antennas over 20 cm, 128 bins, 64^3 stratified-jittered
    samples in [-10,10]^2 x [15,27] cm; 2 boxes (4-8 cm edges) + a 2.5 cm sphere, non-overlapping;
    refl U(0.3,1); 10 dB."""
    seed = 1
    rng = np.random.default_rng(seed)
    ants = plane_antennas(32, 32, 0.20)
    lo, hi = np.array([-0.1, -0.1, 0.15]), np.array([0.1, 0.1, 0.27])
    prims = _random_prims(rng, 3, lo, hi, size_range={"box": (0.04, 0.08), "sphere": (0.025, 0.025)},
                          no_overlap=True, kinds=["box", "box", "sphere"])
    cxy = 0.2 / 64
    cz = 0.12 / 64
    ix, iy = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    px = -0.1 + (ix.ravel() + rng.random(4096)) * cxy           # jitter per column (straight ray)
    py = -0.1 + (iy.ravel() + rng.random(4096)) * cxy
    pz = 0.15 + (np.arange(64)[None, :] + rng.random((4096, 64))) * cz
    X = np.stack([np.broadcast_to(px[:, None], pz.shape), np.broadcast_to(py[:, None], pz.shape), pz], -1)
    S = _pack(X, prims, rng.uniform(0.3, 1.0, 4096 * 64), 4096, 64)
    return Problem("c2", [Bundle(S, ants)], uniform_grid(128), SHARPNESS, 10.0, seed, ("fwd", "bwd"))


def _lensless_bundle(rng, prims, origin_c, R, half_extent, u0, u1, n_rays, n_per_ray):
    """Parallel primary rays along w_p = R[:,2] with starts uniform over the aperture square."""
    wp = R[:, 2]
    st = rng.uniform(-half_extent, half_extent, (n_rays, 2))
    starts = origin_c + st[:, :1] * R[:, 0] + st[:, 1:2] * R[:, 1]
    cross = _first_crossing(prims, starts, wp, u0, u1)
    u = _mixed_depths(rng, cross, u0, u1, n_per_ray)
    X = starts[:, None, :] + u[..., None] * wp
    return X, cross


def make_c3() -> Problem:
    """BASELINE configs[2] (seed 2): 128x128 antennas at lambda/2, 256 bins, 2^20 lensless samples
    (32768 rays x 32, Q19 mix) over [-12,12]^2 x [15,30] cm; 8 spheres/boxes sizes 1-6 cm;
    refl U(0.2,1); 20 dB."""
    seed = 2
    rng = np.random.default_rng(seed)
    ants = plane_antennas(128, 128, HALF_WAVELENGTH_79GHZ, by_extent=False)
    lo, hi = np.array([-0.12, -0.12, 0.15]), np.array([0.12, 0.12, 0.30])
    prims = _random_prims(rng, 8, lo, hi, size_range=(0.01, 0.06))
    X, _ = _lensless_bundle(rng, prims, np.zeros(3), np.eye(3), 0.12, 0.15, 0.30, 32768, 32)
    S = _pack(X, prims, rng.uniform(0.2, 1.0, X.shape[0] * X.shape[1]), 32768, 32)
    return Problem("c3", [Bundle(S, ants)], uniform_grid(256), SHARPNESS, 20.0, seed,
                   ("fwd", "filter", "bwd"))


def make_c4() -> Problem:
    """BASELINE configs[3] (seed 3): 4 planes x 128x128 at lambda/2, centre R_y(90k)(0,0,-25 cm),
    facing the origin; 512 bins; per plane 32768 rays x 32 over the 16 cm cube (Q19, Q20 plane-local);
    12 primitives in [-8,8]^3 cm; refl U(0.2,1); 20 dB."""
    seed = 3
    rng = np.random.default_rng(seed)
    lo, hi = np.full(3, -0.08), np.full(3, 0.08)
    prims = _random_prims(rng, 12, lo, hi, size_range=(0.01, 0.06))
    bundles = []
    for k in range(4):
        R = _rot_y(np.pi / 2 * k)
        centre = R @ np.array([0.0, 0.0, -0.25])
        ants = plane_antennas(128, 128, HALF_WAVELENGTH_79GHZ, center=centre, R=R, by_extent=False)
        X, _ = _lensless_bundle(rng, prims, centre, R, 0.08, 0.17, 0.33, 32768, 32)
        S = _pack(X, prims, rng.uniform(0.2, 1.0, X.shape[0] * X.shape[1]), 32768, 32)
        bundles.append(Bundle(S, ants))
    return Problem("c4", bundles, uniform_grid(512), SHARPNESS, 20.0, seed, ("fwd", "bwd"))


def make_c5() -> Problem:
    """BASELINE configs[4] (seed 4): 64x64 antennas over 20 cm, 256 bins, 256^3 cell-centre grid
    over [-10,10]^2 x [15,35] cm; hollow box (outer 12 cm, wall 3 mm) around a 4 cm sphere;
    refl 0.9 on the box, 0.6 on the sphere."""
    seed = 4
    ants = plane_antennas(64, 64, 0.20)
    prims = [Prim("hollow_box", np.array([0.0, 0.0, 0.25]), np.array([0.06, 0.003]), refl=0.9),
             Prim("sphere", np.array([0.0, 0.0, 0.25]), np.array([0.02]), refl=0.6)]
    c = -0.1 + (np.arange(256) + 0.5) * (0.2 / 256)
    zc = 0.15 + (np.arange(256) + 0.5) * (0.2 / 256)
    Xg, Yg = np.meshgrid(c, c, indexing="ij")
    X = np.empty((65536, 256, 3))
    X[:, :, 0] = Xg.ravel()[:, None]
    X[:, :, 1] = Yg.ravel()[:, None]
    X[:, :, 2] = zc[None, :]
    sdf, nrm, act = scene_eval(prims, X)
    refl = np.where(act == 0, 0.9, 0.6)
    f = lambda a: np.ascontiguousarray(a.reshape(-1), dtype=np.float32)
    S = SampleSet(f(X[..., 0]), f(X[..., 1]), f(X[..., 2]), f(sdf), f(refl), f(nrm[..., 0]),
                  f(nrm[..., 1]), f(nrm[..., 2]), f(np.ones(sdf.shape)), 65536, 256)
    return Problem("c5", [Bundle(S, ants)], uniform_grid(256), SHARPNESS, 20.0, seed, ("fwd", "filter"))


MAKERS = {"c0a": lambda: make_c0("a"), "c0b": lambda: make_c0("b"), "c1": make_c1, "c2": make_c2,
          "c3": make_c3, "c4": make_c4, "c5": make_c5}


def make(name: str) -> Problem:
    return MAKERS[name]()
