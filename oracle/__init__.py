"""ctypes wrapper of the fp64 CPU oracle (oracle/rfr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.  Inputs (float32 arrays from
`synth`) are widened exactly to float64 before the call; every output is float64 / complex128.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "rfr_oracle.c")
FLAG_NO_GAIN = 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fopenmp (plain C, fp64)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", _SO, _SRC, "-lm"])
    return _SO


class _Samples(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in
                ("x", "y", "z", "sdf", "refl", "nx", "ny", "nz", "power", "phi_origin")] + \
               [("n_rays", C.c_int64), ("n_per_ray", C.c_int32)]


class _Antennas(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in
                ("tx_x", "tx_y", "tx_z", "rx_x", "rx_y", "rx_z", "phi_tx", "phi_rx")] + \
               [("n_ant", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        d, i64, i32, u32 = C.c_double, C.c_int64, C.c_int32, C.c_uint32
        pd, pi64 = P(C.c_double), P(C.c_int64)
        _lib.orc_blend.argtypes = [pd, i64, i32, d, pd, pd, pd]
        _lib.orc_pair.argtypes = [P(_Samples), i64, d, P(_Antennas), i64, u32, pd, pd]
        _lib.orc_forward.argtypes = [P(_Samples), d, P(_Antennas), d, d, i32, u32, pi64, i64, pd]
        _lib.orc_forward.restype = C.c_int
        _lib.orc_filter.argtypes = [pd, P(_Antennas), d, d, i32, pd, pd, pd, i64, pd, pd]
        _lib.orc_loss.argtypes = [pd, pd, i64, pd]
        _lib.orc_loss.restype = C.c_double
        _lib.orc_backward_partials.argtypes = [pd, P(_Samples), d, P(_Antennas), d, d, i32, u32,
                                               pi64, i64, pd]
        _lib.orc_backward_finish.argtypes = [pd, P(_Samples), d, pi64, i64] + [pd] * 7
        _lib.orc_filter_backward.argtypes = [pd, pd, pd, d, P(_Antennas), d, d, i32, pd, pd, pd,
                                             i64, pi64, i64, pd]
        _lib.orc_filter_backward.restype = C.c_int
        _lib.orc_heatmap_loss.argtypes = [pd, pd, i64, P(C.c_int32), pd, d, d, pd, P(C.c_uint8)]
        _lib.orc_heatmap_loss.restype = C.c_double
    return _lib


def _f64(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))   # exact widening of float32


def _ptr(a):
    if a is None:
        return C.POINTER(C.c_double)()
    return a.ctypes.data_as(C.POINTER(C.c_double))


class _Keep:
    """Holds the widened arrays alive while the ctypes structs point into them."""

    def __init__(self):
        self.refs = []

    def __call__(self, a):
        a = _f64(a)
        if a is not None:
            self.refs.append(a)
        return _ptr(a)


def _samples(S, keep) -> _Samples:
    return _Samples(keep(S.x), keep(S.y), keep(S.z), keep(S.sdf), keep(S.refl), keep(S.nx),
                    keep(S.ny), keep(S.nz), keep(S.power), keep(S.phi_origin),
                    int(S.n_rays), int(S.n_per_ray))


def _antennas(A, keep) -> _Antennas:
    return _Antennas(keep(A.tx_x), keep(A.tx_y), keep(A.tx_z), keep(A.rx_x), keep(A.rx_y),
                     keep(A.rx_z), keep(A.phi_tx), keep(A.phi_rx), int(A.n))


def _idx(v):
    if v is None:
        return None, C.POINTER(C.c_int64)()
    a = np.ascontiguousarray(np.asarray(v, dtype=np.int64))
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


def blend(sdf, n_rays: int, n_per_ray: int, s: float):
    """O1: (alpha, 1 - alpha, T) per sample."""
    f = _f64(sdf)
    n = n_rays * n_per_ray
    al, om, T = np.empty(n), np.empty(n), np.empty(n)
    lib().orc_blend(_ptr(f), n_rays, n_per_ray, s, _ptr(al), _ptr(om), _ptr(T))
    return al, om, T


def pair(S, j: int, s: float, A, i: int, flags: int = 0):
    """O2: (A_ij, tau_ij) for one pair."""
    keep = _Keep()
    ss, aa = _samples(S, keep), _antennas(A, keep)
    amp, tau = C.c_double(), C.c_double()
    lib().orc_pair(C.byref(ss), j, s, C.byref(aa), i, flags, C.byref(amp), C.byref(tau))
    return amp.value, tau.value


def forward(S, s: float, A, grid, flags: int = 0, rows: Optional[Sequence[int]] = None):
    """O3: signal s(i, m) for the listed antenna rows (all if None), complex128 [rows][n_freq]."""
    keep = _Keep()
    ss, aa = _samples(S, keep), _antennas(A, keep)
    ra, rp = _idx(rows)
    n_rows = A.n if rows is None else len(ra)
    out = np.zeros((n_rows, grid.n_freq, 2))
    rc = lib().orc_forward(C.byref(ss), s, C.byref(aa), grid.f0, grid.df, grid.n_freq, flags, rp,
                           n_rows, _ptr(out))
    if rc < 0:
        raise MemoryError("oracle forward")
    return out[..., 0] + 1j * out[..., 1]


def filter(signal, A, grid, qx, qy, qz):
    """O4: (M complex128 [n_q], P float64 [n_q])."""
    keep = _Keep()
    aa = _antennas(A, keep)
    sig = np.ascontiguousarray(np.stack([np.real(signal), np.imag(signal)], -1), dtype=np.float64)
    qx, qy, qz = _f64(qx), _f64(qy), _f64(qz)
    n_q = qx.shape[0]
    M = np.zeros((n_q, 2))
    P = np.zeros(n_q)
    lib().orc_filter(_ptr(sig), C.byref(aa), grid.f0, grid.df, grid.n_freq, _ptr(qx), _ptr(qy),
                     _ptr(qz), n_q, _ptr(M), _ptr(P))
    return M[:, 0] + 1j * M[:, 1], P


def loss(s, y):
    """O5: (L, G) with G = s - y."""
    a = np.ascontiguousarray(np.stack([np.real(s), np.imag(s)], -1), dtype=np.float64)
    b = np.ascontiguousarray(np.stack([np.real(y), np.imag(y)], -1), dtype=np.float64)
    G = np.zeros_like(a)
    L = lib().orc_loss(_ptr(a), _ptr(b), a.size // 2, _ptr(G))
    return L, G[..., 0] + 1j * G[..., 1]


def backward_partials(G, S, s: float, A, grid, flags: int = 0, samples=None):
    """O6a: per-sample antenna sums [n_sel][5] = (S1, S2, S3x, S3y, S3z) over the antennas in A."""
    keep = _Keep()
    ss, aa = _samples(S, keep), _antennas(A, keep)
    g = np.ascontiguousarray(np.stack([np.real(G), np.imag(G)], -1), dtype=np.float64)
    sa, sp = _idx(samples)
    n_sel = S.n if samples is None else len(sa)
    out = np.zeros((n_sel, 5))
    lib().orc_backward_partials(_ptr(g), C.byref(ss), s, C.byref(aa), grid.f0, grid.df,
                                grid.n_freq, flags, sp, n_sel, _ptr(out))
    return out


def backward_finish(partials, S, s: float, rays=None):
    """O6b: gradients dict for the listed rays (sample order = rays x n_per_ray)."""
    keep = _Keep()
    ss = _samples(S, keep)
    ra, rp = _idx(rays)
    n_r = S.n_rays if rays is None else len(ra)
    n = n_r * S.n_per_ray
    P = np.ascontiguousarray(partials, dtype=np.float64).reshape(n, 5)
    outs = {k: np.zeros(n) for k in ("sdf", "refl", "nx", "ny", "nz", "power")}
    gs = np.zeros(n_r)
    lib().orc_backward_finish(_ptr(P), C.byref(ss), s, rp, n_r, _ptr(outs["sdf"]),
                              _ptr(outs["refl"]), _ptr(outs["nx"]), _ptr(outs["ny"]),
                              _ptr(outs["nz"]), _ptr(outs["power"]), _ptr(gs))
    outs["sharpness_per_ray"] = gs
    outs["sharpness"] = float(gs.sum())
    return outs


def backward(G, S, s: float, A, grid, flags: int = 0, rays=None):
    """O6: full per-sample gradients for the listed rays (all if None)."""
    if rays is None:
        samples = None
    else:
        samples = (np.asarray(rays, np.int64)[:, None] * S.n_per_ray
                   + np.arange(S.n_per_ray)[None, :]).ravel()
    part = backward_partials(G, S, s, A, grid, flags, samples)
    return backward_finish(part, S, s, rays)


def filter_backward(grad_P, M, P, A, grid, qx, qy, qz, eps: float, rows=None):
    """O7: dL/ds(i, m) = sum_q (dL/dP_q) M_q / max(P_q, eps) e^{-j 2 pi f_m tau_iq} for the listed
    antenna rows (all if None), complex128 [rows][n_freq]."""
    keep = _Keep()
    aa = _antennas(A, keep)
    gp, Pp = _f64(grad_P), _f64(P)
    Mm = np.ascontiguousarray(np.stack([np.real(M), np.imag(M)], -1), dtype=np.float64)
    qx, qy, qz = _f64(qx), _f64(qy), _f64(qz)
    ra, rp = _idx(rows)
    n_rows = A.n if rows is None else len(ra)
    out = np.zeros((n_rows, grid.n_freq, 2))
    lib().orc_filter_backward(_ptr(gp), _ptr(Mm), _ptr(Pp), float(eps), C.byref(aa), grid.f0,
                              grid.df, grid.n_freq, _ptr(qx), _ptr(qy), _ptr(qz), qx.shape[0], rp,
                              n_rows, _ptr(out))
    return out[..., 0] + 1j * out[..., 1]


def heatmap_loss(P, P_gt, cell=None, H=None, thr_hi: float = 0.0, ratio: float = 0.0):
    """O8: (L, dL/dP, mask, H_updated) of the masked heatmap L2; H is copied, not modified."""
    Pp, Pg = _f64(P), _f64(P_gt)
    n = Pp.shape[0]
    g = np.zeros(n)
    mask = np.zeros(n, np.uint8)
    Hc = None if H is None else np.array(H, dtype=np.float64, copy=True)
    cl = None if cell is None else np.ascontiguousarray(cell, dtype=np.int32)
    L = lib().orc_heatmap_loss(_ptr(Pp), _ptr(Pg), n,
                               C.POINTER(C.c_int32)() if cl is None else
                               cl.ctypes.data_as(C.POINTER(C.c_int32)),
                               _ptr(Hc), float(thr_hi), float(ratio), _ptr(g),
                               mask.ctypes.data_as(C.POINTER(C.c_uint8)))
    return L, g, mask.astype(bool), Hc
