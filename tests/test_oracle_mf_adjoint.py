"""Pins of the oracle's matched-filter adjoint (O7) and masked heatmap loss (O8), NEXT-1 / NEXT-3.

O7 is pinned by what the mathematics fixes, not by retyping it: central finite differences of the
heatmap loss through the oracle's own forward filter (O4), the adjoint identity of the C-linear
map s -> M, and the observation that the printed App. A.5 form (without M/|M|) fails the
finite-difference check (reading Q15).  O8 is pinned by the closed forms SPEC S:L416-430 lists.
CPU only.
"""
import numpy as np
import pytest

import oracle
import synth
from synth import AntennaSet


def _scene(n_ant=6, n_q=9, n_freq=12, seed=0, bistatic=False):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    P = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)]
    R = np.c_[rng.uniform(-0.03, 0.03, (n_ant, 2)), np.zeros(n_ant)] if bistatic else None
    A = AntennaSet(f32(P[:, 0]), f32(P[:, 1]), f32(P[:, 2]),
                   *([f32(R[:, 0]), f32(R[:, 1]), f32(R[:, 2])] if bistatic else [None] * 3))
    q = [f32(rng.uniform(-0.02, 0.02, n_q)), f32(rng.uniform(-0.02, 0.02, n_q)),
         f32(rng.uniform(0.18, 0.24, n_q))]
    grid = synth.uniform_grid(n_freq)
    s = rng.standard_normal((n_ant, n_freq)) + 1j * rng.standard_normal((n_ant, n_freq))
    return A, q, grid, s, rng


def _heat_loss(s, A, grid, q, Pgt):
    _, P = oracle.filter(s, A, grid, *q)
    return 0.5 * np.sum((P - Pgt) ** 2)


@pytest.mark.parametrize("bistatic", [False, True])
def test_o7_matches_central_finite_differences(bistatic):
    """dL/dRe s + j dL/dIm s of L = 1/2 sum (|M_q| - Pgt_q)^2, every coordinate, fp64 FD."""
    A, q, grid, s, rng = _scene(bistatic=bistatic)
    M, P = oracle.filter(s, A, grid, *q)
    Pgt = P * rng.uniform(0.2, 1.8, P.shape)
    g = oracle.filter_backward(P - Pgt, M, P, A, grid, *q, eps=1e-30)
    h = 1e-6 * np.abs(s).max()
    fd = np.zeros_like(s)
    for i in range(s.shape[0]):
        for m in range(s.shape[1]):
            for unit in (1.0, 1j):
                e = np.zeros_like(s)
                e[i, m] = unit * h
                d = (_heat_loss(s + e, A, grid, q, Pgt) - _heat_loss(s - e, A, grid, q, Pgt)) / (2 * h)
                fd[i, m] += d * (1.0 if unit == 1.0 else 1j)
    assert np.linalg.norm(g - fd) / np.linalg.norm(fd) < 1e-6


def test_o7_printed_form_without_m_over_p_fails_fd():
    """Q15: the printed gradient (1/P) dL/dP e^{-j phi} is not the derivative of
    |M|; it differs from FD by O(1) -- the reason the oracle uses G_M = dL/dP * M / P."""
    A, q, grid, s, rng = _scene(seed=3)
    M, P = oracle.filter(s, A, grid, *q)
    Pgt = P * rng.uniform(0.2, 1.8, P.shape)
    good = oracle.filter_backward(P - Pgt, M, P, A, grid, *q, eps=1e-30)
    # printed form = same adjoint applied to the REAL weight (dL/dP)/P, i.e. with M replaced by 1
    printed = oracle.filter_backward(P - Pgt, np.ones_like(M), P, A, grid, *q, eps=1e-30)
    assert np.linalg.norm(printed - good) / np.linalg.norm(good) > 0.3


def test_o7_adjoint_identity_of_the_filter_map():
    """Re<F(s), c> = Re<s, F^H(c)> for the C-linear map F: s -> M (Eq. 3); F^H is O7 with
    G_M = c (P = |c|, dL/dP = |c|, M = c)."""
    A, q, grid, s, rng = _scene(n_ant=5, n_q=13, n_freq=9, seed=7)
    c = rng.standard_normal(13) + 1j * rng.standard_normal(13)
    M, _ = oracle.filter(s, A, grid, *q)
    FH = oracle.filter_backward(np.abs(c), c, np.abs(c), A, grid, *q, eps=1e-300)
    lhs = np.real(np.vdot(c, M))           # Re sum conj(c) M
    rhs = np.real(np.vdot(FH, s))          # Re sum conj(F^H c) s
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_o7_zero_upstream_and_eps_guard():
    A, q, grid, s, _ = _scene()
    M, P = oracle.filter(s, A, grid, *q)
    assert np.all(oracle.filter_backward(np.zeros_like(P), M, P, A, grid, *q, eps=1e-12) == 0)
    # P = 0 (zero signal): finite thanks to eps, and zero because M = 0
    Z = np.zeros_like(s)
    M0, P0 = oracle.filter(Z, A, grid, *q)
    g = oracle.filter_backward(np.ones_like(P0), M0, P0, A, grid, *q, eps=1e-30)
    assert np.all(np.isfinite(g)) and np.all(g == 0)
    # reading Q15b: with eps = 0 a query at P = 0 takes the subgradient 0 of |M| at M = 0 (no 0/0),
    # and the other queries are untouched (one zeroed query leaves the rest of the sum as is)
    g0 = oracle.filter_backward(np.ones_like(P0), M0, P0, A, grid, *q, eps=0.0)
    assert np.all(np.isfinite(g0)) and np.all(g0 == 0)
    Mz, Pz = M.copy(), P.copy()
    Mz[3], Pz[3] = 0.0, 0.0
    keep = np.ones(P.shape[0], bool)
    keep[3] = False
    gz = oracle.filter_backward(np.ones_like(Pz), Mz, Pz, A, grid, *q, eps=0.0)
    gk = oracle.filter_backward(np.ones_like(Pz[keep]), M[keep], P[keep], A, grid,
                                *[c[keep] for c in q], eps=0.0)
    assert np.all(np.isfinite(gz)) and np.allclose(gz, gk, rtol=1e-12, atol=0)


def test_o7_row_subset_equals_full_rows():
    A, q, grid, s, rng = _scene()
    M, P = oracle.filter(s, A, grid, *q)
    gp = rng.standard_normal(P.shape)
    full = oracle.filter_backward(gp, M, P, A, grid, *q, eps=1e-30)
    rows = [4, 1]
    sub = oracle.filter_backward(gp, M, P, A, grid, *q, eps=1e-30, rows=rows)
    assert np.array_equal(sub, full[rows])


# ------------------------------------------------------------------------------------------ O8
def test_o8_closed_forms():
    P = np.array([1.0, 2.0, 3.0, 4.0])
    L, g, mask, _ = oracle.heatmap_loss(P, P)
    assert L == 0 and np.all(g == 0) and mask.all()                       # rendered = gt -> 0
    c = 0.5
    L, g, mask, _ = oracle.heatmap_loss(P + c, P)
    assert L == pytest.approx(4 * 0.5 * c * c, rel=1e-15) and np.allclose(g, c)


def test_o8_masking_rule_spec_examples():
    """empty history masks nothing; history 1.0 with current 0.01 and ratio 0.1 is
    masked; a cell never above the high threshold is never masked; history = running max."""
    P = np.array([0.01, 0.5, 0.02, 0.9])
    Pgt = np.array([0.3, 0.3, 0.3, 0.3])
    cell = np.array([0, 1, 2, 0])
    H0 = np.zeros(3)
    L, g, mask, H1 = oracle.heatmap_loss(P, Pgt, cell, H0, thr_hi=0.5, ratio=0.1)
    assert mask.all()                                                      # first iteration
    assert np.array_equal(H1, [0.9, 0.5, 0.02])                            # running max per cell
    H = np.array([1.0, 0.4, 1.0])
    L, g, mask, H2 = oracle.heatmap_loss(P, Pgt, cell, H, thr_hi=0.5, ratio=0.1)
    # q0: H=1.0 > 0.5, 0.01 < 0.1 -> masked; q1: cell history 0.4 <= 0.5 -> kept;
    # q2: H=1.0, 0.02 < 0.1 -> masked; q3: 0.9 >= 0.1 -> kept
    assert list(mask) == [False, True, False, True]
    exp = [not (H[c] > 0.5 and p < 0.1 * H[c]) for p, c in zip(P, cell)]
    assert list(mask) == exp
    assert g[0] == 0 and L == pytest.approx(0.5 * sum((P[k] - Pgt[k]) ** 2 for k in range(4) if exp[k]))
    assert np.all(H2 >= H)
