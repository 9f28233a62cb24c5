"""Host-side pins of the Chebyshev-moment factorisation used by the sm_100a path (rfr_cheb.cu,
DESIGN.md section 5b): the Jacobi-Anger identity with the truncation rule the device applies, and
the fp32 accuracy of Reinsch's stabilised Chebyshev recurrence.  Pure numpy/scipy (no GPU)."""
import numpy as np
import pytest
from scipy.special import jv

# device rule (k_cheb_setup): P moments for |z| <= Z_MAX[P]
Z_MAX = {16: 4.7, 24: 9.9, 28: 12.9, 32: 15.8, 48: 28.6}


def tail(P, z):
    return sum(2 * abs(jv(q, z)) for q in range(P, P + 120))


@pytest.mark.parametrize("P", sorted(Z_MAX))
def test_truncation_rule_bounds_the_tail(P):
    """sum_{p>=P} eps_p |J_p(z)| < 1e-7 for every |z| up to the threshold: the error of the
    truncated expansion relative to sum_j |c_j| (|T_p| <= 1), 10^3 below the 1e-4 tolerance."""
    for z in np.linspace(0.0, Z_MAX[P], 60):
        assert tail(P, z) < 1e-7, (P, z)


# r2 engine rule (rfr_tiled.cu t2_select_P): per-tile Horner expansions, tail < 1e-5 (below the
# ~2e-5 rad per-pair phase error of the unreduced fp32 carrier angle); global expansion t2_select_Pg
Z_MAX_TILE = {8: 1.632, 10: 2.681, 12: 3.866, 14: 4.812}
Z_MAX_GLOBAL = {16: 4.812, 20: 7.33, 24: 10.061, 28: 12.946, 32: 15.948, 48: 28.6}


@pytest.mark.parametrize("P", sorted(Z_MAX_TILE))
def test_r2_tile_rule_bounds_the_tail(P):
    for z in np.linspace(0.0, Z_MAX_TILE[P], 60):
        assert tail(P, z) < 1e-5, (P, z)
    # and the rule is not looser than needed by more than the next even P
    assert tail(P - 2, Z_MAX_TILE[P]) > 1e-5


@pytest.mark.parametrize("P", sorted(Z_MAX_GLOBAL))
def test_r2_global_rule_bounds_the_tail(P):
    for z in np.linspace(0.0, Z_MAX_GLOBAL[P], 60):
        assert tail(P, z) < 1e-7, (P, z)


def test_r2_tile_rule_matches_device_source():
    """the thresholds above are the ones compiled into t2_select_P / t2_select_Pg"""
    import os
    import re
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2605_29097_b200", "csrc",
                            "rfr_tiled.cu")).read()
    def rule(name):
        body = src[src.index(name + "(double z)"):]
        body = body[:body.index("return 0;")]
        return {int(p): float(z) for z, p in re.findall(r"z <= ([0-9.]+)\) return (\d+);", body)}
    assert rule("t2_select_P") == Z_MAX_TILE
    assert rule("t2_select_Pg") == Z_MAX_GLOBAL


@pytest.mark.parametrize("sign", [-1, 1])
def test_jacobi_anger_expansion_matches_exponential(sign):
    """exp(sign j z x) = sum_p eps_p (sign j)^p J_p(z) T_p(x): the forward uses sign = -1, the
    adjoint sign = +1 (a[m][p] and its conjugate)."""
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, 400)
    for z in (0.0, 1.7, 8.3, 13.3):
        P = 32
        T = np.cos(np.outer(np.arange(P), np.arccos(x)))
        coef = np.array([(1 if p == 0 else 2) * (sign * 1j) ** p * jv(p, z) for p in range(P)])
        approx = coef @ T
        exact = np.exp(sign * 1j * z * x)
        assert np.max(np.abs(approx - exact)) < 1e-7


def test_reinsch_recurrence_fp32_error_is_uniform_up_to_the_ends():
    """T_p(|x|) by d_{p+1} = 2(|x|-1) T_p + d_p, T_{p+1} = T_p + d_{p+1} in fp32 (as k_cheb_fwd /
    k_cheb_adj): absolute error < 3e-6 for p < 48 over all of [-1, 1], including |x| -> 1 where
    the plain three-term recurrence loses ~p^2 ulp."""
    f = np.float32
    xs = np.concatenate([np.linspace(0, 1, 4001), 1 - np.logspace(-8, -1, 100)])
    worst = 0.0
    for x in xs:
        xm1 = f(f(x) - f(1))
        t, d = f(1), xm1
        vals = [1.0]
        t = f(t + d)
        vals.append(t)
        for _ in range(2, 48):
            d = f(f(f(2) * xm1) * t + d)
            t = f(t + d)
            vals.append(t)
        exact = np.cos(np.arange(48) * np.arccos(np.float64(f(x))))
        worst = max(worst, np.max(np.abs(np.array(vals, dtype=np.float64) - exact)))
    assert worst < 3e-6, worst
