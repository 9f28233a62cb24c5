"""The r2 engine's dense contractions on tcgen05 (rfr_tc_gemm.cu): the global
expansion of the adjoint rows G_i = Y_i conj(a) (k2_gexp_tc) and the forward's bins
s_i = e^{-j 2 pi m' u_g} a M_g,i (k2_bins_tc), both against the shared Bessel table.

Every forward / filter / backward parity test already runs them (they are the default path); here
the same calls are repeated in a subprocess with RFR_T2TC=0 (the SIMT contractions) and the two are
compared element by element, on shapes that exercise the GEMMs' edges: antenna counts that leave a
ragged last block of 128 rows, bin counts with a partial K chunk (32 bins) and a partial N chunk
(128 bins), and the oracle pins both at sampled rows / queries.  3xFP16 keeps ~22 significant bits,
so the two agree far inside the north_star tolerances (1e-4 signals, 1e-3 gradients)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [(200, 300), (256, 130), (96, 64)]     # (bins, antennas)


def problem(n_freq, n_ant, seed=7):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    npr, n_rays = 8, 500
    xy = rng.uniform(-0.04, 0.04, (n_rays, 2))
    z = np.sort(rng.uniform(0.2, 0.27, (n_rays, npr)), 1)
    X = np.concatenate([np.repeat(xy[:, None], npr, 1), z[..., None]], -1).reshape(-1, 3)
    c = np.array([0.0, 0.0, 0.235])
    d = np.linalg.norm(X - c, axis=1)
    nrm = (X - c) / d[:, None]
    S = synth.SampleSet(f32(X[:, 0]), f32(X[:, 1]), f32(X[:, 2]), f32(d - 0.025),
                        f32(rng.uniform(0.3, 1, len(X))), f32(nrm[:, 0]), f32(nrm[:, 1]),
                        f32(nrm[:, 2]), f32(rng.uniform(0.5, 1, len(X))), n_rays, npr)
    P = np.c_[rng.uniform(-0.06, 0.06, (n_ant, 2)), np.zeros(n_ant)]
    A = synth.AntennaSet(f32(P[:, 0]), f32(P[:, 1]), f32(P[:, 2]))
    return S, A, synth.uniform_grid(n_freq), 300.0


def run_case(n_freq, n_ant, out):
    """forward, filter at the samples and the fused filter + backward through the C ABI; saves
    the outputs and the plan state to `out` (npz)"""
    import torch
    from paper_2605_29097_b200 import rfr
    rfr.load()
    dev = torch.device("cuda:0")
    S, A, grid, s = problem(n_freq, n_ant)
    DS, DA = rfr.DeviceSamples.from_host(S, dev), rfr.DeviceAntennas.from_host(A, dev)
    ws = rfr.workspace(S.n, A.n, n_freq, S.n, dev)
    sig = torch.empty(A.n, n_freq, 2, device=dev)
    rfr.rfr_forward(DS, s, DA, grid, sig, ws)
    plan_fwd = rfr.rfr_plan_state(ws)
    rng = np.random.default_rng(n_freq)
    G = rng.standard_normal((A.n, n_freq, 2)).astype(np.float32)
    Gd = torch.as_tensor(G).to(dev)
    P = torch.empty(S.n, device=dev)
    M = torch.empty(S.n, 2, device=dev)
    out_g = rfr.Grads.empty(S.n, dev)
    rfr.rfr_backward_filter(Gd, sig, DS, s, DA, grid, out_g, P, ws, mf=M)
    plan_flt = rfr.rfr_plan_state(ws)
    torch.cuda.synchronize()
    np.savez(out, sig=sig.cpu().numpy(), M=M.cpu().numpy(), G=G,
             plans=json.dumps([plan_fwd, plan_flt]),
             **{k: getattr(out_g, k).cpu().numpy() for k in rfr.Grads.NAMES})


def both(n_freq, n_ant, tmp_path):
    res = {}
    for tag, v in (("tc", "1"), ("simt", "0")):
        out = str(tmp_path / f"{tag}_{n_freq}_{n_ant}.npz")
        subprocess.check_call([sys.executable, __file__, str(n_freq), str(n_ant), out], cwd=ROOT,
                              env=dict(os.environ, RFR_T2TC=v), timeout=600)
        res[tag] = np.load(out)
    return res["tc"], res["simt"]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n_freq,n_ant", CASES)
def test_tc_contractions_match_simt_and_oracle(n_freq, n_ant, tmp_path):
    tc, simt = both(n_freq, n_ant, tmp_path)
    plans = json.loads(str(tc["plans"]))
    assert all(p["applied"] == 1 and p["Pg"] > 0 for p in plans), plans   # the GEMMs ran
    for k in ("sig", "M", "sdf", "refl", "nx", "ny", "nz", "power"):
        assert np.all(np.isfinite(tc[k])), k
        assert rel(tc[k].astype(np.float64), simt[k].astype(np.float64)) <= 2e-5, k
    S, A, grid, s = problem(n_freq, n_ant)
    rows = np.unique(np.r_[0, 127, 128, n_ant - 1, np.random.default_rng(1).integers(0, n_ant, 4)])
    rows = rows[rows < n_ant]
    ref = oracle.forward(S, s, A, grid, rows=rows)
    got = tc["sig"][rows][..., 0] + 1j * tc["sig"][rows][..., 1]
    assert rel(got, ref) <= 1e-4
    q = np.sort(np.random.default_rng(2).choice(S.n, 256, replace=False))
    Sig = tc["sig"][..., 0].astype(np.float64) + 1j * tc["sig"][..., 1]
    Mr, _ = oracle.filter(Sig, A, grid, S.x[q], S.y[q], S.z[q])
    Mg = tc["M"][q][:, 0] + 1j * tc["M"][q][:, 1]
    assert rel(Mg, Mr) <= 1e-4


if __name__ == "__main__":
    run_case(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3])
