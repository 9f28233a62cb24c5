"""Accuracy margin of the matched filter at full size (the test_filter_sampled_queries_full_size
setting, more queries): rel-L2 of M and P against the oracle on sampled queries.  The kernel variant
comes from the environment (RFR_STDREC=0, RFR_F32G=0, RFR_TILE=0 for the A/B).
  python tests/diag_flt_acc.py [config] [n_queries]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2605_29097_b200 import rfr  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    rfr.load()
    dev = torch.device("cuda:0")
    p = synth.make(name)
    b = p.bundles[0]
    S = b.samples
    sig = p.random_grad()
    DA = rfr.DeviceAntennas.from_host(b.antennas, dev)
    q = [torch.as_tensor(np.ascontiguousarray(v, np.float32)).to(dev) for v in (S.x, S.y, S.z)]
    ws = rfr.workspace(0, b.antennas.n, p.grid.n_freq, S.n, dev)
    P = torch.empty(S.n, device=dev)
    M = torch.empty(S.n, 2, device=dev)
    X = torch.as_tensor(np.stack([sig.real, sig.imag], -1).astype(np.float32)).to(dev)
    rfr.rfr_filter(X, DA, p.grid, *q, P, ws, mf=M)
    torch.cuda.synchronize()
    st = rfr.cheb_state(ws)
    sel = np.sort(np.random.default_rng(5).choice(S.n, nq, replace=False))
    Mr, Pr = oracle.filter(sig.astype(np.complex128), b.antennas, p.grid, S.x[sel], S.y[sel],
                           S.z[sel])
    Mg = M.cpu().numpy().astype(np.float64)
    Mg = Mg[sel, 0] + 1j * Mg[sel, 1]
    Pg = P.cpu().numpy().astype(np.float64)[sel]
    rel = lambda a, r: float(np.linalg.norm(a - r) / np.linalg.norm(r))
    print(f"{name} nq={nq} env(T2RED={os.environ.get('RFR_T2RED', '1')}, V2={os.environ.get('RFR_V2', '1')}, STDREC={os.environ.get('RFR_STDREC', '1')}, "
          f"F32G={os.environ.get('RFR_F32G', '1')}, TILE={os.environ.get('RFR_TILE', '1')}) "
          f"P_tiled={st['P_tiled_filter']} plan={rfr.rfr_plan_state(ws)} relM={rel(Mg, Mr):.3e} relP={rel(Pg, Pr):.3e} "
          f"max_abs_rel={float(np.max(np.abs(Mg - Mr)) / np.max(np.abs(Mr))):.3e}")


if __name__ == "__main__":
    main()
