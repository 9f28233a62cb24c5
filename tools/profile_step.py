"""One renderer step on one config, each hot kernel launched exactly once after one warm-up step:
the target for `ncu --set full -k regex:... -s <warm-up launches> -c 3`.
  python tools/profile_step.py --config c3
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2605_29097_b200 import rfr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--ants", type=int, default=0, help="profile on the first N antennas only")
    ap.add_argument("--separate", action="store_true", help="filter and backward as two sweeps")
    a = ap.parse_args()
    p = synth.make(a.config)
    b = p.bundles[0]
    dev = torch.device("cuda:0")
    S = rfr.DeviceSamples.from_host(b.samples, dev)
    A = rfr.DeviceAntennas.from_host(b.antennas, dev)
    if a.ants:
        A = A.slice(0, a.ants)
    n, na, nf = b.samples.n, A.n, p.grid.n_freq
    ws = rfr.workspace(n, na, nf, n, dev)
    sig = torch.empty(na, nf, 2, device=dev)
    g = p.random_grad()[:na]
    G = torch.as_tensor(np.stack([g.real, g.imag], -1)).contiguous().to(dev)
    M = torch.empty(n, 2, device=dev)
    P = torch.empty(n, device=dev)
    part = torch.empty(5, n, device=dev)
    out = rfr.Grads.empty(n, dev)
    for _ in range(a.steps):
        rfr.rfr_forward(S, p.sharpness, A, p.grid, sig, ws)
        if a.separate:
            rfr.rfr_filter(sig, A, p.grid, S.x, S.y, S.z, P, ws, mf=M)
            rfr.rfr_backward_partial(G, S, p.sharpness, A, p.grid, part, ws,
                                     flags=rfr.RFR_REUSE_BLEND)
            rfr.rfr_backward_finish(part, S, p.sharpness, out, ws, flags=rfr.RFR_REUSE_BLEND)
        else:
            rfr.rfr_backward_filter(G, sig, S, p.sharpness, A, p.grid, out, P, ws, mf=M,
                                    flags=rfr.RFR_REUSE_BLEND)
        rfr.rfr_filter_backward(P, M, A, p.grid, S.x, S.y, S.z, G, ws, power=P, eps=1e-20)
    torch.cuda.synchronize()
    print("profile_step ok", a.config, rfr.rfr_launch_count())


if __name__ == "__main__":
    main()
