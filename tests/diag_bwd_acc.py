"""Accuracy diagnostic of the backward on sampled rays of a config: per-field rel-L2 against the
oracle for the separate backward, the fused backward+filter, for several ray draws.
  python tests/diag_bwd_acc.py --config c4 --draws 4 --rays 2"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2605_29097_b200 import rfr  # noqa: E402

FIELDS = ("sdf", "refl", "nx", "ny", "nz", "power")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--draws", type=int, default=4)
    ap.add_argument("--rays", type=int, default=2)
    ap.add_argument("--ray-list", default="", help="comma-separated ray ids (one extra draw)")
    a = ap.parse_args()
    p = synth.make(a.config)
    b = p.bundles[0]
    S, A = b.samples, b.antennas
    dev = torch.device("cuda:0")
    DS, DA = rfr.DeviceSamples.from_host(S, dev), rfr.DeviceAntennas.from_host(A, dev)
    G = p.random_grad()
    Gt = torch.as_tensor(np.stack([G.real, G.imag], -1).astype(np.float32)).to(dev)
    ws = rfr.workspace(S.n, A.n, p.grid.n_freq, S.n, dev)
    o1, o2 = rfr.Grads.empty(S.n, dev), rfr.Grads.empty(S.n, dev)
    rfr.rfr_backward(Gt, DS, p.sharpness, DA, p.grid, o1, ws)
    P = torch.empty(S.n, device=dev)
    rfr.rfr_backward_filter(Gt, Gt, DS, p.sharpness, DA, p.grid, o2, P, ws)
    torch.cuda.synchronize()
    g1 = {k: getattr(o1, k).cpu().numpy().astype(np.float64) for k in FIELDS}
    g2 = {k: getattr(o2, k).cpu().numpy().astype(np.float64) for k in FIELDS}
    print("fused vs separate max rel diff per field:",
          {k: float(np.linalg.norm(g1[k] - g2[k]) / max(np.linalg.norm(g1[k]), 1e-30)) for k in FIELDS})
    f = S.sdf.reshape(S.n_rays, S.n_per_ray)
    crossing = np.nonzero((f.min(1) < 0) & (f.max(1) > 0))[0]
    draws = [np.sort(np.random.default_rng(100 + d).choice(crossing, a.rays, replace=False))
             for d in range(a.draws)]
    if a.ray_list:
        draws.insert(0, np.array([int(v) for v in a.ray_list.split(",")]))
    for d, rays in enumerate(draws):
        idx = (rays[:, None] * S.n_per_ray + np.arange(S.n_per_ray)[None, :]).ravel()
        ref = oracle.backward(G.astype(np.complex128), S, p.sharpness, A, p.grid, rays=rays)
        e1 = {k: float(np.linalg.norm(g1[k][idx] - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300)) for k in FIELDS}
        e2 = {k: float(np.linalg.norm(g2[k][idx] - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300)) for k in FIELDS}
        print("draw", d, "rays", rays.tolist())
        print("  sep  ", {k: f"{v:.2e}" for k, v in e1.items()})
        print("  fused", {k: f"{v:.2e}" for k, v in e2.items()})
        # which sample dominates the sdf error
        k = "sdf"
        err = np.abs(g1[k][idx] - ref[k])
        i = int(np.argmax(err))
        print(f"  sdf worst sample {idx[i]}: gpu {g1[k][idx][i]:.6e} ref {ref[k][i]:.6e}; |ref| max {np.abs(ref[k]).max():.3e}")
        if d == 0 and a.ray_list:
            np.set_printoptions(linewidth=200, precision=6)
            for k in ("sdf", "refl", "power"):
                print(" ", k, "gpu", g1[k][idx]); print(" ", k, "ref", ref[k])
            # the raw partials: S1 for these samples from the separate path
            part = torch.empty(5, S.n, device=dev)
            rfr.rfr_backward_partial(Gt, DS, p.sharpness, DA, p.grid, part, ws)
            torch.cuda.synchronize()
            pc = part.cpu().numpy().astype(np.float64)[:, idx]
            print("  S1", pc[0]); print("  S2", pc[1])
            pr = oracle.backward_partials(G.astype(np.complex128), S, p.sharpness, A, p.grid,
                                          samples=idx)
            pr = np.asarray(pr).reshape(len(idx), 5)
            print("  S1 ref", pr[:, 0]); print("  S2 ref", pr[:, 1])
            for c in range(5):
                print("  partial", c, "rel-L2", np.linalg.norm(pc[c] - pr[:, c]) / np.linalg.norm(pr[:, c]))


if __name__ == "__main__":
    main()
