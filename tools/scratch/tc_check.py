"""A/B of the tcgen05 contractions (rfr_tc_gemm.cu) against the SIMT ones (RFR_T2TC=0) on c3:
forward signal, filter M and the fused call's gradients; prints rel-L2 of TC vs SIMT."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def run(tag):
    import numpy as np
    import torch
    import synth
    from paper_2605_29097_b200 import rfr
    dev = torch.device("cuda:0")
    rfr.load()
    prob = synth.make("c3")
    b = prob.bundles[0]
    S = rfr.DeviceSamples.from_host(b.samples, dev)
    A = rfr.DeviceAntennas.from_host(b.antennas, dev)
    n, na, nf = b.samples.n, b.antennas.n, prob.grid.n_freq
    ws = rfr.workspace(n, na, nf, n, dev)
    sig = torch.empty(na, nf, 2, device=dev)
    rfr.rfr_forward(S, prob.sharpness, A, prob.grid, sig, ws)
    g = torch.Generator(device="cpu").manual_seed(5)
    G = (torch.randn(na, nf, 2, generator=g) * sig.abs().mean().cpu()).to(dev)
    out = rfr.Grads.empty(n, dev)
    P = torch.empty(n, device=dev)
    M = torch.empty(n, 2, device=dev)
    rfr.rfr_backward_filter(G, sig, S, prob.sharpness, A, prob.grid, out, P, ws, mf=M)
    torch.cuda.synchronize()
    np.savez(f"/tmp/tc_{tag}.npz", sig=sig.cpu().numpy(), M=M.cpu().numpy(),
             **{k: getattr(out, k).cpu().numpy() for k in rfr.Grads.NAMES})


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1])
        sys.exit(0)
    for tag, v in (("tc", "1"), ("simt", "0")):
        subprocess.check_call([sys.executable, __file__, tag], env=dict(os.environ, RFR_T2TC=v))
    import numpy as np
    a, b = np.load("/tmp/tc_tc.npz"), np.load("/tmp/tc_simt.npz")
    for k in a.files:
        x, y = a[k].astype(np.float64), b[k].astype(np.float64)
        print(f"{k:10s} rel-L2(tc vs simt) {np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300):.3e}")
