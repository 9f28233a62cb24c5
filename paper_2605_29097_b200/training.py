"""Training-loop mechanics around the renderer.

Everything numeric below runs in librfr's kernels through the C ABI; this module only arranges
device buffers and calls:

* ``AperturePatches`` -- the Signal Tracing Bank's aperture partition ("we divide the
  antenna aperture into patches, analogous to convolutional processing"; SPEC S:L184-191
  partition_aperture): contiguous grid patches of a row-major antenna grid.  The antennas are
  permuted patch-major once, so that every patch is a contiguous index range and a patch is a
  pointer offset + count at the ABI.
* ``SignalBank`` -- the memory bank: the full-aperture signal [n_ant][n_freq] lives on
  the device; each iteration traces ONE patch fresh with rfr_forward writing straight into that
  patch's rows, the other rows are the cached results of earlier iterations.
* ``RenderHeatmapLoss`` -- torch.autograd.Function for the paper's training loss:
  trace the active patch (K1, K2) -> matched filter over the whole bank at the sample points (K4)
  -> masked heatmap L2 against the ground-truth filter power (K7, dynamic masking P:L392-402);
  backward: matched-filter adjoint on the active patch rows only (K5; cached rows are constants,
  SPEC S:L195) -> tracing backward over the active patch (K3) -> blend backward (K1').
* ``FieldModel`` / ``train_step`` -- the paper's fields: SDF MLP 8x256 and
  reflectivity MLP 4x256 on a 10-level sinusoidal positional encoding, one trainable
  power scalar, normals = normalised SDF gradient.  These are plain PyTorch (cuBLAS):
  outside the renderer's hot path, which is librfr.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import torch

from . import rfr


# ------------------------------------------------------------------------------------ aperture
class AperturePatches:
    """Contiguous grid patches of a row-major n_u x n_v antenna grid (index = u * n_v + v).

    ``perm[k]`` is the original index of the k-th antenna in patch-major order; patch p occupies
    ``bounds[p] = (lo, hi)`` of that order.  Edge patches may be smaller."""

    def __init__(self, n_u: int, n_v: int, patch_u: int, patch_v: int):
        if min(n_u, n_v, patch_u, patch_v) <= 0:
            raise ValueError("grid and patch sizes must be positive")
        order: List[int] = []
        self.bounds: List[Tuple[int, int]] = []
        for pu in range(0, n_u, patch_u):
            for pv in range(0, n_v, patch_v):
                lo = len(order)
                for u in range(pu, min(pu + patch_u, n_u)):
                    for v in range(pv, min(pv + patch_v, n_v)):
                        order.append(u * n_v + v)
                self.bounds.append((lo, len(order)))
        self.perm = torch.tensor(order, dtype=torch.int64)
        self.n_ant = n_u * n_v

    @property
    def n_patches(self) -> int:
        return len(self.bounds)

    def permute_antennas(self, ants: rfr.DeviceAntennas) -> rfr.DeviceAntennas:
        idx = self.perm.to(ants.tx_x.device)
        return rfr.DeviceAntennas(*(None if getattr(ants, f) is None else
                                    getattr(ants, f).index_select(0, idx).contiguous()
                                    for f in rfr.DeviceAntennas.NAMES))

    def permute_rows(self, rows: torch.Tensor) -> torch.Tensor:
        """Rows of an [n_ant][...] array (e.g. measured signals) into patch-major order."""
        return rows.index_select(0, self.perm.to(rows.device)).contiguous()


# ------------------------------------------------------------------------------------ bank
class SignalBank:
    """Signal Tracing Bank: the full-aperture complex64 signal, one patch refreshed per call."""

    def __init__(self, ants: rfr.DeviceAntennas, patches: AperturePatches, grid, device="cuda"):
        self.ants, self.patches, self.grid = ants, patches, grid
        self.signal = torch.zeros(ants.n, grid.n_freq, 2, dtype=torch.float32, device=device)
        self.fresh = [False] * patches.n_patches       # staleness bookkeeping

    def patch_ants(self, p: int) -> rfr.DeviceAntennas:
        lo, hi = self.patches.bounds[p]
        return self.ants.slice(lo, hi)

    def trace(self, p: int, samples: rfr.DeviceSamples, sharpness: float, ws: torch.Tensor,
              flags: int = 0) -> torch.Tensor:
        """K1 + K2 for patch p, written in place into its rows of the bank (bank_step)."""
        lo, hi = self.patches.bounds[p]
        rfr.rfr_forward(samples, sharpness, self.patch_ants(p), self.grid, self.signal[lo:hi], ws,
                        flags)
        self.fresh[p] = True
        return self.signal

    def sweep(self, samples: rfr.DeviceSamples, sharpness: float, ws: torch.Tensor):
        """First full sweep: every patch traced once ("bank initialized")."""
        for p in range(self.patches.n_patches):
            self.trace(p, samples, sharpness, ws)
        return self.signal


# ------------------------------------------------------------------------------------ loss
@dataclasses.dataclass
class LossState:
    """Device-resident inputs of one RenderHeatmapLoss call that are not differentiated."""
    x: torch.Tensor
    y: torch.Tensor
    z: torch.Tensor
    n_rays: int
    n_per_ray: int
    bank: SignalBank
    patch: int
    power_gt: torch.Tensor                 # ground-truth filter power at the sample points
    ws: torch.Tensor
    cell: Optional[torch.Tensor] = None    # int32 [n_s] history cell of every sample
    history: Optional[torch.Tensor] = None # float32 [n_cells] running max of rendered power
    thr_hi: float = 0.0
    ratio: float = 0.0
    eps: float = 1e-30
    flags: int = 0
    # filled by the forward, for inspection
    power: Optional[torch.Tensor] = None
    mask: Optional[torch.Tensor] = None


class RenderHeatmapLoss(torch.autograd.Function):
    """L = 1/2 sum_q keep_q (|M_q| - Pgt_q)^2 with M = filter(bank signal) at the sample points,
    differentiable w.r.t. the per-sample fields (sdf, refl, nx, ny, nz, power) and sharpness."""

    @staticmethod
    def forward(ctx, sdf, refl, nx, ny, nz, power, sharpness: torch.Tensor, st: LossState):
        dev = sdf.device
        s_val = float(sharpness.detach().reshape(-1)[0].item())
        S = rfr.DeviceSamples(st.x, st.y, st.z, *(t.detach().contiguous() for t in
                                                  (sdf, refl, nx, ny, nz, power)),
                              n_rays=st.n_rays, n_per_ray=st.n_per_ray)
        bank = st.bank
        bank.trace(st.patch, S, s_val, st.ws, st.flags)                          # K1, K2
        n = S.n
        P = torch.empty(n, device=dev)
        M = torch.empty(n, 2, device=dev)
        rfr.rfr_filter(bank.signal, bank.ants, bank.grid, st.x, st.y, st.z, P, st.ws, mf=M)  # K4
        gP = torch.empty(n, device=dev)
        L = torch.empty(1, device=dev)
        mask = torch.empty(n, dtype=torch.uint8, device=dev)
        rfr.rfr_heatmap_loss(P, st.power_gt, gP, L, st.ws, cell=st.cell, history=st.history,
                             thr_hi=st.thr_hi, ratio=st.ratio, mask=mask)        # K7
        st.power, st.mask = P, mask
        ctx.st, ctx.S, ctx.s_val, ctx.s_shape = st, S, s_val, sharpness.shape
        ctx.save_for_backward(M, P, gP)
        return L.reshape(())

    @staticmethod
    def backward(ctx, gL):
        M, P, gP = ctx.saved_tensors
        st, S = ctx.st, ctx.S
        bank = st.bank
        lo, hi = bank.patches.bounds[st.patch]
        A = bank.patch_ants(st.patch)
        gPs = (gP * gL).contiguous()
        G = torch.empty(hi - lo, bank.grid.n_freq, 2, device=gP.device)
        rfr.rfr_filter_backward(gPs, M, A, bank.grid, st.x, st.y, st.z, G, st.ws, power=P,
                                eps=st.eps)                                      # K5
        out = rfr.Grads.empty(S.n, gP.device)
        # K1 re-runs here (no RFR_REUSE_BLEND): another call may have used st.ws between this
        # Function's forward and backward (a second loss term, an eval render), and K1 is cheap
        rfr.rfr_backward(G, S, ctx.s_val, A, bank.grid, out, st.ws, flags=st.flags)  # K1, K3, K1'
        return (out.sdf, out.refl, out.nx, out.ny, out.nz, out.power,
                out.sharpness.reshape(ctx.s_shape), None)


def render_heatmap_loss(sdf, refl, nx, ny, nz, power, sharpness, st: LossState):
    return RenderHeatmapLoss.apply(sdf, refl, nx, ny, nz, power, sharpness, st)


# ------------------------------------------------------------------------------------ fields
class PositionalEncoding(torch.nn.Module):
    """gamma(x) = (x, sin(2^k pi x), cos(2^k pi x)) for k < n_levels (N_level = 10)."""

    def __init__(self, n_levels: int = 10, scale: float = 1.0):
        super().__init__()
        self.n_levels, self.scale = n_levels, scale

    @property
    def out_dim(self) -> int:
        return 3 + 6 * self.n_levels

    def forward(self, x):
        xs = x * self.scale
        feats = [x]
        for k in range(self.n_levels):
            w = (2.0 ** k) * math.pi
            feats += [torch.sin(w * xs), torch.cos(w * xs)]
        return torch.cat(feats, -1)


def _mlp(d_in, width, depth, d_out):
    layers, d = [], d_in
    for _ in range(depth):
        layers += [torch.nn.Linear(d, width), torch.nn.Softplus(beta=100)]
        d = width
    layers.append(torch.nn.Linear(d, d_out))
    return torch.nn.Sequential(*layers)


class FieldModel(torch.nn.Module):
    """SDF MLP 8x256 + reflectivity MLP 4x256 on PE(10) and a power scalar."""

    def __init__(self, center=(0.0, 0.0, 0.25), extent=0.15, n_levels=10, width=256,
                 sdf_depth=8, refl_depth=4, init_radius=0.05):
        super().__init__()
        self.register_buffer("center", torch.tensor(center, dtype=torch.float32))
        self.extent = extent
        self.pe = PositionalEncoding(n_levels)
        self.sdf_net = _mlp(self.pe.out_dim, width, sdf_depth, 1)
        self.refl_net = _mlp(self.pe.out_dim, width, refl_depth, 1)
        self.log_power = torch.nn.Parameter(torch.zeros(()))
        self.init_radius = init_radius
        self.log_sharp = torch.nn.Parameter(torch.tensor(math.log(2e4)))

    def fields(self, X):
        """(sdf, refl, normal, power) per point; normal = grad f / |grad f|."""
        X = X.detach().requires_grad_(True)
        u = (X - self.center) / self.extent
        h = self.pe(u)
        # sphere-initialised SDF: |x - c| - r plus the learned residual
        f = (torch.linalg.norm(X - self.center, dim=-1) - self.init_radius
             + 0.01 * self.sdf_net(h).squeeze(-1))
        g, = torch.autograd.grad(f.sum(), X, create_graph=True)
        n = g / torch.linalg.norm(g, dim=-1, keepdim=True).clamp_min(1e-12)
        a = torch.sigmoid(self.refl_net(h).squeeze(-1))
        p = torch.exp(self.log_power).expand_as(a)
        return f, a, n, p


def train_step(model: FieldModel, opt: torch.optim.Optimizer, X: torch.Tensor, st: LossState):
    """One iteration: fields -> renderer loss -> backward -> optimizer step."""
    opt.zero_grad(set_to_none=True)
    f, a, n, p = model.fields(X)
    s = torch.exp(model.log_sharp)
    L = render_heatmap_loss(f.float().contiguous(), a.float().contiguous(),
                            n[:, 0].contiguous(), n[:, 1].contiguous(), n[:, 2].contiguous(),
                            p.float().contiguous(), s.reshape(1), st)
    L.backward()
    opt.step()
    return L.detach()
