#!/usr/bin/env python
"""Benchmark of the renderer's hot path: one step = blend (K1) + forward (K2) + matched filter (K4)
+ loss (K6) + backward (K3, K1') over one synthetic batch, on N GPUs of one node.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl librfr|reference]
  (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N)

Metric (BASELINE.json): render fwd+bwd G contributions/s, one contribution = one (sample x antenna
x frequency-bin) term.  value = N_c / t_step where N_c = sum over bundles of N_s * N_a * N_f and
t_step is the device time of the whole step (filter and loss included, max over ranks).  Antennas
are sharded across ranks (strong scaling); the backward partials and the filter's complex M are
all-reduced with NCCL.  --impl reference times the fp64 CPU oracle on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")
METRIC = "render fwd+bwd G contributions/s (pts×antennas×freqs) at 1/2/4/8 B200"
N_SM = 148
FP32_LANES_PER_SM = 128
# FP32-pipe lane-operations per contribution:
#   forward  : 1 FFMA2 + 1 FADD2 = 4 lane-ops (Chebyshev step + accumulate)
#   backward : 2 FFMA2           = 4 lane-ops (complex Horner step)
#   filter   : 2 FFMA2           = 4 lane-ops
OPS_PER_CONTRIB = 4
# K3/K4 on tensor cores: D = A.B^T per 16-bin block, 4 real MACs per contribution, 3 fp16 products
# (3xFP16 split, tcgen05.mma kind::f16 with fp32 accumulation)
TC_FLOP_PER_CONTRIB = 24


def peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0, "fallback": True}


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(self.rows)}


# ===================================================================================== oracle arm
def oracle_sample_rates(prob, budget_s: float = 20.0, threads: int | None = None):
    """Time the fp64 oracle, as it stands, on bounded samples of the workload: a few antenna rows
    of the forward, a few queries of the filter, a few rays of the backward.  Returns per-pass
    contributions/s and the description of the sample."""
    import oracle
    b = prob.bundles[0]
    S, A, grid = b.samples, b.antennas, prob.grid
    per_row = S.n * grid.n_freq
    cores = threads or os.cpu_count()
    rate_guess = 3e7 * cores                      # ~30 ns / contribution / core
    rows = max(1, int(budget_s / 3 * rate_guess / per_row))
    rows = min(rows, A.n)
    t = time.perf_counter()
    oracle.forward(S, prob.sharpness, A, grid, rows=np.arange(rows))
    t_f = time.perf_counter() - t
    r_f = rows * per_row / t_f
    nq = max(1, min(S.n, int(budget_s / 3 * r_f / (A.n * grid.n_freq))))
    sig = prob.random_grad().astype(np.complex128)
    t = time.perf_counter()
    oracle.filter(sig, A, grid, S.x[:nq], S.y[:nq], S.z[:nq])
    t_q = time.perf_counter() - t
    r_q = nq * A.n * grid.n_freq / t_q
    n_rays = max(1, min(S.n_rays, int(budget_s / 3 * r_f / (S.n_per_ray * A.n * grid.n_freq))))
    t = time.perf_counter()
    oracle.backward(sig, S, prob.sharpness, A, grid, rays=np.arange(n_rays))
    t_b = time.perf_counter() - t
    r_b = n_rays * S.n_per_ray * A.n * grid.n_freq / t_b
    sample = (f"{prob.name} bundle 0: forward {rows} antenna rows x {S.n} samples x "
              f"{grid.n_freq} bins; filter {nq} queries x {A.n} antennas; backward {n_rays} rays "
              f"x {S.n_per_ray} samples x {A.n} antennas")
    return {"fwd": r_f, "filter": r_q, "bwd": r_b, "sample": sample, "cores": cores,
            "seconds": t_f + t_q + t_b}


def step_rate(r):
    """contributions/s of a step (fwd + filter + bwd over the same N_c each), as value = N_c/t."""
    return 1.0 / (1.0 / r["fwd"] + 1.0 / r["filter"] + 1.0 / r["bwd"])


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synth
    prob = synth.make(args.config)
    vals = []
    t0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        r = oracle_sample_rates(prob, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append(step_rate(r))
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v / 1e9, "unit": "G contributions/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": prob.n_contrib / v * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n_contrib_per_pass": prob.n_contrib,
                       "note": "fp64 CPU oracle on bounded samples; ms_per_step projected"},
            "cpu_baseline": {"value": v / 1e9, "unit": "G contributions/s", "cores": r["cores"],
                             "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": v / 1e9, "unit": "G contributions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


# ===================================================================================== GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2605_29097_b200 import rfr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rfr.load()
    # librfr's own NCCL communicator carries the data-path all-reduces (a4 M, a7 partials)
    comm = rfr.Comm.create() if world > 1 else None
    prob = synth.make(args.config)
    grid = prob.grid
    st = torch.cuda.current_stream()

    # ---------------- per-bundle device state
    B = []
    sum_F2 = torch.zeros(1, dtype=torch.float64, device=dev)
    n_F = 0
    for k, b in enumerate(prob.bundles):
        lo, hi = rfr.shard_range(b.antennas.n, rank, world)
        DS = rfr.DeviceSamples.from_host(b.samples, dev)
        DA = rfr.DeviceAntennas.from_host(b.antennas, dev).slice(lo, hi)
        n, na = b.samples.n, hi - lo
        ws = rfr.workspace(n, na, grid.n_freq, n, dev)
        st_k = dict(k=k, lo=lo, hi=hi, S=DS, A=DA, n=n, na=na, ws=ws,
                    sig=torch.empty(na, grid.n_freq, 2, device=dev),
                    G=torch.empty(na, grid.n_freq, 2, device=dev),
                    loss=torch.empty(1, device=dev),
                    M=torch.empty(n, 2, device=dev), P=torch.empty(n, device=dev),
                    part=torch.empty(5, n, device=dev), out=rfr.Grads.empty(n, dev))
        # target y = F(scene) + complex noise at the config's SNR (reading Q18), built untimed
        rfr.rfr_forward(DS, prob.sharpness, DA, grid, st_k["sig"], ws)
        sum_F2 += (st_k["sig"].double() ** 2).sum()
        n_F += na * grid.n_freq
        B.append(st_k)
    if world > 1:
        dist.all_reduce(sum_F2)
    n_F_tot = sum(b.antennas.n for b in prob.bundles) * grid.n_freq
    sigma = float(torch.sqrt(sum_F2 / n_F_tot / 10 ** (prob.snr_db / 10)).item())
    for st_k in B:
        nz = prob.noise_unit(st_k["k"])[st_k["lo"]:st_k["hi"]]
        noise = torch.as_tensor(np.stack([nz.real, nz.imag], -1).astype(np.float32)).to(dev)
        st_k["y"] = st_k["sig"] + sigma * noise
    torch.cuda.synchronize()

    ev = lambda: torch.cuda.Event(enable_timing=True)

    heat = args.step == "heatmap"
    fused = not args.separate and not heat
    if heat:
        # NEXT-1: the paper's heatmap-domain L2.  Ground-truth heatmap = the filter of
        # the noisy target y at the same queries (the samples), built untimed
        for s in B:
            s["P_gt"] = torch.empty(s["n"], device=dev)
            s["gP"] = torch.empty(s["n"], device=dev)
            rfr.rfr_filter(s["y"], s["A"], grid, s["S"].x, s["S"].y, s["S"].z, s["P_gt"], s["ws"],
                           comm=comm)
        torch.cuda.synchronize()

    def step(rec=None):
        # fused (default): K2 forward, K6 loss, then K3 + K4 in one tensor-core sweep
        # (rfr_backward_filter: filter queries = the samples).  --separate: rfr_filter before the
        # loss and rfr_backward after it, as two sweeps.
        for s in B:
            e = [ev() for _ in range(5)] if rec is not None else None
            if e: e[0].record(st)
            rfr.rfr_forward(s["S"], prob.sharpness, s["A"], grid, s["sig"], s["ws"])
            if e: e[1].record(st)
            if not fused:
                rfr.rfr_filter(s["sig"], s["A"], grid, s["S"].x, s["S"].y, s["S"].z, s["P"],
                               s["ws"], mf=s["M"], comm=comm)
            if e: e[2].record(st)
            if heat:
                # K7 heatmap L2, then K5 (matched-filter adjoint) turns dL/dP into dL/ds
                rfr.rfr_heatmap_loss(s["P"], s["P_gt"], s["gP"], s["loss"], s["ws"])
                rfr.rfr_filter_backward(s["gP"], s["M"], s["A"], grid, s["S"].x, s["S"].y,
                                        s["S"].z, s["G"], s["ws"], power=s["P"], eps=1e-20)
            else:
                rfr.rfr_loss(s["sig"], s["y"], s["G"], s["loss"], s["ws"])
            if e: e[3].record(st)
            if fused:
                rfr.rfr_backward_filter(s["G"], s["sig"], s["S"], prob.sharpness, s["A"], grid,
                                        s["out"], s["P"], s["ws"], mf=s["M"],
                                        flags=rfr.RFR_REUSE_BLEND, comm=comm)
            else:
                rfr.rfr_backward(s["G"], s["S"], prob.sharpness, s["A"], grid, s["out"], s["ws"],
                                 flags=rfr.RFR_REUSE_BLEND, comm=comm)
            if e:
                e[4].record(st)
                rec.append(e)

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # which path the device chose (Chebyshev moments or direct kernels): one forward and one
    # backward on bundle 0, read back from the workspace header (untimed diagnostic)
    s0 = B[0]
    rfr.rfr_forward(s0["S"], prob.sharpness, s0["A"], grid, s0["sig"], s0["ws"])
    cf = rfr.cheb_state(s0["ws"])
    p_flt_sep = p_k5 = 0
    if not fused:
        rfr.rfr_filter(s0["sig"], s0["A"], grid, s0["S"].x, s0["S"].y, s0["S"].z, s0["P"],
                       s0["ws"], mf=s0["M"])
        cq = rfr.cheb_state(s0["ws"])
        p_flt_sep = cq["P_tiled_filter"] if cq["sel"] else 0
    if heat:
        rfr.rfr_heatmap_loss(s0["P"], s0["P_gt"], s0["gP"], s0["loss"], s0["ws"])
        rfr.rfr_filter_backward(s0["gP"], s0["M"], s0["A"], grid, s0["S"].x, s0["S"].y, s0["S"].z,
                                s0["G"], s0["ws"], power=s0["P"], eps=1e-20)
        ck = rfr.cheb_state(s0["ws"])
        # tiled K5 (DESIGN 6b) publishes its own P like the tiled filter; RFR_TILE=0: untiled
        p_k5 = ((ck["P_tiled_filter"] if os.environ.get("RFR_TILE") != "0" else ck["P"])
                if ck["sel"] else 0)
    if fused:
        rfr.rfr_backward_filter(s0["G"], s0["sig"], s0["S"], prob.sharpness, s0["A"], grid,
                                s0["out"], s0["P"], s0["ws"], mf=s0["M"], flags=rfr.RFR_REUSE_BLEND)
    else:
        rfr.rfr_backward_partial(s0["G"], s0["S"], prob.sharpness, s0["A"], grid, s0["part"],
                                 s0["ws"], flags=rfr.RFR_REUSE_BLEND)
    ca = rfr.cheb_state(s0["ws"])
    cheb_fwd_P = cf["P"] if cf["sel"] else 0
    cheb_adj_P = ca["P"] if ca["sel"] else 0
    # empty-space skipping: samples that carry forward / backward work (bundle 0)
    act_fwd = cf["n_active_fwd"] / s0["n"]
    act_bwd = ca["n_active_bwd"] / s0["n"]
    barrier()

    # ---------------- timed region: K steps, per-step events, L2 flushed between steps
    n0 = rfr.rfr_launch_count()
    step_ms, seg = [], {"fwd": 0.0, "filter": 0.0, "loss": 0.0, "bwd": 0.0}
    with ClockSampler(local) as clk:
        barrier()
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            s0, s1 = ev(), ev()
            recs = []
            s0.record(st)
            step(recs)
            s1.record(st)
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            for e in recs:
                seg["fwd"] += e[0].elapsed_time(e[1])
                seg["filter"] += e[1].elapsed_time(e[2])
                seg["loss"] += e[2].elapsed_time(e[3])
                seg["bwd"] += e[3].elapsed_time(e[4])
        barrier()
        t_wall = time.perf_counter() - t_wall
    launches = rfr.rfr_launch_count() - n0
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms, seg["fwd"], seg["filter"], seg["loss"], seg["bwd"]], device=dev,
                     dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, f_ms, q_ms, l_ms, b_ms = (float(v) for v in t.tolist())
    ms_per_step = tot_ms / args.steps
    Nc = prob.n_contrib
    value = Nc / (ms_per_step * 1e-3)

    # ---------------- e2e: same step through the ABI with host buffers (pinned) every step
    e2e = run_e2e(args, prob, B, rfr, torch, dist, world, dev, st, step)

    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return 0
    pk = peaks()
    clocks = clk.summary()
    peak_ops = N_SM * FP32_LANES_PER_SM * pk.get("sm_max_mhz", 1965.0) * 1e6
    # fp16 tensor peak (kind::f16 runs at the bf16 rate): the measured bf16 burst peak
    bf16 = pk.get("bf16_tflops", 1590.0)
    peak_f16 = bf16 * 1e12
    tc = os.environ.get("RFR_ADJOINT", "tc") != "simt" and grid.n_freq in (128, 256, 512)
    per_step = lambda ms: ms / args.steps
    clk_ratio = (clocks["sm_mhz"] / pk.get("sm_max_mhz", 1965.0)) if clocks.get("sm_mhz") else None
    roofs = []
    n_pairs = sum(b.samples.n * b.antennas.n for b in prob.bundles) / world
    if cheb_fwd_P:
        # Chebyshev-moment forward: per pair P steps of 1 FFMA + 1 FADD (Reinsch recurrence) +
        # 1 FFMA2 (complex-real moment update) = 4 P FP32 lane-ops, over
        # the pairs of the samples that carry an amplitude (empty-space skipping, section 5c)
        ach = 4 * cheb_fwd_P * n_pairs * act_fwd / (per_step(f_ms) * 1e-3)
        roofs.append({"kernel": f"k_cheb_fwd<P={cheb_fwd_P}> (rfr_forward)", "bound": "alu",
                      "achieved": ach / 1e12, "peak": peak_ops / 1e12,
                      "unit": "T FP32 lane-ops/s", "frac": ach / peak_ops,
                      "lane_ops_per_pair": 4 * cheb_fwd_P, "active_sample_fraction": act_fwd,
                      "ms_per_step": per_step(f_ms)})
    else:
        # K2 forward: FP32-pipe bound, 4 lane-ops per contribution (1 FFMA2 + 1 FADD2)
        ach = OPS_PER_CONTRIB * (Nc / world) / (per_step(f_ms) * 1e-3)
        roofs.append({"kernel": "k_trace_fwd (K2, rfr_forward)", "bound": "alu",
                      "achieved": ach / 1e12, "peak": peak_ops / 1e12, "unit": "T FP32 lane-ops/s",
                      "frac": ach / peak_ops,
                      "frac_at_measured_clock": ach / (peak_ops * clk_ratio) if clk_ratio else None,
                      "ms_per_step": per_step(f_ms)})
    tiled = os.environ.get("RFR_TILE") != "0"

    def lops(P):
        # FP32 lane-ops per (point, antenna) pair of one tiled Chebyshev sweep: per moment one
        # complex-real FFMA2 (2) + the recurrence: plain three-term at P <= 16 (1, DESIGN 5d),
        # Reinsch otherwise (2)
        return (3 if (P <= 16 and os.environ.get("RFR_STDREC") != "0") else 4) * P

    if cheb_adj_P:
        # fused call: the tiled filter over every pair + the tiled backward over the pairs of the
        # samples with alpha != 0 (section 5c), both at the tiled P published by the call
        p_t = (ca.get("P_tiled_filter") or cheb_adj_P) if tiled else cheb_adj_P
        ops = lops(p_t) if tiled else 4 * cheb_adj_P
        work = n_pairs * ((1.0 + act_bwd) if fused else act_bwd)
        for name, ms in ([("k_tile_flt4+k_tile_bwd (filter + backward, rfr_backward_filter)", b_ms)]
                         if fused else [("k_tile_bwd (backward, rfr_backward)", b_ms)]):
            ach = ops * work / (per_step(ms) * 1e-3)
            roofs.append({"kernel": (f"{name.split()[0]}<P={p_t}> " if tiled else
                                     f"k_cheb_adj<P={cheb_adj_P}> ") + " ".join(name.split()[1:]),
                          "bound": "alu", "achieved": ach / 1e12, "peak": peak_ops / 1e12,
                          "unit": "T FP32 lane-ops/s", "frac": ach / peak_ops,
                          "lane_ops_per_pair": ops, "active_sample_fraction": act_bwd,
                          "ms_per_step": per_step(ms)})
    if p_flt_sep:
        # tiled Chebyshev filter (section 5d) over every (sample, antenna) pair
        ach = lops(p_flt_sep) * n_pairs / (per_step(q_ms) * 1e-3)
        roofs.append({"kernel": f"k_tile_flt4<P={p_flt_sep}> (K4, rfr_filter)", "bound": "alu",
                      "achieved": ach / 1e12, "peak": peak_ops / 1e12,
                      "unit": "T FP32 lane-ops/s", "frac": ach / peak_ops,
                      "lane_ops_per_pair": lops(p_flt_sep), "ms_per_step": per_step(q_ms)})
    if p_k5:
        # K5 = a forward-shaped Chebyshev sweep over the queries, per
        # (query, antenna) pair; its segment also holds the (negligible) K7 heatmap loss
        o5 = lops(p_k5) if tiled else 4 * p_k5
        ach = o5 * n_pairs / (per_step(l_ms) * 1e-3)
        k5 = "k_tile_fwd" if tiled else "k_cheb_fwd"
        roofs.append({"kernel": f"{k5}<P={p_k5},MFAdj> (K5+K7, rfr_filter_backward)",
                      "bound": "alu", "achieved": ach / 1e12, "peak": peak_ops / 1e12,
                      "unit": "T FP32 lane-ops/s", "frac": ach / peak_ops,
                      "lane_ops_per_pair": o5, "ms_per_step": per_step(l_ms)})
    if cheb_adj_P:
        pass
    elif fused:
        adj = [("k_adjoint_tc<both> (K3+K4 fused +K1', rfr_backward_filter)", b_ms, 2)]
    else:
        adj = [("k_adjoint_tc<bwd> (K3+K1', rfr_backward)", b_ms, 1),
               ("k_adjoint_tc<flt> (K4, rfr_filter)", q_ms, 1)]
    if cheb_adj_P:
        adj = []
    for name, ms, npass in adj:
        rate = npass * (Nc / world) / (per_step(ms) * 1e-3)     # contributions of all its passes
        if tc:
            # exact 16-bin block factorisation on tcgen05 kind::f16, 3xFP16: per contribution
            # 4 real MACs x 3 products = 24 tensor FLOP
            ach = TC_FLOP_PER_CONTRIB * rate
            roofs.append({"kernel": name, "bound": "tensor", "achieved": ach / 1e12,
                          "peak": peak_f16 / 1e12, "unit": "T f16 FLOP/s", "frac": ach / peak_f16,
                          "alu_equivalent_frac": OPS_PER_CONTRIB * rate / peak_ops,
                          "ms_per_step": per_step(ms)})
        else:
            ach = OPS_PER_CONTRIB * rate
            roofs.append({"kernel": name.replace("_tc", ""), "bound": "alu", "achieved": ach / 1e12,
                          "peak": peak_ops / 1e12, "unit": "T FP32 lane-ops/s",
                          "frac": ach / peak_ops, "ms_per_step": per_step(ms)})
    dom = max(roofs, key=lambda r: r["ms_per_step"])
    traffic = None
    try:   # bytes per launch from the committed full-size ncu capture (profiles/traffic.json)
        key = dom["kernel"].split()[0].split("<P=")[0]
        traffic = json.load(open(TRAFFIC_PATH)).get(args.config, {}).get(key)
    except Exception:
        pass
    roof = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
            "unit": dom["unit"], "frac": dom["frac"], "traffic": traffic, "kernel": dom["kernel"],
            "peak_note": ("148 SM x 128 FP32 lanes x sm_max_mhz (MEASURED_PEAKS.json); "
                          + (f"{dom['lane_ops_per_pair']} lane-ops per (sample, antenna) pair "
                             "(Chebyshev moments)" if "lane_ops_per_pair" in dom else
                             "4 lane-ops per contribution") if dom["bound"] == "alu" else
                          "measured bf16 burst peak (kind::f16 runs at the bf16 rate); 24 tensor "
                          "FLOP per contribution (3xFP16)")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = oracle_sample_rates(prob, budget_s=args.ref_budget)
        cpu = {"value": step_rate(r) / 1e9, "unit": "G contributions/s", "cores": r["cores"],
               "kind": "oracle", "sample": r["sample"],
               "per_pass_G_per_s": {k: r[k] / 1e9 for k in ("fwd", "filter", "bwd")}}
    line = {"metric": METRIC, "value": value / 1e9, "unit": "G contributions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n_contrib_per_pass": Nc,
                       "bundles": len(prob.bundles),
                       "n_samples": [b.samples.n for b in prob.bundles][0],
                       "n_antennas": [b.antennas.n for b in prob.bundles][0],
                       "n_freq": grid.n_freq, "parallelism": f"antenna-shard x{world}",
                       "l2": "flushed between steps (512 MiB memset, outside the step events)",
                       "loss": "heatmap L2 (NEXT-1)" if heat else "signal-domain complex residual",
                       "step": ("K1 blend + forward + K4 filter (+NCCL all-reduce of M) + K7 "
                                "heatmap loss + K5 matched-filter adjoint + K3 backward (+NCCL "
                                "all-reduce of partials) + K1' finish" if heat else
                                "K1 blend + forward + K6 loss + K3/K4 fused backward + "
                                "matched filter at the samples (+NCCL all-reduce of partials and "
                                "M) + K1' finish" if fused else
                                "K1 blend + forward + K4 filter (+NCCL all-reduce of M) + K6 "
                                "loss + K3 backward (+NCCL all-reduce of partials) + K1' finish")},
            "passes": ({"fwd_G_per_s": Nc / (per_step(f_ms) * 1e-3) / 1e9,
                        "filter_plus_bwd_fused_G_per_s": Nc / (per_step(b_ms) * 1e-3) / 1e9,
                        "loss_ms": per_step(l_ms), "fwd_ms": per_step(f_ms),
                        "filter_plus_bwd_ms": per_step(b_ms)} if fused else
                       {"fwd_ms": per_step(f_ms), "filter_ms": per_step(q_ms),
                        "heat_loss_plus_k5_ms": per_step(l_ms), "bwd_ms": per_step(b_ms),
                        "k5_G_per_s": Nc / (per_step(l_ms) * 1e-3) / 1e9} if heat else
                       {"fwd_G_per_s": Nc / (per_step(f_ms) * 1e-3) / 1e9,
                        "filter_G_per_s": Nc / (per_step(q_ms) * 1e-3) / 1e9,
                        "bwd_G_per_s": Nc / (per_step(b_ms) * 1e-3) / 1e9,
                        "fwd_plus_bwd_G_per_s": Nc / (per_step(f_ms + b_ms) * 1e-3) / 1e9,
                        "loss_ms": per_step(l_ms)}),
            "method": {"forward": f"chebyshev-moments P={cheb_fwd_P} (delta={cf['delta']:.4g} cycles)"
                       if cheb_fwd_P else "direct recurrence (K2)",
                       "adjoint": (f"chebyshev-moments P={cheb_adj_P} (delta={ca['delta']:.4g} "
                                   f"cycles); tiled filter P={ca.get('P_tiled_filter')}")
                       if cheb_adj_P else "tensor-core 16-bin block GEMM",
                       "empty_space_skipping": {
                           "forward_active_samples": act_fwd, "backward_active_samples": act_bwd,
                           "note": "samples whose amplitude (forward) or alpha (backward) is exactly "
                                   "0 in fp32 are skipped; value still counts every (sample, "
                                   "antenna, bin) of the batch (the metric's definition)"}},
            "roofline": roof, "rooflines": roofs, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "wall_s_timed": t_wall}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, prob, B, rfr, torch, dist, world, dev, st, step):
    """Same step measured end to end through the public API: every step copies its inputs
    (samples, local antennas, local target rows) host->device from pinned buffers and reads the
    result (loss + per-sample gradients) device->host."""
    host_in, dev_in, host_out, dev_out = [], [], [], []
    for s in B:
        for f in rfr.DeviceSamples.FIELDS:
            d = getattr(s["S"], f)
            host_in.append(d.cpu().pin_memory()); dev_in.append(d)
        for f in ("tx_x", "tx_y", "tx_z"):
            d = getattr(s["A"], f)
            host_in.append(d.cpu().pin_memory()); dev_in.append(d)
        tgt = s["P_gt"] if "P_gt" in s else s["y"]      # heatmap step: the target heatmap
        host_in.append(tgt.cpu().pin_memory()); dev_in.append(tgt)
        for f in ("sdf", "refl", "nx", "ny", "nz", "power", "sharpness"):
            d = getattr(s["out"], f)
            host_out.append(torch.empty(d.shape, dtype=d.dtype).pin_memory()); dev_out.append(d)
        host_out.append(torch.empty(1).pin_memory()); dev_out.append(s["loss"])
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        e0, e1 = ev(), ev()
        e0.record(st)
        for h, d in zip(host_in, dev_in):
            d.copy_(h, non_blocking=True)
        step()
        for h, d in zip(host_out, dev_out):
            h.copy_(d, non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(ms) / steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    v = prob.n_contrib / (float(t.item()) * 1e-3)
    return {"value": v / 1e9, "unit": "G contributions/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="librfr", choices=["librfr", "reference"])
    ap.add_argument("--ref-budget", type=float, default=20.0,
                    help="seconds of oracle work per reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--step", default="signal", choices=["signal", "heatmap"],
                    help="signal: the north_star step (signal-domain residual, default); heatmap: "
                         "the paper's heatmap-domain L2 through the matched-filter adjoint K5 "
                         "(SURVEY 8f NEXT-1)")
    ap.add_argument("--separate", action="store_true",
                    help="filter and backward as two sweeps (rfr_filter + rfr_backward)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
