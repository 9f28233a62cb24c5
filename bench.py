#!/usr/bin/env python
"""Benchmark of the renderer's hot path on N GPUs of one node.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl librfr|reference]
  (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N)

One step = the config's passes (BASELINE.json configs / synth Problem.passes) over one synthetic
batch: K1 blend + forward (a1-a3), then
  fwd + filter + bwd (c1, c3): loss (a5) + the fused filter at the samples and backward (a4, a6-a8);
  fwd + bwd (c2, c4):          loss + backward;
  fwd + filter (c5):           the matched filter at the samples.
Metric (BASELINE.json): render fwd+bwd G contributions/s, one contribution = one (sample x antenna
x frequency-bin) term.  value = N_c / t_step, N_c = sum over bundles of N_s * N_a * N_f, t_step the
device time of the whole step (max over ranks).  Antennas are sharded across ranks; the backward
partials and the filter's complex M are all-reduced with NCCL (or, --filter-collective gather, the
signal rows are all-gathered and the queries sharded).  --impl reference times the fp64 CPU oracle
on bounded samples.  --emulate-world N --emulate-rank r times rank r's whole share of an N-GPU run
on one GPU (collectives excluded, reported as such).  --dense runs c3 with s = 200 / m, where no
sample is skipped (every alpha is non-zero: the early-training regime).
"""
from __future__ import annotations

import argparse
import dataclasses
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
METRIC = "render fwd+bwd G contributions/s (pts\u00d7antennas\u00d7freqs) at 1/2/4/8 B200"
N_SM = 148
FP32_LANES_PER_SM = 128
XU_LANES_PER_SM = 16


# Algorithmic work per (point, antenna) pair of the r2 engine's sweeps, in
# FP32 lane-operations (one fp32 FMA / MUL / ADD on one lane) and XU operations (MUFU):
#   pair geometry (all sweeps): delta = |q'|^2 - 2 a'.q' (3), s2 = D + delta (1), d = s2 rsqrt(s2)
#     (1), d + d_a (1), d - d_a = delta / (d + d_a) (1), cycles (1), reduction to [-1/2, 1/2] (3),
#     angle (1), x (1)                                             = 13 lane-ops, 4 XU (rsqrt, rcp,
#                                                                    sin, cos)
#   filter:   Horner over P monomial coefficients: (P - 1) complex x real FMAs = 2 (P - 1);
#             carrier M += E h (complex MAC)                       = 4
#   backward: Horner 2 (P - 1); R = Re(E h) (2); Eq. 5 sums U, V (gain 3, gamma 2, U 1, F 2,
#             sum F 1, W 3)                                        = 14
#   forward:  per moment one complex x real FMA (2) + the recurrence (1) = 3 P; amplitude
#             (n.d 3, gain 3, gamma / A 3, c = A E 2)              = 11
def lane_ops_per_pair(sweep: str, P: int) -> int:
    geo = 13
    if sweep == "filter":
        return geo + 2 * (P - 1) + 4
    if sweep == "backward":
        return geo + 2 * (P - 1) + 2 + 14
    return geo + 3 * P + 11


def moment_ops_per_pair(sweep: str, P: int) -> int:
    """The moment / polynomial part alone (the r1 accounting, for comparison)."""
    return 2 * (P - 1) + (4 if sweep == "filter" else 2) if sweep != "forward" else 3 * P


# MUFU per pair: rsqrt, rcp, sin, cos; the filter's default geometry (t2_geo1: one Newton step on the FMA
# pipe instead of the rcp) issues 3
XU_PER_PAIR = {"filter": 3, "backward": 4, "forward": 4}


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
    prob = make_problem(args)
    vals = []
    t0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        r = oracle_sample_rates(prob, budget_s=args.ref_step_budget)
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
def make_problem(args):
    import synth
    prob = synth.make(args.config)
    if args.dense:
        # the early-training regime: a soft NeuS density (s = 200 / m), every alpha non-zero, so
        # empty-space skipping removes nothing (DESIGN 5c)
        prob.sharpness = 200.0
        prob.name = prob.name + "-dense"
    return prob


def run_gpu(args):
    import torch
    import torch.distributed as dist

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
    # librfr's own NCCL communicator carries the data-path collectives (a4 M, a7 partials)
    comm = rfr.Comm.create() if world > 1 else None
    # emulation of one rank of an N-GPU run on this GPU: rank r's antenna shard, no collective
    ew, er = (args.emulate_world, args.emulate_rank) if args.emulate_world else (world, rank)
    prob = make_problem(args)
    grid = prob.grid
    st = torch.cuda.current_stream()
    passes = set(prob.passes) if not args.passes else set(args.passes.split(","))
    has_flt, has_bwd = "filter" in passes, "bwd" in passes
    heat = args.step == "heatmap"
    if heat:
        has_flt = has_bwd = True
    fused = has_flt and has_bwd and not args.separate and not heat
    gather = args.filter_collective == "gather" and has_flt and not has_bwd

    # ---------------- per-bundle device state
    B = []
    sum_F2 = torch.zeros(1, dtype=torch.float64, device=dev)
    for k, b in enumerate(prob.bundles):
        lo, hi = rfr.shard_range(b.antennas.n, er, ew)
        DS = rfr.DeviceSamples.from_host(b.samples, dev)
        DA_full = rfr.DeviceAntennas.from_host(b.antennas, dev)
        DA = DA_full.slice(lo, hi)
        n, na = b.samples.n, hi - lo
        qlo, qhi = rfr.shard_range(n, er, ew) if gather else (0, n)
        ws = rfr.workspace(n, b.antennas.n if gather else na, grid.n_freq, n, dev)
        st_k = dict(k=k, lo=lo, hi=hi, S=DS, A=DA, A_full=DA_full, n=n, na=na, ws=ws, qlo=qlo,
                    qhi=qhi, sig_full=(torch.randn(b.antennas.n, grid.n_freq, 2, device=dev)
                                       if gather and args.emulate_world else None),
                    sig=torch.empty(na, grid.n_freq, 2, device=dev),
                    G=torch.empty(na, grid.n_freq, 2, device=dev),
                    loss=torch.empty(1, device=dev),
                    M=torch.empty(n, 2, device=dev), P=torch.empty(n, device=dev),
                    part=torch.empty(5, n, device=dev), out=rfr.Grads.empty(n, dev))
        # target y = F(scene) + complex noise at the config's SNR (reading Q18), built untimed
        rfr.rfr_forward(DS, prob.sharpness, DA, grid, st_k["sig"], ws)
        sum_F2 += (st_k["sig"].double() ** 2).sum()
        B.append(st_k)
    if world > 1:
        dist.all_reduce(sum_F2)
    n_F_tot = sum(b.antennas.n for b in prob.bundles) * grid.n_freq
    # (emulation: the local rows stand for the full set in the noise level)
    scale = 1.0 if (world > 1 or ew == 1) else float(ew)
    sigma = float(torch.sqrt(sum_F2 * scale / n_F_tot / 10 ** (prob.snr_db / 10)).item())
    for st_k in B:
        nz = prob.noise_unit(st_k["k"])[st_k["lo"]:st_k["hi"]]
        noise = torch.as_tensor(np.stack([nz.real, nz.imag], -1).astype(np.float32)).to(dev)
        st_k["y"] = st_k["sig"] + sigma * noise
    torch.cuda.synchronize()
    if heat:
        # NEXT-1: the paper's heatmap-domain L2.  Ground-truth heatmap = the filter of
        # the noisy target y at the same queries (the samples), built untimed
        for s in B:
            s["P_gt"] = torch.empty(s["n"], device=dev)
            s["gP"] = torch.empty(s["n"], device=dev)
            rfr.rfr_filter(s["y"], s["A"], grid, s["S"].x, s["S"].y, s["S"].z, s["P_gt"], s["ws"],
                           comm=comm)
        torch.cuda.synchronize()

    ev = lambda: torch.cuda.Event(enable_timing=True)

    def filt(s):
        if gather and args.emulate_world:
            # the emulated rank's share of the query-sharded filter: every antenna (the gathered
            # rows; their values do not change the work) x this rank's query slice
            q = slice(s["qlo"], s["qhi"])
            rfr.rfr_filter(s["sig_full"], s["A_full"], grid, s["S"].x[q], s["S"].y[q], s["S"].z[q],
                           s["P"][q], s["ws"], mf=s["M"][q])
        elif gather:
            rfr.rfr_filter_gather(s["sig"], s["A"], grid, s["S"].x, s["S"].y, s["S"].z,
                                  s["P"][s["qlo"]:s["qhi"]], s["ws"], comm=comm,
                                  n_ant_total=prob.bundles[s["k"]].antennas.n,
                                  mf=s["M"][s["qlo"]:s["qhi"]])
        else:
            rfr.rfr_filter(s["sig"], s["A"], grid, s["S"].x, s["S"].y, s["S"].z, s["P"],
                           s["ws"], mf=s["M"], comm=comm)

    def step(rec=None):
        for s in B:
            e = [ev() for _ in range(5)] if rec is not None else None
            if e: e[0].record(st)
            rfr.rfr_forward(s["S"], prob.sharpness, s["A"], grid, s["sig"], s["ws"])
            if e: e[1].record(st)
            if has_flt and not fused:
                filt(s)
            if e: e[2].record(st)
            if heat:
                # K7 heatmap L2, then K5 (matched-filter adjoint) turns dL/dP into dL/ds
                rfr.rfr_heatmap_loss(s["P"], s["P_gt"], s["gP"], s["loss"], s["ws"])
                rfr.rfr_filter_backward(s["gP"], s["M"], s["A"], grid, s["S"].x, s["S"].y,
                                        s["S"].z, s["G"], s["ws"], power=s["P"], eps=1e-20)
            elif has_bwd:
                rfr.rfr_loss(s["sig"], s["y"], s["G"], s["loss"], s["ws"])
            if e: e[3].record(st)
            if fused:
                rfr.rfr_backward_filter(s["G"], s["sig"], s["S"], prob.sharpness, s["A"], grid,
                                        s["out"], s["P"], s["ws"], mf=s["M"],
                                        flags=rfr.RFR_REUSE_BLEND, comm=comm)
            elif has_bwd:
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
    # untimed diagnostics (bundle 0): the r2 plan of each call type, active-sample counts
    s0 = B[0]
    rfr.rfr_forward(s0["S"], prob.sharpness, s0["A"], grid, s0["sig"], s0["ws"])
    plan_fwd = rfr.rfr_plan_state(s0["ws"])
    n_act_fwd = rfr.cheb_state(s0["ws"])["n_active_fwd"]
    plan_flt = plan_bwd = plan_k5 = None
    n_act_bwd = 0
    if has_flt and not fused:
        filt(s0)
        plan_flt = rfr.rfr_plan_state(s0["ws"])
    if heat:
        rfr.rfr_heatmap_loss(s0["P"], s0["P_gt"], s0["gP"], s0["loss"], s0["ws"])
        rfr.rfr_filter_backward(s0["gP"], s0["M"], s0["A"], grid, s0["S"].x, s0["S"].y, s0["S"].z,
                                s0["G"], s0["ws"], power=s0["P"], eps=1e-20)
        plan_k5 = rfr.rfr_plan_state(s0["ws"])
    if has_bwd:
        rfr.rfr_loss(s0["sig"], s0["y"], s0["G"], s0["loss"], s0["ws"])
        if fused:
            rfr.rfr_backward_filter(s0["G"], s0["sig"], s0["S"], prob.sharpness, s0["A"], grid,
                                    s0["out"], s0["P"], s0["ws"], mf=s0["M"],
                                    flags=rfr.RFR_REUSE_BLEND)
            plan_flt = plan_bwd = rfr.rfr_plan_state(s0["ws"])
        else:
            rfr.rfr_backward_partial(s0["G"], s0["S"], prob.sharpness, s0["A"], grid, s0["part"],
                                     s0["ws"], flags=rfr.RFR_REUSE_BLEND)
            plan_bwd = rfr.rfr_plan_state(s0["ws"])
        n_act_bwd = rfr.cheb_state(s0["ws"])["n_active_bwd"]
    act_fwd = n_act_fwd / s0["n"]
    act_bwd = n_act_bwd / s0["n"] if has_bwd else 0.0
    barrier()

    # ---------------- timed region: K steps, per-step events, L2 flushed between steps
    n0 = rfr.rfr_launch_count()
    step_ms, seg = [], {"fwd": 0.0, "filter": 0.0, "loss": 0.0, "bwd": 0.0}
    rfr.rfr_profile_enable(True)
    with ClockSampler(local) as clk:
        barrier()
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            s0e, s1e = ev(), ev()
            recs = []
            s0e.record(st)
            step(recs)
            s1e.record(st)
            torch.cuda.synchronize()
            step_ms.append(s0e.elapsed_time(s1e))
            for e in recs:
                seg["fwd"] += e[0].elapsed_time(e[1])
                seg["filter"] += e[1].elapsed_time(e[2])
                seg["loss"] += e[2].elapsed_time(e[3])
                seg["bwd"] += e[3].elapsed_time(e[4])
        barrier()
        t_wall = time.perf_counter() - t_wall
    sweeps = {k: rfr.rfr_profile_read(k) for k in rfr.SWEEPS}
    rfr.rfr_profile_enable(False)
    launches = rfr.rfr_launch_count() - n0
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms, seg["fwd"], seg["filter"], seg["loss"], seg["bwd"]], device=dev,
                     dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, f_ms, q_ms, l_ms, b_ms = (float(v) for v in t.tolist())
    ms_per_step = tot_ms / args.steps
    Nc = prob.n_contrib
    share = (1.0 / ew) if args.emulate_world else 1.0      # the emulated rank's share of N_c
    value = Nc * share / (ms_per_step * 1e-3)
    active_frac = {"fwd": act_fwd, "bwd": act_bwd}

    # ---------------- e2e: same step through the ABI with host buffers (pinned) every step
    e2e = run_e2e(args, prob, B, rfr, torch, dist, world, dev, st, step, share)

    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return 0
    pk = peaks()
    clocks = clk.summary()
    mhz = pk.get("sm_max_mhz", 1965.0)
    peak_ops = N_SM * FP32_LANES_PER_SM * mhz * 1e6
    peak_xu = N_SM * XU_LANES_PER_SM * mhz * 1e6
    per_step = lambda ms: ms / args.steps
    # pairs per step of each sweep on this rank (every bundle has the same shape)
    na_loc = sum(s["na"] for s in B)
    n_pts = B[0]["n"]
    pairs = {"filter": sum(s["n"] * (s["hi"] - s["lo"]) for s in B) if has_flt else 0,
             "backward": act_bwd * n_pts * na_loc if has_bwd else 0,
             # the heatmap step's K5 (matched-filter adjoint) runs the forward sweep over every
             # query (the samples) too, timed under the same sweep id
             "forward": act_fwd * n_pts * na_loc + (n_pts * na_loc if heat else 0)}
    if gather:
        pairs["filter"] = sum((s["qhi"] - s["qlo"]) * prob.bundles[s["k"]].antennas.n for s in B)
    plans = {"filter": plan_flt, "backward": plan_bwd, "forward": plan_fwd}
    roofs = []
    for sw in ("filter", "backward", "forward"):
        ms_tot, nl = sweeps[sw]
        pl = plans[sw]
        if not nl or not pl or not pl["applied"] or not pairs[sw]:
            continue
        ms = ms_tot / args.steps
        P = pl["P"]
        ops = lane_ops_per_pair(sw, P)
        ach = ops * pairs[sw] / (ms * 1e-3)
        xu = XU_PER_PAIR[sw] * pairs[sw] / (ms * 1e-3)
        kern = {"filter": "k2_filter", "backward": "k2_bwd", "forward": "k2_fwd"}[sw]
        roofs.append({"kernel": f"{kern}<P={P}>", "sweep": sw, "bound": "alu",
                      "achieved": ach / 1e12, "peak": peak_ops / 1e12, "unit": "T FP32 lane-ops/s",
                      "frac": ach / peak_ops, "lane_ops_per_pair": ops,
                      "frac_moments_only": moment_ops_per_pair(sw, P) * pairs[sw] / (ms * 1e-3) / peak_ops,
                      "xu_frac": xu / peak_xu, "pairs_per_step": pairs[sw],
                      "ms_per_step": ms, "launches_per_step": nl / args.steps,
                      "tiles": [pl["lx"], pl["ly"], pl["lz"]], "Pg": pl["Pg"]})
    dom = max(roofs, key=lambda r: r["ms_per_step"]) if roofs else None
    roof = None
    if dom:
        traffic = None
        try:   # DRAM bytes per launch from the committed full-size ncu capture
            traffic = json.load(open(TRAFFIC_PATH)).get(args.config, {}).get(dom["kernel"].split("<")[0])
        except Exception:
            pass
        roof = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
                "unit": dom["unit"], "frac": dom["frac"], "traffic": traffic,
                "kernel": dom["kernel"], "xu_frac": dom["xu_frac"],
                "frac_moments_only": dom["frac_moments_only"],
                "peak_note": (f"148 SM x 128 FP32 lanes x sm_max_mhz (MEASURED_PEAKS.json); "
                              f"{dom['lane_ops_per_pair']} lane-ops per (point, antenna) pair "
                              "(DESIGN 5e work model: pair geometry + Horner / moments + epilogue), "
                              "timed live per launch with CUDA events on the launching stream "
                              f"(rfr_profile); xu_frac: {XU_PER_PAIR[dom['sweep']]} MUFU per pair against 148 x 16 XU lanes")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.emulate_world:
        r = oracle_sample_rates(prob, budget_s=args.ref_budget)
        cpu = {"value": step_rate(r) / 1e9, "unit": "G contributions/s", "cores": r["cores"],
               "kind": "oracle", "sample": r["sample"],
               "per_pass_G_per_s": {k: r[k] / 1e9 for k in ("fwd", "filter", "bwd")}}
    desc = ("K1 blend + forward + K4 filter (+NCCL all-reduce of M) + K7 heatmap loss + K5 "
            "matched-filter adjoint + K3 backward (+NCCL all-reduce of partials) + K1' finish"
            if heat else
            "K1 blend + forward + K6 loss + fused backward + matched filter at the samples "
            "(+NCCL all-reduce of partials and M) + K1' finish" if fused else
            "K1 blend + forward + K4 filter + K6 loss + K3 backward + K1' finish"
            if (has_flt and has_bwd) else
            "K1 blend + forward + K6 loss + K3 backward (+NCCL all-reduce of partials) + K1' finish"
            if has_bwd else
            "K1 blend + forward + K4 matched filter at the samples (" +
            ("all-gather of the signal rows, query-sharded" if gather else "+NCCL all-reduce of M")
            + ")")
    n_active_contrib = (pairs["forward"] + pairs["backward"] + pairs["filter"]) * grid.n_freq
    # per-pass rates in the metric's units -- N_c / t_fwd (the forward call: K1 +
    # plan + sweep + bins), N_q N_a N_f / t_filter and N_c / t_bwd; inside the fused call the filter
    # is its sweep time and the backward the rest of the call (plan, prep, sweep, K1')
    sw_ms = {k: v[0] / args.steps for k, v in sweeps.items()}
    n_q_tot = sum((s["qhi"] - s["qlo"]) for s in B) if gather else sum(s["n"] for s in B)
    nqf = n_q_tot * (prob.bundles[0].antennas.n if gather else na_loc) * grid.n_freq
    t_f, t_q, t_b = per_step(f_ms), per_step(q_ms), per_step(b_ms)
    if fused:
        t_q, t_b = sw_ms.get("filter", 0.0), per_step(b_ms) - sw_ms.get("filter", 0.0)
    Nc_loc = Nc * share
    per_pass = {"fwd": Nc_loc / (t_f * 1e-3) / 1e9 if t_f > 0 else None,
                "filter": nqf / (t_q * 1e-3) / 1e9 if (has_flt and t_q > 0) else None,
                "bwd": Nc_loc / (t_b * 1e-3) / 1e9 if (has_bwd and t_b > 0) else None}
    line = {"metric": METRIC, "value": value / 1e9, "unit": "G contributions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": prob.name, "n_contrib_per_pass": Nc,
                       "passes": sorted(passes), "bundles": len(prob.bundles),
                       "n_samples": n_pts, "n_antennas": prob.bundles[0].antennas.n,
                       "n_freq": grid.n_freq, "sharpness_per_m": prob.sharpness,
                       "parallelism": f"antenna-shard x{ew}" + (" (emulated rank "
                                                                  f"{er} on one GPU)" if args.emulate_world else ""),
                       "l2": "flushed between steps (512 MiB memset, outside the step events)",
                       "loss": "heatmap L2 (NEXT-1)" if heat else "signal-domain complex residual",
                       "step": desc},
            "value_active": {"value": n_active_contrib / (ms_per_step * 1e-3) / 1e9,
                             "unit": "G contributions/s",
                             "note": "(point, antenna, bin) terms the kernels evaluate: every "
                                     "sample for the filter, the alpha != 0 / amplitude != 0 samples "
                                     "for the backward / forward (empty-space skipping, DESIGN 5c), "
                                     "summed over the step's passes"},
            "passes": {"fwd_ms": per_step(f_ms), "filter_ms": per_step(q_ms),
                       "loss_ms": per_step(l_ms), "bwd_or_fused_ms": per_step(b_ms)},
            "sweeps_ms_per_step": {k: v[0] / args.steps for k, v in sweeps.items()},
            "per_pass_G_per_s": per_pass,
            "method": {"engine": "r2 tiled (DESIGN 5e)",
                       "plans": {k: v for k, v in (("forward", plan_fwd), ("filter", plan_flt),
                                                   ("backward", plan_bwd), ("k5", plan_k5)) if v},
                       "empty_space_skipping": {
                           "forward_active_samples": act_fwd, "backward_active_samples": act_bwd,
                           "note": "samples whose amplitude (forward) or alpha (backward) is exactly "
                                   "0 in fp32 are skipped; value still counts every (sample, "
                                   "antenna, bin) of the batch (the metric's definition)"}},
            "roofline": roof, "rooflines": roofs, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "wall_s_timed": t_wall}
    if args.emulate_world:
        line["emulated"] = {"world": ew, "rank": er, "note": "one rank's share on one GPU: "
                            "value = that rank's contributions / its step time; collectives excluded"}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, prob, B, rfr, torch, dist, world, dev, st, step, share):
    """Same step measured end to end through the public API: every step copies its inputs
    (samples, local antennas, local target rows) host->device from pinned buffers and reads the
    result (loss + per-sample gradients, or the heatmap) device->host.

    Pipelined the way a training loop feeds the renderer: two device slots of inputs and outputs;
    step k+1's H2D runs on a copy stream while step k computes, and step k's D2H on the copy stream
    while step k+1 computes.  The timed region (events on the compute stream, the copy stream
    joined at both ends) holds every step's H2D and D2H: the first step's H2D is not hidden, nor
    the last step's D2H.  `serial_value` is the same loop with the copies in line on the compute
    stream (no overlap)."""
    has_bwd = "bwd" in prob.passes or args.step == "heatmap"

    def io_of(s):
        """(inputs, outputs) device tensors of bundle state s, in a fixed order"""
        ins, outs = [], []
        for f in rfr.DeviceSamples.FIELDS:
            ins.append(getattr(s["S"], f))
        for f in ("tx_x", "tx_y", "tx_z"):
            ins.append(getattr(s["A"], f))
        if has_bwd:
            ins.append(s["P_gt"] if "P_gt" in s else s["y"])   # heatmap step: the target heatmap
            for f in rfr.Grads.NAMES:
                outs.append(getattr(s["out"], f))
            outs.append(s["loss"])
        else:
            outs.append(s["P"][s["qlo"]:s["qhi"]])
        return ins, outs

    # slot 0 = the bench's own buffers; slot 1 = fresh device buffers of the same shapes
    keys = ("S", "A", "y", "P_gt", "out", "loss", "P", "M")
    slots = [{k: s[k] for k in keys if k in s} for s in B]
    slots1 = []
    for s in B:
        d = {"S": dataclasses.replace(s["S"], **{f: torch.empty_like(getattr(s["S"], f))
                                                 for f in rfr.DeviceSamples.FIELDS}),
             "A": dataclasses.replace(s["A"], **{f: torch.empty_like(getattr(s["A"], f))
                                                 for f in ("tx_x", "tx_y", "tx_z")}),
             "out": rfr.Grads.empty(s["n"], dev), "loss": torch.empty_like(s["loss"]),
             "P": torch.empty_like(s["P"]), "M": torch.empty_like(s["M"])}
        for k in ("y", "P_gt"):
            if k in s:
                d[k] = torch.empty_like(s[k])
        slots1.append(d)
    host_in, host_out, dev_in, dev_out = [], [], [[], []], [[], []]
    for j, s in enumerate(B):
        ins, outs = io_of(s)
        host_in += [t.cpu().pin_memory() for t in ins]
        host_out += [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in outs]
        dev_in[0] += ins
        dev_out[0] += outs
        s1 = dict(s)
        s1.update(slots1[j])
        i1, o1 = io_of(s1)
        dev_in[1] += i1
        dev_out[1] += o1
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)

    def use_slot(k):
        for s, a, b in zip(B, slots, slots1):
            s.update(a if k == 0 else b)

    ev = lambda: torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 5))
    cs = torch.cuda.Stream(device=dev)

    def serial():
        e0, e1 = ev(), ev()
        e0.record(st)
        for _ in range(steps):
            for h, d in zip(host_in, dev_in[0]):
                d.copy_(h, non_blocking=True)
            step()
            for h, d in zip(host_out, dev_out[0]):
                h.copy_(d, non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    def pipelined():
        e0, e1 = ev(), ev()
        h2d_done = [torch.cuda.Event() for _ in range(steps)]
        d2h_done = [torch.cuda.Event() for _ in range(steps)]
        comp_done = [torch.cuda.Event() for _ in range(steps)]

        def issue_h2d(k):
            if k == 0:
                cs.wait_stream(st)
            if k >= 2:
                cs.wait_event(comp_done[k - 2])      # slot k % 2 is free once step k-2 computed
            with torch.cuda.stream(cs):
                for h, d in zip(host_in, dev_in[k % 2]):
                    d.copy_(h, non_blocking=True)
            h2d_done[k].record(cs)

        e0.record(st)
        issue_h2d(0)
        for k in range(steps):
            if k + 1 < steps:
                issue_h2d(k + 1)
            st.wait_event(h2d_done[k])
            if k >= 2:
                st.wait_event(d2h_done[k - 2])       # outputs of slot k % 2 were read back
            use_slot(k % 2)
            step()
            comp_done[k].record(st)
            cs.wait_event(comp_done[k])
            with torch.cuda.stream(cs):
                for h, d in zip(host_out, dev_out[k % 2]):
                    h.copy_(d, non_blocking=True)
            d2h_done[k].record(cs)
        st.wait_event(d2h_done[steps - 1])
        st.wait_stream(cs)
        e1.record(st)
        torch.cuda.synchronize()
        use_slot(0)
        return e0.elapsed_time(e1) / steps

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    pipelined()                                      # warm the second slot (plans, workspaces)
    t_ser = serial()
    t_pip = pipelined()
    t = torch.tensor([t_pip, t_ser], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_pip, t_ser = (float(v) for v in t.tolist())
    conv = lambda ms: prob.n_contrib * share / (ms * 1e-3) / 1e9
    return {"value": conv(t_pip), "unit": "G contributions/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "ms_per_step": t_pip,
            "serial_value": conv(t_ser), "serial_ms_per_step": t_ser,
            "note": "pinned host buffers every step; pipelined over two device slots (H2D of step "
                    "k+1 and D2H of step k-1 on a copy stream during step k), the first H2D and "
                    "the last D2H exposed; serial_value: copies in line on the compute stream"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="librfr", choices=["librfr", "reference"])
    ap.add_argument("--ref-budget", type=float, default=20.0,
                    help="seconds of oracle work for the cpu_baseline sample")
    ap.add_argument("--ref-step-budget", type=float, default=4.0,
                    help="seconds of oracle work per step of --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--step", default="signal", choices=["signal", "heatmap"],
                    help="signal: the north_star step (signal-domain residual, default); heatmap: "
                         "the paper's heatmap-domain L2 through the matched-filter adjoint K5 "
                         "(SURVEY 8f NEXT-1)")
    ap.add_argument("--separate", action="store_true",
                    help="filter and backward as two sweeps (rfr_filter + rfr_backward)")
    ap.add_argument("--passes", default="", help="override the config's passes, e.g. fwd,filter")
    ap.add_argument("--dense", action="store_true",
                    help="s = 200 / m: no empty space to skip (early-training regime)")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="time one rank's share of an N-GPU run on this GPU")
    ap.add_argument("--emulate-rank", type=int, default=0)
    ap.add_argument("--filter-collective", default="auto", choices=["auto", "allreduce", "gather"],
                    help="multi-GPU filter: all-reduce M, or all-gather the signal rows and shard "
                         "the queries; auto = the smaller payload (SURVEY 8e)")
    args = ap.parse_args()
    if args.filter_collective == "auto":
        import synth
        p = synth.make(args.config)
        b = p.bundles[0]
        # all-reduce of M: 8 B x N_q; all-gather of the signal rows: 8 B x N_a x N_f (+ positions)
        args.filter_collective = ("gather" if 8 * b.antennas.n * p.grid.n_freq + 12 * b.antennas.n
                                  < 8 * b.samples.n else "allreduce")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
