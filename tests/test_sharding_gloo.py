"""Multi-rank host logic on CPU (world_size 2 and 3, gloo): antenna sharding with rfr.shard_range, an
all-reduce (sum) of the per-sample backward partials and of the filter's complex M, then the finish
step -- the same composition bench.py runs over NCCL, with the oracle standing in for the kernels;
the query-sharded filter (rfr_filter_gather's composition: the ranks' antenna slices and signal
rows gathered in rank order, each rank filtering its query slice); and librfr's communicator
plumbing (rank 0's NCCL unique id from rfr_comm_unique_id, broadcast over the process group)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_29097_b200.rfr import shard_range
        p = synth.make("c0b")
        b = p.bundles[0]
        S, A = b.samples, b.antennas
        rng = np.random.default_rng(0)
        G = rng.standard_normal((A.n, p.grid.n_freq)) + 1j * rng.standard_normal((A.n, p.grid.n_freq))
        lo, hi = shard_range(A.n, rank, world)
        part = torch.from_numpy(oracle.backward_partials(G[lo:hi], S, p.sharpness, A.slice(lo, hi),
                                                         p.grid))
        dist.all_reduce(part)                                  # sum over antenna shards
        grads = oracle.backward_finish(part.numpy(), S, p.sharpness)
        M, _ = oracle.filter(G[lo:hi], A.slice(lo, hi), p.grid, S.x, S.y, S.z)
        Mt = torch.from_numpy(np.stack([M.real, M.imag], -1))
        dist.all_reduce(Mt)
        if rank == 0:
            ref = oracle.backward(G, S, p.sharpness, A, p.grid)
            Mr, Pr = oracle.filter(G, A, p.grid, S.x, S.y, S.z)
            err = max(np.linalg.norm(grads[k] - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300)
                      for k in ("sdf", "refl", "nx", "ny", "nz", "power"))
            P = np.hypot(Mt[:, 0].numpy(), Mt[:, 1].numpy())
            q.put((float(err), float(np.max(np.abs(P - Pr) / Pr))))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_backward_and_filter_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(180)
        assert pr.exitcode == 0
    err_g, err_p = q.get(timeout=5)
    assert err_g < 1e-12 and err_p < 1e-12


def _worker_gather(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_29097_b200 import rfr
        # communicator plumbing: every rank holds rank 0's 128-byte id
        uid = rfr.Comm.unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        same_id = all(i == ids[0] for i in ids) and len(uid) == 128 and any(uid)
        p = synth.make("c1")
        b = p.bundles[0]
        S, A = b.samples.subset_rays(np.arange(0, 256, 17)), b.antennas
        rng = np.random.default_rng(3)
        sig = rng.standard_normal((A.n, p.grid.n_freq)) + 1j * rng.standard_normal((A.n, p.grid.n_freq))
        lo, hi = rfr.shard_range(A.n, rank, world)
        # gather the local rows and positions in rank order (rfr_filter_gather's broadcasts)
        local = (sig[lo:hi], A.tx_x[lo:hi], A.tx_y[lo:hi], A.tx_z[lo:hi])
        parts = [None] * world
        dist.all_gather_object(parts, local)
        g_sig = np.concatenate([pp[0] for pp in parts])
        g_ant = synth.AntennaSet(*[np.concatenate([pp[c] for pp in parts]) for c in (1, 2, 3)])
        qlo, qhi = rfr.shard_range(S.n, rank, world)
        M, P = oracle.filter(g_sig, g_ant, p.grid, S.x[qlo:qhi], S.y[qlo:qhi], S.z[qlo:qhi])
        slices = [None] * world
        dist.all_gather_object(slices, (qlo, qhi, P))
        if rank == 0:
            _, Pr = oracle.filter(sig, A, p.grid, S.x, S.y, S.z)
            Pq = np.concatenate([sl[2] for sl in slices])
            cover = [sl[:2] for sl in slices]
            contiguous = cover[0][0] == 0 and cover[-1][1] == S.n and all(
                cover[k][1] == cover[k + 1][0] for k in range(world - 1))
            q.put((bool(same_id), bool(contiguous), float(np.max(np.abs(Pq - Pr) / Pr))))
    finally:
        dist.destroy_process_group()


def test_query_sharded_filter_and_comm_plumbing_gloo():
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker_gather, args=(r, world, port, q)) for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(180)
            assert pr.exitcode == 0
        same_id, contiguous, err = q.get(timeout=5)
        assert same_id and contiguous and err < 1e-12, (world, same_id, contiguous, err)
