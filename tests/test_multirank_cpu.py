"""World-size-2 CPU tests (gloo) of the data-parallel host logic:
shards are disjoint and complete, and the all-reduced per-rank normal
equations equal the full system (what the NCCL all-reduce in libmis relies on:
H, b and E are linear in the per-rank sums; graph terms on rank 0 only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1803_02009_b200 import shard
from tests.common import random_state, scene_problem


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, pb, fr, _ = scene_problem("c1")
        m = pb.g.shape[0]
        idx = shard.shard_indices(pb.idx, m, world, rank)
        # partition: disjoint and complete
        all_idx = [torch.zeros(1)] * world
        got = torch.from_numpy(idx.astype(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(idx)]))
        mx = int(max(s.item() for s in sizes))
        pad = torch.full((mx,), -1, dtype=torch.int64)
        pad[:len(idx)] = got
        bufs = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(bufs, pad)
        merged = np.concatenate([b.numpy()[b.numpy() >= 0] for b in bufs])
        ok_part = len(merged) == pb.xyz.shape[0] and len(np.unique(merged)) == pb.xyz.shape[0]
        # per-rank system, graph terms only on rank 0, then all-reduce (sum)
        Rt = random_state(m, np.random.default_rng(7), 0.01, 0.2)
        prm = O.params()
        nbr = pb.nbr if shard.graph_terms_on(rank) else np.full_like(pb.nbr, -1)
        feats = (pb.fsrc, pb.fdst) if shard.graph_terms_on(rank) else (None, None)
        sub = O.Problem(pb.xyz[idx], pb.nrm[idx], pb.idx[idx], pb.w[idx], pb.g, nbr, *feats)
        s = O.system(prm, sub, fr, Rt)
        H = torch.from_numpy(O.dense_H(s, m))
        b = torch.from_numpy(s["rhs"].copy())
        E = torch.from_numpy(s["energy"].copy())
        for t in (H, b, E):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        if rank == 0:
            full = O.system(prm, pb, fr, Rt)
            Hf = O.dense_H(full, m)
            q.put((ok_part,
                   float(np.abs(H.numpy() - Hf).max() / np.abs(Hf).max()),
                   float(np.abs(b.numpy() - full["rhs"]).max() / np.abs(full["rhs"]).max()),
                   float(np.abs(E.numpy() - full["energy"]).max() / full["energy"][4]),
                   len(idx)))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_and_allreduced_system_equal_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok_part, eH, eb, eE, n0 = res
    assert ok_part
    assert 0 < n0 < 5000
    assert eH < 1e-10 and eb < 1e-10 and eE < 1e-10, (eH, eb, eE)


def test_node_ranges_balanced():
    rng = np.random.default_rng(0)
    primary = np.sort(rng.integers(0, 100, 10000))
    for world in (1, 2, 4, 8):
        b = shard.node_ranges(primary, 100, world)
        assert b[0] == 0 and b[-1] == 100 and (np.diff(b) >= 0).all()
        counts = [((primary >= b[r]) & (primary < b[r + 1])).sum() for r in range(world)]
        assert sum(counts) == 10000
        assert max(counts) - min(counts) <= 2 * 10000 / 100 + 1   # within ~one node's points
