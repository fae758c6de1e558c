"""World-size-2 CPU tests (gloo) of the data-parallel host logic:
shards are disjoint and complete, and the reduction protocol libmis uses gives the
full system: every rank assembles the point terms of its shard and the graph terms
(regulariser, features) of the whole graph; only the point terms (H, b, E_data, E_pt,
the association count) are all-reduced, then each rank adds its own graph terms."""
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
        # per-rank point terms (the shard, no graph terms) all-reduced; graph terms local on every rank
        Rt = random_state(m, np.random.default_rng(7), 0.01, 0.2)
        prm = O.params()
        no_nbr = np.full_like(pb.nbr, -1)
        sub = O.Problem(pb.xyz[idx], pb.nrm[idx], pb.idx[idx], pb.w[idx], pb.g, no_nbr)
        s = O.system(prm, sub, fr, Rt)
        H = torch.from_numpy(O.dense_H(s, m))
        b = torch.from_numpy(s["rhs"].copy())
        E = torch.from_numpy(s["energy"][:2].copy())   # E_data, E_pt
        for t in (H, b, E):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        none = np.zeros(0, np.int64)
        gsub = O.Problem(pb.xyz[none], pb.nrm[none], pb.idx[none], pb.w[none], pb.g, pb.nbr, pb.fsrc, pb.fdst)
        gs = O.system(prm, gsub, fr, Rt)   # the graph terms, identical on every rank
        H = H + torch.from_numpy(O.dense_H(gs, m))
        b = b + torch.from_numpy(gs["rhs"])
        E = torch.from_numpy(np.concatenate([E.numpy(), gs["energy"][2:4]]))
        E = torch.cat([E, torch.tensor([prm.w_data * E[0] + prm.w_pt * E[1] + prm.w_reg * E[2] + prm.w_corr * E[3]],
                                       dtype=E.dtype)])
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
