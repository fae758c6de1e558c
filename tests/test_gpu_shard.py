"""P15 on the GPU path (SURVEY §8(c) pins; A15 shard reduction): the normal equations
assembled by the CUDA kernels on S virtual shards of one model -- points split by primary
node range (paper_1803_02009_b200.shard, what each rank passes in a sharded run), the
regulariser and feature terms on shard 0 only -- sum to the single-context system, and to
the fp64 oracle's full system within the north_star J^T J gate.  This is the linearity the
NCCL all-reduce of the accumulators relies on, checked on one GPU with
independent contexts instead of ranks."""
import numpy as np
import pytest

import oracle as O
from paper_1803_02009_b200 import shard
from tests.common import random_state, scene_problem, state_f32
from tests.test_gpu_parity import check_system, dense_from_bsr, oracle_params

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def shard_ctx(sc, pb, idx, graph_terms):
    c = sc["cfg"]
    prm = M.mis_default_params(k=pb.k, n_nbr=pb.n_nbr, gn_iters=c.gn_iters, pcg_iters=c.pcg_iters)
    ctx = M.Context(prm)
    n = len(idx)
    rgb = sc["rgb"][idx] if sc.get("rgb") is not None else None
    M.mis_set_model(ctx.ptr, pb.xyz[idx], pb.nrm[idx], rgb, None, None, None, capacity=n + c.H * c.W)
    nbr = pb.nbr if graph_terms else np.full_like(pb.nbr, -1)
    M.mis_set_graph(ctx.ptr, pb.g, nbr, np.ascontiguousarray(pb.idx[idx]),
                    np.ascontiguousarray(pb.w[idx], np.float32))
    it = sc["intr"]
    M.mis_set_frame(ctx.ptr, sc["depth"], M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"]),
                    sc["pose"])
    if graph_terms and pb.fsrc.shape[0]:
        M.mis_set_features(ctx.ptr, pb.fsrc, pb.fdst)
    return ctx


@pytest.mark.parametrize("S", [2, 3])
def test_virtual_shards_sum_to_full_system(S):
    sc, pb, fr, _ = scene_problem("c2")
    m = pb.g.shape[0]
    Rt = state_f32(random_state(m, np.random.default_rng(21), 0.01, 0.3))
    parts = [shard.shard_indices(pb.idx, m, S, r) for r in range(S)]
    merged = np.concatenate(parts)
    assert len(merged) == pb.xyz.shape[0] and len(np.unique(merged)) == len(merged)
    H = np.zeros((6 * m, 6 * m))
    b = np.zeros(6 * m)
    E = np.zeros(5)
    for r in range(S):
        ctx = shard_ctx(sc, pb, parts[r], shard.graph_terms_on(r))
        M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
        gs = M.mis_dbg_system(ctx.ptr, m)
        H += dense_from_bsr(gs, m)
        b += gs["rhs"]
        E += gs["energy"]
    full = shard_ctx(sc, pb, np.arange(pb.xyz.shape[0]), True)
    M.mis_dbg_set_nodes(full.ptr, Rt.astype(np.float32))
    gf = M.mis_dbg_system(full.ptr, m)
    Hf = dense_from_bsr(gf, m)
    # sum over shards == one context (fp32 sums in another order)
    d = np.sqrt(np.maximum(np.diag(Hf), 1e-30))
    assert (np.abs(H - Hf) / np.outer(d, d)).max() < 1e-5
    Ef = gf["energy"][4]
    assert (np.abs(b - gf["rhs"]) / np.sqrt(np.diag(Hf) * 2 * Ef)).max() < 1e-5
    assert np.abs(E[:4] - gf["energy"][:4]).max() <= 1e-5 * Ef
    # and the summed system passes the oracle gate
    prm = oracle_params(full.params)
    osys = O.system(prm, pb, fr, Rt)
    osys["prm"] = prm
    gsum = {"row_ptr": gf["row_ptr"], "col": gf["col"], "val": None, "rhs": b, "energy": E}
    rp, col = gf["row_ptr"], gf["col"]
    val = np.zeros((len(col), 6, 6))
    for r in range(m):
        for e in range(rp[r], rp[r + 1]):
            val[e] = H[6 * r:6 * r + 6, 6 * col[e]:6 * col[e] + 6]
    gsum["val"] = val
    check_system(gsum, osys, m)


def test_multi_gpu_payload_path_parity():
    """The multi-GPU reduction path (point part of H and b formed before the cross-rank sum,
    scattered back as pre-weighted accumulators, graph terms per rank) on one GPU:
    MIS_SHARD_PROTOCOL=1 runs its kernels in every assembly (without the NCCL call, a sum over one
    rank), and the system / registration parity suites must pass unchanged through it."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MIS_SHARD_PROTOCOL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "system_parity or register_parity_mirror or association_parity"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
