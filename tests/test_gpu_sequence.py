"""NEXT-1 on the GPU: Alg. 2 Step 5 node regeneration (mis_regenerate_nodes, K15; reading A36)
and the per-frame pipeline of a sequence (BASELINE configs[2]: the C3 100-frame register + fuse
sequence; SURVEY §8(c) "Sequences (C3)": per-frame parity by state injection).

State injection: before each checked stage the GPU state (model, skinning, nodes, graph) is read
back and handed to the oracle, so every stage is compared on identical inputs:
  register  -> converged nodes <= 0.01 mm / 1e-4 rad (MIRROR, same G and P)
  warp      -> live model <= 0.05 mm, normals 1e-4
  fuse      -> tests.common.check_fusion (exact outside ties)
  filter    -> box count / survivors / ids / weights / stamps exact, positions 1e-3 mm (as test_gpu_filter)
  regenerate-> node count exact, centroids <= 1e-4 mm, N(j) exact outside near-ties, Eq. 2 skinning
               of every point exact outside near-ties, identity transforms
"""
import numpy as np
import pytest

import oracle as O
from paper_1803_02009_b200 import synth
from tests.common import check_fusion, scene_problem
from tests.test_gpu_parity import make_ctx, oracle_params, rot_err

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def node_spacing(xyz, m):
    ext = xyz.max(0) - xyz.min(0)
    return float(np.sqrt(ext[0] * ext[1] / m))


def check_regeneration(ctx, k, n_nbr, grid):
    """mis_regenerate_nodes against O8 on the GPU's own model floats (state injection)."""
    mod = M.mis_get_model(ctx.ptr, k)
    og, onbr, omg = O.regenerate_nodes(mod["xyz"], grid, n_nbr)
    m = M.mis_regenerate_nodes(ctx.ptr, grid)
    assert m == og.shape[0]
    g = M.mis_get_graph(ctx.ptr, np.zeros((m, 3), np.float32))
    assert np.abs(g - og).max() < 1e-4
    nbr = M.mis_get_nbr(ctx.ptr, np.zeros((m, n_nbr), np.int32))
    sure = omg > 1e-5
    assert sure.mean() > 0.95
    assert (np.sort(nbr[sure], 1) == np.sort(onbr[sure], 1)).all()
    assert (M.mis_get_nodes_f64(ctx.ptr, m) == O.identity_state(m)).all()
    # every point re-skinned (Eq. 2) against the new nodes: the oracle on the GPU's fp32 nodes
    mod2 = M.mis_get_model(ctx.ptr, k)
    order = np.argsort(mod2["ids"])
    assert (np.sort(mod2["ids"]) == np.sort(mod["ids"])).all()      # same points, regrouped
    oi, ow, om = O.skin(mod2["xyz"], g, k)
    oi = np.sort(oi, 1)
    keep = om > 1e-5
    assert keep.mean() > 0.99
    assert (mod2["knn_idx"][keep] == oi[keep]).all()
    assert order.size == mod["ids"].size
    return m, g, nbr


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("scale", [1.0, 1.6])
def test_regenerate_parity(cfg, scale):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    grid = scale * node_spacing(pb.xyz, pb.g.shape[0])
    m, g, nbr = check_regeneration(ctx, pb.k, pb.n_nbr, grid)
    # the next registration runs on the regenerated graph and matches the oracle on the same inputs
    mod = M.mis_get_model(ctx.ptr, pb.k)
    pb2 = O.Problem(mod["xyz"], mod["nrm"], mod["knn_idx"], mod["knn_w"], g, nbr)
    rep = M.report_dict(M.mis_register(ctx.ptr, None, None, None, np.zeros((0, 3), np.float32),
                                       np.zeros((0, 3), np.float32)))
    assert rep["status"] == 0
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    Ro, _, _ = O.register(oracle_params(ctx.params), pb2, fr)
    assert np.abs(Rg[:, 9:] - Ro[:, 9:]).max() < 0.01
    assert max(rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)) < 1e-4


def test_regenerate_errors_leave_graph():
    sc, pb, fr, _ = scene_problem("c1")
    ctx = make_ctx(sc, pb)
    m0 = pb.g.shape[0]
    with pytest.raises(M.MisError):
        M.mis_regenerate_nodes(ctx.ptr, 1e4)            # one occupied cell < k + 1 nodes
    with pytest.raises(M.MisError):
        M.mis_regenerate_nodes(ctx.ptr, -1.0)
    g = M.mis_get_graph(ctx.ptr, np.zeros((m0, 3), np.float32))
    assert np.array_equal(g, pb.g)
    rep = M.report_dict(M.mis_register(ctx.ptr))       # the old graph is still bound
    assert rep["status"] == 0


def _state(ctx, k, m, n_nbr):
    mod = M.mis_get_model(ctx.ptr, k)
    g = M.mis_get_graph(ctx.ptr, np.zeros((m, 3), np.float32))
    nbr = M.mis_get_nbr(ctx.ptr, np.zeros((m, n_nbr), np.int32))
    return mod, g, nbr


@pytest.mark.parametrize("cfg,frames,checked", [("c1", 6, (1, 2, 3, 6)), ("c3", 50, (1, 2, 3, 50))])
def test_sequence_state_injection(cfg, frames, checked):
    """Alg. 2 per frame (register -> warp -> fuse -> filter -> regenerate), every stage of the
    checked frames against the oracle on the GPU's pre-stage state (SURVEY §8(c) Sequences)."""
    base, fl = synth.make_sequence_frames(cfg, frames)
    c = base["cfg"]
    k, nn = c.k, c.n_nbr
    prm = M.mis_default_params(k=k, n_nbr=nn, gn_iters=c.gn_iters, pcg_iters=c.pcg_iters)
    ctx = M.Context(prm)
    n0 = base["xyz"].shape[0]
    M.mis_set_model(ctx.ptr, base["xyz"], base["nrm"], base["rgb"], base["weight"], base["stamp"],
                    capacity=n0 + 4 * c.H * c.W)
    M.mis_set_graph(ctx.ptr, base["g"], base["nbr"])
    m = base["g"].shape[0]
    it = base["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    box = node_spacing(base["xyz"], n0)                 # the model's point spacing (P:597 point density)
    node_grid = 1.3 * node_spacing(base["xyz"], m)      # ~ the initial node density
    op = oracle_params(prm)
    O.set_threads(8)
    try:
        for f in fl:
            fi = f["frame"]
            chk = fi in checked
            if chk:
                mod, g, nbr = _state(ctx, k, m, nn)
                pb = O.Problem(mod["xyz"], mod["nrm"], mod["knn_idx"], mod["knn_w"], g, nbr)
                fr = O.Frame(f["depth"], it, f["pose"])
            rep = M.report_dict(M.mis_register(ctx.ptr, f["depth"], intr, f["pose"], f["feat_src"], f["feat_dst"]))
            assert rep["status"] == 0
            if chk:
                Rg = M.mis_get_nodes_f64(ctx.ptr, m)
                Ro, Eo, _ = O.register(op, pb, fr)
                assert np.abs(Rg[:, 9:] - Ro[:, 9:]).max() < 0.01, fi
                assert max(rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)) < 1e-4, fi
                M.mis_dbg_set_nodes(ctx.ptr, Ro.astype(np.float32))   # warp both sides with the same field
                Rt = Ro.astype(np.float32).astype(np.float64)
            M.mis_warp(ctx.ptr)
            if chk:
                w = M.mis_get_model(ctx.ptr, k)
                xo, no, go = O.warp_model(pb, Rt)
                pos = {int(i): p for p, i in enumerate(mod["ids"])}
                src = np.array([pos[int(i)] for i in w["ids"]])
                assert np.abs(w["xyz"] - xo[src]).max() < 0.05, fi
                assert np.abs(w["nrm"] - no[src]).max() < 1e-4, fi
                # fusion on the warped GPU model (state injection)
                H, W_ = c.H, c.W
                owner, why = M.mis_dbg_fuse_register(ctx.ptr, H, W_, w["xyz"].shape[0])
                gn = M.mis_get_graph(ctx.ptr, np.zeros((m, 3), np.float32))
                o = O.fuse(op, w["xyz"], w["nrm"], w["rgb"], w["weight"], w["stamp"], fr, f["rgb_obs"], fi, gn)
                ids_before = np.arange(w["xyz"].shape[0])            # oracle indices = GPU internal order here
            n_out, st = M.mis_fuse(ctx.ptr, f["rgb_obs"], fi)
            if chk:
                # check_fusion matches points by caller id: map the GPU ids to their pre-fusion position
                check_fusion(_IdShim(w["ids"]), ctx, k, o, fr, owner, why, ids_before, fi, n_out, st)
            pre = M.mis_get_model(ctx.ptr, k) if chk else None
            nf, fst = M.mis_filter(ctx.ptr, box, fi, 10, 3.0)
            if chk:
                of = O.filter_points(pre["xyz"], pre["nrm"], pre["rgb"], pre["weight"], pre["stamp"], pre["ids"], box,
                                     fi, 10, 3.0, prm.omega_max)
                fm = M.mis_get_model(ctx.ptr, k)
                assert nf == len(of["ids"]) and (fm["ids"] == of["ids"]).all(), fi
                assert (fm["weight"] == of["weight"].astype(np.float32)).all() and (fm["stamp"] == of["stamp"]).all()
                assert np.abs(fm["xyz"] - of["xyz"]).max() < 1e-3
                m, _, _ = check_regeneration(ctx, k, nn, node_grid)
            else:
                m = M.mis_regenerate_nodes(ctx.ptr, node_grid)
    finally:
        O.set_threads(1)
    assert 0.5 * n0 < nf < 4 * n0          # the model stays bounded over the sequence (Alg. 3)


class _IdShim:
    """check_fusion reads the model through M.mis_get_model and matches caller ids; in a sequence
    the ids are those of earlier frames, so translate them to the oracle's indices: a point present
    before the fusion -> its pre-fusion position, a lifted point -> n + its rank among the new ids
    (fresh ids are handed out in row-major pixel order, the oracle's lift order)."""

    def __init__(self, ids_before):
        self._old = np.asarray(ids_before)
        self._pos = {int(i): p for p, i in enumerate(self._old)}

    def mis_get_model(self, ptr, k):
        mod = M.mis_get_model(ptr, k)
        ids = mod["ids"]
        old = np.isin(ids, self._old)
        out = np.empty_like(ids)
        out[old] = [self._pos[int(i)] for i in ids[old]]
        out[~old] = self._old.size + np.argsort(np.argsort(ids[~old]))
        mod["ids"] = out
        return mod
