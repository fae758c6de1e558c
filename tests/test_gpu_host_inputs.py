"""Host-memory frame inputs go through the context's copy stream (depth before the frame prep,
colours before the fusion's update kernel; DESIGN.md §5 host synchronisation): two consecutive
frames with pinned host inputs must give the same registration (within fp32 atomic-order
rounding) and, bit for bit, the same fused model and lifted points as the same frames with
device inputs, including the reuse of the staging buffers by the second frame.  (The node state is
reset to the identity after each registration, so the warp and the fusion -- fp64 decisions, no
float atomics -- are deterministic and the two runs must agree exactly.)"""
import numpy as np
import pytest

from tests.common import scene_problem

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def _run(sc, pb, host, stage=False):
    torch = pytest.importorskip("torch")
    prm = M.mis_default_params(k=pb.k, n_nbr=pb.n_nbr)
    ctx = M.Context(prm)
    c = sc["cfg"]
    M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], None,
                    capacity=pb.xyz.shape[0] + 3 * c.H * c.W)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr, pb.idx, np.ascontiguousarray(pb.w, np.float32))
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    if host:
        cv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    else:
        cv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    depth, rgb, fs, fd = cv(sc["depth"]), cv(sc["rgb_obs"]), cv(pb.fsrc), cv(pb.fdst)
    energies, sizes = [], []
    for frame in (1, 2):
        if stage and frame == 2:   # the colour upload issued before the registration (mis_stage_colour)
            M.mis_stage_colour(ctx.ptr, rgb)
        rep = M.report_dict(M.mis_register(ctx.ptr, depth, intr, sc["pose"], fs, fd))
        assert rep["status"] == 0
        energies.append(rep["energy"][:, 4])
        ident = np.zeros((pb.g.shape[0], 12), np.float32)
        ident[:, [0, 4, 8]] = 1.0                       # R_j = I, t_j = 0
        M.mis_dbg_set_nodes(ctx.ptr, ident)
        M.mis_warp(ctx.ptr)
        n_out, stats = M.mis_fuse(ctx.ptr, rgb, frame)
        sizes.append((n_out, stats.copy()))
    md = M.mis_get_model(ctx.ptr, pb.k)
    order = np.argsort(md["ids"])
    return energies, sizes, md["xyz"][order], md["rgb"][order]


def test_host_inputs_match_device_inputs():
    sc, pb, fr, _ = scene_problem("c2")
    eh, sh, xh, ch = _run(sc, pb, True)
    ed, sd, xd, cd = _run(sc, pb, False)
    for a, b in zip(eh, ed):
        assert np.allclose(a, b, rtol=1e-3)
    for (na, sa), (nb, sb) in zip(sh, sd):
        assert na == nb and (sa == sb).all()
    assert (xh == xd).all() and (ch == cd).all()


def test_staged_colour_matches_device_inputs():
    """mis_stage_colour (the next fusion's host colour uploaded while the registration runs) gives the
    same fused model, bit for bit, as device colours; its argument errors."""
    torch = pytest.importorskip("torch")
    sc, pb, fr, _ = scene_problem("c2")
    es, ss, xs, cs = _run(sc, pb, True, stage=True)
    ed, sd, xd, cd = _run(sc, pb, False)
    for (na, sa), (nb, sb) in zip(ss, sd):
        assert na == nb and (sa == sb).all()
    assert (xs == xd).all() and (cs == cd).all()
    ctx = M.Context(M.mis_default_params())
    with pytest.raises(M.MisError):   # no frame size known yet
        M.mis_stage_colour(ctx.ptr, np.zeros((4, 4, 3), np.float32))
    with pytest.raises(ValueError):   # device colours are read in place, not staged
        M.mis_stage_colour(ctx.ptr, torch.zeros((4, 4, 3), device="cuda"))
