"""Host-memory frame inputs go through the context's copy stream (depth before the frame prep,
colours before the fusion's update kernel; DESIGN.md §5 host synchronisation): two consecutive
frames with pinned host inputs must give the same registration, fused model and lifted points
as the same frames with device inputs (within fp32 atomic-order rounding), including the reuse
of the staging buffers by the second frame."""
import numpy as np
import pytest

from tests.common import scene_problem

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def _run(sc, pb, host):
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
        rep = M.report_dict(M.mis_register(ctx.ptr, depth, intr, sc["pose"], fs, fd))
        assert rep["status"] == 0
        energies.append(rep["energy"][:, 4])
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
        assert abs(na - nb) <= max(5, 1e-4 * nb)
        assert np.abs(sa - sb).max() <= max(5, 1e-4 * nb)
    # the caller's points (ids < n0): lifted points get ids in pixel order, so one pixel registered
    # in one run and lifted in the other (atomic-order rounding deciding a |dz| tie) shifts every
    # later id; two fusions in a row can also move an occasional winner, so the gate is on 99.9 %
    n = pb.xyz.shape[0]
    dx = np.abs(xh[:n] - xd[:n]).max(axis=1)
    assert np.quantile(dx, 0.999) < 0.05, np.quantile(dx, 0.999)   # mm, the warped / fused gate
    assert dx.max() < 1.0, dx.max()
    dc = np.abs(ch[:n] - cd[:n]).max(axis=1)
    assert np.quantile(dc, 0.999) < 1e-3
