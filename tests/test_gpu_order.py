"""K13 model ordering on the GPU.  For k <= 4 and m < 65535 the model is grouped by exact kNN
tuple through a hash table (no sort): every tuple's points must be one contiguous run
(segments == distinct tuples, no split), the permutation must be a bijection (ids), and the
registration must equal the radix-sort ordering's (MIS_ORDER_BY_SORT=1) within fp32 rounding."""
import os

import numpy as np
import pytest

from tests.common import scene_problem
from tests.test_gpu_parity import make_ctx, rot_err

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_grouped_order_contiguous_tuples(cfg):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    md = M.mis_get_model(ctx.ptr, pb.k)
    n = pb.xyz.shape[0]
    assert np.array_equal(np.sort(md["ids"]), np.arange(n))                 # a permutation
    tup = np.sort(np.asarray(md["knn_idx"]).reshape(n, pb.k), axis=1)
    change = np.any(tup[1:] != tup[:-1], axis=1)
    runs = 1 + int(change.sum())
    distinct = len(np.unique(tup, axis=0))
    assert runs == distinct                                                 # one run per tuple
    assert rep["n_segments"] == distinct
    # internal order carries the caller's points: positions and skinning follow the ids
    assert np.allclose(md["xyz"], pb.xyz[md["ids"]])


def test_grouped_matches_sorted_registration():
    sc, pb, fr, _ = scene_problem("c2")
    m = pb.g.shape[0]
    out = {}
    for mode in ("0", "1"):
        os.environ["MIS_ORDER_BY_SORT"] = mode
        try:
            ctx = make_ctx(sc, pb)
            rep = M.report_dict(M.mis_register(ctx.ptr))
            out[mode] = (M.mis_get_nodes_f64(ctx.ptr, m), rep)
        finally:
            os.environ.pop("MIS_ORDER_BY_SORT", None)
    (Ra, ra), (Rb, rb) = out["0"], out["1"]
    assert ra["n_segments"] <= rb["n_segments"]   # hashing may split a segment, grouping never
    assert np.abs(Ra[:, 9:] - Rb[:, 9:]).max() < 1e-3
    assert max(rot_err(Ra[j, :9].reshape(3, 3), Rb[j, :9].reshape(3, 3)) for j in range(m)) < 1e-5
    assert np.allclose(ra["energy"][:, 4], rb["energy"][:, 4], rtol=1e-3)   # as the MIRROR gate (fp32 atomics order)
