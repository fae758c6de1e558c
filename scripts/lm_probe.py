import numpy as np, sys
sys.path.insert(0, "/root/repo")
import oracle as O
from paper_1803_02009_b200 import mis as M
from tests.common import scene_problem
from tests.test_gpu_parity import make_ctx, oracle_params, rot_err
from tests.test_gpu_lm import _near_ties
for cfg, G in [("c1", 8), ("c2", 6), ("c1", 12), ("c3", 5)]:
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb, flags=M.MIS_F_LM, gn_iters=G)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G)
    Ro, Eo, nao, acco = O.register(prm, pb, fr, with_accepted=True)
    ties = _near_ties(Eo[:, 4], acco, 1e-5)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1).max()
    rerr = max(rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m))
    print(cfg, G, "gpu", rep["accepted"].astype(int), "ora", acco, "ties", ties, "terr %.2e rerr %.2e" % (terr, rerr),
          "Erel %.1e" % np.abs(rep["energy"][:, 4] / Eo[:, 4] - 1).max())
