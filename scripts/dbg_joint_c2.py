import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from tests.common import scene_problem
from tests.test_gpu_pose import perturbed_pose, joint_ctx, ofr
from tests.test_gpu_parity import M, oracle_params, rot_err
sc, pb, fr, _ = scene_problem("c2")
prior = perturbed_pose(np.array(fr.s.pose[:]))
res = []
Ro = None
for rep_i in range(4):
    ctx, sc2 = joint_ctx(sc, pb, prior)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    if Ro is None:
        prm = oracle_params(ctx.params, joint_pose=1, w_r=ctx.params.w_r, w_p=ctx.params.w_p)
        Ro, po, Eo, nao = O.register_pose(prm, pb, ofr(sc2))
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    print(rep_i, "terr", terr.max(), "rerr", rerr.max(), "res", rep["pcg_rel_res"])
    ctx.close()
