/* oracle.h -- plain, slow, fp64 CPU oracle of the MIS-SLAM (arXiv 1803.02009)
 * non-rigid registration + fusion hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call it.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1803_02009_b200/csrc, include/mis.h); neither side includes the other.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "R-An" = the
 * reading An of DESIGN.md §3.  Units are mm throughout.
 * All arithmetic is fp64; fp32 inputs are upcast exactly.
 */
#ifndef MIS_ORACLE_H
#define MIS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t k;            /* nodes per point (Eq. 1 "k"), R-A5                         */
  int32_t n_nbr;        /* regulariser neighbours per node (Eq. 6 N(j)), R-A15       */
  double w_data, w_pt, w_reg, w_corr;   /* P:598 (w_pt: R-A13)                      */
  double eps_d, eps_n_deg;              /* Eq. 7 thresholds                   */
  double tau_z, delta_deg, trunc, omega_max; /* Alg. 1 / Eq. 11 / Eq. 15 */
  int32_t gn_iters, pcg_iters;
  double lambda;                        /* GN damping, R-A16                         */
  int32_t solve_mode;                   /* 0 = EXACT, 1 = MIRROR (same P as GPU)     */
  int32_t lm;                           /* 1: Levenberg-Marquardt, R-A29 */
  double lm_mu0;                        /* initial Marquardt damping (1e-3)    */
  int32_t joint_pose;                   /* 1: joint global-pose refinement (NEXT-2, below) */
  double w_r, w_p;                      /* Eq. 10 prior weights, P:598 (1e6, 1000)    */
  double w_rot;                         /* Eq. 4 weight, P:598 (1000); the _aff functions */
} or_params;
/* joint_pose (NEXT-2, readings A37-A40): the pose of Eq. 1 becomes unknown
 * number m (after the m nodes; "only 6 more variables") with the local increment
 * R <- R Exp(dphi), T <- T + R dtau (A37); or_frame.pose is both its start value and the
 * ORB-SLAM prior of Eq. 10: E_r = |wrap(euler_zyx(R^T) - euler_zyx(R0^T))|^2 (scope
 * orientation as yaw-pitch-roll, A38), E_p = |c - c0|^2 with the scope position
 * c = -R^T T (A39).  Energy rows then have 7 entries: E_data, E_pt, E_reg, E_corr, E_r,
 * E_p, weighted total. */

typedef struct {
  int32_t W, H;
  double fx, fy, cx, cy;
  const float* depth;   /* H*W, mm; <=0 or non-finite = invalid                     */
  double pose[12];      /* world->camera: R row-major (9), T (3); Eq. 1 R_i, T_i      */
} or_frame;

typedef struct {
  int64_t n;
  const float* xyz;     /* n*3 model points v_i (world)                              */
  const float* nrm;     /* n*3 model normals                                        */
  const int32_t* idx;   /* n*k node ids per point (Eq. 1 "k nearest")               */
  const float* w;       /* n*k skinning weights (Eq. 2), normalised in the warp     */
  int32_t m;
  const float* g;       /* m*3 node positions g_j                                   */
  const int32_t* nbr;   /* m*n_nbr neighbour ids, -1 = none                         */
  int32_t nf;
  const float* fsrc;    /* nf*3 feature model positions V_i (world, frame n-1)      */
  const float* fdst;    /* nf*3 feature observed positions (camera, frame n)        */
} or_problem;

/* why-bits of one association (Eq. 7 / Alg. 1 gates), evaluated in order and
 * short-circuited at the first failure. */
enum { OR_Z = 1, OR_FRAME = 2, OR_DEPTH = 4, OR_NORMAL = 8, OR_DIST = 16, OR_ANGLE = 32, OR_ALL = 63 };

/* Host threads of the oracle (default 1): independent points / pixels / queries are split over
 * them; per-thread partial normal equations are merged in thread order.  bench.py's all-cores
 * column only -- the pins and the parity tests run single-threaded. */
void or_set_threads(int32_t n);
/* O0: back-projection and central-difference normals of a depth map. */
void or_frame_prep(const or_frame* f, double* q, double* N, uint8_t* dvalid, uint8_t* nvalid);
/* O1: Eq. 2 skinning of nq query points against m nodes. idx/w: nq*k, nearest
 * first; margin[i] = relative gap deciding the k-set (for tie exclusion). */
void or_skin(int64_t nq, const float* p, int32_t m, const float* g, int32_t k,
             int32_t* idx, double* w, double* margin);
/* A18: Rodrigues exponential. */
void or_exp(const double w[3], double R[9]);
/* O3a: warp every point (Eq. 1).  x_hat: world (before the pose), vt/nt:
 * camera frame.  ok[i]=0 when the weights sum to <= 0 or the normal vanishes. */
void or_warp(const or_problem* p, int32_t k, const double* Rt, const double pose[12],
             double* x_hat, double* n_hat, double* vt, double* nt, uint8_t* ok);
/* O3b: projective association (Eq. 7). */
void or_associate(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                  int32_t* pix, uint8_t* why, double* margin);
/* O3c-g: normal equations in 6x6 node blocks (upper triangle j<=l, full 6x6
 * each, sorted by (row, col)).  Returns the number of blocks; writes at most
 * cap of them.  energy[5] = E_data, E_pt, E_reg, E_corr, weighted total.
 * fidx/fw: feature skinning (nf*k) from or_skin. */
int64_t or_system(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                  const int32_t* fidx, const double* fw, int64_t cap,
                  int32_t* brow, int32_t* bcol, double* bval, double* rhs, double energy[5],
                  int64_t* n_assoc);
/* Dense Jacobian / residual stack for small problems (pins P6, P7).  Rows:
 * per associated point 1 (plane) + 3 (point), per directed edge 3, per feature
 * 3, each scaled by sqrt(weight).  pix_frozen (n) fixes the association (-1 =
 * none) so that finite differences see a smooth function.  J: rows*6m. */
int64_t or_residuals(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                     const int32_t* pix_frozen, const int32_t* fidx, const double* fw,
                     int64_t cap_rows, double* r, double* J);
/* O3h: solve (H + lambda I) x = rhs from or_system's blocks. mode 0 EXACT, 1 MIRROR. */
int32_t or_solve(int32_t m, int64_t nblk, const int32_t* brow, const int32_t* bcol, const double* bval,
                 const double* rhs, double lambda, int32_t mode, int32_t pcg_iters, double* x);
/* O3: fixed-iteration Gauss-Newton registration.  Rt (m*12, R row-major + t)
 * is the initial state on entry and the result on exit.  energy: (G+1)*5 (start
 * of each iteration, then final), n_assoc: G+1.
 * prm->lm = 1: Levenberg-Marquardt instead ("Levenberg-Marquardt"; damping
 * and schedule S:290; R-A29): iteration it evaluates the energy of the trial
 * state (energy[it], it = 0 is the start), accepts it if it = 0 or the total is
 * strictly lower than the last accepted one (accepted[it] = 1; mu *= 0.5 for it > 0),
 * else restores the last accepted state and keeps its system (mu *= 10); then solves
 * (H' + lambda I) x = b with H' = H whose diagonal entries are scaled by (1 + mu) and
 * steps from the accepted state.  Entry G is the final trial, kept if it is accepted.
 * accepted (G+1) may be NULL. */
void or_register(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt,
                 double* energy, int64_t* n_assoc, int32_t* accepted);
/* ---- NEXT-2: joint global pose (see or_params.joint_pose) ---- */
/* ZYX Euler angles (yaw psi, pitch theta, roll phi) of a rotation O = Rz(psi) Ry(theta) Rx(phi). */
void or_euler_zyx(const double O[9], double e[3]);
/* Eq. 10 prior residuals at the current pose cur (world->camera R row-major 9, T 3) against
 * prior: r[0..3) = wrap(euler_zyx(R^T) - euler_zyx(R0^T)), r[3..6) = c - c0, c = -R^T T;
 * J (6x6 row-major) w.r.t. [dphi, dtau] of A37.  Returns 0, or 1 at gimbal lock
 * (|cos theta| < 1e-6: the E_r rows are zero). */
int32_t or_pose_prior(const double prior[12], const double cur[12], double r[6], double J[36]);
/* or_system / or_residuals / or_register with the pose: pose_cur (12) is the current pose
 * (or_frame.pose the prior); blocks over m + 1 unknowns (the pose is unknown m), rhs 6(m+1),
 * energy[7]; J: rows x 6(m+1) incl. the 6 sqrt-weighted prior rows (last).  or_register_pose:
 * pose_io = start pose on entry (normally the prior), the refined pose on exit; energy (G+1)*7. */
int64_t or_system_pose(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                       const double pose_cur[12], const int32_t* fidx, const double* fw, int64_t cap,
                       int32_t* brow, int32_t* bcol, double* bval, double* rhs, double energy[7],
                       int64_t* n_assoc);
int64_t or_residuals_pose(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                          const double pose_cur[12], const int32_t* pix_frozen, const int32_t* fidx,
                          const double* fw, int64_t cap_rows, double* r, double* J);
void or_register_pose(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt, double* pose_io,
                      double* energy, int64_t* n_assoc, int32_t* accepted);
/* ---- NEXT-4: affine nodes A_j + E_rot (Eq. 1, Eq. 4-6; readings A41-A45) ----
 * At: m x 12 (A_j row-major 9, t_j 3); 12 unknowns per node [dA_j row-major, dt_j], additive
 * update; normals warp by A_j^-T (A itself if |det| < 1e-9).  Blocks 12 x 12 (144 doubles),
 * rhs 12m, energy[6] = E_data, E_pt, E_reg, E_corr, E_rot, weighted total (w_rot). */
void or_warp_aff(const or_problem* p, int32_t k, const double* At, const double pose[12], double* x_hat,
                 double* n_hat, double* vt, double* nt, uint8_t* ok);
void or_associate_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At, int32_t* pix,
                      uint8_t* why, double* margin);
/* Eq. 5 residuals r[6] (c1.c2, c1.c3, c2.c3, |c1|^2-1, |c2|^2-1, |c3|^2-1) and J (6 x 9, A row-major) */
void or_rot(const double A[9], double r[6], double J[54]);
int64_t or_system_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At,
                      const int32_t* fidx, const double* fw, int64_t cap, int32_t* brow, int32_t* bcol, double* bval,
                      double* rhs, double energy[6], int64_t* n_assoc);
int64_t or_residuals_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At,
                         const int32_t* pix_frozen, const int32_t* fidx, const double* fw, int64_t cap_rows, double* r,
                         double* J);
int32_t or_solve_aff(int32_t m, int64_t nblk, const int32_t* brow, const int32_t* bcol, const double* bval,
                     const double* rhs, double lambda, int32_t mode, int32_t pcg_iters, double* x);
/* prm->lm: Levenberg-Marquardt with the schedule of or_register (R-A29); accepted (G+1) nullable */
void or_register_aff(const or_params* prm, const or_problem* p, const or_frame* f, double* At, double* energy,
                     int64_t* n_assoc, int32_t* accepted);
void or_warp_model_aff(const or_problem* p, int32_t k, const double* At, double* xyz_out, double* nrm_out,
                       double* g_out);
/* O4: apply the field: live world state x_hat, unit normals; advanced nodes g+t. */
void or_warp_model(const or_problem* p, int32_t k, const double* Rt, double* xyz_out, double* nrm_out,
                   double* g_out);

typedef struct {
  int64_t n;
  const float* xyz; const float* nrm; const float* rgb; const float* weight; const int32_t* stamp;
} or_model;

/* O5 + O6: Alg. 1 registration, Eq. 12-15 fusion, Alg. 2 Step 3 lift.
 * Outputs for the n existing points (fused in place of the copies) and the
 * lifted points appended after them (capacity n + W*H).  owner: W*H point id
 * or -1; key_margin: W*H gap between the two best keys (mm, +inf if < 2).
 * Returns the number of lifted points. */
int64_t or_fuse(const or_params* prm, const or_model* mdl, const or_frame* f, const float* rgb_obs,
                int32_t frame_index, int32_t m, const float* g,
                double* xyz_out, double* nrm_out, double* rgb_out, double* weight_out, int32_t* stamp_out,
                int32_t* lift_idx, double* lift_w, double* lift_margin,
                int64_t* owner, double* key_margin, uint8_t* why, double* gate_margin);

/* O7 (NEXT-1): Alg. 3 point filtering with the downsampling of
 * P:597 and the reading of S:369 (A30-A34).  Cells: (floor(x/grid),
 * floor(y/grid), floor(z/grid)), each quotient an IEEE fp32 division and floor
 * (A30).  Per non-empty cell, members in ascending input index: position,
 * normal and colour weighted by omega (unweighted if the cell's omega sum is
 * 0), the normal renormalised (the first member's if the sum is 0), omega =
 * min(sum omega, omega_max), stamp = max, id = the first member's (A31).
 * Then Alg. 3: delete the merged point iff stamp < frame - tau_time and
 * omega < tau_weight; stable = omega >= tau_weight (A32).  Survivors are
 * written in ascending (kx, ky, kz) order (A33).  Outputs sized n.
 * cells_out (nullable): the number of non-empty cells.  Returns survivors. */
int64_t or_filter(int64_t n, const float* xyz, const float* nrm, const float* rgb, const float* weight,
                  const int32_t* stamp, const int64_t* ids, float grid, int32_t frame_index, int32_t tau_time,
                  float tau_weight, float omega_max, double* xyz_out, double* nrm_out, double* rgb_out,
                  double* weight_out, int32_t* stamp_out, int64_t* ids_out, uint8_t* stable_out,
                  int64_t* cells_out);

/* O8 (NEXT-1): Alg. 2 Step 5 node regeneration as S:102-104 (reading A36): the
 * centroids of the occupied grid cells (fp32 floor(x/grid) per axis, A30) in ascending (kx, ky, kz)
 * order, identity transforms, N(j) = the n_nbr nearest other nodes (ties to the lower index, -1
 * padded).  g_out: n*3 capacity; nbr_out: n*n_nbr; nbr_margin: n (relative gap at the n_nbr cut).
 * Returns the node count. */
int64_t or_regenerate_nodes(int64_t n, const float* xyz, float grid, int32_t n_nbr, double* g_out,
                            int32_t* nbr_out, double* nbr_margin);

#ifdef __cplusplus
}
#endif
#endif
