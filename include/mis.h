/* mis.h -- C-ABI of the B200 (sm_100a) MIS-SLAM registration + fusion hot path.
 *
 * MIS-SLAM: "MIS-SLAM: Real-time Large Scale Dense Deformable SLAM System in
 * Minimal Invasive Surgery Based on Heterogeneous Computing", arXiv 1803.02009.
 * Citations: P:n = PAPER.md line n (equation / algorithm named), S:n = SPEC.md
 * line n, "reading An" = DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Units: millimetres; angles in degrees in mis_params, radians elsewhere.
 *  - mis_mem says where every pointer argument of the call lives:
 *    MIS_MEM_HOST (pageable or pinned host memory) or MIS_MEM_DEVICE (device
 *    memory of the context's GPU, e.g. a torch tensor's data_ptr()).  Device
 *    inputs are read in stream order on the context stream: a device buffer
 *    must stay valid until the work the call enqueued has run (as with any
 *    asynchronous CUDA call; freeing it through the same stream is safe).
 *  - Ownership: the library keeps its state in context-owned device memory
 *    (allocated with cudaMalloc on the context's device) and never retains a
 *    caller pointer after the enqueued work of the call has run (the depth
 *    map and colours are read in place by the frame's kernels, everything
 *    else is copied).  Outputs are written into caller buffers.  Calls with
 *    host outputs synchronise the context stream before returning; calls with
 *    device outputs do not.
 *  - Errors: every call returns a mis_status; no exception crosses the
 *    boundary.  mis_last_error() gives a human-readable message for the last
 *    failing call on that context.  Per-point degeneracies (z <= 0, invalid
 *    depth, vanishing warped normal) are masked, never errors.
 *  - Threading: a context is not re-entrant; distinct contexts are independent.
 *  - Layouts: xyz-like arrays are n x 3 row-major float32 (x, y, z), node
 *    states are m x 12 float32 (R row-major 9, t 3), pose[12] is the
 *    world->camera transform (R row-major 9, T 3) of Eq. 1.
 *  - Internal point order: points are kept grouped by their canonical kNN
 *    tuple, every tuple's points contiguous (K13: exact-tuple hash grouping
 *    for k <= 4 and m < 65535, where the order of the groups and within a
 *    group is unspecified; else a stable radix sort of a tuple hash); every
 *    per-point output is in that internal order and mis_get_model returns the
 *    caller ids that map it back.
 */
#ifndef MIS_H
#define MIS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define MIS_ABI_VERSION 2
#define MIS_MAX_GN 32
#define MIS_MAX_K 8

typedef struct mis_ctx mis_ctx;

typedef enum {
  MIS_OK = 0,
  MIS_E_ARG = 1,       /* invalid argument (value, size, range)                     */
  MIS_E_STATE = 2,     /* call out of order (e.g. register before set_graph)        */
  MIS_E_CUDA = 3,      /* CUDA runtime error (message in mis_last_error)            */
  MIS_E_NCCL = 4,      /* NCCL error or NCCL unavailable with world > 1             */
  MIS_E_NOMEM = 5,     /* device allocation failed                                  */
  MIS_E_CAPACITY = 6,  /* Group-2 growth would exceed the model capacity            */
  MIS_E_NUMERIC = 7    /* non-finite GN step or PCG scalar (e.g. a NaN input): the node
                          state is rolled back to before that GN iteration and no later
                          iteration of the registration updates it                    */
} mis_status;

typedef enum { MIS_MEM_HOST = 0, MIS_MEM_DEVICE = 1 } mis_mem;

/* Pinhole intrinsics: fx, fy > 0; 0 <= cx < width; 0 <= cy < height. */
typedef struct { float fx, fy, cx, cy; int32_t width, height; } mis_intrinsics;

/* Flags */
#define MIS_F_FINAL_ENERGY 1u   /* mis_register also evaluates the energy after the last update */
#define MIS_F_GRID_SOLVER  4u   /* force the grid-wide PCG kernel (else the cluster-resident one
                                   whenever the system fits in one cluster's shared memory)       */
#define MIS_F_STANDARD_PCG 8u   /* cluster kernel: textbook PCG recurrences (2 barriers/iteration)
                                   instead of the pipelined variant (1 barrier/iteration)         */
#define MIS_F_LM          16u   /* Levenberg-Marquardt instead of Gauss-Newton (SURVEY
                                   NEXT-3; reading A29): iteration it evaluates the trial state,
                                   accepts it if it = 0 or its weighted total energy is strictly
                                   lower than the last accepted one (damping mu x 0.5, mu_0 =
                                   1e-3) else restores the last accepted state and its
                                   system (mu x 10), then solves (H' + lambda I) x = b, H' = H
                                   with its diagonal entries times (1 + mu), from that state.
                                   The last trial is evaluated too (energy row [iters]) and kept
                                   only if accepted.  Per-iteration decisions in report n_guard.
                                   Runs in the register-resident pipelined cluster PCG (systems
                                   of C1-C3 size) or else the pipelined grid PCG (the damped
                                   block-Jacobi inverses built there); combines with
                                   MIS_F_JOINT_POSE and MIS_F_AFFINE; single GPU (MIS_E_ARG)        */
#define MIS_F_JOINT_POSE  32u   /* NEXT-2 (readings A37-A40): the global pose (R, T) of
                                   Eq. 1 is refined jointly with the nodes as unknown number m
                                   ("only 6 more variables"): increment R <- R Exp(dphi),
                                   T <- T + R dtau; the pose given to mis_register / mis_set_frame
                                   is the start value and the ORB-SLAM prior of Eq. 10:
                                   E_r = |wrap(euler_zyx(R^T) - euler_zyx(R0^T))|^2 (scope
                                   orientation as yaw, pitch, roll), E_p = |c - c0|^2 with the
                                   scope position c = -R^T T, weights w_r, w_p.  The pose enters
                                   every point / feature row (Jacobian R [-[x_hat]x, I]), the
                                   block-Jacobi preconditioner and lambda like a node.  The refined
                                   pose is used by mis_warp / mis_fuse of the frame and read with
                                   mis_get_pose.  Solved by the grid-wide PCG (the pose row is
                                   dense).  Requires k <= 7 and world == 1 (MIS_E_ARG)              */
#define MIS_F_AFFINE      64u   /* NEXT-4 (Eq. 1, Eq. 4-6; readings A41-A45): every node carries
                                   the paper's general 3x3 matrix A_j instead of a rotation -- 12
                                   unknowns per node [dA_j row-major, dt_j], additive update,
                                   12 x 12 blocks -- with E_rot (Eq. 4-5: the columns' Gram matrix
                                   minus I, weight w_rot) and Eq. 6 with A_j; normals warp by
                                   A_j^-T (A_j itself if |det A_j| < 1e-9).  Node states in the
                                   R9_t3 arrays of mis_get_nodes / mis_dbg_set_nodes are then
                                   A (row-major 9), t.  Gauss-Newton with the grid-wide PCG;
                                   requires k <= 4 and world == 1; not with MIS_F_JOINT_POSE
                                   (MIS_E_ARG)                                                      */

/* Method parameters; defaults (mis_default_params) are the paper's. */
typedef struct {
  int32_t k;            /* nodes per point, Eq. 1 (reading A5), 1..8                       */
  int32_t n_nbr;        /* regulariser neighbours per node, Eq. 6 N(j) (reading A15)       */
  float w_data;         /* Eq. 8 weight, 1                                         */
  float w_point;        /* dense point-to-point weight, 1 (reading A13)                    */
  float w_reg;          /* Eq. 6 weight, 1e4                                       */
  float w_corr;         /* Eq. 9 weight, 10                                        */
  float eps_d_mm;       /* Eq. 7 distance gate, 15 mm                              */
  float eps_n_deg;      /* Eq. 7 angle gate, 10 deg (reading A8)                    */
  float tau_z_mm;       /* Alg. 1 depth gate, 10 mm                                */
  float delta_deg;      /* Alg. 1 angle gate, 10 deg                               */
  float trunc_mm;       /* Eq. 11 truncation, 40 mm (reading A20)                   */
  float omega_max;      /* Eq. 15 weight cap, 10 (reading A22)                      */
  int32_t gn_iters;     /* Gauss-Newton iterations G, 1..MIS_MAX_GN (reading A3)           */
  int32_t pcg_iters;    /* PCG iterations P per GN iteration, >= 1                         */
  float lambda;         /* GN damping, 1e-4 (reading A16)                                  */
  uint32_t flags;       /* MIS_F_*                                                         */
  float w_r;            /* Eq. 10 orientation prior weight, 1e6, MIS_F_JOINT_POSE  */
  float w_p;            /* Eq. 10 position prior weight, 1000, MIS_F_JOINT_POSE    */
  float w_rot;          /* Eq. 4 E_rot weight, 1000, MIS_F_AFFINE                  */
} mis_params;

/* Per-registration report (all host memory). */
typedef struct {
  int32_t iters;                       /* GN iterations run                                  */
  int32_t status;                      /* mis_status of the registration                    */
  double energy[MIS_MAX_GN + 1][5];    /* per iteration (state before its update): E_data,
                                          E_point, E_reg, E_corr, weighted total; row
                                          [iters] = after the last update (MIS_F_FINAL_ENERGY) */
  int64_t n_assoc[MIS_MAX_GN + 1];     /* associated points per iteration                   */
  float pcg_rel_res[MIS_MAX_GN];       /* sqrt(r.z / r0.z0) after the last PCG iteration    */
  int64_t nnzb;                        /* nonzero 6x6 blocks of H (both triangles)           */
  int64_t n_segments;                  /* distinct kNN tuples in the model                  */
  int32_t solver_cluster;              /* CTAs of the cluster-resident PCG (0: grid kernel)  */
  int32_t reserved;
  int64_t n_guard[MIS_MAX_GN + 1];     /* MIS_F_LM: 1 if the trial of iteration i (row [iters]: the
                                          final one) was accepted, else 0; Gauss-Newton: 0        */
  double energy_pose[MIS_MAX_GN + 1][2]; /* MIS_F_JOINT_POSE: E_r, E_p per iteration (unweighted;
                                          their weighted sum is part of energy[i][4]); else 0     */
  double energy_rot[MIS_MAX_GN + 1];   /* MIS_F_AFFINE: E_rot per iteration (unweighted; w_rot E_rot
                                          is part of energy[i][4]); else 0                        */
} mis_report;

int32_t mis_abi_version(void);
void mis_default_params(mis_params* out);

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t to
 * adopt (e.g. torch.cuda.current_stream().cuda_stream) or NULL to create one.
 * rank/world: this process' place in a data-parallel job (world >= 1);
 * nccl_unique_id: 128 bytes from mis_nccl_unique_id on rank 0 (broadcast by
 * the caller), NULL when world == 1.  With world > 1 every rank must pass its
 * own point shard to mis_set_model and the same node graph to mis_set_graph;
 * the node-block system is all-reduced over NCCL each GN iteration. */
mis_status mis_create(const mis_params* params, int device, void* cuda_stream, int rank, int world,
                      const void* nccl_unique_id, mis_ctx** out);
mis_status mis_destroy(mis_ctx* ctx);
const char* mis_last_error(const mis_ctx* ctx);
/* 128-byte NCCL unique id (rank 0 only).  MIS_E_NCCL if libnccl cannot be loaded. */
mis_status mis_nccl_unique_id(void* out128);
mis_status mis_set_params(mis_ctx* ctx, const mis_params* params);

/* Caller-provided device memory (e.g. torch.empty(bytes, dtype=torch.uint8,
 * device='cuda')).  mis_workspace_bytes: an upper bound of the device memory the context
 * allocates for a model capacity n_cap, m nodes and H x W frames, assuming at most
 * m (2 n_nbr + 1 + 4 k^2) nonzero 6x6 blocks (the node pairs sharing a kNN tuple or a
 * regulariser edge; surface-like graphs have 14 m at k = 4, 32 m at k = 8) and at most
 * max(4096, H W / 64) feature pairs.  mis_bind_workspace: from then on every buffer of the
 * context is carved from [dev_ptr, dev_ptr + bytes) (first fit, 256-byte aligned) instead of
 * cudaMalloc; must precede mis_set_model (MIS_E_STATE), dev_ptr must be 256-byte aligned device
 * memory of the context's GPU (MIS_E_ARG).  The caller owns the region and frees it after
 * mis_destroy.  A request the region cannot hold fails with MIS_E_NOMEM (the call's state is
 * unchanged up to the failing allocation; mis_last_error names the size).  mis_create's own
 * ~4 KB (report block, counters) stay cudaMalloc'ed. */
mis_status mis_workspace_bytes(const mis_ctx* ctx, int64_t n_cap, int32_t m, int32_t H, int32_t W, size_t* bytes);
mis_status mis_bind_workspace(mis_ctx* ctx, void* dev_ptr, size_t bytes);

/* Model points, Sec. II-A "five domains" + normal.  n >= 0 points,
 * capacity >= n bounds Group-2 growth in mis_fuse.  xyz: world positions v_i;
 * nrm: unit normals; rgb (n x 3, [0,1], NULL = 0); weight: fusion weights
 * omega (NULL = 1); stamp: frame stamps t_i (NULL = 0); ids: caller ids
 * (NULL = 0..n-1).  Invalidates the graph binding (call mis_set_graph next). */
mis_status mis_set_model(mis_ctx* ctx, int64_t n, mis_mem mem, const float* xyz, const float* nrm,
                         const float* rgb, const float* weight, const int32_t* stamp, const int64_t* ids,
                         int64_t capacity);

/* ED graph (Sec. II-D).  node_pos: m x 3 positions g_j; node_nbr:
 * m x n_nbr neighbour ids of Eq. 6, -1 padded, never self (MIS_E_ARG);
 * knn_idx / knn_w: n x k skinning of the model points in the caller's point
 * order (distinct ids per point, weights >= 0, normalised in the warp,
 * reading A6).  knn_idx == NULL: the skinning is computed on the device by
 * Eq. 2 (k+1 nearest nodes, ties to the lower id; requires m >= k+1).
 * Resets every node transform to the identity (R_j = I, t_j = 0).  Groups the
 * points by their canonical kNN tuple (internal order, see above).
 * Validation (MIS_E_ARG): with MIS_MEM_HOST inputs before returning; with
 * MIS_MEM_DEVICE inputs without a host synchronisation -- invalid ids are
 * clamped / dropped on the device and the next mis_register (or mis_dbg_*)
 * returns MIS_E_ARG and unbinds the graph. */
mis_status mis_set_graph(mis_ctx* ctx, int32_t m, mis_mem mem, const float* node_pos, const int32_t* node_nbr,
                         const int32_t* knn_idx, const float* knn_w);

/* Current observation: depth (H x W mm, <= 0 or non-finite = invalid),
 * intrinsics and the world->camera pose (the ORB-SLAM input of P:85, fixed
 * during registration, reading A2).  Computes the normal map (K1). */
mis_status mis_set_frame(mis_ctx* ctx, mis_mem mem, const float* depth_mm, const mis_intrinsics* intr,
                         const float pose[12]);
/* Sparse ORB feature pairs (Eq. 9): feat_src n_feat x 3 model-side
 * positions V_i (world, frame n-1), feat_dst n_feat x 3 observed positions
 * (camera frame, frame n).  Skinned on the device by Eq. 2. */
mis_status mis_set_features(mis_ctx* ctx, mis_mem mem, int32_t n_feat, const float* feat_src,
                            const float* feat_dst);

/* One registration (Sec. II-E/F): mis_set_frame + mis_set_features + G
 * Gauss-Newton iterations of warp (Eq. 1), association (Eq. 7), residuals
 * (Eq. 6, 8, 9, point-to-point), 6x6 block normal equations, block-Jacobi PCG
 * (P iterations, x0 = 0) and the node update R_j <- Exp(dtheta) R_j, t_j += dt
 * (reading A18), starting from the current node state.  depth_mm == NULL
 * keeps the frame of the last mis_set_frame; n_feat < 0 keeps the features.
 * rep (host, nullable) receives the report (synchronises). */
mis_status mis_register(mis_ctx* ctx, mis_mem mem, const float* depth_mm, const mis_intrinsics* intr,
                        const float pose[12], int32_t n_feat, const float* feat_src, const float* feat_dst,
                        mis_report* rep);

/* Node transforms: R9_t3 m x 12 float32 (mem) or fp64 master copy (host). */
mis_status mis_get_nodes(mis_ctx* ctx, mis_mem mem, float* R9_t3);
mis_status mis_get_nodes_f64(mis_ctx* ctx, double* R9_t3_host);
/* The pose of the last registration (host, 12 doubles: R row-major, T; world -> camera):
 * with MIS_F_JOINT_POSE the refined pose, else the frame's input pose. */
mis_status mis_get_pose(mis_ctx* ctx, double pose[12]);
/* Current node positions g_j (m x 3). */
mis_status mis_get_graph(mis_ctx* ctx, mis_mem mem, float* node_pos);
/* Current regulariser neighbour lists N(j) (m x n_nbr, -1 padded). */
mis_status mis_get_nbr(mis_ctx* ctx, mis_mem mem, int32_t* node_nbr);

/* Alg. 2 Step 2: apply the converged field to every point and
 * normal; the model becomes the live world-frame state x_hat_i; the nodes
 * advance g_j += t_j and reset (reading A26).  xyz_cam / nrm_cam (n x 3,
 * nullable, internal order) receive R x_hat + T and the camera-frame normals. */
mis_status mis_warp(mis_ctx* ctx, mis_mem mem, float* xyz_cam, float* nrm_cam);

/* Alg. 1 + Alg. 2 Step 3 on the current frame: exclusive
 * point-to-pixel registration (gates |z - D| < tau_z, < trunc, angle < delta;
 * smallest |dz| then lower internal index wins, reading A19), Eq. 12-15
 * weighted-average fusion of the winners, and lifting of every valid,
 * unregistered pixel into a new point (row-major order, omega = 1, stamp =
 * frame_index, skinned by Eq. 2).  rgb: H x W x 3 observed colour (mem;
 * NULL = no colour fusion, lifted colour 0).  n_out (host): new model size;
 * stats (host, nullable): [registered, lifted, valid pixels, model size].
 * MIS_E_CAPACITY (model unchanged) if the lift exceeds the capacity. */
mis_status mis_fuse(mis_ctx* ctx, mis_mem mem, const float* rgb, int32_t frame_index, int64_t* n_out,
                    int64_t stats[4]);

/* Start the upload of the next mis_fuse's host colour (H x W x 3 float, the current camera's H x W)
 * now, on the context's copy stream, so it overlaps whatever is issued before the fusion (e.g. the
 * registration); a following mis_fuse with the same host pointer uses the staged copy.  The buffer
 * must stay unchanged until that mis_fuse returns.  MIS_E_ARG: rgb NULL, a device pointer (device
 * colours are read in place anyway) or no frame size known yet (before the first frame). */
mis_status mis_stage_colour(mis_ctx* ctx, const float* rgb);

/* NEXT-1: Alg. 3 point filtering with the grid-box downsampling of
 * P:597 (readings A30-A34).  The model points are binned into the boxes
 * (floor(x/grid_mm), floor(y/grid_mm), floor(z/grid_mm)) of the world frame (fp32
 * division); each non-empty box becomes one point: omega-weighted average of
 * position, colour and normal (renormalised), omega = min(sum omega, omega_max),
 * stamp = max, id = the member's with the lowest internal index.  The merged
 * point is deleted iff stamp < frame_index - tau_time and omega < tau_weight
 * (Alg. 3 line 3); the stability flag S_i is omega >= tau_weight (not
 * stored).  Survivors are written in ascending (kx, ky, kz) box order; merged
 * boxes are re-skinned by Eq. 2 against the current nodes (requires m >= k+1),
 * single-member boxes keep their point's position and skinning; the node
 * graph is unchanged (Step 5 regeneration is a separate call).  Single GPU only
 * (world > 1: MIS_E_ARG, a box may span several ranks' shards).  grid_mm > 0,
 * tau_time >= 0.  n_out (host): new model size; stats (host, nullable):
 * [boxes, deleted, stable survivors, model size].  Two host synchronisations
 * (the box range, the survivor count).  MIS_E_ARG (model unchanged) if a
 * position is not finite, a box coordinate leaves (-2^30, 2^30) or the boxes'
 * range needs more than 63 key bits. */
mis_status mis_filter(mis_ctx* ctx, float grid_mm, int32_t frame_index, int32_t tau_time, float tau_weight,
                      int64_t* n_out, int64_t stats[4]);

/* NEXT-1: Alg. 2 Step 5 "Regenerate node and corresponding rotation and translation"
 * in the form of S:102-104 (reading A36): the nodes become the centroids (fp64 mean,
 * stored fp32) of the occupied cells (floor(x/g), floor(y/g), floor(z/g)) of the model points,
 * g = node_grid_mm (the paper's node density: 4 mm / 10 mm), each quotient an IEEE fp32
 * division (as mis_filter), in ascending (kx, ky, kz) order, with identity transforms (R_j = I,
 * t_j = 0); N(j) = the n_nbr nearest other nodes (ties to the lower index, -1 padded); every
 * point is re-skinned by Eq. 2 against the new nodes and the model regrouped -- i.e. exactly
 * mis_set_graph with these nodes and device skinning.  *m_out (host): the node count.  Two host
 * synchronisations (the cell range, the node count).  MIS_E_ARG (graph unchanged) for
 * node_grid_mm <= 0, a non-finite position, cells spanning more than 63 key bits, fewer than k+1
 * occupied cells or points, n_nbr > 16, or world > 1. */
mis_status mis_regenerate_nodes(mis_ctx* ctx, float node_grid_mm, int32_t* m_out);

/* Read the model (internal order).  Any output may be NULL.  knn_idx/knn_w:
 * n x k in the canonical per-point order (ids ascending). */
mis_status mis_get_model(mis_ctx* ctx, mis_mem mem, float* xyz, float* nrm, float* rgb, float* weight,
                         int32_t* stamp, int64_t* ids, int32_t* knn_idx, float* knn_w, int64_t* n_host);

/* Eq. 2 skinning (k+1 nearest of the current nodes, ties to the lower id,
 * d_max = 0 -> 1/k) of nq query points: idx / w n x k, ids ascending. */
mis_status mis_skin(mis_ctx* ctx, mis_mem mem, int64_t nq, const float* pts, int32_t* idx, float* w);

/* ---- stage outputs for parity tests (same kernels as the hot path) ---- */
/* Inject a node state (m x 12 float32: R row-major, t); fp64 master = upcast. */
mis_status mis_dbg_set_nodes(mis_ctx* ctx, mis_mem mem, const float* R9_t3);
/* NEXT-2: inject the current pose (host, 12 doubles, R row-major + T) of a joint registration; the
 * prior stays the frame's input pose.  The next mis_dbg_system / mis_dbg_associate with
 * MIS_F_JOINT_POSE and mis_warp / mis_fuse use it (mis_register restarts from the prior). */
mis_status mis_dbg_set_pose(mis_ctx* ctx, const double pose[12]);
/* Normal map of the current frame: H x W x 4 (nx, ny, nz, D); n = 0 when the
 * normal is invalid, D = 0 when the depth is invalid. */
mis_status mis_dbg_frame(mis_ctx* ctx, mis_mem mem, float* nmap);
/* Association of every point under the current node state (Eq. 7): pix =
 * py*W + px or -1; why = passed gates, bit0 z>0, bit1 in frame, bit2 depth
 * valid, bit3 normal valid, bit4 distance, bit5 angle (short-circuit). */
mis_status mis_dbg_associate(mis_ctx* ctx, mis_mem mem, int32_t* pix, uint8_t* why);
/* The normal equations at the current state: full BSR (both triangles,
 * rows sorted by column): row_ptr (m+1), col (nnzb), val (nnzb x 36,
 * row-major 6x6, unknowns [dtheta, dt] per node), rhs (6m) = -J^T r, energy[5].
 * With MIS_F_JOINT_POSE the pose is unknown m: row_ptr (m+2), rhs 6(m+1), and
 * energy[4] includes w_r E_r + w_p E_p.  With MIS_F_AFFINE the blocks are 12 x 12
 * (val nnzb x 144, unknowns [dA row-major, dt] per node), rhs 12m, energy[4]
 * includes w_rot E_rot.
 * With val == NULL only *nnzb is returned.  Host memory only. */
mis_status mis_dbg_system(mis_ctx* ctx, int32_t* row_ptr, int32_t* col, float* val, float* rhs,
                          double energy[5], int64_t* nnzb);
/* The fusion registration of the current frame without applying it: owner
 * (H*W, internal point index or -1), why (n). Host memory only. */
mis_status mis_dbg_fuse_register(mis_ctx* ctx, int64_t* owner, uint8_t* why);

/* ---- instrumentation (bench / profiling) ---- */
#define MIS_PROF_NCAT 16
/* Kernel groups: 0 frame_prep (K1), 1 skin (K2), 2 sort_order (K13), 3 pattern,
 * 4 assemble_points (K3), 5 assemble_graph (K4/K5), 6 solve (K6-K8),
 * 7 warp_model (K9), 8 fuse_register (K10), 9 fuse_apply (K11), 10 lift (K12),
 * 11 io (uploads, layout conversion), 12 reduce_records (K3 chunk records -> blocks),
 * 13 accum_points, 14 filter (K14 + the survivors' K2), 15 regenerate (K15 node regeneration). */
const char* mis_prof_name(int cat);
/* on = 1: record a CUDA event pair on the context stream around every kernel
 * group launched by this context; on = 2: only around the K3 and solver groups
 * (less host work per step); 0: off.  Adds no synchronisation. */
mis_status mis_prof_enable(mis_ctx* ctx, int on);
/* Accumulated device milliseconds and launches per group since the last reset
 * (synchronises the context stream).  ms / launches: MIS_PROF_NCAT entries. */
mis_status mis_prof_read(mis_ctx* ctx, double* ms, int64_t* launches, int reset);
/* Kernels of this library launched so far in this process (all contexts;
 * CUB library kernels of the setup sort are not counted). */
int64_t mis_launch_count(void);
/* %globaltimer stamps (ns) of the last cluster-PCG launch, 8 per CTA (16 CTAs):
 * start, system built, preconditioner built, PCG start, PCG end, nodes updated,
 * z replicated, partial published (host memory, 128 entries). */
mis_status mis_dbg_solver_phases(mis_ctx* ctx, uint64_t* out128);

#ifdef __cplusplus
}
#endif
#endif /* MIS_H */
