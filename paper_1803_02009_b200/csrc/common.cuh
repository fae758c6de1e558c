// common.cuh -- internal declarations of libmis (B200 / sm_100a).
// Device-side structs, small vector helpers and the kernel launchers shared
// between the .cu files of the library.  Nothing here is visible through the
// C-ABI (include/mis.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mis.h"

namespace mis {

// Programmatic dependent launch (sm_90+): kernels of the Gauss-Newton chain are launched with
// programmatic stream serialisation, so a kernel's launch and block scheduling overlap the tail
// of its predecessor; pdl_wait() (before reading anything the predecessor wrote) blocks until the
// predecessor grid has completed and its writes are visible; pdl_trigger() lets the successor
// launch.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ------------------------------------------------------------- device views
struct FrameView {
  int W, H;
  float fx, fy, cx, cy;
  double fxd, fyd, cxd, cyd;
  double ifxd, ifyd;     // 1 / fx, 1 / fy
  const float* depth;    // H*W
  const float4* nmap;    // H*W: (nx, ny, nz, D); n = 0 invalid normal, D = 0 invalid depth
  const double4* nmapd;  // H*W: the same in fp64 (the association's precision)
  float R[9], T[3];      // world -> camera (fp32 copy)
  double Rd[9], Td[3];   // fp64 copy (the association and fusion decisions)
  const double* pose_dev;   // NEXT-2: the refined pose on the device (R row-major 9, T 3), else null
};

// The frame's world -> camera pose in fp64: the device copy refined by a joint registration
// (MIS_F_JOINT_POSE) when there is one, else the input pose passed by value.
__device__ __forceinline__ void frame_pose(const FrameView& f, double* R, double* T) {
  if (f.pose_dev) {
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = f.pose_dev[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) T[i] = f.pose_dev[9 + i];
  } else {
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = f.Rd[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) T[i] = f.Td[i];
  }
}

struct ModelView {
  int64_t n, cap;
  float *px, *py, *pz, *nx, *ny, *nz;   // SoA, internal (tuple-sorted) order
  float *cr, *cg, *cb, *w;              // colour, fusion weight omega
  int32_t* stamp;
  int64_t* ids;
  int32_t* kidx;                        // slot-major [s*cap + i], ids ascending per point
  float* kw;                            // slot-major raw skinning weights
};

struct NodeView {
  int m;
  const float* g;        // m*3 node positions
  float* node32;         // m*16: R (9) t (3) g (3) pad -- what the kernels read
  double* Rt64;          // m*12 fp64 master state (R row-major, t)
};

// pair index of slot positions (j <= l) within a k-tuple
__host__ __device__ inline int pair_index(int j, int l, int K) { return j * K - (j * (j - 1)) / 2 + (l - j); }
__host__ __device__ inline int n_pairs(int K) { return K * (K + 1) / 2; }

// ------------------------------------------------------------- accumulator layout
// acc region (float), zeroed every GN iteration, all-reduced across ranks:
//   data[nnzu*36] | mom[nnzu*16] | graph[nnzu*36] | rhs_data[m*6] | node_mom[m*12] | rhs_graph[m*6]
// energy region (double): E_data, E_pt, E_reg, E_corr ; n_assoc (u64 as double slot 4)
struct AccView {
  float* data;
  float* mom;
  float* graph;
  float* rhs_data;
  float* node_mom;
  float* rhs_graph;
  double* energy;              // [0..3] energies, [4] n_assoc, [6] K3b work counter (u64);
                               // [8 + 64 q + s]: striped partials of quantity q (0 E_data, 1 E_pt, 2 E_reg,
                               // 3 E_corr, 4 n_assoc, 5 E_rot), summed by the finalisation
};
constexpr int kEnergyStripes = 64;
constexpr int kEnergyQ = 6;
constexpr int kEnergyDoubles = 8 + kEnergyQ * kEnergyStripes;
// one fp64 atomic per warp into a stripe picked by the warp index: no same-address serialisation
__device__ __forceinline__ void energy_add(double* energy, int q, double v) {
  const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (v != 0.0) atomicAdd(energy + 8 + kEnergyStripes * q + (w % kEnergyStripes), v);
}

// ------------------------------------------------------------- host-side launchers
struct Ctx;   // defined in api.cu

void launch_frame_prep(const FrameView& f, float4* nmap, double4* nmapd, cudaStream_t s);
void launch_skin(int64_t nq, const float* px, const float* py, const float* pz, int64_t stride_xyz,
                 const float* g, int m, int K, int32_t* idx, float* w, int64_t out_stride, cudaStream_t s);
// K2 over spatially coherent 256-query blocks with a per-block candidate-node bound (exact Eq. 2)
void launch_skin_boxed(int64_t nq, const uint32_t* order, int out_at_q, const float* px, const float* py,
                       const float* pz, int64_t sxyz, const float* g, int m, int K, int32_t* idx, float* w, int64_t os,
                       cudaStream_t s);

struct AsmPointsArgs {
  ModelView md;
  const int32_t* seg_nodes;   // nseg*K
  const int4* chunks;         // (seg, start, end, -)
  int64_t nchunk;
  const int32_t* seg_slot;    // nseg*P
  NodeView nd;
  FrameView fr;
  float eps_d, cos_eps_n;
  double eps_dd, cos_eps_nd;
  AccView acc;                // K3 commits atomically into the BSR accumulators
  float4* pstate;             // K3a -> K3b per-point factor state: (K + 2) planes of pstride float4
  int64_t pstride;
  unsigned long long* work_counter;   // zeroed before the launch (dynamic chunk scheduling)
  int32_t* dbg_pix;           // nullable: per point association outputs
  uint8_t* dbg_why;
  // NEXT-2 (MIS_F_JOINT_POSE): the current pose (12 doubles) -- K3a warps with it and writes the
  // pose as one more factor slot (x_hat, 1) after the K node slots; K3b then runs with K + 1 slots
  // whose last node id is m (seg_nodes / seg_slot of the joint pattern).  null: fixed pose
  const double* pose_cur;
  int32_t* chunk_live;        // non-null: K3a runs by chunk and flags the chunks with an associated point
                              // (the tcgen05 K3b skips the others: no staging, no commit)
  int sparse_state;           // the tcgen05 K3b consumes the factor state: K3a writes the (n', associated)
                              // plane for every point and the other K + 1 planes only for associated points
  int affine;                 // NEXT-4 (MIS_F_AFFINE): the node matrices are general A_j; K3a writes
                              // (w_j d_j, w_j), d_j = v - g_j, and warps normals by A_j^-T
};
// K3a (per point), then K3b (per chunk)
struct AsmGraphArgs;
// K3a (per point; with K4/K5 items in the same launch when ga != null), then K3b (per chunk)
void launch_assoc_points(int K, const AsmPointsArgs& a, const AsmGraphArgs* ga, cudaStream_t s);
// fused (k <= 4, no debug outputs): K3a + K3b in one kernel, the K4 / K5 items (ga) in extra CTAs
void launch_accum_points(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s, bool fused = false,
                         const AsmGraphArgs* ga = nullptr);
// K3b for 5 <= k <= 8 on tcgen05 (k3b_umma.cu; chunks of <= 128 points); MIS_K3B_UMMA=0 in the
// environment selects the FP32 register-tile kernel instead
bool umma_k3b_enabled();
void launch_accum_points_umma(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s);

// Per-chunk tile dump order of K3 ("record" floats, mapped to accumulator
// addresses at commit): P pairs x [36 data (6x6, upper for the diagonal pair) |
// 16 point-to-point moments], K slots x [6 rhs_data | 12 node moments], tail
// [E_data, E_pt x, E_pt y, E_pt z, n_assoc]; padded to 4.
__host__ __device__ inline int rec_stride(int K) { return (52 * (K * (K + 1) / 2) + 18 * K + 5 + 3) & ~3; }

// Levenberg-Marquardt state on the device (MIS_F_LM, reading A29): the
// Marquardt damping, the last accepted energy and which of the two system buffers
// (0: Hval / rhs, 1: the alternates) holds the last accepted normal equations.
struct LmDev {
  double mu, E_acc;
  int32_t acc_buf, pad;
};

struct FinalArgs {
  int64_t nnzb;
  int64_t nup;                // off-diagonal upper entries ((nnzb - m) / 2)
  const int2* ulist;          // nup x (entry, mirror)
  int m;
  const int32_t* upper_of;
  const int32_t* lower_of;    // upper entry -> its mirror (-1 on the diagonal)
  const int32_t* diag_pos;    // m: BSR entry of each diagonal block
  float w_data, w_pt;
  int pre_weighted;           // data holds the weighted point part of H (rhs_data: -b), mom / node_mom zero
                              // (the multi-GPU payload, k_shard_scatter): H = data + graph, b = -rhs_data + graph
  AccView acc;                // K3 / K4 / K5 sums in
  float* Hval;                // nnzb*36 final blocks (both triangles)
  float* rhs;                 // 6m final right-hand side
  float* Minv;                // m*36 block-Jacobi inverses
  float lambda, w_reg, w_corr;
  int slot;                   // report slot of this assembly (-1: none)
  // NEXT-2: unknown pose_node (= m; -1: none) is the pose; its diagonal block and rhs get the
  // Eq. 10 priors at pose_cur against pose_prior (w_r, w_p), its energies go to rep_pose
  int pose_node;
  const double *pose_cur, *pose_prior;
  float w_r, w_p;
  double* rep_pose;           // (MIS_MAX_GN+1)*2
  float w_rot;                // NEXT-4: E_rot weight (its energy goes to rep_rot)
  double* rep_rot;            // (MIS_MAX_GN+1)
  double* rep_energy;         // (MIS_MAX_GN+1)*5
  double* rep_nassoc;         // 2*(MIS_MAX_GN+1): association counts, fp64 guard counts
  const LmDev* lm;            // LM: write the system into the buffer not holding the accepted one
  float *Hval_alt, *rhs_alt;
};
void launch_finalize(const FinalArgs& r, cudaStream_t s);
// multi-GPU reduction payload (assemble.cu): point part of H (upper blocks) and b before the all-reduce,
// scattered back as accumulators after it
void launch_shard_partial(const FinalArgs& r, float* HU, float* RU, cudaStream_t s);
void launch_shard_scatter(const FinalArgs& r, const float* HU, const float* RU, cudaStream_t s);
// NEXT-4 (affine.cu): K3b over the 12-unknown node blocks, the graph terms (Eq. 6 with A_j, Eq. 9,
// Eq. 4-5 E_rot) and the 12 x 12 finalisation
void launch_accum_points_aff(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s);
void launch_assemble_graph_aff(const struct AsmGraphArgs& a, cudaStream_t s);
void launch_finalize_aff(const FinalArgs& r, cudaStream_t s);

struct AsmGraphArgs {
  NodeView nd;
  int n_nbr;
  const int32_t* nbr;         // m*n_nbr
  const int32_t* edge_slot;   // m*n_nbr (slot of (min, max)), -1 if none
  const int32_t* diag_slot;   // m
  int nf;
  const float* fsrc; const float* fdst;
  const int32_t* fidx; const float* fw;   // K*nf (slot-major: [s*nf + f]), ids ascending
  const int32_t* feat_slot;   // nf*P
  FrameView fr;
  float w_reg, w_corr;
  AccView acc;
  int K;
  int KS;                     // feature slots: K, or K + 1 with the pose (fidx row K = m, NEXT-2)
  const double* pose_cur;     // NEXT-2: the current pose (null: fr's)
  float w_rot;                // NEXT-4 (affine kernels): E_rot weight
};
void launch_assemble_graph(const AsmGraphArgs& a, cudaStream_t s);

struct SolveArgs {
  int m, K;
  int64_t nnzb;
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* upper_of;    // nnzb: index of the (min, max) entry
  const int32_t* diag_pos;    // m
  AccView acc;
  float w_data, w_pt, lambda;
  int pcg_iters;
  float* Hval;                // nnzb*36
  float* rhs;                 // 6m
  float* Minv;                // m*36
  float *x, *r, *z, *p, *Ap;  // 6m
  float* pv;                  // grid pipelined PCG: 9 planes of B m floats (r u w z q s p m m)
  double* dots;               // 2*pcg_iters + 4
  NodeView nd;
  int do_update;              // 0: only build the system (debug)
  int gn_it;                  // report slot
  float* rep_res;             // MIS_MAX_GN
  int* numeric_flag;
  // cluster-resident variant (pcg_cluster.cu); cluster_size == 0 -> grid variant
  int cluster_size;
  const int32_t* part;        // cluster_size+1 row boundaries (balanced by nnz)
  int max_rows, max_nnz;      // per-CTA maxima (uniform smem layout)
  size_t smem_bytes;
  int write_global;           // also write x to global memory (debug)
  int pipelined;              // cluster variant: pipelined PCG (1 barrier / iteration) instead of standard
  int minv_ready;             // Minv already built by the record reduction (single GPU)
  unsigned long long* tstamp; // 8 %globaltimer stamps of the phases (rank 0, thread 0)
  const int32_t *pptr, *pc, *push, *npush;   // cluster variant: per-rank SpMV pieces and halo lists (per frame)
  // Levenberg-Marquardt (cluster kernel, register-resident variant only): accept / reject the
  // trial whose energy the finalisation just wrote, pick the system, damp, keep the base state
  LmDev* lm;                  // nullptr: Gauss-Newton
  float lm_mu0;
  const float *Hval_alt, *rhs_alt;
  double* Rt_acc;             // m x 12: last accepted state
  int pose_node;              // NEXT-2: unknown index of the pose (m), -1: none
  int block;                  // unknowns per node: 6 (SE(3)), 12 (NEXT-4 affine; additive update)
  double* pose;               // its state (R row-major 9, T 3): R <- R Exp(dphi), T <- T + R dtau
  const double* rep_energy;   // (MIS_MAX_GN+1) x 5, the trial energies
  double* rep_flags;          // MIS_MAX_GN+1: 1 = trial accepted
};
void launch_lm_finish(int m, int slot, const LmDev* lm, const double* rep_energy, double* rep_flags, double* Rt64,
                      const double* Rt_acc, float* node32, cudaStream_t s, double* pose = nullptr);

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
cudaError_t launch_solve(const SolveArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_solve_cluster(const SolveArgs& a, cudaStream_t s);
// per frame, after the pattern: the cluster ranks' SpMV pieces and halo push lists
void launch_pcg_prep(const int32_t* row_ptr, const int32_t* col, const int32_t* part, int cs, int max_rows, int max_nnz,
                     int32_t* pptr, int32_t* pc, int32_t* push, int32_t* npush, uint32_t* mask, cudaStream_t s,
                     bool marked = false);
int pcg_max_pieces(int max_rows, int max_nnz);
// cluster partition (row boundaries balancing nnz) computed on the device; cl_size 0 = does not fit
struct PlanOut { int32_t cl_size, max_rows, max_nnz, pad; int64_t smem; };
void launch_plan_cluster(const int32_t* row_ptr, int m, int max_cluster, PlanOut* out, int32_t* part, int64_t* nnz_out,
                         cudaStream_t s);

// ---- fusion (fuse.cu)
void launch_warp_model(int K, const ModelView& md, const NodeView& nd, const FrameView& fr, float* xyz_cam,
                       float* nrm_cam, cudaStream_t s, bool affine = false);
void launch_advance_nodes(const NodeView& nd, float* g_mut, cudaStream_t s);
struct FuseArgs {
  ModelView md;
  FrameView fr;
  double tz, cos_delta, omega_max;
  double key_scale;           // (2^32 - 1) / tz: |dz| < tz quantised to the key's 32 high bits
  const float* rgb_obs;       // H*W*3 or null
  int32_t frame_index;
  unsigned long long* pixkey; // H*W
  int32_t* pix;               // n
  uint8_t* why;               // n (nullable)
  uint32_t rank_tag;          // rank << 27 in the key's index bits (0 on one GPU): keys unique across ranks
  unsigned long long* n_reg;  // registered-pixel counter (zeroed by K10, filled by the lift count)
  const long long* fits;      // nullable: 0 when the frame's lift would exceed the capacity (K11 skips)
};
void launch_fuse_register(const FuseArgs& a, cudaStream_t s);
void launch_fuse_apply(const FuseArgs& a, cudaStream_t s);
// lift: count pass (per-block counts) then write pass; returns via device counters
void launch_lift_count(const FuseArgs& a, int32_t* block_counts, int nblocks, long long* ids_dev,
                       unsigned long long* n_registered, int do_lift, int64_t base, int64_t cap, cudaStream_t s);
void launch_lift_write(const FuseArgs& a, const int32_t* block_offsets, int nblocks, int64_t base, int64_t cap,
                       const long long* ids_dev, int32_t* lift_pos, cudaStream_t s);
// K2 (Eq. 2) of the lifted points, per pixel tile with a candidate-node bound (exact)
void launch_skin_lifted(int K, int W, int H, const int32_t* lift_pos, const ModelView& md, const float* g, int m,
                        cudaStream_t s);
int lift_blocks(int W, int H);

// ---- model order / pattern (sort.cu)
struct SortWork;   // temp storage owner (in api.cu)
}  // namespace mis
