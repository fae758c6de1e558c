// ctx.cuh -- the library context (host side) shared by api.cu and sort.cu.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "common.cuh"

struct mis_ctx;   // opaque in mis.h; defined as mis::Ctx below

namespace mis {

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool reg = false;   // in Ctx::bufs (freed by mis_destroy)
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct ModelBufs {
  DBuf px, py, pz, nx, ny, nz, cr, cg, cb, w, stamp, ids, kidx, kw;
};

struct NcclApi;   // dlopen'ed NCCL entry points (api.cu)

struct Ctx {
  mis_params prm{};
  int device = 0, num_sms = 148;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  cudaStream_t st_copy = nullptr;      // host->device copies of frame inputs (overlap the model ordering)
  cudaEvent_t ev_depth_free = nullptr, ev_depth_ready = nullptr, ev_rgb_free = nullptr, ev_rgb_ready = nullptr;
  const float* rgb_staged = nullptr;    // host colour already on its way into rgb_obs (mis_stage_colour)
  const float* rgb_pending = nullptr;   // staged colour whose upload the next frame upload issues
  int rank = 0, world = 1;
  void* nccl_comm = nullptr;
  std::string err;

  // ---- memory: every device buffer of the context is registered here on its first allocation
  // (mis_destroy frees exactly this list); with a bound workspace (mis_bind_workspace) buffers are
  // carved first-fit from the caller's region instead of cudaMalloc
  std::vector<DBuf*> bufs;
  char* ws_base = nullptr;
  size_t ws_bytes = 0;
  std::map<size_t, size_t> ws_free;   // offset -> bytes of the free extents (coalesced)

  // ---- model (internal, tuple-sorted order); two buffer sets for the sort gather
  int64_t n = 0, cap = 0, next_id = 0;
  int K = 4;
  ModelBufs mb[2];
  int cur = 0;
  bool have_model = false, have_graph = false, dirty = false;
  bool graph_check = false;   // device-memory set_graph: validation flags still to be read back
  int graph_flags = 0;

  // ---- graph
  int m = 0;
  DBuf g, nbr, node32, Rt64;

  // ---- NEXT-2 joint global pose (MIS_F_JOINT_POSE): unknown number m of the system
  bool joint = false;           // the flag, as of the last prepare()
  bool pattern_joint = false;   // the current pattern / accumulator layout includes the pose
  bool pose_valid = false;      // posebuf holds this frame's pose (registered jointly or injected)
  DBuf posebuf;                 // 24 doubles: current pose (R 9, T 3) | prior (the frame's input pose)
  DBuf seg_nodes_j;             // nseg x (k + 1): segment tuples + the pose id m

  // ---- NEXT-4 affine nodes (MIS_F_AFFINE): 12 unknowns per node
  bool affine = false;          // the flag, as of the last prepare()
  bool pattern_affine = false;  // the accumulator / system layout has 12 x 12 blocks

  // ---- order: segments and chunks (K13)
  int64_t nseg = 0, nchunk = 0;
  DBuf keys, keys2, vals, vals2, flags, scan, seg_start, seg_nodes, chunks, chunk_off;
  // grouping by exact tuple (k <= 4, m < 65535): hash table (keys | group ids, empty at rest),
  // per-group key / slot / count (count zero at rest) and the group counter
  DBuf gtab, gkeys, gslot, gcount;
  int64_t gtab_slots = 0, gsize_cap = 0;
  bool order_by_sort = false;   // MIS_ORDER_BY_SORT=1 in the environment: the radix-sort path
  bool k3_split = false;        // MIS_K3_SPLIT=1 in the environment: K3a + K3b as two kernels

  // ---- pattern
  int64_t nnzb = 0;
  bool pattern_valid = false;
  DBuf bitmap, bitmap_all, row_cnt, row_ptr, col, row_of, diag_pos, upper_of, lower_of, seg_slot, edge_slot, feat_slot;
  DBuf ulist;   // int2 (entry, mirror) of every off-diagonal upper entry: the finalisation's work list
  bool bitmap_clean = false;   // pattern bitmap all-zero (cleared by k_row_fill) -> no memset
  int64_t bitmap_words = 0;
  DBuf nnz_dev;   // int64 info: [0] nnz, [1] nseg, [2] nchunk, [3] set_graph validation flags, [4..6] plan

  // ---- system and solver
  int cl_size = 0, cl_max_rows = 0, cl_max_nnz = 0;   // cluster-resident PCG plan (0: grid variant)
  size_t cl_smem = 0;
  bool cluster_ok = true;
  std::string solver_note;
  int last_solver = 0;   // cluster size of the last PCG launch (0: grid kernel)
  DBuf part, tstamp;
  DBuf pcg_pptr, pcg_pc, pcg_push, pcg_npush, pcg_mask;   // cluster PCG lists (per frame)
  size_t acc_floats = 0;
  DBuf pstate;   // K3a -> K3b per-point factor state
  DBuf chunk_live;   // per chunk: any point associated (K3a by chunk -> the tcgen05 K3b skips the rest)
  bool acc_dirty = true;   // accumulators may be nonzero (set while an assembly is in flight)
  DBuf acc, energy, Hval, rhs, Minv, x, r, z, p, Ap, dots, pvec;   // pvec: grid pipelined PCG vectors
  DBuf shard_buf;   // multi-GPU reduction payload: point part of H (upper blocks) and b
  DBuf lm, Hval2, rhs2, Rt_acc;   // Levenberg-Marquardt (MIS_F_LM): state, second system buffer, kept nodes

  // ---- frame
  bool have_frame = false;
  bool frame_pending = false;        // mis_register's frame prep, launched behind the pattern readback
  const float* frame_src = nullptr;  // its depth source
  int64_t* hpin = nullptr;           // pinned readback buffer (16 x int64)
  cudaEvent_t rb_ev = nullptr;       // completion of a readback copy
  int W = 0, H = 0;
  mis_intrinsics intr{};
  float pose[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
  DBuf depth, nmap, nmapd, rgb_obs, stage;

  // ---- features
  int nf = 0;
  DBuf fsrc, fdst, fidx, fw;

  // ---- fuse
  DBuf pixkey, pix, why, lift_counts, counter;
  DBuf lift_pos;   // per pixel: the lifted point's model index (-1: none)
  bool pixkey_clean = false;   // pixel keys all-ones (reset by the lift write) -> no memset before K10
  DBuf ids_dev;   // int64 [0] next fresh point id, [1] id base of the last lift, [2] lifted points written

  // ---- report
  DBuf rep;   // report block (one memset / one readback per registration), layout below

  DBuf cub_tmp;
  DBuf finfo;   // mis_filter: int64 [survivors, boxes, stable, boxes to re-skin] + int32 range [7]
  DBuf fl_xyz, fl_idx, fl_kidx, fl_kw;   // mis_filter: re-skinning list (positions, model index, K2 output)
  DBuf rg_nbr, rg_sums;   // mis_regenerate_nodes: N(j) of the new nodes (positions: fl_xyz), fp64 cell sums

  // ---- instrumentation
  bool prof = false, prof_light = false;   // light: only the K3 and solver groups
  struct PEv { int cat; cudaEvent_t a, b; };
  std::vector<PEv> pev;
  std::vector<cudaEvent_t> pool;
  double prof_ms[MIS_PROF_NCAT] = {0};
  int64_t prof_n[MIS_PROF_NCAT] = {0};
};

enum { P_FRAME = 0, P_SKIN, P_ORDER, P_PATTERN, P_POINTS, P_GRAPH, P_SOLVE, P_WARP, P_FREG, P_FAPPLY, P_LIFT, P_IO,
       P_REDUCE, P_ACCUM, P_FILTER, P_REGEN };
void count_launches(int64_t k);

// report block: [energy (MIS_MAX_GN+1) x 5 | n_assoc, n_guard 2 x (MIS_MAX_GN+1) | PCG residual
// MIS_MAX_GN floats | numeric flag | E_r, E_p (MIS_MAX_GN+1) x 2], doubles
constexpr size_t kRepN = 5 * (MIS_MAX_GN + 1), kRepR = kRepN + 2 * (MIS_MAX_GN + 1), kRepF = kRepR + MIS_MAX_GN / 2,
                 kRepP = kRepF + 1, kRepO = kRepP + 2 * (MIS_MAX_GN + 1), kRepBytes = (kRepO + MIS_MAX_GN + 1) * 8;
// per-point scratch is sized for the model capacity (fixed at mis_set_model), not the current size:
// a growing sequence (fuse / filter / regenerate every frame) then allocates it once
inline int64_t ncap(const Ctx* c, int64_t n) { return n > c->cap ? n : c->cap; }
// unknown blocks of the current system: the m nodes, plus the pose with the joint pattern (NEXT-2)
inline int sys_m(const Ctx* c) { return c->m + (c->pattern_joint ? 1 : 0); }
// unknowns per node block of the current system: 6 (SE(3)), 12 (affine, NEXT-4)
inline int sys_b(const Ctx* c) { return c->pattern_affine ? 12 : 6; }
inline double* rep_energy(Ctx* c) { return c->rep.as<double>(); }
inline double* rep_nassoc(Ctx* c) { return c->rep.as<double>() + kRepN; }
inline float* rep_res(Ctx* c) { return reinterpret_cast<float*>(c->rep.as<double>() + kRepR); }
inline int* numeric_flag(Ctx* c) { return reinterpret_cast<int*>(c->rep.as<double>() + kRepF); }
inline double* rep_pose(Ctx* c) { return c->rep.as<double>() + kRepP; }
inline double* rep_rot(Ctx* c) { return c->rep.as<double>() + kRepO; }

// Records an event pair around a group of `nk` kernel launches on the context
// stream when profiling is on; always adds nk to the launch counter.
struct ProfScope {
  Ctx* c;
  int cat;
  cudaEvent_t b = nullptr;
  int64_t l0 = 0;
  ProfScope(Ctx* c_, int cat_, int nk);
  ~ProfScope();
};

// buffer management (api.cu)
cudaError_t ensure(Ctx* c, DBuf& b, size_t bytes);
void free_buf(Ctx* c, DBuf& b);
size_t cub_tmp_bound(int64_t n);   // sort.cu: CUB temporary storage of the largest sort / scan over n items

// views
ModelView model_view(Ctx* c);
ModelView model_view_of(Ctx* c, ModelBufs& B);
NodeView node_view(Ctx* c);
FrameView frame_view(Ctx* c);
AccView acc_view(Ctx* c);

// sort.cu
cudaError_t build_order(Ctx* c);      // K13: tuple sort, gather, segments, chunks
cudaError_t flush_frame(Ctx* c);      // a deferred frame prep (api.cu)
cudaError_t build_pattern(Ctx* c);    // BSR pattern + slot tables (incl. features)
// filter.cu (NEXT-1)
cudaError_t run_filter_range(Ctx* c, float grid, int32_t* range_host);
int filter_key_bits(const int32_t* range, int* sh_x, int* sh_y);
cudaError_t run_filter(Ctx* c, float grid, const int32_t* range, int sh_x, int sh_y, int bits, int32_t frame,
                       int32_t tau_time, float tau_weight);
cudaError_t run_filter_skin(Ctx* c, int64_t nl);
cudaError_t run_regen_centroids(Ctx* c, float grid, const int32_t* range, int sh_x, int sh_y, int bits, int64_t* m_out);
cudaError_t run_regen_knn(Ctx* c, int m, int nn);
cudaError_t nccl_allreduce_sum_f32(Ctx* c, float* buf, size_t count);
cudaError_t nccl_allreduce_sum_f64(Ctx* c, double* buf, size_t count);
cudaError_t nccl_allreduce_max_i64(Ctx* c, int64_t* buf, size_t count);
cudaError_t nccl_allgather_u64(Ctx* c, const uint64_t* send, uint64_t* recv, size_t count);

#ifndef MIS_KCHUNK
#define MIS_KCHUNK 128   // measured: C5 K3b 18.8 -> 16.5 ms per step vs 64, C3 unchanged; 256 slower at C3
#endif
constexpr int kChunk = MIS_KCHUNK;   // max points per K3 chunk (a segment splits into equal chunks)
}  // namespace mis
