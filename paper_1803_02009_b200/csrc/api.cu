// api.cu -- the C-ABI of libmis (include/mis.h): context, argument checking,
// uploads, orchestration of the kernels of one frame, NCCL plumbing.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <iterator>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "ctx.cuh"

struct mis_ctx : public mis::Ctx {};

namespace mis {

// ------------------------------------------------------------ buffers
#ifndef MIS_ENSURE_SLACK_DIV
#define MIS_ENSURE_SLACK_DIV 2   // a (re)allocation takes 1 + 1/DIV times the request (growing sequences: fewer reallocations)
#endif
static constexpr size_t kWsAlign = 256;

// first-fit allocation from the bound workspace (mis_bind_workspace); nullptr when it is exhausted
static void* ws_alloc(Ctx* c, size_t bytes) {
  bytes = (bytes + kWsAlign - 1) & ~(kWsAlign - 1);
  for (auto it = c->ws_free.begin(); it != c->ws_free.end(); ++it) {
    if (it->second < bytes) continue;
    const size_t off = it->first, left = it->second - bytes;
    c->ws_free.erase(it);
    if (left) c->ws_free[off + bytes] = left;
    return c->ws_base + off;
  }
  return nullptr;
}
static void ws_release(Ctx* c, void* p, size_t bytes) {
  bytes = (bytes + kWsAlign - 1) & ~(kWsAlign - 1);
  size_t off = (size_t)(static_cast<char*>(p) - c->ws_base);
  auto nx = c->ws_free.lower_bound(off);
  if (nx != c->ws_free.end() && off + bytes == nx->first) {   // merge with the next extent
    bytes += nx->second;
    nx = c->ws_free.erase(nx);
  }
  if (nx != c->ws_free.begin()) {                              // and with the previous one
    auto pv = std::prev(nx);
    if (pv->first + pv->second == off) { pv->second += bytes; return; }
  }
  c->ws_free[off] = bytes;
}
static bool in_ws(const Ctx* c, const void* p) {
  return c->ws_base && p >= c->ws_base && p < c->ws_base + c->ws_bytes;
}

cudaError_t ensure(Ctx* c, DBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.p && b.bytes >= bytes) return cudaSuccess;
  if (b.p) {
    static const bool dbg = getenv("MIS_DEBUG_ALLOC") != nullptr;
    if (dbg) fprintf(stderr, "mis: realloc %zu -> %zu bytes (buffer %p)\n", b.bytes, bytes, (void*)&b);
    cudaError_t e = cudaStreamSynchronize(c->st);   // the old buffer may still be in use
    if (e != cudaSuccess) return e;
    free_buf(c, b);
  }
  size_t alloc = bytes + bytes / MIS_ENSURE_SLACK_DIV + 256;
  if (c->ws_base) {
    b.p = ws_alloc(c, alloc);
    if (!b.p) {
      c->err = "workspace exhausted (" + std::to_string(alloc) + " more bytes needed; see mis_workspace_bytes)";
      return cudaErrorMemoryAllocation;
    }
  } else {
    cudaError_t e = cudaMalloc(&b.p, alloc);
    if (e != cudaSuccess) { b.p = nullptr; return e; }
  }
  b.bytes = alloc;
  if (!b.reg) { b.reg = true; c->bufs.push_back(&b); }
  return cudaSuccess;
}

void free_buf(Ctx* c, DBuf& b) {
  if (b.p) {
    if (in_ws(c, b.p)) ws_release(c, b.p, b.bytes);
    else cudaFree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
}

ModelView model_view(Ctx* c) { return model_view_of(c, c->mb[c->cur]); }

ModelView model_view_of(Ctx* c, ModelBufs& B) {
  ModelView v;
  v.n = c->n; v.cap = c->cap;
  v.px = B.px.as<float>(); v.py = B.py.as<float>(); v.pz = B.pz.as<float>();
  v.nx = B.nx.as<float>(); v.ny = B.ny.as<float>(); v.nz = B.nz.as<float>();
  v.cr = B.cr.as<float>(); v.cg = B.cg.as<float>(); v.cb = B.cb.as<float>(); v.w = B.w.as<float>();
  v.stamp = B.stamp.as<int32_t>(); v.ids = B.ids.as<int64_t>();
  v.kidx = B.kidx.as<int32_t>(); v.kw = B.kw.as<float>();
  return v;
}

NodeView node_view(Ctx* c) {
  NodeView v;
  v.m = c->m; v.g = c->g.as<float>(); v.node32 = c->node32.as<float>(); v.Rt64 = c->Rt64.as<double>();
  return v;
}

FrameView frame_view(Ctx* c) {
  FrameView f;
  f.W = c->W; f.H = c->H;
  f.fx = c->intr.fx; f.fy = c->intr.fy; f.cx = c->intr.cx; f.cy = c->intr.cy;
  f.fxd = c->intr.fx; f.fyd = c->intr.fy; f.cxd = c->intr.cx; f.cyd = c->intr.cy;
  f.ifxd = 1.0 / f.fxd; f.ifyd = 1.0 / f.fyd;
  f.depth = nullptr;   // only K1 reads the depth (the caller's buffer or its staged copy)
  f.nmap = c->nmap.as<float4>();
  f.nmapd = c->nmapd.as<double4>();
  for (int i = 0; i < 9; ++i) { f.R[i] = c->pose[i]; f.Rd[i] = c->pose[i]; }
  for (int i = 0; i < 3; ++i) { f.T[i] = c->pose[9 + i]; f.Td[i] = c->pose[9 + i]; }
  f.pose_dev = c->pose_valid ? c->posebuf.as<double>() : nullptr;   // NEXT-2: the refined pose
  return f;
}

AccView acc_view(Ctx* c) {
  AccView a;
  float* base = c->acc.as<float>();
  const size_t nz = (size_t)c->nnzb, m = (size_t)sys_m(c), B = (size_t)sys_b(c);
  // all accumulated atomically (K3 float4 / float2 adds, K4 / K5), zeroed every iteration:
  // data | mom | rhs_data (padded to 4 floats: 16-byte aligned node moments) | node_mom | graph | rhs_graph
  // (B x B blocks, B = 6, or 12 for the affine nodes of NEXT-4)
  a.data = base;
  a.mom = a.data + nz * B * B;
  a.rhs_data = a.mom + nz * 16;
  a.node_mom = a.rhs_data + ((B * m + 3) & ~(size_t)3);
  a.graph = a.node_mom + 12 * m;
  a.rhs_graph = a.graph + nz * B * B;
  a.energy = c->energy.as<double>();
  return a;
}

// ------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  std::string why;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, char[128], int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
// ncclDataType_t / ncclRedOp_t values (nccl.h, NCCL 2.x)
enum { kNcclInt64 = 4, kNcclUint64 = 5, kNcclFloat32 = 7, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.why = "libnccl.so.2 not found"; return; }
    api.GetUniqueId = (int (*)(void*))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (int (*)(void**, int, char[128], int))dlsym(h, "ncclCommInitRank");
    api.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclAllReduce");
    api.AllGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(h, "ncclAllGather");
    api.CommDestroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
    api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.CommDestroy;
    if (!api.ok) api.why = "libnccl symbols missing";
  });
  return api;
}

static cudaError_t nccl_ret(Ctx* c, int r) {
  if (r == 0) return cudaSuccess;
  c->err = std::string("NCCL error: ") + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
  return cudaErrorUnknown;
}
cudaError_t nccl_allreduce_sum_f32(Ctx* c, float* buf, size_t count) {
  return nccl_ret(c, nccl().AllReduce(buf, buf, count, kNcclFloat32, kNcclSum, c->nccl_comm, c->st));
}
cudaError_t nccl_allreduce_sum_f64(Ctx* c, double* buf, size_t count) {
  return nccl_ret(c, nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, c->nccl_comm, c->st));
}
cudaError_t nccl_allreduce_max_i64(Ctx* c, int64_t* buf, size_t count) {
  return nccl_ret(c, nccl().AllReduce(buf, buf, count, kNcclInt64, kNcclMax, c->nccl_comm, c->st));
}
cudaError_t nccl_allgather_u64(Ctx* c, const uint64_t* send, uint64_t* recv, size_t count) {
  return nccl_ret(c, nccl().AllGather(send, recv, count, kNcclUint64, c->nccl_comm, c->st));
}

// ------------------------------------------------------------ small kernels
__global__ void k_interleave3(int64_t n, const float* x, const float* y, const float* z, float* aos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  aos[3 * i] = x[i]; aos[3 * i + 1] = y[i]; aos[3 * i + 2] = z[i];
}
// mis_set_model in one pass: AoS xyz / nrm / rgb -> SoA, weight / stamp / ids
// copied or defaulted, next fresh id = max(ids) + 1 (ids_dev zeroed before).
struct LoadSrc {
  const float *xyz, *nrm, *rgb, *w;
  const int32_t* stamp;
  const int64_t* ids;
};
__global__ void k_load_model(int64_t n, LoadSrc src, ModelView md, long long* ids_dev) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ long long bm;
  if (threadIdx.x == 0) bm = -1;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !src.ids) ids_dev[0] = n;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    md.px[i] = src.xyz[3 * i]; md.py[i] = src.xyz[3 * i + 1]; md.pz[i] = src.xyz[3 * i + 2];
    md.nx[i] = src.nrm[3 * i]; md.ny[i] = src.nrm[3 * i + 1]; md.nz[i] = src.nrm[3 * i + 2];
    if (src.rgb) { md.cr[i] = src.rgb[3 * i]; md.cg[i] = src.rgb[3 * i + 1]; md.cb[i] = src.rgb[3 * i + 2]; }
    else { md.cr[i] = 0.f; md.cg[i] = 0.f; md.cb[i] = 0.f; }
    md.w[i] = src.w ? src.w[i] : 1.0f;
    md.stamp[i] = src.stamp ? src.stamp[i] : 0;
    const int64_t id = src.ids ? src.ids[i] : i;
    md.ids[i] = id;
    if (src.ids) atomicMax(&bm, (long long)id);
  }
  if (!src.ids) return;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(ids_dev, bm + 1);
}
// point-major (n x K) caller skinning -> slot-major, ids ascending; validation flags
__global__ void k_canon_knn(int64_t n, int K, int m, const int32_t* idx_pm, const float* w_pm, int64_t cap,
                            int32_t* kidx, float* kw, int* flag) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int id[MIS_MAX_K];
  float w[MIS_MAX_K];
  for (int s = 0; s < K; ++s) { id[s] = idx_pm[i * K + s]; w[s] = w_pm[i * K + s]; }
  for (int a = 1; a < K; ++a)
    for (int b = a; b > 0 && id[b] < id[b - 1]; --b) {
      int t = id[b]; id[b] = id[b - 1]; id[b - 1] = t;
      float tw = w[b]; w[b] = w[b - 1]; w[b - 1] = tw;
    }
  int f = 0;
  for (int s = 0; s < K; ++s) {
    if (id[s] < 0 || id[s] >= m) f |= 1;
    if (s > 0 && id[s] == id[s - 1]) f |= 2;
    if (!(w[s] >= 0.f) || !isfinite(w[s])) f |= 4;
    kidx[s * cap + i] = id[s] < 0 ? 0 : (id[s] >= m ? m - 1 : id[s]);
    kw[s * cap + i] = w[s];
  }
  if (f) atomicOr(flag, f);
}
__global__ void k_to_point_major(int64_t n, int K, int64_t cap, const int32_t* kidx, const float* kw, int32_t* idx_pm,
                                 float* w_pm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int s = 0; s < K; ++s) {
    if (idx_pm) idx_pm[i * K + s] = kidx[s * cap + i];
    if (w_pm) w_pm[i * K + s] = kw[s * cap + i];
  }
}
__global__ void k_copy2(int64_t n, const float* a, const float* b, float* a_out, float* b_out) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) { a_out[t] = a[t]; b_out[t] = b[t]; }
}

// mis_set_graph's inputs in one pass: node positions copied, neighbour lists copied and
// validated (an invalid entry is flagged and neutralised so later kernels stay in bounds), and the
// node states initialised to the identity (from the source positions; one launch, not two)
__global__ void k_graph_in(int m, int n_nbr, const float* g_src, const int32_t* nbr_src, float* g, int32_t* nbr,
                           int* flag, double* Rt64, float* node32) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 3 * m) g[t] = g_src[t];
  if (t < m) {
    for (int i = 0; i < 12; ++i) Rt64[12 * t + i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
    for (int i = 0; i < 12; ++i) node32[16 * t + i] = (i == 0 || i == 4 || i == 8) ? 1.f : 0.f;
    for (int c = 0; c < 3; ++c) node32[16 * t + 12 + c] = g_src[3 * t + c];
    node32[16 * t + 15] = 0.f;
  }
  if (t >= m * n_nbr) return;
  int l = nbr_src[t];
  if (l < -1 || l >= m || l == t / n_nbr) {
    atomicOr(flag, 8);
    l = -1;
  }
  nbr[t] = l;
}
__global__ void k_set_nodes(int m, const float* Rt, double* Rt64, float* node32) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (int i = 0; i < 12; ++i) {
    Rt64[12 * j + i] = (double)Rt[12 * j + i];
    node32[16 * j + i] = Rt[12 * j + i];
  }
}
__global__ void k_get_nodes(int m, const float* node32, float* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (int i = 0; i < 12; ++i) out[12 * j + i] = node32[16 * j + i];
}
// ids_dev[0] = max(ids) + 1 (ids == null: n); grid-wide max by atomicMax after a block max
__global__ void k_next_id(int64_t n, const int64_t* ids, long long* ids_dev) {
  __shared__ long long bm;
  if (threadIdx.x == 0) bm = -1;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !ids) ids_dev[0] = n;
  __syncthreads();
  if (!ids) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicMax(&bm, (long long)ids[i]);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(ids_dev, bm + 1);
}


static inline int nb(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------------ instrumentation
static std::atomic<int64_t> g_launches{0};
void count_launches(int64_t k) { g_launches += k; }

static cudaEvent_t pool_get(Ctx* c) {
  if (!c->pool.empty()) { cudaEvent_t e = c->pool.back(); c->pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(Ctx* c_, int cat_, int nk) : c(c_), cat(cat_) {
  l0 = g_launches;
  g_launches += nk;
  if (c->prof && (!c->prof_light || cat == P_POINTS || cat == P_ACCUM || cat == P_SOLVE)) {
    cudaEvent_t a = pool_get(c);
    b = pool_get(c);
    cudaEventRecord(a, c->st);
    c->pev.push_back({cat, a, b});
  }
}
ProfScope::~ProfScope() {
  c->prof_n[cat] += g_launches - l0;   // includes count_launches() calls made inside the scope
  if (b) cudaEventRecord(b, c->st);
}

static void prof_collect(Ctx* c) {
  cudaStreamSynchronize(c->st);
  for (auto& e : c->pev) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) c->prof_ms[e.cat] += ms;
    c->pool.push_back(e.a);
    c->pool.push_back(e.b);
  }
  c->pev.clear();
}

// copy stream for host-memory frame inputs, created with the first one
cudaError_t copy_stream(Ctx* c) {
  if (c->st_copy) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->st_copy, cudaStreamNonBlocking)) != cudaSuccess) return e;
  cudaEvent_t* evs[] = {&c->ev_depth_free, &c->ev_depth_ready, &c->ev_rgb_free, &c->ev_rgb_ready};
  for (cudaEvent_t* ev : evs)
    if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  return cudaSuccess;
}

// K1 of a frame whose launch mis_register deferred (see set_frame_impl)
cudaError_t flush_frame(Ctx* c) {
  if (!c->frame_pending) return cudaSuccess;
  c->frame_pending = false;
  ProfScope ps(c, P_FRAME, 1);
  FrameView fv = frame_view(c);
  fv.depth = c->frame_src;
  launch_frame_prep(fv, c->nmap.as<float4>(), c->nmapd.as<double4>(), c->st);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && c->frame_src == c->depth.p)   // host-staged depth: the buffer may be overwritten
    e = cudaEventRecord(c->ev_depth_free, c->st);     // (device inputs record nothing: no break in the PDL chain)
  return e;
}

}  // namespace mis

using namespace mis;

// ------------------------------------------------------------ error helpers
static mis_status fail(Ctx* c, mis_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}
static mis_status cuda_fail(Ctx* c, cudaError_t e, const char* where) {
  if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e) + (c->err.empty() ? "" : " (" + c->err + ")");
  return e == cudaErrorMemoryAllocation ? MIS_E_NOMEM : MIS_E_CUDA;
}
#define TRY(c, call)                                              \
  do {                                                            \
    cudaError_t e__ = (call);                                     \
    if (e__ != cudaSuccess) return cuda_fail((c), e__, #call);    \
  } while (0)

static cudaError_t run_build_order(Ctx* c) {
  ProfScope ps(c, P_ORDER, 0);   // build_order counts its own launches
  return build_order(c);
}

static cudaMemcpyKind kind_in(mis_mem mem) { return mem == MIS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice; }
static cudaMemcpyKind kind_out(mis_mem mem) { return mem == MIS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice; }

static mis_status check_params(const mis_params* p) {
  if (!p) return MIS_E_ARG;
  if (p->k < 1 || p->k > MIS_MAX_K || p->n_nbr < 0 || p->gn_iters < 1 || p->gn_iters > MIS_MAX_GN ||
      p->pcg_iters < 0 || !(p->eps_d_mm > 0) || !(p->eps_n_deg > 0) || !(p->tau_z_mm > 0) || !(p->trunc_mm > 0) ||
      !(p->omega_max >= 1) || !(p->lambda >= 0) || !std::isfinite(p->tau_z_mm) || !std::isfinite(p->trunc_mm) ||
      !std::isfinite(p->eps_d_mm) || !(p->delta_deg > 0) || !(p->delta_deg < 180) || !(p->eps_n_deg < 180) ||
      !std::isfinite(p->omega_max) || !std::isfinite(p->lambda) || p->n_nbr > 64 || !(p->w_r >= 0) ||
      !(p->w_p >= 0) || !std::isfinite(p->w_r) || !std::isfinite(p->w_p) || !(p->w_rot >= 0) ||
      !std::isfinite(p->w_rot))
    return MIS_E_ARG;
  if ((p->flags & MIS_F_AFFINE) && (p->k > 4 || (p->flags & MIS_F_JOINT_POSE))) return MIS_E_ARG;
  if ((p->flags & MIS_F_JOINT_POSE) && p->k > MIS_MAX_K - 1) return MIS_E_ARG;
  return MIS_OK;
}

// ------------------------------------------------------------ C-ABI
extern "C" {

int32_t mis_abi_version(void) { return MIS_ABI_VERSION; }

void mis_default_params(mis_params* o) {
  if (!o) return;
  o->k = 4; o->n_nbr = 4;
  o->w_data = 1.0f; o->w_point = 1.0f; o->w_reg = 1e4f; o->w_corr = 10.0f;
  o->eps_d_mm = 15.0f; o->eps_n_deg = 10.0f;
  o->tau_z_mm = 10.0f; o->delta_deg = 10.0f; o->trunc_mm = 40.0f; o->omega_max = 10.0f;
  o->gn_iters = 5; o->pcg_iters = 10; o->lambda = 1e-4f; o->flags = 0;
  o->w_r = 1e6f; o->w_p = 1000.0f;   // Eq. 10 prior weights, MIS_F_JOINT_POSE
  o->w_rot = 1000.0f;                 // Eq. 4 weight, MIS_F_AFFINE
}

const char* mis_last_error(const mis_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

mis_status mis_nccl_unique_id(void* out128) {
  if (!out128) return MIS_E_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return MIS_E_NCCL;
  return api.GetUniqueId(out128) == 0 ? MIS_OK : MIS_E_NCCL;
}

mis_status mis_create(const mis_params* params, int device, void* cuda_stream, int rank, int world,
                      const void* nccl_unique_id, mis_ctx** out) {
  if (!out) return MIS_E_ARG;
  *out = nullptr;
  if (check_params(params) != MIS_OK || world < 1 || rank < 0 || rank >= world) return MIS_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return MIS_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return MIS_E_CUDA;
  mis_ctx* c = new mis_ctx();
  c->prm = *params;
  c->K = params->k;
  c->device = device;
  c->rank = rank;
  c->world = world;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    c->st = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) { delete c; return MIS_E_CUDA; }
    c->own_stream = true;
  }
  if (const char* e = getenv("MIS_ORDER_BY_SORT")) c->order_by_sort = atoi(e) != 0;
  if (const char* e = getenv("MIS_K3_SPLIT")) c->k3_split = atoi(e) != 0;

  if (world > 1) {
    NcclApi& api = nccl();
    if (!api.ok || !nccl_unique_id) { delete c; return MIS_E_NCCL; }
    char id[128];
    memcpy(id, nccl_unique_id, 128);
    if (api.CommInitRank(&c->nccl_comm, world, id, rank) != 0) { delete c; return MIS_E_NCCL; }
  }
  if (ensure(c, c->rep, kRepBytes) != cudaSuccess ||
      ensure(c, c->tstamp, 2048) != cudaSuccess || cudaMemset(c->tstamp.p, 0, 2048) != cudaSuccess ||
      ensure(c, c->counter, 64) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->hpin), 16 * sizeof(int64_t)) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->rb_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return MIS_E_NOMEM;
  }
  *out = c;
  return MIS_OK;
}

mis_status mis_destroy(mis_ctx* c) {
  if (!c) return MIS_E_ARG;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  for (DBuf* b : c->bufs) free_buf(c, *b);   // every buffer ensure() ever allocated
  c->bufs.clear();
  if (c->nccl_comm && nccl().ok) nccl().CommDestroy(c->nccl_comm);
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->rb_ev) cudaEventDestroy(c->rb_ev);
  if (c->st_copy) { cudaStreamSynchronize(c->st_copy); cudaStreamDestroy(c->st_copy); }
  for (cudaEvent_t ev : {c->ev_depth_free, c->ev_depth_ready, c->ev_rgb_free, c->ev_rgb_ready})
    if (ev) cudaEventDestroy(ev);
  if (c->own_stream) cudaStreamDestroy(c->st);

  delete c;
  return MIS_OK;
}

// Upper bound of the device memory the context's buffers take for a model capacity n_cap, m nodes
// and H x W frames (mis.h).  Every buffer ensure() may allocate is listed at its largest size; the
// pattern-dependent ones assume nnzb <= m (2 n_nbr + 1 + 4 k^2) blocks (measured: 14 m at C3, 32 m
// at C5) and n_feat <= max(4096, H W / 64) feature pairs.
static size_t workspace_plan(const Ctx* c, int64_t n, int64_t m, int64_t H, int64_t W) {
  const int64_t K = c->K + 1, P = K * (K + 1) / 2, nn = std::max<int32_t>(c->prm.n_nbr, 1), px = H * W;
  // sized for a joint-pose pattern (NEXT-2): k + 1 factor slots, m + 1 unknowns, 2m + 1 more blocks
  const int64_t nnz = std::min<int64_t>(m * m, m * (2 * nn + 1 + 4 * K * K)) + 2 * m + 1;
  m += 1;
  const int64_t nf = std::max<int64_t>(4096, px / 64);
  const int64_t mr = m, cs = 16, mp = nnz / 4 + mr + 1;   // cluster PCG lists (pcg_cluster.cu max_pieces)
  int64_t slots = 1024;
  while (slots < 2 * n) slots <<= 1;
  std::vector<int64_t> b = {
      // model, two buffer sets: 10 float planes, stamp, ids, skinning (MIS_MAX_K slots)
      2 * 10 * 4 * n, 2 * 4 * n, 2 * 8 * n, 2 * 4 * n * MIS_MAX_K, 2 * 4 * n * MIS_MAX_K,
      32, 64, 64, 64,                                                        // ids_dev, nnz_dev, finfo, lm
      12 * m, 4 * m * nn, 64 * m, 96 * m,                                    // graph, node states
      std::max(std::max(n * 64 + 64, n * (12 + 16 * K) + 64), m * 48),       // staging
      slots * 12, 8 * n, 4 * n + 64, 4 * n + 64,                            // K13 grouping
      4 * n, 4 * n, 8 * n, 8 * n, 4 * (n + 1), 4 * n * K, 16 * n, 8 * n, 4 * n, 4 * (n + 1),   // order
      (int64_t)cub_tmp_bound(std::max<int64_t>(n, m + 1)) + 256,
      m * ((m + 63) / 64) * 8 * (c->world > 1 ? 1 + c->world : 1),         // pattern bitmap(s)
      4 * (m + 1), 4 * (m + 1), 4 * m, 128, 4 * nnz + 4, 4 * nnz + 4, 4 * nnz + 4, 4 * nnz + 4,
      ((nnz - m) / 2 + 1) * 8, (n * P + 1) * 4, (m * nn + 1) * 4, (nf * P + 1) * 4,
      cs * (mr + 1) * 4, cs * mp * 4, cs * mr * 64, 128, 4 * m,              // cluster PCG lists
      // accumulators, system and PCG sized for 12 x 12 blocks (the affine nodes of NEXT-4)
      nnz * 304 * 4 + (12 * m + 3) * 4 + 48 * m + 48 * m, kEnergyDoubles * 8,  // accumulators
      576 * nnz, 48 * m, 576 * m, 14 * 48 * m, (8 * (int64_t)c->prm.pcg_iters + 16) * 8,   // system, PCG
      144 * nnz, 24 * m, 96 * m,                                            // LM second system, kept nodes
      (K + 2) * 16 * n,                                                     // K3a -> K3b state
      4 * px, 16 * px, 32 * px, 12 * px, 8 * px, 4 * px, (2 * ((px + 255) / 256) + 4) * 4,   // frame, fusion
      4 * n, n,                                                             // pix, why
      12 * nf + 16, 12 * nf + 16, 4 * nf * K + 16, 4 * nf * K + 16,         // features
      12 * n, 4 * n, 4 * n * K, 4 * n * K,                                  // filter re-skinning list
      32 * n, 4 * m * nn,                                                   // node regeneration: cell sums, N(j)
      24 * 8, 4 * n * K,                                                    // joint pose: state, tuples
  };
  size_t total = 0;
  for (int64_t x : b) {
    const size_t bytes = (size_t)std::max<int64_t>(x, 16);
    total += ((bytes + bytes / MIS_ENSURE_SLACK_DIV + 256) + kWsAlign - 1) & ~(kWsAlign - 1);   // ensure()'s slack
  }
  return total + total / 8 + (1 << 20);   // first-fit fragmentation margin
}

mis_status mis_workspace_bytes(const mis_ctx* c, int64_t n_cap, int32_t m, int32_t H, int32_t W, size_t* bytes) {
  if (!c || !bytes || n_cap < 0 || m < 1 || H < 0 || W < 0) return MIS_E_ARG;
  *bytes = workspace_plan(c, std::max<int64_t>(n_cap, 1), m, H, W);
  return MIS_OK;
}

mis_status mis_bind_workspace(mis_ctx* c, void* dev_ptr, size_t bytes) {
  if (!c) return MIS_E_ARG;
  if (!dev_ptr || bytes < (1 << 20) || ((uintptr_t)dev_ptr & (kWsAlign - 1)))
    return fail(c, MIS_E_ARG, "bind_workspace: null, < 1 MiB or not 256-byte aligned");
  if (c->ws_base) return fail(c, MIS_E_STATE, "bind_workspace: a workspace is already bound");
  if (c->have_model) return fail(c, MIS_E_STATE, "bind_workspace must precede mis_set_model");
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, dev_ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice || at.device != c->device) {
    cudaGetLastError();
    return fail(c, MIS_E_ARG, "bind_workspace: not device memory of the context's GPU");
  }
  c->ws_base = static_cast<char*>(dev_ptr);
  c->ws_bytes = bytes & ~(kWsAlign - 1);
  c->ws_free.clear();
  c->ws_free[0] = c->ws_bytes;
  return MIS_OK;
}

mis_status mis_set_params(mis_ctx* c, const mis_params* p) {
  if (!c) return MIS_E_ARG;
  if (check_params(p) != MIS_OK) return fail(c, MIS_E_ARG, "invalid parameters");
  if (p->k != c->prm.k && c->have_graph) return fail(c, MIS_E_STATE, "k cannot change after mis_set_graph");
  if (p->n_nbr != c->prm.n_nbr && c->have_graph) return fail(c, MIS_E_STATE, "n_nbr cannot change after mis_set_graph");
  c->prm = *p;
  c->K = p->k;
  c->pattern_valid = false;
  return MIS_OK;
}

mis_status mis_set_model(mis_ctx* c, int64_t n, mis_mem mem, const float* xyz, const float* nrm, const float* rgb,
                         const float* weight, const int32_t* stamp, const int64_t* ids, int64_t capacity) {
  if (!c) return MIS_E_ARG;
  if (n < 0 || capacity < n || (n > 0 && (!xyz || !nrm)) || capacity > (int64_t)0x7fffffff)
    return fail(c, MIS_E_ARG, "set_model: bad sizes or null xyz/nrm");
  cudaSetDevice(c->device);
  const int K = c->K;
  if (capacity < 1) capacity = 1;
  for (int s = 0; s < 2; ++s) {
    ModelBufs& B = c->mb[s];
    DBuf* f[] = {&B.px, &B.py, &B.pz, &B.nx, &B.ny, &B.nz, &B.cr, &B.cg, &B.cb, &B.w};
    for (DBuf* b : f) TRY(c, ensure(c, *b, capacity * 4));
    TRY(c, ensure(c, B.stamp, capacity * 4));
    TRY(c, ensure(c, B.ids, capacity * 8));
    TRY(c, ensure(c, B.kidx, capacity * 4 * MIS_MAX_K));
    TRY(c, ensure(c, B.kw, capacity * 4 * MIS_MAX_K));
  }
  c->cur = 0;
  c->cap = capacity;
  c->n = n;
  ModelView md = model_view(c);
  TRY(c, ensure(c, c->ids_dev, 32));
  TRY(c, cudaMemsetAsync(c->ids_dev.p, 0, 32, c->st));
  if (n > 0) {
    LoadSrc src{xyz, nrm, rgb, weight, stamp, ids};
    if (mem == MIS_MEM_HOST) {   // stage the host arrays once, then the same single pass
      TRY(c, ensure(c, c->stage, n * 56));
      char* st = c->stage.as<char>();
      cudaError_t err = cudaSuccess;
      auto put = [&](const void* h, size_t bytes, size_t off) -> const void* {
        if (!h) return nullptr;
        const cudaError_t e = cudaMemcpyAsync(st + off, h, bytes, cudaMemcpyHostToDevice, c->st);
        if (e != cudaSuccess) err = e;
        return st + off;
      };
      src.xyz = (const float*)put(xyz, n * 12, 0);
      src.nrm = (const float*)put(nrm, n * 12, n * 12);
      src.rgb = (const float*)put(rgb, n * 12, n * 24);
      src.w = (const float*)put(weight, n * 4, n * 36);
      src.stamp = (const int32_t*)put(stamp, n * 4, n * 40);
      src.ids = (const int64_t*)put(ids, n * 8, n * 48);
      TRY(c, err);
    }
    ProfScope ps(c, P_IO, 1);
    launch_pdl(k_load_model, dim3(nb(n)), dim3(256), 0, c->st, n, src, md, c->ids_dev.as<long long>());
  } else {
    ProfScope ps(c, P_IO, 1);
    k_next_id<<<1, 256, 0, c->st>>>(0, nullptr, c->ids_dev.as<long long>());
  }
  TRY(c, cudaGetLastError());
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  c->have_model = true;
  c->have_graph = false;
  c->pattern_valid = false;
  return MIS_OK;
}

static cudaError_t skin(Ctx* c, int64_t nq, const float* px, const float* py, const float* pz, int64_t sxyz,
                        int32_t* idx, float* w, int64_t os) {
  launch_skin(nq, px, py, pz, sxyz, c->g.as<float>(), c->m, c->K, idx, w, os, c->st);
  return cudaGetLastError();
}

static std::string graph_flag_message(int f) {
  return std::string("set_graph: invalid") + ((f & 1) ? " node id" : "") + ((f & 2) ? " duplicate id" : "") +
         ((f & 4) ? " weight" : "") + ((f & 8) ? " neighbour list" : "");
}

// skin_order (internal, mis_regenerate_nodes): the points in a spatially coherent order (sorted by node
// cell), skinned by the boxed K2 instead of the brute-force one
static mis_status set_graph_impl(mis_ctx* c, int32_t m, mis_mem mem, const float* node_pos, const int32_t* node_nbr,
                                 const int32_t* knn_idx, const float* knn_w, const uint32_t* skin_order);

mis_status mis_set_graph(mis_ctx* c, int32_t m, mis_mem mem, const float* node_pos, const int32_t* node_nbr,
                         const int32_t* knn_idx, const float* knn_w) {
  return set_graph_impl(c, m, mem, node_pos, node_nbr, knn_idx, knn_w, nullptr);
}

static mis_status set_graph_impl(mis_ctx* c, int32_t m, mis_mem mem, const float* node_pos, const int32_t* node_nbr,
                                 const int32_t* knn_idx, const float* knn_w, const uint32_t* skin_order) {
  if (!c) return MIS_E_ARG;
  if (!c->have_model) return fail(c, MIS_E_STATE, "set_graph before set_model");
  const int K = c->K, nn = c->prm.n_nbr;
  if (m < 1 || !node_pos || (nn > 0 && !node_nbr) || (knn_idx && !knn_w))
    return fail(c, MIS_E_ARG, "set_graph: bad arguments");
  if (!knn_idx && m < K + 1) return fail(c, MIS_E_ARG, "device skinning needs m >= k+1 (Eq. 2)");
  if (knn_idx && m < K) return fail(c, MIS_E_ARG, "k distinct nodes per point need m >= k");
  cudaSetDevice(c->device);
  c->m = m;
  TRY(c, ensure(c, c->g, (size_t)m * 12));
  TRY(c, ensure(c, c->nbr, (size_t)m * (nn > 0 ? nn : 1) * 4));
  TRY(c, ensure(c, c->node32, (size_t)m * 64));
  TRY(c, ensure(c, c->Rt64, (size_t)m * 96));
  const float* g_src = node_pos;            // device inputs are read in place by k_graph_in
  const int32_t* nbr_src = node_nbr;
  if (mem == MIS_MEM_HOST) {
    TRY(c, cudaMemcpyAsync(c->g.p, node_pos, (size_t)m * 12, cudaMemcpyHostToDevice, c->st));
    if (nn > 0) TRY(c, cudaMemcpyAsync(c->nbr.p, node_nbr, (size_t)m * nn * 4, cudaMemcpyHostToDevice, c->st));
    g_src = c->g.as<float>();
    nbr_src = c->nbr.as<int32_t>();
  }
  if (!c->nnz_dev.p) {
    TRY(c, ensure(c, c->nnz_dev, 64));
    TRY(c, cudaMemsetAsync(c->nnz_dev.p, 0, 64, c->st));
  }
  int* flag = reinterpret_cast<int*>(c->nnz_dev.as<int64_t>() + 3);   // validation flags (info[3], zero at rest)
  {
    ProfScope ps(c, P_IO, 1);
    launch_pdl(k_graph_in, dim3(nb(std::max<int64_t>((int64_t)m * nn, 3 * (int64_t)m))), dim3(256), 0, c->st, m, nn,
               g_src, nbr_src, c->g.as<float>(), c->nbr.as<int32_t>(), flag, c->Rt64.as<double>(),
               c->node32.as<float>());
  }
  ModelView md = model_view(c);
  const int64_t n = c->n;
  if (n > 0) {
    ProfScope ps(c, knn_idx ? P_IO : P_SKIN, 1);
    if (knn_idx) {
      const int32_t* si = knn_idx;
      const float* sw = knn_w;
      if (mem == MIS_MEM_HOST) {   // device pointers are read in place
        TRY(c, ensure(c, c->stage, n * K * 8));
        int32_t* di = c->stage.as<int32_t>();
        float* dw = reinterpret_cast<float*>(di + n * K);
        TRY(c, cudaMemcpyAsync(di, knn_idx, n * K * 4, cudaMemcpyHostToDevice, c->st));
        TRY(c, cudaMemcpyAsync(dw, knn_w, n * K * 4, cudaMemcpyHostToDevice, c->st));
        si = di;
        sw = dw;
      }
      launch_pdl(k_canon_knn, dim3(nb(n)), dim3(256), 0, c->st, n, K, m, si, sw, c->cap, md.kidx, md.kw, flag);
    } else if (skin_order) {
      launch_skin_boxed(n, skin_order, 1, md.px, md.py, md.pz, 1, c->g.as<float>(), m, K, md.kidx, md.kw, c->cap,
                        c->st);
      TRY(c, cudaGetLastError());
    } else {
      TRY(c, skin(c, n, md.px, md.py, md.pz, 1, md.kidx, md.kw, c->cap));
    }
  }
  if (mem == MIS_MEM_HOST) {   // host inputs: validate now (the copies synchronise anyway)
    int hflag = 0;
    TRY(c, cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, c->st));
    TRY(c, cudaStreamSynchronize(c->st));
    if (hflag) {
      TRY(c, cudaMemsetAsync(flag, 0, 8, c->st));   // back to zero at rest
      c->have_graph = false;
      return fail(c, MIS_E_ARG, graph_flag_message(hflag));
    }
    c->graph_check = false;
  } else {
    // device inputs: no host synchronisation here; invalid ids were clamped / neutralised on
    // the device and the flags come back with the pattern readback (the next mis_register
    // fails with MIS_E_ARG)
    c->graph_check = true;
  }
  TRY(c, cudaGetLastError());   // (the identity node states were written by k_graph_in)
  TRY(c, run_build_order(c));
  c->have_graph = true;
  return MIS_OK;
}


// defer: mis_register only -- K1 is queued behind the frame's pattern readback so it runs
// while the host waits for it (the depth is still read within the same API call)
static cudaError_t issue_colour_copy(Ctx* c, const float* rgb);
static mis_status set_frame_impl(mis_ctx* c, mis_mem mem, const float* depth_mm, const mis_intrinsics* it,
                                 const float pose[12], bool defer);
mis_status mis_set_frame(mis_ctx* c, mis_mem mem, const float* depth_mm, const mis_intrinsics* it, const float pose[12]) {
  return set_frame_impl(c, mem, depth_mm, it, pose, false);
}
static mis_status set_frame_impl(mis_ctx* c, mis_mem mem, const float* depth_mm, const mis_intrinsics* it,
                                 const float pose[12], bool defer) {
  if (!c) return MIS_E_ARG;
  if (!depth_mm || !it || !pose) return fail(c, MIS_E_ARG, "set_frame: null argument");
  if (!(it->fx > 0) || !(it->fy > 0) || it->width < 3 || it->height < 3 || !(it->cx >= 0) || !(it->cx < it->width) ||
      !(it->cy >= 0) || !(it->cy < it->height))
    return fail(c, MIS_E_ARG, "set_frame: invalid intrinsics (S:24)");
  cudaSetDevice(c->device);
  c->intr = *it;
  c->W = it->width;
  c->H = it->height;
  memcpy(c->pose, pose, 48);   // pose is host memory (12 floats) in every mode
  c->pose_valid = false;       // a new input pose (NEXT-2: the next joint registration refines it)
  const size_t px = (size_t)c->W * c->H;
  const float* dsrc = depth_mm;   // device depth is read in place by K1 (stream order)
  if (mem == MIS_MEM_HOST) {
    TRY(c, ensure(c, c->depth, px * 4));
    dsrc = c->depth.as<float>();
  }
  TRY(c, ensure(c, c->nmap, px * 16));
  TRY(c, ensure(c, c->nmapd, px * 32));
  if (mem == MIS_MEM_HOST) {
    // on the copy stream, after the previous frame prep has read the buffer: the transfer overlaps
    // whatever the context stream is still running (e.g. the model ordering of mis_set_graph);
    // the context stream waits for it before K1
    TRY(c, copy_stream(c));
    TRY(c, cudaStreamWaitEvent(c->st_copy, c->ev_depth_free, 0));
    TRY(c, cudaMemcpyAsync(c->depth.p, depth_mm, px * 4, cudaMemcpyHostToDevice, c->st_copy));
    TRY(c, cudaEventRecord(c->ev_depth_ready, c->st_copy));
    TRY(c, cudaStreamWaitEvent(c->st, c->ev_depth_ready, 0));
  }
  if (c->rgb_pending) {   // a staged colour (mis_stage_colour): its upload right behind the depth's
    TRY(c, issue_colour_copy(c, c->rgb_pending));
    c->rgb_pending = nullptr;
  }
  c->frame_src = dsrc;
  c->frame_pending = true;
  if (!defer || c->prof) TRY(c, flush_frame(c));   // (profiling: K1 in its own group)
  c->have_frame = true;
  return MIS_OK;
}

mis_status mis_set_features(mis_ctx* c, mis_mem mem, int32_t n_feat, const float* src, const float* dst) {
  if (!c) return MIS_E_ARG;
  if (n_feat < 0 || (n_feat > 0 && (!src || !dst))) return fail(c, MIS_E_ARG, "set_features: bad arguments");
  if (!c->have_graph) return fail(c, MIS_E_STATE, "set_features before set_graph");
  if (n_feat > 0 && c->m < c->K + 1) return fail(c, MIS_E_ARG, "feature skinning needs m >= k+1");
  cudaSetDevice(c->device);
  c->nf = n_feat;
  const int K = c->K;
  TRY(c, ensure(c, c->fsrc, (size_t)n_feat * 12 + 16));
  TRY(c, ensure(c, c->fdst, (size_t)n_feat * 12 + 16));
  TRY(c, ensure(c, c->fidx, (size_t)n_feat * (K + 1) * 4 + 16));   // + the pose row of a joint pattern
  TRY(c, ensure(c, c->fw, (size_t)n_feat * K * 4 + 16));
  if (n_feat > 0) {
    if (mem == MIS_MEM_HOST) {
      TRY(c, cudaMemcpyAsync(c->fsrc.p, src, (size_t)n_feat * 12, cudaMemcpyHostToDevice, c->st));
      TRY(c, cudaMemcpyAsync(c->fdst.p, dst, (size_t)n_feat * 12, cudaMemcpyHostToDevice, c->st));
    } else {   // both copies in one launch
      ProfScope ps(c, P_IO, 1);
      launch_pdl(k_copy2, dim3(nb(3 * (int64_t)n_feat)), dim3(256), 0, c->st, 3 * (int64_t)n_feat, src, dst,
                 c->fsrc.as<float>(), c->fdst.as<float>());
    }
    const float* s = c->fsrc.as<float>();
    ProfScope ps(c, P_SKIN, 1);
    TRY(c, skin(c, n_feat, s, s + 1, s + 2, 3, c->fidx.as<int32_t>(), c->fw.as<float>(), n_feat));
    TRY(c, cudaGetLastError());
  }
  c->pattern_valid = false;
  return MIS_OK;
}

// K3 (+ K4/K5 on rank 0) into the zeroed accumulators, all-reduce across ranks, finalise
// (which writes report slot `slot` if >= 0 and re-zeroes everything it read)
static mis_status assemble(Ctx* c, bool dbg, int slot) {
  AccView acc = acc_view(c);
  c->acc_dirty = true;   // until the finalisation below has re-zeroed them
  const double d2r = M_PI / 180.0;
  AsmPointsArgs a;
  a.md = model_view(c);
  a.seg_nodes = c->seg_nodes.as<int32_t>();
  a.chunks = c->chunks.as<int4>();
  a.nchunk = c->nchunk;
  a.seg_slot = c->seg_slot.as<int32_t>();
  a.nd = node_view(c);
  a.fr = frame_view(c);
  a.eps_d = c->prm.eps_d_mm;
  a.eps_dd = c->prm.eps_d_mm;
  a.cos_eps_nd = cos(c->prm.eps_n_deg * d2r);
  a.cos_eps_n = (float)a.cos_eps_nd;
  a.acc = acc;
  const bool joint = c->pattern_joint;   // NEXT-2: the pose as factor slot k / unknown m
  const int KS = c->K + (joint ? 1 : 0);
  a.pose_cur = joint ? c->posebuf.as<double>() : nullptr;
  const bool aff = c->pattern_affine;   // NEXT-4
  a.affine = aff ? 1 : 0;
  // the tcgen05 K3b (k > 4) reads the factor state of associated points only (MIS_K3B_SPARSE=0 writes
  // every point's planes, for comparison)
  static const bool sparse_env = [] {
    const char* e = getenv("MIS_K3B_SPARSE");
    return e ? atoi(e) != 0 : true;
  }();
  a.sparse_state = (KS > 4 && !aff && kChunk <= 128 && umma_k3b_enabled() && sparse_env) ? 1 : 0;
  // K3a by chunk (MIS_K3A_CHUNKED=0: per point) for the tcgen05 K3b's k > 4 (joint: k + 1 > 4) slots
  static const bool chunked_env = [] {
    const char* e = getenv("MIS_K3A_CHUNKED");
    return e ? atoi(e) != 0 : true;
  }();
  a.chunk_live = nullptr;
  if (a.sparse_state && chunked_env && !dbg && c->nchunk > 0 && (joint ? c->K < MIS_MAX_K : c->K > 4)) {
    TRY(c, ensure(c, c->chunk_live, (size_t)c->nchunk * 4));
    a.chunk_live = c->chunk_live.as<int32_t>();
  }
  if (joint) a.seg_nodes = c->seg_nodes_j.as<int32_t>();
  TRY(c, ensure(c, c->pstate, (size_t)(KS + 2) * 16 * (size_t)std::max<int64_t>(ncap(c, c->n), 1)));
  a.pstate = c->pstate.as<float4>();
  a.pstride = std::max<int64_t>(c->n, 1);
  a.work_counter = reinterpret_cast<unsigned long long*>(c->energy.as<double>() + 6);   // zeroed with the energies
  a.dbg_pix = dbg ? c->pix.as<int32_t>() : nullptr;
  a.dbg_why = dbg ? c->why.as<uint8_t>() : nullptr;
  // K4/K5 (regulariser, features) on every rank: they are O(m n_nbr + n_f), identical everywhere, and
  // stay out of the cross-rank reduction (only the point terms are summed over the shards)
  const bool graph_terms = (int64_t)c->m * c->prm.n_nbr + c->nf > 0;
  AsmGraphArgs gA;
  {   // (filled always: the affine model's E_rot terms need it without edges or features)
    gA.nd = node_view(c);
    gA.n_nbr = c->prm.n_nbr;
    gA.nbr = c->nbr.as<int32_t>();
    gA.edge_slot = c->edge_slot.as<int32_t>();
    gA.diag_slot = c->diag_pos.as<int32_t>();
    gA.nf = c->nf;
    gA.fsrc = c->fsrc.as<float>();
    gA.fdst = c->fdst.as<float>();
    gA.fidx = c->fidx.as<int32_t>();
    gA.fw = c->fw.as<float>();
    gA.feat_slot = c->feat_slot.as<int32_t>();
    gA.fr = frame_view(c);
    gA.w_reg = c->prm.w_reg;
    gA.w_corr = c->prm.w_corr;
    gA.acc = acc;
    gA.K = c->K;
    gA.KS = KS;
    gA.pose_cur = a.pose_cur;
    gA.w_rot = c->prm.w_rot;
  }
  // K3a + K3b fused into one kernel (k <= 4 SE(3), no debug outputs; MIS_K3_SPLIT=1 in the
  // environment keeps the two-kernel path for comparison), the K4/K5 items in its extra CTAs
  // (k > 4 fused into the FP32 register-tile SYRK spills ~1.3 KB per thread and measured slower at C5:
  // 39.2 vs 30.1 ms per step of K3, so k > 4 keeps the two kernels)
  const bool fused = !dbg && !joint && !aff && c->K <= 4 && !c->k3_split;
  if (fused) {
    if (a.nchunk > 0 || graph_terms) {
      ProfScope ps(c, P_ACCUM, 1);
      launch_accum_points(KS, a, c->num_sms, c->st, true, graph_terms ? &gA : nullptr);
    }
  } else {
    if (c->n > 0 || graph_terms) {   // K3a + K4/K5 in one launch (affine: K4/K5/E_rot in their own)
      ProfScope ps(c, P_POINTS, 1);
      launch_assoc_points(c->K, a, graph_terms ? &gA : nullptr, c->st);
    }
    if (aff) {   // the affine graph terms include E_rot on every node: always (rank 0)
      ProfScope ps(c, P_GRAPH, 1);
      launch_assemble_graph_aff(gA, c->st);
    }
    if (a.nchunk > 0) {
      ProfScope ps(c, P_ACCUM, 1);
      if (aff) launch_accum_points_aff(c->K, a, c->num_sms, c->st);
      else if (KS > 4 && kChunk <= 128 && umma_k3b_enabled()) launch_accum_points_umma(KS, a, c->num_sms, c->st);
      else launch_accum_points(KS, a, c->num_sms, c->st);
    }
  }
  TRY(c, cudaGetLastError());
  // multi-GPU: the point part of H (upper 6x6 blocks) and b is formed on every rank,
  // all-reduced (36 (m + nup) + 6 m floats) with the point energies, and scattered back as pre-weighted
  // accumulators; the graph terms are every rank's own.  MIS_SHARD_PROTOCOL=1 runs the same kernels on
  // one GPU (without the NCCL call), so the parity tests check the payload path.
  static const bool shard_protocol = getenv("MIS_SHARD_PROTOCOL") != nullptr;
  const bool sharded = (c->world > 1 || shard_protocol) && !c->pattern_affine && !c->pattern_joint &&
                       !(c->prm.flags & MIS_F_LM);
  if (sharded) {
    FinalArgs rp{};
    rp.m = sys_m(c);
    rp.nup = (c->nnzb - sys_m(c)) / 2;
    rp.ulist = c->ulist.as<int2>();
    rp.diag_pos = c->diag_pos.as<int32_t>();
    rp.w_data = c->prm.w_data;
    rp.w_pt = c->prm.w_point;
    rp.acc = acc;
    const size_t nh = 36 * (size_t)(rp.m + rp.nup), nr = 6 * (size_t)rp.m;
    TRY(c, ensure(c, c->shard_buf, (nh + nr) * 4));
    float* HU = c->shard_buf.as<float>();
    launch_shard_partial(rp, HU, HU + nh, c->st);
    if (c->world > 1) {
      if (nccl_allreduce_sum_f32(c, HU, nh + nr) != cudaSuccess) return MIS_E_NCCL;
      double* E = c->energy.as<double>();
      if (nccl_allreduce_sum_f64(c, E + 8, 2 * kEnergyStripes) != cudaSuccess) return MIS_E_NCCL;   // E_data, E_pt
      if (nccl_allreduce_sum_f64(c, E + 8 + 4 * kEnergyStripes, kEnergyStripes) != cudaSuccess) return MIS_E_NCCL;
    }
    launch_shard_scatter(rp, HU, HU + nh, c->st);
    count_launches(2);
  }
  {   // accumulators -> final H (both triangles), b, block-Jacobi inverses
    ProfScope ps(c, P_REDUCE, 1);
    FinalArgs r;
    r.pre_weighted = sharded ? 1 : 0;
    r.nnzb = c->nnzb;
    r.nup = (c->nnzb - sys_m(c)) / 2;
    r.ulist = c->ulist.as<int2>();
    r.m = sys_m(c);
    r.pose_node = joint ? c->m : -1;
    r.pose_cur = joint ? c->posebuf.as<double>() : nullptr;
    r.pose_prior = joint ? c->posebuf.as<double>() + 12 : nullptr;
    r.w_r = c->prm.w_r;
    r.w_p = c->prm.w_p;
    r.rep_pose = rep_pose(c);
    r.w_rot = c->prm.w_rot;
    r.rep_rot = rep_rot(c);
    r.upper_of = c->upper_of.as<int32_t>();
    r.lower_of = c->lower_of.as<int32_t>();
    r.diag_pos = c->diag_pos.as<int32_t>();
    r.w_data = c->prm.w_data;
    r.w_pt = c->prm.w_point;
    r.acc = acc;
    r.Hval = c->Hval.as<float>();
    r.rhs = c->rhs.as<float>();
    r.Minv = c->Minv.as<float>();
    r.lambda = c->prm.lambda;
    r.w_reg = c->prm.w_reg;
    r.w_corr = c->prm.w_corr;
    r.slot = slot;
    r.rep_energy = rep_energy(c);
    r.rep_nassoc = rep_nassoc(c);
    const bool lm = (c->prm.flags & MIS_F_LM) && !dbg;
    r.lm = lm ? reinterpret_cast<const LmDev*>(c->lm.p) : nullptr;
    r.Hval_alt = lm ? c->Hval2.as<float>() : nullptr;
    r.rhs_alt = lm ? c->rhs2.as<float>() : nullptr;
    if (lm) r.Minv = nullptr;   // the damped inverses are built by the solver once it has decided
    if (aff) launch_finalize_aff(r, c->st);
    else launch_finalize(r, c->st);
  }
  c->acc_dirty = false;
  TRY(c, cudaGetLastError());
  return MIS_OK;
}

static SolveArgs solve_args(Ctx* c, int it, bool update, int pcg_iters) {
  SolveArgs s;
  s.m = sys_m(c);
  s.K = c->K;
  s.pose_node = c->pattern_joint ? c->m : -1;   // NEXT-2
  s.pose = c->pattern_joint ? c->posebuf.as<double>() : nullptr;
  s.block = sys_b(c);   // NEXT-4: 12 x 12 blocks
  s.nnzb = c->nnzb;
  s.row_ptr = c->row_ptr.as<int32_t>();
  s.col = c->col.as<int32_t>();
  s.upper_of = c->upper_of.as<int32_t>();
  s.diag_pos = c->diag_pos.as<int32_t>();
  s.acc = acc_view(c);
  s.w_data = c->prm.w_data;
  s.w_pt = c->prm.w_point;
  s.lambda = c->prm.lambda;
  s.pcg_iters = pcg_iters;
  s.Hval = c->Hval.as<float>();
  s.rhs = c->rhs.as<float>();
  s.Minv = c->Minv.as<float>();
  s.x = c->x.as<float>(); s.r = c->r.as<float>(); s.z = c->z.as<float>(); s.p = c->p.as<float>(); s.Ap = c->Ap.as<float>();
  s.pv = c->pvec.as<float>();
  s.dots = c->dots.as<double>();
  s.nd = node_view(c);
  s.do_update = update ? 1 : 0;
  s.gn_it = it;
  s.rep_res = rep_res(c);
  s.numeric_flag = numeric_flag(c);
  const bool lm_flag = (c->prm.flags & MIS_F_LM) != 0;
  // LM runs in the register-resident pipelined cluster kernel or in the pipelined grid kernel
  const bool cl_lm_ok = 6 * c->cl_max_rows <= 512 && !(c->prm.flags & MIS_F_STANDARD_PCG);
  const bool cl = c->cl_size > 0 && c->cluster_ok && !(c->prm.flags & MIS_F_GRID_SOLVER) && (!lm_flag || cl_lm_ok);
  s.cluster_size = cl ? c->cl_size : 0;
  s.part = c->part.as<int32_t>();
  s.max_rows = c->cl_max_rows;
  s.max_nnz = c->cl_max_nnz;
  s.smem_bytes = c->cl_smem;
  s.write_global = update ? 0 : 1;
  s.pipelined = (c->prm.flags & MIS_F_STANDARD_PCG) && !lm_flag ? 0 : 1;
  s.minv_ready = 1;   // built by the finalisation (after the all-reduce when sharded)
  s.tstamp = c->tstamp.as<unsigned long long>();
  s.pptr = c->pcg_pptr.as<int32_t>();
  s.pc = c->pcg_pc.as<int32_t>();
  s.push = c->pcg_push.as<int32_t>();
  s.npush = c->pcg_npush.as<int32_t>();
  const bool lm = (c->prm.flags & MIS_F_LM) && update;
  s.lm = lm ? reinterpret_cast<LmDev*>(c->lm.p) : nullptr;
  s.lm_mu0 = 1e-3f;
  s.Hval_alt = lm ? c->Hval2.as<float>() : nullptr;
  s.rhs_alt = lm ? c->rhs2.as<float>() : nullptr;
  s.Rt_acc = lm ? c->Rt_acc.as<double>() : nullptr;
  s.rep_energy = rep_energy(c);
  s.rep_flags = rep_nassoc(c) + MIS_MAX_GN + 1;   // the report's n_guard row
  return s;
}

// cluster launch first; fall back to the grid-wide kernel if the device refuses it
static cudaError_t run_solve(Ctx* c, const SolveArgs& s) {
  cudaError_t e = launch_solve(s, c->num_sms, c->st);
  if (e != cudaSuccess && s.cluster_size > 0) {
    cudaGetLastError();
    c->cluster_ok = false;
    c->solver_note = std::string("cluster PCG unavailable (") + cudaGetErrorString(e) + "), using the grid kernel";
    SolveArgs g = s;
    g.cluster_size = 0;
    e = launch_solve(g, c->num_sms, c->st);
    c->last_solver = 0;
  } else {
    c->last_solver = s.cluster_size;
  }
  return e;
}

// NEXT-2: posebuf = [current pose | prior]; the prior is the frame's input pose, the current one
// `cur` (fp64, host) or the prior.  One tiny launch (by-value arguments, no host buffer to keep).
struct Pose24 { double v[24]; };
__global__ void k_pose_init(Pose24 p, double* out) {
  if (threadIdx.x < 24) out[threadIdx.x] = p.v[threadIdx.x];
}
static cudaError_t pose_init(Ctx* c, const double* cur) {
  cudaError_t e = ensure(c, c->posebuf, 24 * 8);
  if (e != cudaSuccess) return e;
  Pose24 p;
  for (int i = 0; i < 12; ++i) {
    p.v[12 + i] = (double)c->pose[i];
    p.v[i] = cur ? cur[i] : (double)c->pose[i];
  }
  launch_pdl(k_pose_init, dim3(1), dim3(32), 0, c->st, p, c->posebuf.as<double>());
  count_launches(1);
  c->pose_valid = true;
  return cudaGetLastError();
}

static mis_status prepare(Ctx* c) {
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph (mis_set_graph)");
  if (!c->have_frame) return fail(c, MIS_E_STATE, "no frame (mis_set_frame / depth)");
  c->joint = (c->prm.flags & MIS_F_JOINT_POSE) != 0;
  if (c->joint && c->world > 1) return fail(c, MIS_E_ARG, "MIS_F_JOINT_POSE: single GPU only");
  if (c->joint != c->pattern_joint) c->pattern_valid = false;   // the pose row / column come or go
  c->affine = (c->prm.flags & MIS_F_AFFINE) != 0;
  if (c->affine && c->world > 1) return fail(c, MIS_E_ARG, "MIS_F_AFFINE: single GPU only");
  if (c->affine != c->pattern_affine) c->pattern_valid = false;   // 12 x 12 blocks come or go
  if (c->dirty) TRY(c, run_build_order(c));
  if (!c->pattern_valid) {
    {
      ProfScope ps(c, P_PATTERN, 0);   // build_pattern counts its own launches
      TRY(c, build_pattern(c));
    }
    if (c->graph_check) {   // deferred validation of a device-memory mis_set_graph
      c->graph_check = false;
      if (c->graph_flags) {
        c->have_graph = false;
        c->pattern_valid = false;
        return fail(c, MIS_E_ARG, graph_flag_message(c->graph_flags));
      }
    }
  }
  TRY(c, flush_frame(c));   // if the pattern was still valid (no readback to hide it behind)
  if (c->nf > 0 && !c->fidx.p) return fail(c, MIS_E_STATE, "features not set");
  if (c->joint && !c->pose_valid) TRY(c, pose_init(c, nullptr));
  return MIS_OK;
}

static mis_status fill_report(Ctx* c, mis_report* rep, int iters) {
  memset(rep, 0, sizeof(*rep));
  double blk[kRepBytes / 8];
  TRY(c, cudaMemcpyAsync(blk, c->rep.p, kRepBytes, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  const double* e = blk;
  const double* na = blk + kRepN;
  memcpy(rep->pcg_rel_res, blk + kRepR, sizeof(rep->pcg_rel_res));
  int flag = 0;
  memcpy(&flag, blk + kRepF, 4);
  rep->iters = iters;
  rep->status = flag ? MIS_E_NUMERIC : MIS_OK;
  for (int i = 0; i <= MIS_MAX_GN; ++i) {
    for (int q = 0; q < 5; ++q) rep->energy[i][q] = e[5 * i + q];
    rep->n_assoc[i] = (int64_t)llround(na[i]);
    rep->n_guard[i] = (int64_t)llround(na[MIS_MAX_GN + 1 + i]);
    rep->energy_pose[i][0] = blk[kRepP + 2 * i];
    rep->energy_pose[i][1] = blk[kRepP + 2 * i + 1];
    rep->energy_rot[i] = blk[kRepO + i];
  }
  rep->nnzb = c->nnzb;
  rep->n_segments = c->nseg;
  rep->solver_cluster = c->last_solver;
  return flag ? MIS_E_NUMERIC : MIS_OK;
}

mis_status mis_register(mis_ctx* c, mis_mem mem, const float* depth_mm, const mis_intrinsics* intr,
                        const float pose[12], int32_t n_feat, const float* feat_src, const float* feat_dst,
                        mis_report* rep) {
  if (!c) return MIS_E_ARG;
  cudaSetDevice(c->device);
  mis_status s;
  // the report block is zeroed first: enqueued while the device is still busy with earlier work,
  // it is not a host-bound step between the pattern and the first assembly
  TRY(c, cudaMemsetAsync(c->rep.p, 0, kRepBytes, c->st));
  if (depth_mm) {
    if ((s = set_frame_impl(c, mem, depth_mm, intr, pose, true)) != MIS_OK) return s;
  } else if (pose) {
    memcpy(c->pose, pose, 48);
    c->pose_valid = false;
  }
  if (n_feat >= 0)
    if ((s = mis_set_features(c, mem, n_feat, feat_src, feat_dst)) != MIS_OK) return s;
  if ((c->prm.flags & MIS_F_JOINT_POSE) && c->pose_valid) TRY(c, pose_init(c, nullptr));   // start at the prior
  if ((s = prepare(c)) != MIS_OK) return s;
  const int G = c->prm.gn_iters;
  const bool lm = c->prm.flags & MIS_F_LM;
  if (lm) {   // the LM decisions live in the register-resident pipelined cluster PCG and in the
              // pipelined grid PCG (solve_args picks one of them)
    if (c->world != 1) return fail(c, MIS_E_ARG, "MIS_F_LM: single GPU only");
    const bool fresh = !c->lm.p;
    const size_t B = (size_t)sys_b(c), mu = (size_t)sys_m(c);
    TRY(c, ensure(c, c->lm, 64));
    if (fresh) TRY(c, cudaMemsetAsync(c->lm.p, 0, 64, c->st));
    TRY(c, ensure(c, c->Hval2, (size_t)c->nnzb * B * B * 4));
    TRY(c, ensure(c, c->rhs2, mu * B * 4));
    TRY(c, ensure(c, c->Rt_acc, mu * 96));   // the kept node states (+ the pose, NEXT-2)
  }
  for (int it = 0; it < G; ++it) {
    if ((s = assemble(c, false, it)) != MIS_OK) return s;
    ProfScope ps(c, P_SOLVE, 1);
    const SolveArgs sa = solve_args(c, it, true, c->prm.pcg_iters);
    TRY(c, run_solve(c, sa));
  }
  if ((c->prm.flags & MIS_F_FINAL_ENERGY) || lm)
    if ((s = assemble(c, false, G)) != MIS_OK) return s;
  if (lm) {   // the last trial is kept only if accepted
    ProfScope ps(c, P_SOLVE, 1);
    launch_lm_finish(c->m, G, reinterpret_cast<const LmDev*>(c->lm.p), rep_energy(c), rep_nassoc(c) + MIS_MAX_GN + 1,
                     c->Rt64.as<double>(), c->Rt_acc.as<double>(), c->node32.as<float>(), c->st,
                     c->pattern_joint ? c->posebuf.as<double>() : nullptr);
  }
  TRY(c, cudaGetLastError());
  if (rep) return fill_report(c, rep, G);
  return MIS_OK;
}

mis_status mis_get_nodes(mis_ctx* c, mis_mem mem, float* out) {
  if (!c || !out) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  cudaSetDevice(c->device);
  TRY(c, ensure(c, c->stage, (size_t)c->m * 48));
  ProfScope ps(c, P_IO, 1);
  k_get_nodes<<<nb(c->m), 256, 0, c->st>>>(c->m, c->node32.as<float>(), c->stage.as<float>());
  TRY(c, cudaMemcpyAsync(out, c->stage.p, (size_t)c->m * 48, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_get_nodes_f64(mis_ctx* c, double* out) {
  if (!c || !out) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  cudaSetDevice(c->device);
  TRY(c, cudaMemcpyAsync(out, c->Rt64.p, (size_t)c->m * 96, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_get_pose(mis_ctx* c, double pose[12]) {
  if (!c || !pose) return MIS_E_ARG;
  cudaSetDevice(c->device);
  if (c->pose_valid) {
    TRY(c, cudaMemcpyAsync(pose, c->posebuf.p, 96, cudaMemcpyDeviceToHost, c->st));
    TRY(c, cudaStreamSynchronize(c->st));
  } else {
    for (int i = 0; i < 12; ++i) pose[i] = (double)c->pose[i];
  }
  return MIS_OK;
}

mis_status mis_dbg_set_pose(mis_ctx* c, const double pose[12]) {
  if (!c || !pose) return MIS_E_ARG;
  if (!c->have_frame) return fail(c, MIS_E_STATE, "no frame");
  cudaSetDevice(c->device);
  TRY(c, pose_init(c, pose));
  return MIS_OK;
}

mis_status mis_get_graph(mis_ctx* c, mis_mem mem, float* node_pos) {
  if (!c || !node_pos) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  cudaSetDevice(c->device);
  TRY(c, cudaMemcpyAsync(node_pos, c->g.p, (size_t)c->m * 12, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_get_nbr(mis_ctx* c, mis_mem mem, int32_t* node_nbr) {
  if (!c || !node_nbr) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  if (c->prm.n_nbr == 0) return MIS_OK;
  cudaSetDevice(c->device);
  TRY(c, cudaMemcpyAsync(node_nbr, c->nbr.p, (size_t)c->m * c->prm.n_nbr * 4, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_dbg_set_nodes(mis_ctx* c, mis_mem mem, const float* Rt) {
  if (!c || !Rt) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  cudaSetDevice(c->device);
  TRY(c, ensure(c, c->stage, (size_t)c->m * 48));
  TRY(c, cudaMemcpyAsync(c->stage.p, Rt, (size_t)c->m * 48, kind_in(mem), c->st));
  ProfScope ps(c, P_IO, 1);
  k_set_nodes<<<nb(c->m), 256, 0, c->st>>>(c->m, c->stage.as<float>(), c->Rt64.as<double>(), c->node32.as<float>());
  TRY(c, cudaGetLastError());
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_dbg_frame(mis_ctx* c, mis_mem mem, float* nmap) {
  if (!c || !nmap) return MIS_E_ARG;
  if (!c->have_frame) return fail(c, MIS_E_STATE, "no frame");
  TRY(c, flush_frame(c));
  cudaSetDevice(c->device);
  TRY(c, cudaMemcpyAsync(nmap, c->nmap.p, (size_t)c->W * c->H * 16, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_dbg_associate(mis_ctx* c, mis_mem mem, int32_t* pix, uint8_t* why) {
  if (!c || !pix || !why) return MIS_E_ARG;
  cudaSetDevice(c->device);
  mis_status s;
  if ((s = prepare(c)) != MIS_OK) return s;
  TRY(c, ensure(c, c->pix, c->cap * 4));
  TRY(c, ensure(c, c->why, c->cap));
  if ((s = assemble(c, true, -1)) != MIS_OK) return s;
  TRY(c, cudaMemcpyAsync(pix, c->pix.p, c->n * 4, kind_out(mem), c->st));
  TRY(c, cudaMemcpyAsync(why, c->why.p, c->n, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_dbg_system(mis_ctx* c, int32_t* row_ptr, int32_t* col, float* val, float* rhs, double energy[5],
                          int64_t* nnzb) {
  if (!c || !nnzb) return MIS_E_ARG;
  cudaSetDevice(c->device);
  mis_status s;
  if ((s = prepare(c)) != MIS_OK) return s;
  *nnzb = c->nnzb;
  if (!val) return MIS_OK;
  if ((s = assemble(c, false, 0)) != MIS_OK) return s;
  if (row_ptr) TRY(c, cudaMemcpyAsync(row_ptr, c->row_ptr.p, (size_t)(sys_m(c) + 1) * 4, cudaMemcpyDeviceToHost, c->st));
  if (col) TRY(c, cudaMemcpyAsync(col, c->col.p, (size_t)c->nnzb * 4, cudaMemcpyDeviceToHost, c->st));
  const size_t B = (size_t)sys_b(c);
  TRY(c, cudaMemcpyAsync(val, c->Hval.p, (size_t)c->nnzb * B * B * 4, cudaMemcpyDeviceToHost, c->st));
  if (rhs) TRY(c, cudaMemcpyAsync(rhs, c->rhs.p, (size_t)sys_m(c) * B * 4, cudaMemcpyDeviceToHost, c->st));
  if (energy) TRY(c, cudaMemcpyAsync(energy, rep_energy(c), 40, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_warp(mis_ctx* c, mis_mem mem, float* xyz_cam, float* nrm_cam) {
  if (!c) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  cudaSetDevice(c->device);
  if (c->dirty) TRY(c, run_build_order(c));
  float* xc = nullptr;
  float* nc = nullptr;
  if (xyz_cam || nrm_cam) {
    TRY(c, ensure(c, c->stage, (size_t)c->n * 24 + 16));
    xc = c->stage.as<float>();
    nc = xc + 3 * c->n;
  }
  {
    ProfScope ps(c, P_WARP, (c->n > 0) + 1);
    launch_warp_model(c->K, model_view(c), node_view(c), frame_view(c), xyz_cam ? xc : nullptr,
                      nrm_cam ? nc : nullptr, c->st, (c->prm.flags & MIS_F_AFFINE) != 0);
    launch_advance_nodes(node_view(c), c->g.as<float>(), c->st);
  }
  TRY(c, cudaGetLastError());
  if (xyz_cam) TRY(c, cudaMemcpyAsync(xyz_cam, xc, (size_t)c->n * 12, kind_out(mem), c->st));
  if (nrm_cam) TRY(c, cudaMemcpyAsync(nrm_cam, nc, (size_t)c->n * 12, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST && (xyz_cam || nrm_cam)) TRY(c, cudaStreamSynchronize(c->st));
  c->pattern_valid = false;   // feature skinning refers to the old node positions
  return MIS_OK;
}

static FuseArgs fuse_args(Ctx* c, const float* rgb, int32_t frame) {
  FuseArgs a;
  a.md = model_view(c);
  a.fr = frame_view(c);
  a.tz = fmin((double)c->prm.tau_z_mm, (double)c->prm.trunc_mm);
  a.key_scale = 4294967295.0 / a.tz;   // dz * key_scale < 2^32 - 1 for dz < tz
  a.cos_delta = cos(c->prm.delta_deg * M_PI / 180.0);
  a.omega_max = c->prm.omega_max;
  a.rgb_obs = rgb;
  a.frame_index = frame;
  a.pixkey = c->pixkey.as<unsigned long long>();
  a.pix = c->pix.as<int32_t>();
  a.why = c->why.as<uint8_t>();
  a.rank_tag = c->world > 1 ? ((uint32_t)c->rank << 27) : 0u;
  const int nbk = lift_blocks(c->W, c->H);   // lift counts: [nbk counts | nbk + 1 offsets | u64 n_reg]
  a.fits = nullptr;
  a.n_reg = c->lift_counts.bytes >= (size_t)(2 * nbk + 4) * 4
                ? reinterpret_cast<unsigned long long*>(c->lift_counts.as<int32_t>() + 2 * nbk + 2)
                : nullptr;
  return a;
}

static mis_status fuse_register(Ctx* c, const float* rgb, int32_t frame) {
  const size_t px = (size_t)c->W * c->H;
  TRY(c, ensure(c, c->lift_counts, (size_t)(2 * lift_blocks(c->W, c->H) + 4) * 4));
  if (c->pixkey.bytes < px * 8) c->pixkey_clean = false;
  TRY(c, ensure(c, c->pixkey, px * 8));
  TRY(c, ensure(c, c->pix, c->cap * 4));
  TRY(c, ensure(c, c->why, c->cap));
  if (!c->pixkey_clean) TRY(c, cudaMemsetAsync(c->pixkey.p, 0xff, px * 8, c->st));   // else reset by K12
  c->pixkey_clean = false;
  ProfScope ps(c, P_FREG, c->n > 0 ? 1 : 0);
  launch_fuse_register(fuse_args(c, rgb, frame), c->st);
  TRY(c, cudaGetLastError());
  if (c->world > 1) {   // the exclusive winner per pixel over all ranks' shards (keys carry the rank)
    if (c->n >= (1 << 27) || c->world > 32) return fail(c, MIS_E_ARG, "sharded fusion: > 2^27 points or > 32 ranks");
    if (nccl_ret(c, nccl().AllReduce(c->pixkey.p, c->pixkey.p, px, kNcclUint64, kNcclMin, c->nccl_comm, c->st)) !=
        cudaSuccess)
      return MIS_E_NCCL;
  }
  return MIS_OK;
}

mis_status mis_dbg_fuse_register(mis_ctx* c, int64_t* owner, uint8_t* why) {
  if (!c || !owner) return MIS_E_ARG;
  if (!c->have_graph || !c->have_frame) return fail(c, MIS_E_STATE, "no graph or frame");
  TRY(c, flush_frame(c));
  cudaSetDevice(c->device);
  if (c->dirty) TRY(c, run_build_order(c));
  mis_status s;
  if ((s = fuse_register(c, nullptr, 0)) != MIS_OK) return s;
  const size_t px = (size_t)c->W * c->H;
  std::vector<unsigned long long> k(px);
  TRY(c, cudaMemcpyAsync(k.data(), c->pixkey.p, px * 8, cudaMemcpyDeviceToHost, c->st));
  if (why) TRY(c, cudaMemcpyAsync(why, c->why.p, c->n, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  for (size_t p = 0; p < px; ++p) owner[p] = (k[p] == ~0ull) ? -1 : (int64_t)(k[p] & 0xffffffffull);
  return MIS_OK;
}

// the host colour's upload on the copy stream, after the previous fusion has read the buffer
static cudaError_t issue_colour_copy(Ctx* c, const float* rgb) {
  const size_t px = (size_t)c->W * c->H;
  cudaError_t e;
  if ((e = ensure(c, c->rgb_obs, px * 12)) != cudaSuccess) return e;
  if ((e = copy_stream(c)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(c->st_copy, c->ev_rgb_free, 0)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(c->rgb_obs.p, rgb, px * 12, cudaMemcpyHostToDevice, c->st_copy)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(c->ev_rgb_ready, c->st_copy)) != cudaSuccess) return e;
  c->rgb_staged = rgb;
  return cudaSuccess;
}

mis_status mis_stage_colour(mis_ctx* c, const float* rgb) {
  if (!c) return MIS_E_ARG;
  if (!rgb) return fail(c, MIS_E_ARG, "stage_colour: rgb is NULL");
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, rgb) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
    return fail(c, MIS_E_ARG, "stage_colour: a device pointer (device colours are read in place)");
  cudaGetLastError();   // (a pageable host pointer may leave an error on older drivers)
  if ((size_t)c->W * c->H == 0) return fail(c, MIS_E_ARG, "stage_colour: no frame size known yet");
  // issued by the next frame upload right behind its depth (the registration needs the depth first),
  // or by mis_fuse if no frame comes in between
  c->rgb_pending = rgb;
  c->rgb_staged = nullptr;
  return MIS_OK;
}

mis_status mis_fuse(mis_ctx* c, mis_mem mem, const float* rgb, int32_t frame_index, int64_t* n_out, int64_t stats[4]) {
  if (!c || !n_out) return MIS_E_ARG;
  if (!c->have_graph || !c->have_frame) return fail(c, MIS_E_STATE, "no graph or frame");
  TRY(c, flush_frame(c));
  cudaSetDevice(c->device);
  if (c->dirty) TRY(c, run_build_order(c));
  const size_t px = (size_t)c->W * c->H;
  const float* rgb_dev = rgb;   // device colours are read in place by K11 / K12 (stream order)
  if (rgb && mem == MIS_MEM_HOST) {
    // on the copy stream, after the previous fusion read the buffer: the transfer overlaps the
    // registration of the model points (K10); the colours are first read by K11.  Already issued
    // by mis_stage_colour for this pointer: nothing to do
    if (c->rgb_staged != rgb || c->rgb_obs.bytes < px * 12) TRY(c, issue_colour_copy(c, rgb));
    rgb_dev = c->rgb_obs.as<float>();
  }
  c->rgb_staged = nullptr;
  c->rgb_pending = nullptr;
  mis_status s;
  if ((s = fuse_register(c, rgb_dev, frame_index)) != MIS_OK) return s;
  const bool rgb_staged = rgb && mem == MIS_MEM_HOST;
  if (rgb_staged) TRY(c, cudaStreamWaitEvent(c->st, c->ev_rgb_ready, 0));
  FuseArgs a = fuse_args(c, rgb_dev, frame_index);
  const int nbk = lift_blocks(c->W, c->H);
  int32_t* counts = c->lift_counts.as<int32_t>();
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(counts + 2 * nbk + 2);   // zeroed by K10
  if (c->n == 0) TRY(c, cudaMemsetAsync(cnt, 0, 8, c->st));   // (K10 not launched)
  // lift count + offsets first: the scan decides on the device whether the lift fits the
  // capacity, and K11 (Eq. 12-15) and the lift write apply nothing when it does not, so
  // MIS_E_CAPACITY leaves the model unchanged.  One host readback (the API returns the new model
  // size); the writes and K2 of the new points run behind it (overlapping the host's wait)
  const int64_t base = c->n;
  const int do_lift = (c->world == 1 || c->rank == 0) ? 1 : 0;   // sharded model: rank 0 owns the lifted points
  long long* ids_dev = c->ids_dev.as<long long>();
  {
    ProfScope ps(c, P_LIFT, 2);
    launch_lift_count(a, counts, nbk, ids_dev, cnt, do_lift, base, c->cap, c->st);
  }
  a.fits = ids_dev + 3;
  {
    ProfScope ps(c, P_FAPPLY, c->n > 0 ? 1 : 0);
    launch_fuse_apply(a, c->st);
  }
  // one readback of [lifted total, registered pixels (u64)] (pinned, asynchronous).  Lifting
  // ranks queue the lifted points' writes (+ pixel-key reset) and their K2 behind it, so they
  // run while the host waits for the count; they write only below the capacity, and points
  // past an exceeded capacity are ignored (MIS_E_CAPACITY, model size unchanged)
  TRY(c, cudaMemcpyAsync(c->hpin, counts + 2 * nbk + 1, 12, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaEventRecord(c->rb_ev, c->st));
  if (do_lift) {
    ProfScope ps(c, P_LIFT, 2);
    ModelView md = model_view(c);
    TRY(c, ensure(c, c->lift_pos, px * 4));
    launch_lift_write(a, counts + nbk + 1, nbk, base, c->cap, ids_dev, c->lift_pos.as<int32_t>(), c->st);   // + key reset
    launch_skin_lifted(c->K, c->W, c->H, c->lift_pos.as<int32_t>(), md, c->g.as<float>(), c->m, c->st);
  } else {
    TRY(c, cudaMemsetAsync(c->pixkey.p, 0xff, px * 8, c->st));
  }
  TRY(c, cudaEventSynchronize(c->rb_ev));
  int32_t hb[3];
  memcpy(hb, c->hpin, 12);
  const int32_t n_lift = hb[0];
  unsigned long long n_reg = 0;
  memcpy(&n_reg, hb + 1, 8);
  if (rgb_staged) TRY(c, cudaEventRecord(c->ev_rgb_free, c->st));   // K11 / K12 have read the staged colours
  c->pixkey_clean = true;
  if (c->n + n_lift > c->cap) {
    *n_out = c->n;
    return fail(c, MIS_E_CAPACITY, "mis_fuse: lifted points exceed the model capacity (model unchanged)");
  }
  if (n_lift > 0) c->dirty = true;
  TRY(c, cudaGetLastError());
  c->n += n_lift;
  *n_out = c->n;
  if (stats) {
    stats[0] = (int64_t)n_reg;
    stats[1] = n_lift;
    stats[2] = (int64_t)n_reg + n_lift;
    stats[3] = c->n;
  }
  c->pattern_valid = false;
  return MIS_OK;
}

mis_status mis_filter(mis_ctx* c, float grid_mm, int32_t frame_index, int32_t tau_time, float tau_weight,
                      int64_t* n_out, int64_t stats[4]) {
  if (!c || !n_out || !(grid_mm > 0.f) || tau_time < 0 || !(tau_weight == tau_weight)) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  if (c->m < c->K + 1) return fail(c, MIS_E_ARG, "mis_filter: re-skinning needs m >= k+1");
  if (c->world > 1)   // a box may hold points of several ranks' shards: not merged across ranks (yet)
    return fail(c, MIS_E_ARG, "mis_filter: single-GPU only (world > 1 would filter per-rank partial boxes)");
  TRY(c, flush_frame(c));
  cudaSetDevice(c->device);
  TRY(c, ensure(c, c->finfo, 64));
  const int64_t n0 = c->n;
  if (n0 == 0) {
    *n_out = 0;
    if (stats) stats[0] = stats[1] = stats[2] = stats[3] = 0;
    return MIS_OK;
  }
  // K14a + readback: validate the box coordinates before the model is touched, size the sort key
  int32_t range[7];
  {
    ProfScope ps(c, P_FILTER, 1);
    TRY(c, run_filter_range(c, grid_mm, range));
  }
  int sh_x = 0, sh_y = 0;
  const int bits = range[6] ? -1 : filter_key_bits(range, &sh_x, &sh_y);
  if (bits < 0) {
    *n_out = n0;
    return fail(c, MIS_E_ARG, "mis_filter: a position is not finite or the boxes span more than 63 key bits");
  }
  {
    ProfScope ps(c, P_FILTER, 3);
    TRY(c, run_filter(c, grid_mm, range, sh_x, sh_y, bits, frame_index, tau_time, tau_weight));
  }
  TRY(c, cudaMemcpyAsync(c->hpin, c->finfo.p, 32, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  int64_t h[4];
  memcpy(h, c->hpin, 32);
  c->n = h[0];
  {
    ProfScope ps(c, P_FILTER, h[3] > 0 ? 2 : 0);
    TRY(c, run_filter_skin(c, h[3]));
  }
  c->dirty = true;
  c->pattern_valid = false;
  *n_out = c->n;
  if (stats) {
    stats[0] = h[1];
    stats[1] = n0 - h[0];
    stats[2] = h[2];
    stats[3] = c->n;
  }
  return MIS_OK;
}

mis_status mis_regenerate_nodes(mis_ctx* c, float node_grid_mm, int32_t* m_out) {
  if (!c || !m_out || !(node_grid_mm > 0.f) || !std::isfinite(node_grid_mm)) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  if (c->world > 1)   // the cells of a sharded model span ranks: not reduced across ranks (yet)
    return fail(c, MIS_E_ARG, "mis_regenerate_nodes: single-GPU only");
  if (c->prm.n_nbr > 16) return fail(c, MIS_E_ARG, "mis_regenerate_nodes: n_nbr <= 16");
  if (c->n <= c->K) return fail(c, MIS_E_ARG, "mis_regenerate_nodes: fewer than k+1 points");
  TRY(c, flush_frame(c));
  cudaSetDevice(c->device);
  TRY(c, ensure(c, c->finfo, 64));
  int32_t range[7];
  int64_t m = 0;
  {
    ProfScope ps(c, P_REGEN, 1);
    TRY(c, run_filter_range(c, node_grid_mm, range));
  }
  int sh_x = 0, sh_y = 0;
  const int bits = range[6] ? -1 : filter_key_bits(range, &sh_x, &sh_y);
  if (bits < 0)
    return fail(c, MIS_E_ARG, "mis_regenerate_nodes: a position is not finite or the cells span more than 63 key bits");
  {
    ProfScope ps(c, P_REGEN, 4);
    TRY(c, run_regen_centroids(c, node_grid_mm, range, sh_x, sh_y, bits, &m));
  }
  if (m < c->K + 1 || m > 0x7fffffff)
    return fail(c, MIS_E_ARG, "mis_regenerate_nodes: fewer than k+1 occupied cells (graph unchanged)");
  {
    ProfScope ps(c, P_REGEN, c->prm.n_nbr > 0 ? 1 : 0);
    TRY(c, run_regen_knn(c, (int)m, c->prm.n_nbr));
  }
  // the new graph through the device-input path of mis_set_graph: identity transforms, Eq. 2
  // skinning of every point against the new nodes (K2), K13 regrouping
  mis_status s = set_graph_impl(c, (int32_t)m, MIS_MEM_DEVICE, c->fl_xyz.as<float>(), c->rg_nbr.as<int32_t>(), nullptr,
                                nullptr, c->vals2.as<uint32_t>());   // points in node-cell order (K15's sort)
  if (s != MIS_OK) return s;
  *m_out = (int32_t)m;
  return MIS_OK;
}

mis_status mis_get_model(mis_ctx* c, mis_mem mem, float* xyz, float* nrm, float* rgb, float* weight, int32_t* stamp,
                         int64_t* ids, int32_t* knn_idx, float* knn_w, int64_t* n_host) {
  if (!c) return MIS_E_ARG;
  if (!c->have_model) return fail(c, MIS_E_STATE, "no model");
  cudaSetDevice(c->device);
  const int64_t n = c->n;
  if (n_host) *n_host = n;
  if (n == 0) return MIS_OK;
  ModelView md = model_view(c);
  TRY(c, ensure(c, c->stage, (size_t)n * 8 * MIS_MAX_K + 64));
  ProfScope ps(c, P_IO, (xyz != nullptr) + (nrm != nullptr) + (rgb != nullptr) + (knn_idx || knn_w));
  float* st = c->stage.as<float>();
  if (xyz) {
    k_interleave3<<<nb(n), 256, 0, c->st>>>(n, md.px, md.py, md.pz, st);
    TRY(c, cudaMemcpyAsync(xyz, st, n * 12, kind_out(mem), c->st));
    if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  }
  if (nrm) {
    k_interleave3<<<nb(n), 256, 0, c->st>>>(n, md.nx, md.ny, md.nz, st);
    TRY(c, cudaMemcpyAsync(nrm, st, n * 12, kind_out(mem), c->st));
    if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  }
  if (rgb) {
    k_interleave3<<<nb(n), 256, 0, c->st>>>(n, md.cr, md.cg, md.cb, st);
    TRY(c, cudaMemcpyAsync(rgb, st, n * 12, kind_out(mem), c->st));
    if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  }
  if (weight) TRY(c, cudaMemcpyAsync(weight, md.w, n * 4, kind_out(mem), c->st));
  if (stamp) TRY(c, cudaMemcpyAsync(stamp, md.stamp, n * 4, kind_out(mem), c->st));
  if (ids) TRY(c, cudaMemcpyAsync(ids, md.ids, n * 8, kind_out(mem), c->st));
  if (knn_idx || knn_w) {
    if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
    int32_t* si = reinterpret_cast<int32_t*>(st);
    float* sw = reinterpret_cast<float*>(si + n * c->K);
    k_to_point_major<<<nb(n), 256, 0, c->st>>>(n, c->K, c->cap, md.kidx, md.kw, si, sw);
    if (knn_idx) TRY(c, cudaMemcpyAsync(knn_idx, si, n * c->K * 4, kind_out(mem), c->st));
    if (knn_w) TRY(c, cudaMemcpyAsync(knn_w, sw, n * c->K * 4, kind_out(mem), c->st));
  }
  TRY(c, cudaGetLastError());
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

mis_status mis_skin(mis_ctx* c, mis_mem mem, int64_t nq, const float* pts, int32_t* idx, float* w) {
  if (!c || nq < 0 || (nq > 0 && (!pts || !idx || !w))) return MIS_E_ARG;
  if (!c->have_graph) return fail(c, MIS_E_STATE, "no graph");
  if (c->m < c->K + 1) return fail(c, MIS_E_ARG, "skinning needs m >= k+1");
  if (nq == 0) return MIS_OK;
  cudaSetDevice(c->device);
  const int K = c->K;
  TRY(c, ensure(c, c->stage, (size_t)nq * (12 + 16 * K) + 64));
  float* sp = c->stage.as<float>();
  int32_t* si = reinterpret_cast<int32_t*>(sp + 3 * nq);
  float* sw = reinterpret_cast<float*>(si + nq * K);
  int32_t* pi = reinterpret_cast<int32_t*>(sw + nq * K);
  float* pw = reinterpret_cast<float*>(pi + nq * K);
  TRY(c, cudaMemcpyAsync(sp, pts, nq * 12, kind_in(mem), c->st));
  ProfScope ps(c, P_SKIN, 2);
  TRY(c, skin(c, nq, sp, sp + 1, sp + 2, 3, si, sw, nq));
  k_to_point_major<<<nb(nq), 256, 0, c->st>>>(nq, K, nq, si, sw, pi, pw);
  TRY(c, cudaGetLastError());
  TRY(c, cudaMemcpyAsync(idx, pi, nq * K * 4, kind_out(mem), c->st));
  TRY(c, cudaMemcpyAsync(w, pw, nq * K * 4, kind_out(mem), c->st));
  if (mem == MIS_MEM_HOST) TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

const char* mis_prof_name(int cat) {
  static const char* names[MIS_PROF_NCAT] = {"frame_prep", "skin", "sort_order", "pattern", "assoc_points",
                                             "assemble_graph", "solve", "warp_model", "fuse_register", "fuse_apply",
                                             "lift", "io", "finalize", "accum_points", "filter",
                                             "regenerate"};
  return (cat >= 0 && cat < MIS_PROF_NCAT) ? names[cat] : "?";
}

mis_status mis_prof_enable(mis_ctx* c, int on) {
  if (!c) return MIS_E_ARG;
  c->prof = on != 0;
  c->prof_light = on == 2;
  return MIS_OK;
}

mis_status mis_prof_read(mis_ctx* c, double* ms, int64_t* launches, int reset) {
  if (!c) return MIS_E_ARG;
  cudaSetDevice(c->device);
  prof_collect(c);
  for (int i = 0; i < MIS_PROF_NCAT; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_n[i];
    if (reset) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
  }
  return MIS_OK;
}

int64_t mis_launch_count(void) { return g_launches.load(); }

mis_status mis_dbg_solver_phases(mis_ctx* c, uint64_t* out128) {
  if (!c || !out128) return MIS_E_ARG;
  cudaSetDevice(c->device);
  TRY(c, cudaMemcpyAsync(out128, c->tstamp.p, 2048, cudaMemcpyDeviceToHost, c->st));
  TRY(c, cudaStreamSynchronize(c->st));
  return MIS_OK;
}

}  // extern "C"
