// filter.cu -- NEXT-1: Alg. 3 point filtering with the grid-box downsampling of P:597,
// readings A30-A34.  Per frame, after mis_fuse:
//
//   K14a k_cell_range    box coordinates (kx, ky, kz) = floor(v / s) (fp32 IEEE division, A30): their
//                        range and a bad flag, read back (validation before the model is touched; the
//                        key width = the bits the range needs, so the sort runs only the passes it must)
//   K14b k_cell_keys     key = coordinates relative to the range minimum, x-major, + internal index
//   (CUB)                stable radix sort of (key, index): a box's members become contiguous, in
//                        ascending internal index (the oracle's member order)
//   K14c k_cell_decide   one thread per sorted position; a box's first position applies Alg. 3's
//                        deletion test to the merged omega and stamp (A32): keep flag
//   (CUB)                exclusive scan of the keep flags: output positions (ascending box order, A33)
//   K14d k_cell_merge    a surviving box's S:369 weighted averages, omega cap, max stamp, first
//                        member's id (A31) written to the other buffer set at its position, which becomes
//                        the model; merged boxes are listed for re-skinning, single-member boxes keep
//                        theirs (bit-exact position)
//   K2 + K14e            Eq. 2 skinning of the listed boxes against the current nodes (A34), scattered
//
// HBM-bound: every pass is a streaming read / write of the point records (K14).
#include <cub/cub.cuh>

#include <climits>
#include <cstring>

#include "ctx.cuh"

namespace mis {

namespace {

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return e_;          \
  } while (0)

constexpr float kAxisLim = 1073741824.f;   // |box coordinate| < 2^30 (int32 with headroom)

// fp32 IEEE division and floor: the oracle's decision (A30)
__device__ __forceinline__ float box_coord(float v, float s) { return floorf(__fdiv_rn(v, s)); }

// K14a: the box-coordinate range (min / max per axis) and the bad flag.  range: int32 [min x, y, z,
// max x, y, z, bad], initialised to (INT_MAX, INT_MIN, 0) by the caller.
__global__ void __launch_bounds__(256) k_cell_range(ModelView md, float s, int* __restrict__ range) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  bool bad = false;
  if (i < md.n) {
    const float q[3] = {box_coord(md.px[i], s), box_coord(md.py[i], s), box_coord(md.pz[i], s)};
    for (int a = 0; a < 3; ++a) {
      if (!(q[a] > -kAxisLim && q[a] < kAxisLim)) bad = true;   // out of range or non-finite
      else lo[a] = hi[a] = (int)q[a];
    }
  }
  const unsigned full = 0xffffffffu;
  for (int a = 0; a < 3; ++a) {
    lo[a] = __reduce_min_sync(full, lo[a]);
    hi[a] = __reduce_max_sync(full, hi[a]);
  }
  const bool anybad = __any_sync(full, bad);
  if ((threadIdx.x & 31) == 0) {
    for (int a = 0; a < 3; ++a) {
      if (lo[a] != INT_MAX) atomicMin(range + a, lo[a]);
      if (hi[a] != INT_MIN) atomicMax(range + 3 + a, hi[a]);
    }
    if (anybad) atomicOr(range + 6, 1);
  }
}

// K14b: key = box coordinates relative to the range minimum, x-major, by[1] + by[2] + by[0] <= 63
// bits (order-preserving: the same ascending (kx, ky, kz) order, A33), plus the internal index.
__global__ void __launch_bounds__(256) k_cell_keys(ModelView md, float s, int3 lo, int sh_x, int sh_y,
                                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= md.n) return;
  const uint64_t kx = (uint64_t)((int)box_coord(md.px[i], s) - lo.x);
  const uint64_t ky = (uint64_t)((int)box_coord(md.py[i], s) - lo.y);
  const uint64_t kz = (uint64_t)((int)box_coord(md.pz[i], s) - lo.z);
  keys[i] = (kx << sh_x) | (ky << sh_y) | kz;
  vals[i] = (uint32_t)i;
}

struct MergeArgs {
  ModelView a;   // current model (read)
  ModelView b;   // other buffer set: the filtered model, written at the survivors' positions
  const uint64_t* keys;   // sorted
  const uint32_t* vals;   // sorted internal indices
  int32_t* keep;          // n: 1 at a surviving box's first position, else 0
  const int32_t* pos;     // n: exclusive scan of keep (output position)
  int64_t* info;          // [0] survivors, [1] boxes, [2] stable survivors, [3] boxes to re-skin
  float* lxyz;            // re-skinning list: positions (3 floats) ...
  int32_t* lidx;          // ... and output index
  int K;
  int32_t frame, tau_time;
  float tau_weight, omega_max;
};

__device__ __forceinline__ int64_t box_end(const MergeArgs& r, int64_t i, int64_t n) {
  const uint64_t key = r.keys[i];
  int64_t e = i + 1;
  while (e < n && r.keys[e] == key) ++e;
  return e;
}

// K14c: one thread per sorted position; a box's first position decides it: omega = min(sum, omega_max),
// t = max, Alg. 3 line 3 as S:369 -- delete iff t < frame - tau_time and omega < tau_weight (A32).
__global__ void __launch_bounds__(256) k_cell_decide(MergeArgs r) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = r.a.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool head = false, kept = false, stable = false;
  if (i < n) {
    head = (i == 0) || (r.keys[i - 1] != r.keys[i]);
    if (head) {
      const int64_t e = box_end(r, i, n);
      double wsum = 0.0;   // fp64 like the oracle: the deletion test must not flip on rounding
      int32_t t = INT_MIN;
      for (int64_t j = i; j < e; ++j) {
        const uint32_t p = r.vals[j];
        wsum += (double)r.a.w[p];
        t = max(t, r.a.stamp[p]);
      }
      const double om = fmin(wsum, (double)r.omega_max);                          // Eq. 15 cap
      kept = !(((int64_t)t < (int64_t)r.frame - (int64_t)r.tau_time) && (om < (double)r.tau_weight));
      stable = kept && om >= (double)r.tau_weight;                                // S_i (A32)
    }
    r.keep[i] = kept ? 1 : 0;
  }
  // boxes and stable survivors: one atomic per warp
  const unsigned hb = __ballot_sync(0xffffffffu, head), sb = __ballot_sync(0xffffffffu, stable);
  if ((threadIdx.x & 31) == 0) {
    if (hb) atomicAdd(reinterpret_cast<unsigned long long*>(r.info + 1), (unsigned long long)__popc(hb));
    if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(r.info + 2), (unsigned long long)__popc(sb));
  }
}

// K14d: a surviving box's first position merges it (A31) straight into the other buffer set at its
// output position (ascending box order, A33).  A single-member box keeps its position and colour bit
// for bit (the oracle's w*x/w is exact in fp64) and so its Eq. 2 skinning, which is copied; a merged
// box is appended to the re-skinning list.
__global__ void __launch_bounds__(256) k_cell_merge(MergeArgs r) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = r.a.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool skin = false;
  int64_t o = 0;
  float vx = 0.f, vy = 0.f, vz = 0.f;
  if (i < n) {
    if (i == n - 1) r.info[0] = (int64_t)r.pos[i] + r.keep[i];
    if (r.keep[i]) {
      const int64_t e = box_end(r, i, n);
      const ModelView& a = r.a;
      const ModelView& b = r.b;
      const uint32_t p0 = r.vals[i];
      o = r.pos[i];
      double wsum = 0.0;
      for (int64_t j = i; j < e; ++j) wsum += (double)a.w[r.vals[j]];
      const bool weighted = wsum > 0.0;
      float nx = 0.f, ny = 0.f, nz = 0.f, cr = 0.f, cg = 0.f, cb = 0.f, den = 0.f;
      int32_t t = INT_MIN;
      for (int64_t j = i; j < e; ++j) {
        const uint32_t p = r.vals[j];
        const float wi = weighted ? a.w[p] : 1.f;
        vx = fmaf(wi, a.px[p], vx); vy = fmaf(wi, a.py[p], vy); vz = fmaf(wi, a.pz[p], vz);
        nx = fmaf(wi, a.nx[p], nx); ny = fmaf(wi, a.ny[p], ny); nz = fmaf(wi, a.nz[p], nz);
        cr = fmaf(wi, a.cr[p], cr); cg = fmaf(wi, a.cg[p], cg); cb = fmaf(wi, a.cb[p], cb);
        den += wi;
        t = max(t, a.stamp[p]);
      }
      if (e == i + 1) {
        vx = a.px[p0]; vy = a.py[p0]; vz = a.pz[p0];
        cr = a.cr[p0]; cg = a.cg[p0]; cb = a.cb[p0];
        for (int q = 0; q < r.K; ++q) {
          b.kidx[q * b.cap + o] = a.kidx[q * a.cap + p0];
          b.kw[q * b.cap + o] = a.kw[q * a.cap + p0];
        }
      } else {
        const float inv = 1.f / den;
        vx *= inv; vy *= inv; vz *= inv;
        cr *= inv; cg *= inv; cb *= inv;
        skin = true;
      }
      b.px[o] = vx; b.py[o] = vy; b.pz[o] = vz;
      b.cr[o] = cr; b.cg[o] = cg; b.cb[o] = cb;
      const float len2 = nx * nx + ny * ny + nz * nz;
      if (len2 > 0.f) {
        const float il = rsqrtf(len2);
        b.nx[o] = nx * il; b.ny[o] = ny * il; b.nz[o] = nz * il;
      } else {
        b.nx[o] = a.nx[p0]; b.ny[o] = a.ny[p0]; b.nz[o] = a.nz[p0];
      }
      b.w[o] = (float)fmin(wsum, (double)r.omega_max);
      b.stamp[o] = t;
      b.ids[o] = a.ids[p0];
    }
  }
  // warp-aggregated append to the re-skinning list
  const unsigned full = 0xffffffffu, bal = __ballot_sync(full, skin);
  if (!bal) return;
  const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(reinterpret_cast<unsigned long long*>(r.info + 3), (unsigned long long)__popc(bal));
  base = __shfl_sync(full, base, leader);
  if (skin) {
    const int64_t l = (int64_t)base + __popc(bal & ((1u << lane) - 1));
    r.lxyz[3 * l] = vx; r.lxyz[3 * l + 1] = vy; r.lxyz[3 * l + 2] = vz;
    r.lidx[l] = (int32_t)o;
  }
}

// K14e: the re-skinned boxes' Eq. 2 tuples (K2 output, slot-major over the list) into the model.
__global__ void __launch_bounds__(256) k_cell_skin_scatter(int64_t nl, int K, const int32_t* __restrict__ lidx,
                                                           const int32_t* __restrict__ si, const float* __restrict__ sw,
                                                           ModelView a) {
  pdl_wait();
  pdl_trigger();
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  const int64_t o = lidx[l];
  for (int q = 0; q < K; ++q) {
    a.kidx[q * a.cap + o] = si[q * nl + l];
    a.kw[q * a.cap + o] = sw[q * nl + l];
  }
}

template <class F>
cudaError_t cub_call(Ctx* c, F f) {
  size_t need = 0;
  CK(f(nullptr, need));
  CK(ensure(c, c->cub_tmp, std::max(need, cub_tmp_bound(c->cap)) + 256));
  size_t have = c->cub_tmp.bytes;
  return f(c->cub_tmp.p, have);
}

int bits_for_span(int64_t span) {   // bits to hold 0..span-1
  int b = 0;
  while (b < 62 && (int64_t(1) << b) < span) ++b;
  return b;
}

}  // namespace

// K14a on the context stream and one readback: the box-coordinate range.  range_host (7 x int32):
// min x, y, z, max x, y, z, bad flag.  n > 0.
cudaError_t run_filter_range(Ctx* c, float grid, int32_t* range_host) {
  const int64_t n = c->n;
  int32_t* h = reinterpret_cast<int32_t*>(c->hpin);
  for (int a = 0; a < 3; ++a) { h[a] = INT_MAX; h[3 + a] = INT_MIN; }
  h[6] = 0;
  int* range = reinterpret_cast<int*>(c->finfo.as<int64_t>() + 4);
  CK(cudaMemcpyAsync(range, h, 28, cudaMemcpyHostToDevice, c->st));
  launch_pdl(k_cell_range, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, c->st, model_view(c), grid, range);
  CK(cudaMemcpyAsync(h, range, 28, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  memcpy(range_host, h, 28);
  return cudaGetLastError();
}

// Key bits of a validated range: the shifts of x and y and the total (<= 63; -1 if it does not fit).
int filter_key_bits(const int32_t* range, int* sh_x, int* sh_y) {
  const int bx = bits_for_span((int64_t)range[3] - range[0] + 1), by = bits_for_span((int64_t)range[4] - range[1] + 1),
            bz = bits_for_span((int64_t)range[5] - range[2] + 1);
  if (bx + by + bz > 63) return -1;
  *sh_y = bz;
  *sh_x = by + bz;
  return bx + by + bz;
}

// K14b-d and the CUB sort / scan (the other buffer set becomes current) on the context stream; info (finfo[0..3], zeroed here) receives
// [survivors, boxes, stable survivors, boxes to re-skin].  Read back by the caller, which then
// calls run_filter_skin.
cudaError_t run_filter(Ctx* c, float grid, const int32_t* range, int sh_x, int sh_y, int bits, int32_t frame,
                       int32_t tau_time, float tau_weight) {
  const int64_t n = c->n;
  int64_t* info = c->finfo.as<int64_t>();
  CK(cudaMemsetAsync(info, 0, 32, c->st));
  CK(ensure(c, c->keys, ncap(c, n) * 8)); CK(ensure(c, c->keys2, ncap(c, n) * 8));
  CK(ensure(c, c->vals, ncap(c, n) * 4)); CK(ensure(c, c->vals2, ncap(c, n) * 4));
  CK(ensure(c, c->flags, ncap(c, n) * 4)); CK(ensure(c, c->scan, ncap(c, n) * 4));
  CK(ensure(c, c->fl_xyz, ncap(c, n) * 12)); CK(ensure(c, c->fl_idx, ncap(c, n) * 4));
  const int b = (int)((n + 255) / 256);
  ModelView A = model_view(c);
  ModelView B = model_view_of(c, c->mb[1 - c->cur]);
  B.n = n;
  launch_pdl(k_cell_keys, dim3(b), dim3(256), 0, c->st, A, grid, make_int3(range[0], range[1], range[2]), sh_x, sh_y,
             c->keys.as<uint64_t>(), c->vals.as<uint32_t>());
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceRadixSort::SortPairs(t, s, c->keys.as<uint64_t>(), c->keys2.as<uint64_t>(), c->vals.as<uint32_t>(),
                                           c->vals2.as<uint32_t>(), (int)n, 0, std::max(bits, 1), c->st);
  }));
  MergeArgs r{A, B, c->keys2.as<uint64_t>(), c->vals2.as<uint32_t>(), c->flags.as<int32_t>(), c->scan.as<int32_t>(),
              info, c->fl_xyz.as<float>(), c->fl_idx.as<int32_t>(), c->K, frame, tau_time, tau_weight,
              c->prm.omega_max};
  launch_pdl(k_cell_decide, dim3(b), dim3(256), 0, c->st, r);
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceScan::ExclusiveSum(t, s, c->flags.as<int32_t>(), c->scan.as<int32_t>(), (int)n, c->st);
  }));
  launch_pdl(k_cell_merge, dim3(b), dim3(256), 0, c->st, r);
  c->cur = 1 - c->cur;   // the filtered model is the other buffer set
  return cudaGetLastError();
}

// Eq. 2 skinning of the nl merged survivors (A34) against the current nodes, then the scatter into
// the model (2 launches).
cudaError_t run_filter_skin(Ctx* c, int64_t nl) {
  if (nl <= 0) return cudaSuccess;
  CK(ensure(c, c->fl_kidx, (size_t)nl * 4 * c->K)); CK(ensure(c, c->fl_kw, (size_t)nl * 4 * c->K));
  const float* x = c->fl_xyz.as<float>();
  launch_skin_boxed(nl, nullptr, 0, x, x + 1, x + 2, 3, c->g.as<float>(), c->m, c->K, c->fl_kidx.as<int32_t>(),
                    c->fl_kw.as<float>(), nl, c->st);   // the list is in box order: spatially coherent blocks
  launch_pdl(k_cell_skin_scatter, dim3((unsigned)((nl + 255) / 256)), dim3(256), 0, c->st, nl, c->K,
             c->fl_idx.as<int32_t>(), c->fl_kidx.as<int32_t>(), c->fl_kw.as<float>(), model_view(c));
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K15: node regeneration
// NEXT-1, Alg. 2 Step 5 as S:102-104, reading A36: the nodes become the centroids of the
// occupied cells of size s (the same fp32 box coordinates as K14, A30), in ascending (kx, ky, kz)
// order, with identity transforms; N(j) = the n_nbr nearest other nodes (ties to the lower index).
//   K14a k_cell_range + readback   validation and key width (as the filter)
//   K14b k_cell_keys + CUB sort    a cell's members contiguous, cells in ascending key order
//   K15a k_cell_heads + CUB scan   cell id of every sorted position
//   K15b k_cell_accum              segmented warp sums of the members' positions (fp64) + one atomic per
//                                  (warp, cell); k_cell_centroid: fp32 centroids, the node count read back
//   K15c k_node_knn                brute-force n_nbr nearest (fp64 distances of the fp32 centroids)
// then mis_set_graph (device inputs): identity states, Eq. 2 skinning of every point (K2), K13 order.
__global__ void __launch_bounds__(256) k_cell_heads(int64_t n, const uint64_t* __restrict__ keys,
                                                    int32_t* __restrict__ head) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i - 1] != keys[i]) ? 1 : 0;
}

// K15b: every sorted position adds its point to its cell's fp64 sums (x, y, z, count): a segmented
// warp scan over the (non-decreasing) cell ids, then one atomic per (warp, cell) segment -- fully
// parallel whatever the cell sizes (a cell of a 3 mm node grid holds ~500 points at C3).
__global__ void __launch_bounds__(256) k_cell_accum(int64_t n, const uint32_t* __restrict__ vals,
                                                    const int32_t* __restrict__ cid_incl, ModelView md,
                                                    double4* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int cid = -1;
  double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
  if (i < n) {
    const uint32_t p = vals[i];
    cid = cid_incl[i] - 1;
    v = make_double4(md.px[p], md.py[p], md.pz[p], 1.0);
  }
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int cu = __shfl_up_sync(full, cid, off);
    const double ux = __shfl_up_sync(full, v.x, off), uy = __shfl_up_sync(full, v.y, off);
    const double uz = __shfl_up_sync(full, v.z, off), uw = __shfl_up_sync(full, v.w, off);
    if (lane >= off && cu == cid) { v.x += ux; v.y += uy; v.z += uz; v.w += uw; }
  }
  const int cn = __shfl_down_sync(full, cid, 1);
  if (cid >= 0 && (lane == 31 || cn != cid)) {   // the last lane of its segment in this warp
    double* s = reinterpret_cast<double*>(sums + cid);
    atomicAdd(s, v.x); atomicAdd(s + 1, v.y); atomicAdd(s + 2, v.z); atomicAdd(s + 3, v.w);
  }
}

// K15b': the fp32 centroids of the m cells (m = the last inclusive cell id), node count to info[0].
__global__ void __launch_bounds__(256) k_cell_centroid(int64_t n, const int32_t* __restrict__ cid_incl,
                                                       const double4* __restrict__ sums, float* __restrict__ g,
                                                       int64_t* __restrict__ info) {
  pdl_wait();
  pdl_trigger();
  const int64_t m = cid_incl[n - 1];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) info[0] = m;
  if (j >= m) return;
  const double4 s = sums[j];
  const double inv = 1.0 / s.w;
  g[3 * j] = (float)(s.x * inv); g[3 * j + 1] = (float)(s.y * inv); g[3 * j + 2] = (float)(s.z * inv);
}

constexpr int kMaxRegenNbr = 16;
__global__ void __launch_bounds__(256) k_node_knn(int m, int nn, const float* __restrict__ g,
                                                  int32_t* __restrict__ nbr) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 tile[256];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double gj[3] = {0, 0, 0};
  if (j < m) { gj[0] = g[3 * j]; gj[1] = g[3 * j + 1]; gj[2] = g[3 * j + 2]; }
  double bd[kMaxRegenNbr];
  int bi[kMaxRegenNbr];
#pragma unroll
  for (int s = 0; s < kMaxRegenNbr; ++s) { bd[s] = INFINITY; bi[s] = -1; }
  for (int t0 = 0; t0 < m; t0 += 256) {
    __syncthreads();
    const int l = t0 + threadIdx.x;
    if (l < m) tile[threadIdx.x] = make_float4(g[3 * l], g[3 * l + 1], g[3 * l + 2], 0.f);
    __syncthreads();
    const int tn = min(256, m - t0);
    if (j >= m) continue;
    for (int q = 0; q < tn; ++q) {
      const int l2 = t0 + q;
      if (l2 == j) continue;
      const float4 p = tile[q];
      const double dx = (double)p.x - gj[0], dy = (double)p.y - gj[1], dz = (double)p.z - gj[2];
      double cd = dx * dx + dy * dy + dz * dz;
      if (!(cd < bd[nn - 1])) continue;   // ids ascend within the scan: a tie keeps the lower id
      int ci = l2;
#pragma unroll
      for (int s = 0; s < kMaxRegenNbr; ++s) {
        if (s < nn && cd < bd[s]) {
          const double td = bd[s];
          const int ti = bi[s];
          bd[s] = cd; bi[s] = ci; cd = td; ci = ti;
        }
      }
    }
  }
  if (j >= m) return;
  for (int s = 0; s < nn; ++s) nbr[(int64_t)nn * j + s] = bi[s];
}

// K14b + CUB + K15a/b: centroids into c->fl_xyz, node count read back into *m_out.
cudaError_t run_regen_centroids(Ctx* c, float grid, const int32_t* range, int sh_x, int sh_y, int bits, int64_t* m_out) {
  const int64_t n = c->n;
  int64_t* info = c->finfo.as<int64_t>();
  CK(ensure(c, c->keys, ncap(c, n) * 8)); CK(ensure(c, c->keys2, ncap(c, n) * 8));
  CK(ensure(c, c->vals, ncap(c, n) * 4)); CK(ensure(c, c->vals2, ncap(c, n) * 4));
  CK(ensure(c, c->flags, ncap(c, n) * 4)); CK(ensure(c, c->scan, ncap(c, n) * 4));
  CK(ensure(c, c->fl_xyz, ncap(c, n) * 12));
  CK(ensure(c, c->rg_sums, ncap(c, n) * 32));
  CK(cudaMemsetAsync(c->rg_sums.p, 0, n * 32, c->st));
  const int b = (int)((n + 255) / 256);
  ModelView A = model_view(c);
  launch_pdl(k_cell_keys, dim3(b), dim3(256), 0, c->st, A, grid, make_int3(range[0], range[1], range[2]), sh_x, sh_y,
             c->keys.as<uint64_t>(), c->vals.as<uint32_t>());
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceRadixSort::SortPairs(t, s, c->keys.as<uint64_t>(), c->keys2.as<uint64_t>(), c->vals.as<uint32_t>(),
                                           c->vals2.as<uint32_t>(), (int)n, 0, std::max(bits, 1), c->st);
  }));
  launch_pdl(k_cell_heads, dim3(b), dim3(256), 0, c->st, n, (const uint64_t*)c->keys2.as<uint64_t>(), c->flags.as<int32_t>());
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceScan::InclusiveSum(t, s, c->flags.as<int32_t>(), c->scan.as<int32_t>(), (int)n, c->st);
  }));
  launch_pdl(k_cell_accum, dim3(b), dim3(256), 0, c->st, n, (const uint32_t*)c->vals2.as<uint32_t>(),
             (const int32_t*)c->scan.as<int32_t>(), A, c->rg_sums.as<double4>());
  launch_pdl(k_cell_centroid, dim3(b), dim3(256), 0, c->st, n, (const int32_t*)c->scan.as<int32_t>(),
             (const double4*)c->rg_sums.as<double4>(), c->fl_xyz.as<float>(), info);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->hpin, info, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  memcpy(m_out, c->hpin, 8);
  return cudaSuccess;
}

// K15c: N(j) of the m regenerated nodes (in c->fl_xyz) into c->rg_nbr.
cudaError_t run_regen_knn(Ctx* c, int m, int nn) {
  CK(ensure(c, c->rg_nbr, (size_t)m * (nn > 0 ? nn : 1) * 4));
  if (nn > 0)
    launch_pdl(k_node_knn, dim3((unsigned)((m + 255) / 256)), dim3(256), 0, c->st, m, nn,
               (const float*)c->fl_xyz.as<float>(), c->rg_nbr.as<int32_t>());
  return cudaGetLastError();
}

}  // namespace mis
