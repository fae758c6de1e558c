// sort.cu -- K13: canonical kNN-tuple sort of the model, tuple segments and
// K3 work chunks; and the block-sparse (BSR) pattern of the normal equations
// with the slot tables K3 / K4 / K5 commit into.  Setup work, once per model
// change (order) and once per registration (pattern, since the feature tuples
// change every frame).  CUB radix sort / scan are library primitives here.
#include <cub/cub.cuh>

#include <algorithm>

#include "ctx.cuh"

namespace mis {

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return e_;          \
  } while (0)

static int bits_for(int m) {
  int b = 1;
  while ((1ll << b) < (int64_t)m) ++b;
  return b;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

// key: the top kb bits of a 64-bit mix of the (ascending) id tuple.  Equal tuples get
// equal keys, so the stable radix sort makes every tuple's points contiguous up to
// key collisions; a collision only interleaves the points of two tuples, which
// k_seg_flags (comparing whole tuples) then splits into more, shorter segments --
// never a wrong one.  kb ~ log2(#tuples) + 7 keeps collisions rare with 8-bit
// radix passes: 3 passes at c3 instead of 5 for the exact 40-bit packing.
__global__ void k_tuple_keys(int64_t n, int64_t cap, const int32_t* kidx, int K, int kb, uint64_t* keys,
                             uint32_t* vals) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (int s = 0; s < K; ++s) h = mix64(h ^ (uint64_t)(uint32_t)kidx[s * cap + i]);
  keys[i] = kb >= 64 ? h : (h >> (64 - kb));
  vals[i] = (uint32_t)i;
}

// all model arrays in one launch: dst[i] = src[perm[i]]
__global__ void k_gather_model(int64_t n, const uint32_t* perm, ModelView a, ModelView b, int K) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
  b.px[i] = a.px[j]; b.py[i] = a.py[j]; b.pz[i] = a.pz[j];
  b.nx[i] = a.nx[j]; b.ny[i] = a.ny[j]; b.nz[i] = a.nz[j];
  b.cr[i] = a.cr[j]; b.cg[i] = a.cg[j]; b.cb[i] = a.cb[j]; b.w[i] = a.w[j];
  b.stamp[i] = a.stamp[j]; b.ids[i] = a.ids[j];
  for (int s = 0; s < K; ++s) {
    b.kidx[s * a.cap + i] = a.kidx[s * a.cap + j];
    b.kw[s * a.cap + i] = a.kw[s * a.cap + j];
  }
}

__global__ void k_seg_flags(int64_t n, int64_t cap, const int32_t* kidx, int K, int32_t* flags) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f = (i == 0);
  if (!f)
    for (int s = 0; s < K; ++s)
      if (kidx[s * cap + i] != kidx[s * cap + i - 1]) { f = 1; break; }
  flags[i] = f;
}

// scan = inclusive sum of flags; seg id = scan - 1
__global__ void k_seg_write(int64_t n, int64_t cap, const int32_t* kidx, int K, const int32_t* flags,
                            const int32_t* scan, int32_t* seg_start, int32_t* seg_nodes) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!flags[i]) return;
  const int32_t s = scan[i] - 1;
  seg_start[s] = (int32_t)i;
  for (int q = 0; q < K; ++q) seg_nodes[(int64_t)s * K + q] = kidx[q * cap + i];
  if (i == 0) seg_start[scan[n - 1]] = (int32_t)n;   // sentinel
}

__global__ void k_chunk_count(int64_t n, const int32_t* nseg_dev, const int32_t* seg_start, int32_t* cnt) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if (s >= *nseg_dev) { cnt[s] = 0; return; }
  const int32_t len = seg_start[s + 1] - seg_start[s];
  cnt[s] = (len + kChunk - 1) / kChunk;
}

__global__ void k_chunk_write(int64_t n, const int32_t* nseg_dev, const int32_t* seg_start, const int32_t* off,
                              int4* chunks, int64_t* info) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) { info[1] = *nseg_dev; info[2] = off[n - 1]; }   // device-resident counts (read back with the pattern)
  if (s >= n || s >= *nseg_dev) return;
  const int32_t a = seg_start[s], b = seg_start[s + 1];
  const int32_t nc = (b - a + kChunk - 1) / kChunk, len = b - a;
  const int32_t o = off[s] - nc;   // inclusive scan -> start
  for (int32_t q = 0; q < nc; ++q)   // equal-size chunks: the last one is not a short tail
    chunks[o + q] = make_int4((int)s, a + (int32_t)((int64_t)len * q / nc), a + (int32_t)((int64_t)len * (q + 1) / nc), 0);
}

// ---- grouping by exact tuple (k <= 4, m < 65535): the model only needs every tuple's points
// contiguous, not an order of the tuples, so instead of sorting, each point finds its tuple in
// a hash table (the first finder of a tuple claims a group id), takes a rank inside the group
// with one atomic, and one CTA lays the groups out (prefix sums of sizes and chunk counts,
// segment / chunk tables); a scatter then gives the gather permutation.  Group order and the
// order inside a group follow the atomics (the K3 sums are atomic-order dependent anyway).
constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ uint64_t tuple_key(const int32_t* kidx, int64_t cap, int64_t i, int K) {
  uint64_t key = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint64_t id = s < K ? (uint64_t)(uint32_t)kidx[s * cap + i] : 0xffffull;
    key |= (id & 0xffffull) << (16 * s);
  }
  return key;
}

__global__ void __launch_bounds__(256) k_group_insert(int64_t n, int64_t cap, const int32_t* kidx, int K,
                                                      unsigned long long* tkeys, int32_t* tgid, int64_t tmask,
                                                      int32_t* gcount, uint64_t* gkeys, int32_t* gslot, int32_t* gsize,
                                                      int32_t* gid_out, int32_t* rank_out) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ int32_t nwin, base;
  if (threadIdx.x == 0) nwin = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool valid = i < n;
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  // lanes with the same tuple (a grouped model makes most of a warp one tuple) elect the lowest
  // as their leader: only leaders touch the table and the group sizes
  uint64_t key = 0;
  unsigned mask = 0;
  if (valid) {
    key = tuple_key(kidx, cap, i, K);
    mask = __match_any_sync(vmask, key);
  }
  const int leader = valid ? __ffs(mask) - 1 : lane;
  const bool lead = valid && leader == lane;
  // phase A (never waits): leaders find or insert the tuple's slot
  int64_t h = -1;
  bool won = false;
  if (lead) {
    h = (int64_t)(mix64(key) & (uint64_t)tmask);
    for (;;) {
      unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(tkeys + h);
      if (cur == kEmpty) {
        cur = atomicCAS(tkeys + h, kEmpty, (unsigned long long)key);
        if (cur == kEmpty) { won = true; break; }
      }
      if (cur == key) break;
      h = (h + 1) & tmask;
    }
  }
  // group ids for this block's new tuples: one counter atomic per block
  int my = 0;
  if (won) my = atomicAdd(&nwin, 1);
  __syncthreads();
  if (threadIdx.x == 0 && nwin > 0) base = atomicAdd(gcount, nwin);
  __syncthreads();
  int32_t gid = -1, r0 = 0;
  if (won) {
    gid = base + my;
    gkeys[gid] = key;
    gslot[gid] = (int32_t)h;
    __threadfence();
    *reinterpret_cast<volatile int32_t*>(tgid + h) = gid;
  }
  // phase B: tuples inserted elsewhere (their winner is resident and publishes without waiting)
  if (lead) {
    if (!won) {
      int32_t g;
      while ((g = *reinterpret_cast<volatile int32_t*>(tgid + h)) < 0) {}
      gid = g;
    }
    r0 = atomicAdd(gsize + gid, __popc(mask));
  }
  if (valid) {
    gid = __shfl_sync(vmask, gid, leader);
    r0 = __shfl_sync(vmask, r0, leader);
    gid_out[i] = gid;
    rank_out[i] = r0 + __popc(mask & ((1u << lane) - 1u));
  }
}

// one CTA: segment starts (prefix of group sizes), segment node tuples, chunk table (equal
// chunks of <= kChunk points per segment), the counts for the pattern readback; re-empties the
// hash slots and group sizes it used
__global__ void __launch_bounds__(1024) k_group_layout(int64_t n, const int32_t* gcount, const int32_t* gsize,
                                                       int2* pre, int32_t* seg_start, int64_t* info) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ int32_t wsum[2][32];
  __shared__ int32_t carry[2];
  const int T = *gcount;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) { carry[0] = 0; carry[1] = 0; }
  __syncthreads();
  for (int base = 0; base < T; base += 1024) {
    const int s = base + t;
    const int len = s < T ? gsize[s] : 0, nc = (len + kChunk - 1) / kChunk;
    int a = len, b = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) { a += x; b += y; }
    }
    if (lane == 31) { wsum[0][w] = a; wsum[1][w] = b; }
    __syncthreads();
    if (w == 0) {
      int x = wsum[0][lane], y = wsum[1][lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o), v = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) { x += u; y += v; }
      }
      wsum[0][lane] = x;
      wsum[1][lane] = y;
    }
    __syncthreads();
    const int pre0 = carry[0] + (w > 0 ? wsum[0][w - 1] : 0) + a - len;
    const int pre1 = carry[1] + (w > 0 ? wsum[1][w - 1] : 0) + b - nc;
    if (s < T) pre[s] = make_int2(pre0, pre1);   // one coalesced store: the writes are spread by k_group_write
    __syncthreads();
    if (t == 0) { carry[0] += wsum[0][31]; carry[1] += wsum[1][31]; }
    __syncthreads();
  }
  if (t == 0) {
    seg_start[T] = (int32_t)n;
    info[1] = T;
    info[2] = carry[1];
  }
}

// one thread per group: segment start, node tuple, chunks; re-empties the hash slot and the size
__global__ void k_group_write(int K, const int32_t* gcount, const uint64_t* gkeys, const int32_t* gslot,
                              int32_t* gsize, const int2* pre, unsigned long long* tkeys, int32_t* tgid,
                              int32_t* seg_start, int32_t* seg_nodes, int4* chunks) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int T = *gcount;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= T) return;
  const int len = gsize[s], nc = (len + kChunk - 1) / kChunk;
  const int2 p = pre[s];
  const uint64_t key = gkeys[s];
  const int32_t hs = gslot[s];
  seg_start[s] = p.x;
  for (int q = 0; q < K; ++q) seg_nodes[s * K + q] = (int32_t)((key >> (16 * q)) & 0xffffull);
  for (int q = 0; q < nc; ++q)
    chunks[p.y + q] = make_int4((int)s, p.x + (int32_t)((int64_t)len * q / nc), p.x + (int32_t)((int64_t)len * (q + 1) / nc), 0);
  tkeys[hs] = kEmpty;
  tgid[hs] = -1;
  gsize[s] = 0;
}


__global__ void k_group_perm(int64_t n, const int32_t* gid, const int32_t* rank, const int32_t* seg_start,
                             uint32_t* perm, int32_t* gcount) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *gcount = 0;   // every reader of the group count (the layout kernels) has finished
  if (i >= n) return;
  perm[seg_start[gid[i]] + rank[i]] = (uint32_t)i;
}

// the model grouped by tuple (replaces sort + segment scans when k <= 4 and m < 65535)
static cudaError_t build_order_grouped(Ctx* c) {
  const int64_t n = c->n;
  const int K = c->K;
  ModelBufs& A = c->mb[c->cur];
  ModelBufs& B = c->mb[1 - c->cur];
  int64_t slots = 1024;
  while (slots < 2 * ncap(c, n)) slots <<= 1;   // load factor <= 1/2 even if every point had its own tuple
  if (c->gtab_slots < slots) {
    CK(ensure(c, c->gtab, (size_t)slots * 12));
    CK(cudaMemsetAsync(c->gtab.p, 0xff, (size_t)slots * 12, c->st));   // keys empty, group ids -1
    c->gtab_slots = slots;
  }
  if (c->gcount.bytes < 64 || c->gsize_cap < n) {   // (sized for the capacity: see ncap)
    CK(ensure(c, c->gkeys, (size_t)ncap(c, n) * 8));
    CK(ensure(c, c->gslot, (size_t)ncap(c, n) * 4 + 64));
    CK(ensure(c, c->gcount, (size_t)ncap(c, n) * 4 + 64));   // [0]: group counter, [16..]: group sizes
    CK(cudaMemsetAsync(c->gcount.p, 0, (size_t)ncap(c, n) * 4 + 64, c->st));
    c->gsize_cap = ncap(c, n);
  }
  CK(ensure(c, c->vals, ncap(c, n) * 4)); CK(ensure(c, c->vals2, ncap(c, n) * 4)); CK(ensure(c, c->keys, ncap(c, n) * 8));
  CK(ensure(c, c->seg_start, (ncap(c, n) + 1) * 4));
  CK(ensure(c, c->seg_nodes, (size_t)ncap(c, n) * K * 4));
  CK(ensure(c, c->chunks, (size_t)ncap(c, n) * 16));
  if (!c->nnz_dev.p) {
    CK(ensure(c, c->nnz_dev, 64));
    CK(cudaMemsetAsync(c->nnz_dev.p, 0, 64, c->st));
  }
  unsigned long long* tkeys = reinterpret_cast<unsigned long long*>(c->gtab.p);
  int32_t* tgid = reinterpret_cast<int32_t*>(tkeys + c->gtab_slots);
  int32_t* gcount = c->gcount.as<int32_t>();
  int32_t* gsize = gcount + 16;
  const int b = (int)((n + 255) / 256);
  launch_pdl(k_group_insert, dim3(b), dim3(256), 0, c->st, n, c->cap, A.kidx.as<int32_t>(), K, tkeys, tgid,
             c->gtab_slots - 1, gcount, c->gkeys.as<uint64_t>(), c->gslot.as<int32_t>(), gsize, c->vals.as<int32_t>(),
             c->vals2.as<int32_t>());
  CK(ensure(c, c->scan, (size_t)ncap(c, n) * 8));   // per-group (segment start, chunk start)
  int2* pre = reinterpret_cast<int2*>(c->scan.p);
  launch_pdl(k_group_layout, dim3(1), dim3(1024), 0, c->st, n, gcount, gsize, pre, c->seg_start.as<int32_t>(),
             c->nnz_dev.as<int64_t>());
  launch_pdl(k_group_write, dim3(b), dim3(256), 0, c->st, K, gcount, c->gkeys.as<uint64_t>(), c->gslot.as<int32_t>(),
             gsize, pre, tkeys, tgid, c->seg_start.as<int32_t>(), c->seg_nodes.as<int32_t>(), c->chunks.as<int4>());
  uint32_t* perm = reinterpret_cast<uint32_t*>(c->keys.p);
  launch_pdl(k_group_perm, dim3(b), dim3(256), 0, c->st, n, c->vals.as<int32_t>(), c->vals2.as<int32_t>(),
             c->seg_start.as<int32_t>(), perm, gcount);
  launch_pdl(k_gather_model, dim3(b), dim3(256), 0, c->st, n, perm, model_view(c), model_view_of(c, B), K);
  count_launches(5);
  CK(cudaGetLastError());
  c->cur = 1 - c->cur;
  c->nseg = -1;
  c->nchunk = -1;
  c->dirty = false;
  c->pattern_valid = false;
  return cudaSuccess;
}

template <class F>
static cudaError_t cub_call(Ctx* c, F f) {
  size_t need = 0;
  CK(f(nullptr, need));
  CK(ensure(c, c->cub_tmp, std::max(need, cub_tmp_bound(c->cap)) + 256));
  size_t have = c->cub_tmp.bytes;
  return f(c->cub_tmp.p, have);
}

size_t cub_tmp_bound(int64_t n) {
  size_t a = 0, b = 0, d = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, 64);
  cub::DeviceScan::InclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, d, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return std::max(a, std::max(b, d));
}

cudaError_t build_order(Ctx* c) {
  const int64_t n = c->n;
  const int K = c->K;
  if (n > 0 && K <= 4 && c->m < 65535 && !c->order_by_sort) return build_order_grouped(c);
  ModelBufs& A = c->mb[c->cur];
  ModelBufs& B = c->mb[1 - c->cur];
  if (n > 0) {
    CK(ensure(c, c->keys, ncap(c, n) * 8)); CK(ensure(c, c->keys2, ncap(c, n) * 8));
    CK(ensure(c, c->vals, ncap(c, n) * 4)); CK(ensure(c, c->vals2, ncap(c, n) * 4));
    // tuples expected: the last pattern's segment count (the model changes little between
    // frames), else n / 8; key bits = log2 of that + 7, rounded up to whole 8-bit passes
    const int64_t t_est = c->nseg > 0 ? c->nseg : std::max<int64_t>(n / 8, 1);
    const int kb = std::min(64, (bits_for((int)std::min<int64_t>(t_est, 1 << 30)) + 7 + 7) / 8 * 8);
    const int b = (int)((n + 255) / 256);
    launch_pdl(k_tuple_keys, dim3(b), dim3(256), 0, c->st, n, c->cap, A.kidx.as<int32_t>(), K, kb, c->keys.as<uint64_t>(),
                                        c->vals.as<uint32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceRadixSort::SortPairs(t, s, c->keys.as<uint64_t>(), c->keys2.as<uint64_t>(),
                                             c->vals.as<uint32_t>(), c->vals2.as<uint32_t>(), (int)n, 0, kb, c->st);
    }));
    launch_pdl(k_gather_model, dim3(b), dim3(256), 0, c->st, n, c->vals2.as<uint32_t>(), model_view(c), model_view_of(c, B), K);
    count_launches(2);   // keys, gather (CUB's sort kernels are library code, not counted)
    CK(cudaGetLastError());
    c->cur = 1 - c->cur;
  }
  ModelBufs& S = c->mb[c->cur];
  // segments and chunks, sized by the upper bound n; the counts stay on the device
  // (info[1], info[2]) and reach the host with the single readback of build_pattern
  if (!c->nnz_dev.p) {
    CK(ensure(c, c->nnz_dev, 64));
    CK(cudaMemsetAsync(c->nnz_dev.p, 0, 64, c->st));   // zero at rest afterwards (flags cleared by k_row_fill)
  }
  c->nseg = -1;
  c->nchunk = -1;
  if (n > 0) {
    CK(ensure(c, c->flags, ncap(c, n) * 4)); CK(ensure(c, c->scan, ncap(c, n) * 4));
    CK(ensure(c, c->seg_start, (ncap(c, n) + 1) * 4));
    CK(ensure(c, c->seg_nodes, (size_t)ncap(c, n) * K * 4));
    CK(ensure(c, c->chunk_off, (ncap(c, n) + 1) * 4));
    CK(ensure(c, c->chunks, (size_t)ncap(c, n) * 16));
    const int b = (int)((n + 255) / 256);
    launch_pdl(k_seg_flags, dim3(b), dim3(256), 0, c->st, n, c->cap, S.kidx.as<int32_t>(), K, c->flags.as<int32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceScan::InclusiveSum(t, s, c->flags.as<int32_t>(), c->scan.as<int32_t>(), (int)n, c->st);
    }));
    const int32_t* nseg_dev = c->scan.as<int32_t>() + n - 1;
    launch_pdl(k_seg_write, dim3(b), dim3(256), 0, c->st, n, c->cap, S.kidx.as<int32_t>(), K, c->flags.as<int32_t>(),
                                      c->scan.as<int32_t>(), c->seg_start.as<int32_t>(), c->seg_nodes.as<int32_t>());
    launch_pdl(k_chunk_count, dim3(b), dim3(256), 0, c->st, n, nseg_dev, c->seg_start.as<int32_t>(), c->flags.as<int32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceScan::InclusiveSum(t, s, c->flags.as<int32_t>(), c->chunk_off.as<int32_t>(), (int)n, c->st);
    }));
    launch_pdl(k_chunk_write, dim3(b), dim3(256), 0, c->st, n, nseg_dev, c->seg_start.as<int32_t>(), c->chunk_off.as<int32_t>(),
                                        c->chunks.as<int4>(), c->nnz_dev.as<int64_t>());
    count_launches(4);   // flags, segment write, chunk count, chunk write (+ 2 CUB scans)
    CK(cudaGetLastError());
  } else {
    CK(cudaMemsetAsync(c->nnz_dev.as<int64_t>() + 1, 0, 16, c->st));
  }
  c->dirty = false;
  c->pattern_valid = false;
  return cudaSuccess;
}

// ---------------------------------------------------------------- pattern
// The BSR pattern of the normal equations from a node-pair bitmap (m x m bits,
// 64-bit words): every candidate (segment pair, graph edge, feature pair,
// diagonal) sets its two bits; rows are then read out in column order.  No
// sort, and every count stays on the device until the one host readback.
// info (int64): [0] nnz, [1] nseg, [2] nchunk, [3] set_graph validation flags, [4..6] PlanOut.

// slot position p of a K-tuple -> (j, j + off): pairs (j <= l) in pair_index order
__device__ __forceinline__ void pair_of(int p, int K, int& j, int& off) {
  j = 0;
  while (p >= K - j) { p -= K - j; ++j; }
  off = p;
}

__device__ __forceinline__ void mark(unsigned long long* bm, int64_t W, int a, int b) {
  unsigned long long* w = bm + (int64_t)a * W + (b >> 6);
  const unsigned long long bit = 1ull << (b & 63);
  if (!(*w & bit)) atomicOr(w, bit);
}

// candidates: [tuples ntup*P][edges m*n_nbr][feature pairs nf*P][diagonal mu]; tuples with a
// negative first id are padding (gathered shards).  mu = m unknown blocks, or m + 1 with the pose
// (NEXT-2: tuples and feature slots then carry the pose id m as their last entry)
__global__ void k_mark(const int32_t* tup, const int64_t* ntup_dev, int64_t ntup_host, int K, int m, int mu, int n_nbr,
                       const int32_t* nbr, int nf, const int32_t* fidx, unsigned long long* bm, int64_t W) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int P = K * (K + 1) / 2;
  const int64_t ntup = ntup_dev ? *ntup_dev : ntup_host;
  const int64_t ns = ntup * P, ne = (int64_t)m * n_nbr, nfp = (int64_t)nf * P, total = ns + ne + nfp + mu;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int a, b;
    if (t < ns) {
      const int64_t sg = t / P;
      int j, off;
      pair_of((int)(t % P), K, j, off);
      a = tup[sg * K + j];
      b = tup[sg * K + j + off];
    } else if (t < ns + ne) {
      const int64_t e = t - ns;
      a = (int)(e / n_nbr);
      b = nbr[e];
    } else if (t < ns + ne + nfp) {
      const int64_t e = t - ns - ne, f = e / P;
      int j, off;
      pair_of((int)(e % P), K, j, off);
      a = fidx[(int64_t)j * nf + f];
      b = fidx[(int64_t)(j + off) * nf + f];
    } else {
      a = b = (int)(t - ns - ne - nfp);
    }
    if (a < 0 || b < 0 || a >= mu || b >= mu) continue;
    mark(bm, W, a, b);
    if (a != b) mark(bm, W, b, a);
  }
}

__global__ void k_bitmap_or(int64_t words, int world, const unsigned long long* all, unsigned long long* bm) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = 0;
    for (int r = 0; r < world; ++r) v |= all[(int64_t)r * words + i];
    bm[i] = v;
  }
}

// one warp per row: number of set bits (cnt[m] = 0 for the exclusive scan)
__global__ void k_row_count(const unsigned long long* bm, int64_t W, int m, int32_t* cnt) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r > m) return;
  int s = 0;
  if (r < m)
    for (int64_t w = lane; w < W; w += 32) s += __popcll(bm[r * W + w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) cnt[r] = s;
}

// one warp per row: columns in ascending order, row index of each entry, diagonal position
__global__ void k_row_fill(unsigned long long* bm, int64_t W, int m, const int32_t* row_ptr, int32_t* col,
                           int32_t* row_of, int32_t* diag_pos, int64_t* info) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x == 0) { info[3] = 0; info[7] = 0; }   // (read back already) flags, ulist count
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= m) return;
  int pos = row_ptr[r];
  for (int64_t w0 = 0; w0 < W; w0 += 32) {
    const int64_t w = w0 + lane;
    unsigned long long word = 0ull;
    if (w < W) {
      word = bm[r * W + w];
      bm[r * W + w] = 0ull;   // cleared for the next pattern build (no memset)
    }
    const int cnt = __popcll(word);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int p = pos + inc - cnt;
    while (word) {
      const int b = __ffsll((long long)word) - 1;
      word &= word - 1;
      const int cc = (int)(64 * w + b);
      col[p] = cc;
      row_of[p] = (int32_t)r;
      if (cc == r) diag_pos[r] = p;
      ++p;
    }
    pos += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// entry of (a, b) in the sorted column list of row a (-1 if absent)
__device__ __forceinline__ int find_entry(const int32_t* row_ptr, const int32_t* col, int a, int b) {
  int lo = row_ptr[a], hi = row_ptr[a + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (col[mid] < b) lo = mid + 1; else hi = mid;
  }
  return (lo < row_ptr[a + 1] && col[lo] == b) ? lo : -1;
}

// After k_row_fill, three independent jobs in one launch (block ranges): the mirror / upper maps
// and the finalisation's off-diagonal list (k_upper_lower), the cluster PCG's halo marks (each
// rank marks, in the owner's mask, the rows its blocks read: as k_pcg_mark) and the slot tables
// (k_slots).  One launch instead of three keeps the device fed while the host is still catching
// up after the pattern readback.
struct PostArgs {
  const int32_t *row_ptr, *col, *row_of;
  int m;
  int32_t *upper_of, *lower_of;
  int2* ulist;
  unsigned long long* ucount;
  int64_t nnz, ul_blocks;
  // halo marks (cs = 0: none)
  const int32_t* part;
  int cs;
  uint32_t* mask;
  int32_t* nin;
  // slots
  int64_t nseg;
  const int32_t* seg_nodes;
  int K, n_nbr, nf;
  const int32_t *nbr, *fidx;
  int32_t *seg_slot, *edge_slot, *feat_slot;
  int64_t total;
};
__device__ __forceinline__ void slot_item(const PostArgs& a, int64_t t);
__global__ void k_pattern_post(PostArgs a) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t b = blockIdx.x;
  if (b < a.ul_blocks) {
    for (int64_t e = b * blockDim.x + threadIdx.x; e < a.nnz; e += a.ul_blocks * blockDim.x) {
      const int r = a.row_of[e], cc = a.col[e];
      if (r == cc) {
        a.upper_of[e] = (int32_t)e;
        a.lower_of[e] = -1;
      } else if (r < cc) {
        a.upper_of[e] = (int32_t)e;
        const int lo = find_entry(a.row_ptr, a.col, cc, r);
        a.lower_of[e] = lo;
        a.ulist[atomicAdd(a.ucount, 1ull)] = make_int2((int)e, lo);
      } else {
        a.upper_of[e] = find_entry(a.row_ptr, a.col, cc, r);
      }
    }
    return;
  }
  if (b < a.ul_blocks + a.cs) {
    const int rank = (int)(b - a.ul_blocks), r0 = a.part[rank], r1 = a.part[rank + 1];
    if (rank == 0 && threadIdx.x < 16) a.nin[threadIdx.x] = 0;   // summed by k_pcg_lists
    for (int k = a.row_ptr[r0] + threadIdx.x; k < a.row_ptr[r1]; k += blockDim.x) {
      const int j = a.col[k];
      if (j < r0 || j >= r1) atomicOr(a.mask + j, 1u << rank);
    }
    return;
  }
  const int64_t t = (b - a.ul_blocks - a.cs) * blockDim.x + threadIdx.x;
  if (t < a.total) slot_item(a, t);
}
__device__ __forceinline__ void slot_item(const PostArgs& a, int64_t t) {
  const int K = a.K, P = K * (K + 1) / 2;
  const int64_t ns = a.nseg * P, ne = (int64_t)a.m * a.n_nbr;
  int j, off;
  if (t < ns) {
    const int64_t sg = t / P;
    pair_of((int)(t % P), K, j, off);
    a.seg_slot[t] = find_entry(a.row_ptr, a.col, a.seg_nodes[sg * K + j], a.seg_nodes[sg * K + j + off]);
  } else if (t < ns + ne) {
    const int64_t e = t - ns;
    const int l = a.nbr[e], q = (int)(e / a.n_nbr);
    a.edge_slot[e] = (l >= 0) ? find_entry(a.row_ptr, a.col, min(q, l), max(q, l)) : -1;
  } else {
    const int64_t e = t - ns - ne, f = e / P;
    pair_of((int)(e % P), K, j, off);
    a.feat_slot[e] = find_entry(a.row_ptr, a.col, a.fidx[(int64_t)j * a.nf + f], a.fidx[(int64_t)(j + off) * a.nf + f]);
  }
}

// NEXT-2 (joint pose): the tuples of the joint pattern -- every segment's K nodes, then the pose
// id m -- and the pose row K (= m) of the feature skinning ids (slot-major, row stride nf)
__global__ void k_joint_tuples(const int64_t* nseg_dev, int K, const int32_t* seg_nodes, int m, int32_t* out, int nf,
                               int32_t* fidx) {
  pdl_wait();
  pdl_trigger();
  const int64_t nseg = *nseg_dev, total = nseg * (K + 1) + nf;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nseg * (K + 1)) {
      const int64_t sg = t / (K + 1);
      const int j = (int)(t - sg * (K + 1));
      out[t] = j < K ? seg_nodes[sg * K + j] : m;
    } else {
      fidx[(int64_t)K * nf + (t - nseg * (K + 1))] = m;
    }
  }
}

cudaError_t build_pattern(Ctx* c) {
  const bool joint = c->joint;
  const int K = c->K + (joint ? 1 : 0), P = K * (K + 1) / 2, m = c->m, mu = m + (joint ? 1 : 0);
  c->pattern_joint = joint;
  c->pattern_affine = c->affine;
  const size_t B = c->affine ? 12 : 6, BB = B * B;   // unknowns per node block (NEXT-4: 12)
  const int64_t W = (mu + 63) / 64, words = (int64_t)mu * W;
  int64_t* info = c->nnz_dev.as<int64_t>();
  if (c->bitmap.bytes < (size_t)words * 8 || c->bitmap_words != words) c->bitmap_clean = false;
  CK(ensure(c, c->bitmap, words * 8));
  if (!c->bitmap_clean) CK(cudaMemsetAsync(c->bitmap.p, 0, words * 8, c->st));   // else cleared by k_row_fill
  c->bitmap_clean = false;
  c->bitmap_words = words;
  unsigned long long* bm = c->bitmap.as<unsigned long long>();
  const int grid = c->num_sms * 8;
  const int32_t* tup = c->seg_nodes.as<int32_t>();
  if (joint) {   // tuples + pose id, pose row of the feature ids (K = k + 1 slots from here on)
    CK(ensure(c, c->seg_nodes_j, (size_t)std::max<int64_t>(ncap(c, c->n), 1) * K * 4));
    launch_pdl(k_joint_tuples, dim3(grid), dim3(256), 0, c->st, (const int64_t*)(info + 1), c->K, tup, m,
               c->seg_nodes_j.as<int32_t>(), c->nf, c->fidx.as<int32_t>());
    count_launches(1);
    tup = c->seg_nodes_j.as<int32_t>();
  }
  launch_pdl(k_mark, dim3(grid), dim3(256), 0, c->st, tup, info + 1, 0, K, m, mu, c->prm.n_nbr, c->nbr.as<int32_t>(),
                                  c->nf, c->fidx.as<int32_t>(), bm, W);
  if (c->world > 1) {   // union over the ranks: all-gather the bitmaps and OR them (same pattern everywhere)
    CK(ensure(c, c->bitmap_all, (size_t)words * 8 * c->world));
    CK(nccl_allgather_u64(c, reinterpret_cast<const uint64_t*>(bm), c->bitmap_all.as<uint64_t>(), (size_t)words));
    launch_pdl(k_bitmap_or, dim3(grid), dim3(256), 0, c->st, words, c->world, c->bitmap_all.as<unsigned long long>(), bm);
  }
  count_launches(c->world > 1 ? 2 : 1);
  CK(ensure(c, c->row_cnt, (size_t)(mu + 1) * 4));
  CK(ensure(c, c->row_ptr, (size_t)(mu + 1) * 4));
  CK(ensure(c, c->diag_pos, (size_t)mu * 4));
  CK(ensure(c, c->part, 32 * 4));
  const int wb = (int)(((int64_t)(mu + 1) * 32 + 255) / 256);
  launch_pdl(k_row_count, dim3(wb), dim3(256), 0, c->st, bm, W, mu, c->row_cnt.as<int32_t>());
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceScan::ExclusiveSum(t, s, c->row_cnt.as<int32_t>(), c->row_ptr.as<int32_t>(), mu + 1, c->st);
  }));
  launch_plan_cluster(c->row_ptr.as<int32_t>(), mu, 16, reinterpret_cast<PlanOut*>(info + 4), c->part.as<int32_t>(),
                      info, c->st);
  count_launches(2);   // row count, plan (+ the CUB scan)
  CK(cudaGetLastError());
  // the single host readback of the frame: nnz, segment / chunk counts, cluster plan
  // (pinned, so the copy is asynchronous: a deferred frame prep is queued behind it and runs
  // while the host waits on the copy's event)
  int64_t h[8];
  CK(cudaMemcpyAsync(c->hpin, info, sizeof(h), cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->rb_ev, c->st));
  CK(flush_frame(c));
  CK(cudaEventSynchronize(c->rb_ev));
  memcpy(h, c->hpin, sizeof(h));
  const int64_t nnz = h[0];
  c->nnzb = nnz;
  c->nseg = h[1];
  c->nchunk = h[2];
  c->graph_flags = (int)h[3];
  const PlanOut* plan = reinterpret_cast<const PlanOut*>(h + 4);
  c->cl_size = plan->cl_size;
  c->cl_max_rows = plan->max_rows;
  c->cl_max_nnz = plan->max_nnz;
  c->cl_smem = (size_t)plan->smem;
  if (joint || c->affine) c->cl_size = 0;   // the dense pose row / 12 x 12 blocks: the grid-wide PCG
  CK(ensure(c, c->col, nnz * 4 + 4)); CK(ensure(c, c->row_of, nnz * 4 + 4));
  CK(ensure(c, c->upper_of, nnz * 4 + 4)); CK(ensure(c, c->lower_of, nnz * 4 + 4));
  CK(ensure(c, c->ulist, ((nnz - mu) / 2 + 1) * 8));
  launch_pdl(k_row_fill, dim3(wb), dim3(256), 0, c->st, bm, W, mu, c->row_ptr.as<int32_t>(), c->col.as<int32_t>(),
             c->row_of.as<int32_t>(), c->diag_pos.as<int32_t>(), info);
  c->bitmap_clean = true;
  const int64_t total = c->nseg * P + (int64_t)m * c->prm.n_nbr + (int64_t)c->nf * P;
  CK(ensure(c, c->seg_slot, (c->nseg * P + 1) * 4));
  CK(ensure(c, c->edge_slot, ((int64_t)m * c->prm.n_nbr + 1) * 4));
  CK(ensure(c, c->feat_slot, ((int64_t)c->nf * P + 1) * 4));
  const bool clu = c->cl_size > 0 && nnz > 0;   // cluster PCG: per-rank SpMV pieces and halo lists for the frame
  if (clu) {
    const int cs = c->cl_size, mr = c->cl_max_rows, mp = pcg_max_pieces(c->cl_max_rows, c->cl_max_nnz);
    CK(ensure(c, c->pcg_pptr, (size_t)cs * (mr + 1) * 4));
    CK(ensure(c, c->pcg_pc, (size_t)cs * mp * 4));
    CK(ensure(c, c->pcg_push, (size_t)cs * mr * 16 * 4));
    CK(ensure(c, c->pcg_npush, 32 * 4));   // npush[16] | incoming halo rows nin[16]
    if (c->pcg_mask.bytes < (size_t)mu * 4) {
      CK(ensure(c, c->pcg_mask, (size_t)mu * 4));
      CK(cudaMemsetAsync(c->pcg_mask.p, 0, (size_t)mu * 4, c->st));   // kept zero by k_pcg_lists
    }
  }
  {
    PostArgs pa;
    pa.row_ptr = c->row_ptr.as<int32_t>(); pa.col = c->col.as<int32_t>(); pa.row_of = c->row_of.as<int32_t>();
    pa.m = m; pa.upper_of = c->upper_of.as<int32_t>(); pa.lower_of = c->lower_of.as<int32_t>();
    pa.ulist = c->ulist.as<int2>(); pa.ucount = reinterpret_cast<unsigned long long*>(info + 7);
    pa.nnz = nnz; pa.ul_blocks = nnz > 0 ? std::min<int64_t>(grid, (nnz + 255) / 256) : 0;
    pa.part = c->part.as<int32_t>(); pa.cs = clu ? c->cl_size : 0;
    pa.mask = c->pcg_mask.as<uint32_t>(); pa.nin = c->pcg_npush.as<int32_t>() + 16;
    pa.nseg = c->nseg; pa.seg_nodes = tup; pa.K = K; pa.n_nbr = c->prm.n_nbr; pa.nf = c->nf;
    pa.nbr = c->nbr.as<int32_t>(); pa.fidx = c->fidx.as<int32_t>();
    pa.seg_slot = c->seg_slot.as<int32_t>(); pa.edge_slot = c->edge_slot.as<int32_t>();
    pa.feat_slot = c->feat_slot.as<int32_t>(); pa.total = total;
    const int64_t blocks = pa.ul_blocks + pa.cs + (total + 255) / 256;
    if (blocks > 0) launch_pdl(k_pattern_post, dim3((unsigned)blocks), dim3(256), 0, c->st, pa);
  }
  count_launches(2);
  if (clu) {
    launch_pcg_prep(c->row_ptr.as<int32_t>(), c->col.as<int32_t>(), c->part.as<int32_t>(), c->cl_size, c->cl_max_rows,
                    c->cl_max_nnz, c->pcg_pptr.as<int32_t>(), c->pcg_pc.as<int32_t>(), c->pcg_push.as<int32_t>(),
                    c->pcg_npush.as<int32_t>(), c->pcg_mask.as<uint32_t>(), c->st, /*marked=*/true);
    count_launches(1);
  }
  CK(cudaGetLastError());
  // accumulators (K3 commits atomically into them) and solver buffers
  const size_t m6 = B * (size_t)mu;
  c->acc_floats = (size_t)nnz * (BB + 16 + BB) + ((m6 + 3) & ~(size_t)3) + 12 * (size_t)mu + m6;
  // accumulators: every finalisation re-zeroes what it read, so they need a memset only when
  // (re)allocated or after an assembly that did not reach its finalisation
  if (c->acc.bytes < c->acc_floats * 4 || c->energy.bytes < (size_t)kEnergyDoubles * 8) c->acc_dirty = true;
  CK(ensure(c, c->acc, c->acc_floats * 4));
  CK(ensure(c, c->energy, kEnergyDoubles * 8));
  if (c->acc_dirty) {
    CK(cudaMemsetAsync(c->acc.p, 0, c->acc.bytes, c->st));
    CK(cudaMemsetAsync(c->energy.p, 0, kEnergyDoubles * 8, c->st));
    c->acc_dirty = false;
  }
  CK(ensure(c, c->Hval, (size_t)nnz * BB * 4));
  CK(ensure(c, c->rhs, m6 * 4)); CK(ensure(c, c->Minv, (size_t)mu * BB * 4));
  CK(ensure(c, c->x, m6 * 4)); CK(ensure(c, c->r, m6 * 4)); CK(ensure(c, c->z, m6 * 4));
  CK(ensure(c, c->p, m6 * 4)); CK(ensure(c, c->Ap, m6 * 4));
  CK(ensure(c, c->pvec, 9 * m6 * 4));   // the grid PCG's pipelined vectors (also a fallback of the cluster one)
  CK(ensure(c, c->dots, (8 * (size_t)c->prm.pcg_iters + 16) * 8));   // dots | pose_y (grid PCG)
  c->pattern_valid = true;
  return cudaSuccess;
}

}  // namespace mis
