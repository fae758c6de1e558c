// sort.cu -- K13: canonical kNN-tuple sort of the model, tuple segments and
// K3 work chunks; and the block-sparse (BSR) pattern of the normal equations
// with the slot tables K3 / K4 / K5 commit into.  Setup work, once per model
// change (order) and once per registration (pattern, since the feature tuples
// change every frame).  CUB radix sort / scan are library primitives here.
#include <cub/cub.cuh>

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

// key: exact big-endian packing of the ascending ids when K * bits <= 64,
// else (first id, 64-bits hash of the rest); equal tuples -> equal keys.
__global__ void k_tuple_keys(int64_t n, int64_t cap, const int32_t* kidx, int K, int bits, uint64_t* keys,
                             uint32_t* vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key = 0;
  if (K * bits <= 64) {
    for (int s = 0; s < K; ++s) key = (key << bits) | (uint64_t)kidx[s * cap + i];
  } else {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int s = 1; s < K; ++s) h = mix64(h ^ (uint64_t)kidx[s * cap + i]);
    key = ((uint64_t)kidx[i] << (64 - bits)) | (h >> bits);
  }
  keys[i] = key;
  vals[i] = (uint32_t)i;
}

// all model arrays in one launch: dst[i] = src[perm[i]]
__global__ void k_gather_model(int64_t n, const uint32_t* perm, ModelView a, ModelView b, int K) {
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

template <class T>
__global__ void k_gather(int64_t n, const uint32_t* perm, const T* src, T* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

template <class T>
static void gather(Ctx* c, const uint32_t* perm, const DBuf& src, const DBuf& dst, int64_t n, int slots) {
  const int b = (int)((n + 255) / 256);
  for (int s = 0; s < slots; ++s)
    k_gather<T><<<b, 256, 0, c->st>>>(n, perm, src.as<T>() + s * c->cap, dst.as<T>() + s * c->cap);
}

__global__ void k_seg_flags(int64_t n, int64_t cap, const int32_t* kidx, int K, int32_t* flags) {
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
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!flags[i]) return;
  const int32_t s = scan[i] - 1;
  seg_start[s] = (int32_t)i;
  for (int q = 0; q < K; ++q) seg_nodes[(int64_t)s * K + q] = kidx[q * cap + i];
  if (i == 0) seg_start[scan[n - 1]] = (int32_t)n;   // sentinel
}

__global__ void k_chunk_count(int64_t n, const int32_t* nseg_dev, const int32_t* seg_start, int32_t* cnt) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if (s >= *nseg_dev) { cnt[s] = 0; return; }
  const int32_t len = seg_start[s + 1] - seg_start[s];
  cnt[s] = (len + kChunk - 1) / kChunk;
}

__global__ void k_chunk_write(int64_t n, const int32_t* nseg_dev, const int32_t* seg_start, const int32_t* off,
                              int4* chunks) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n || s >= *nseg_dev) return;
  const int32_t a = seg_start[s], b = seg_start[s + 1];
  int32_t o = off[s] - (b - a + kChunk - 1) / kChunk;   // inclusive scan -> start
  for (int32_t p = a; p < b; p += kChunk) chunks[o++] = make_int4((int)s, p, min(b, p + kChunk), 0);
}

template <class F>
static cudaError_t cub_call(Ctx* c, F f) {
  size_t need = 0;
  CK(f(nullptr, need));
  CK(ensure(c, c->cub_tmp, need + 256));
  size_t have = c->cub_tmp.bytes;
  return f(c->cub_tmp.p, have);
}

cudaError_t build_order(Ctx* c) {
  const int64_t n = c->n;
  const int K = c->K;
  ModelBufs& A = c->mb[c->cur];
  ModelBufs& B = c->mb[1 - c->cur];
  if (n > 0) {
    CK(ensure(c, c->keys, n * 8)); CK(ensure(c, c->keys2, n * 8));
    CK(ensure(c, c->vals, n * 4)); CK(ensure(c, c->vals2, n * 4));
    const int bits = bits_for(c->m);
    const int b = (int)((n + 255) / 256);
    k_tuple_keys<<<b, 256, 0, c->st>>>(n, c->cap, A.kidx.as<int32_t>(), K, bits, c->keys.as<uint64_t>(),
                                        c->vals.as<uint32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceRadixSort::SortPairs(t, s, c->keys.as<uint64_t>(), c->keys2.as<uint64_t>(),
                                             c->vals.as<uint32_t>(), c->vals2.as<uint32_t>(), (int)n, 0, K * bits <= 64 ? K * bits : 64, c->st);
    }));
    k_gather_model<<<b, 256, 0, c->st>>>(n, c->vals2.as<uint32_t>(), model_view(c), model_view_of(c, B), K);
    CK(cudaGetLastError());
    c->cur = 1 - c->cur;
  }
  ModelBufs& S = c->mb[c->cur];
  // segments and chunks, sized by the upper bound n: one host readback at the end
  c->nseg = 0;
  c->nchunk = 0;
  if (n > 0) {
    CK(ensure(c, c->flags, n * 4)); CK(ensure(c, c->scan, n * 4));
    CK(ensure(c, c->seg_start, (n + 1) * 4));
    CK(ensure(c, c->seg_nodes, (size_t)n * K * 4));
    CK(ensure(c, c->chunk_off, (n + 1) * 4));
    CK(ensure(c, c->chunks, (size_t)n * 16));
    const int b = (int)((n + 255) / 256);
    k_seg_flags<<<b, 256, 0, c->st>>>(n, c->cap, S.kidx.as<int32_t>(), K, c->flags.as<int32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceScan::InclusiveSum(t, s, c->flags.as<int32_t>(), c->scan.as<int32_t>(), (int)n, c->st);
    }));
    const int32_t* nseg_dev = c->scan.as<int32_t>() + n - 1;
    k_seg_write<<<b, 256, 0, c->st>>>(n, c->cap, S.kidx.as<int32_t>(), K, c->flags.as<int32_t>(),
                                      c->scan.as<int32_t>(), c->seg_start.as<int32_t>(), c->seg_nodes.as<int32_t>());
    k_chunk_count<<<b, 256, 0, c->st>>>(n, nseg_dev, c->seg_start.as<int32_t>(), c->flags.as<int32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceScan::InclusiveSum(t, s, c->flags.as<int32_t>(), c->chunk_off.as<int32_t>(), (int)n, c->st);
    }));
    k_chunk_write<<<b, 256, 0, c->st>>>(n, nseg_dev, c->seg_start.as<int32_t>(), c->chunk_off.as<int32_t>(),
                                        c->chunks.as<int4>());
    int32_t cnt[2] = {0, 0};
    CK(cudaMemcpyAsync(&cnt[0], nseg_dev, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&cnt[1], c->chunk_off.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->nseg = cnt[0];
    c->nchunk = cnt[1];
    CK(cudaGetLastError());
  }
  c->dirty = false;
  c->pattern_valid = false;
  return cudaSuccess;
}

// ---------------------------------------------------------------- pattern
// (row, col) key with sb = bits_for(m) bits per index: radix sorts need only 2 sb + 1 bits
__device__ __forceinline__ uint64_t pkey(int r, int col, int sb) { return ((uint64_t)(uint32_t)r << sb) | (uint32_t)col; }
constexpr uint64_t kNoKey = ~0ull;

// candidates: [segment pairs nseg*P][edges m*n_nbr][feature pairs nf*P][diagonal m]; 2 keys each
__global__ void k_candidates(int64_t nseg, const int32_t* seg_nodes, int K, int m, int n_nbr, const int32_t* nbr,
                             int nf, const int32_t* fidx, uint64_t* keys, int64_t total, int sb) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int P = K * (K + 1) / 2;
  const int64_t ns = nseg * P, ne = (int64_t)m * n_nbr, nfp = (int64_t)nf * P;
  int a = -1, b = -1;
  if (t < ns) {
    const int64_t s = t / P;
    int p = (int)(t % P), j = 0;
    while (p >= K - j) { p -= K - j; ++j; }
    a = seg_nodes[s * K + j];
    b = seg_nodes[s * K + j + p];
  } else if (t < ns + ne) {
    const int64_t e = t - ns;
    const int l = nbr[e];
    if (l >= 0) { a = (int)(e / n_nbr); b = l; }
  } else if (t < ns + ne + nfp) {
    const int64_t e = t - ns - ne;
    const int64_t f = e / P;
    int p = (int)(e % P), j = 0;
    while (p >= K - j) { p -= K - j; ++j; }
    a = fidx[(int64_t)j * nf + f];
    b = fidx[(int64_t)(j + p) * nf + f];
  } else {
    a = b = (int)(t - ns - ne - nfp);
  }
  if (a < 0) { keys[2 * t] = kNoKey; keys[2 * t + 1] = kNoKey; return; }
  keys[2 * t] = pkey(a, b, sb);
  keys[2 * t + 1] = (a != b) ? pkey(b, a, sb) : kNoKey;
}

__global__ void k_unique_flags(int64_t n, const uint64_t* k, int32_t* f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  f[i] = (k[i] != kNoKey) && (i == 0 || k[i] != k[i - 1]);
}

__global__ void k_unique_write(int64_t n, const uint64_t* k, const int32_t* f, const int32_t* pos, uint64_t* u,
                               int64_t* nnz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (f[i]) u[pos[i] - 1] = k[i];
  if (i == n - 1) *nnz = pos[i];
}

__device__ __forceinline__ int64_t find_key(const uint64_t* u, int64_t nnz, uint64_t key) {
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (u[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < nnz && u[lo] == key) ? lo : -1;
}

__global__ void k_rows(int64_t cap, const int64_t* nnz_dev, const uint64_t* u, int m, int32_t* row_ptr, int32_t* col,
                       int32_t* upper_of, int32_t* lower_of, int32_t* diag_pos, int sb) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nnz = *nnz_dev;
  if (e >= nnz || e >= cap) return;
  const int r = (int)(u[e] >> sb), cc = (int)(u[e] & ((1ull << sb) - 1));
  col[e] = cc;
  const int rp = (e == 0) ? -1 : (int)(u[e - 1] >> sb);
  for (int q = rp + 1; q <= r; ++q) row_ptr[q] = (int32_t)e;
  if (e == nnz - 1)
    for (int q = r + 1; q <= m; ++q) row_ptr[q] = (int32_t)nnz;
  if (r == cc) diag_pos[r] = (int32_t)e;
  upper_of[e] = (r <= cc) ? (int32_t)e : (int32_t)find_key(u, nnz, pkey(cc, r, sb));
  if (r == cc) lower_of[e] = -1;                       // diagonal: no mirror
  else if (r > cc) lower_of[upper_of[e]] = (int32_t)e;   // the upper partner's mirror
}

__global__ void k_slots(int64_t nseg, const int32_t* seg_nodes, int K, int m, int n_nbr, const int32_t* nbr, int nf,
                        const int32_t* fidx, const uint64_t* u, const int64_t* nnz_dev, int32_t* seg_slot, int32_t* edge_slot,
                        int32_t* feat_slot, int64_t total, int sb) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nnz = *nnz_dev;
  if (t >= total) return;
  const int P = K * (K + 1) / 2;
  const int64_t ns = nseg * P, ne = (int64_t)m * n_nbr, nfp = (int64_t)nf * P;
  if (t < ns) {
    const int64_t s = t / P;
    int p = (int)(t % P), j = 0;
    while (p >= K - j) { p -= K - j; ++j; }
    seg_slot[t] = (int32_t)find_key(u, nnz, pkey(seg_nodes[s * K + j], seg_nodes[s * K + j + p], sb));
  } else if (t < ns + ne) {
    const int64_t e = t - ns;
    const int l = nbr[e], j = (int)(e / n_nbr);
    edge_slot[e] = (l >= 0) ? (int32_t)find_key(u, nnz, pkey(min(j, l), max(j, l), sb)) : -1;
  } else if (t < ns + ne + nfp) {
    const int64_t e = t - ns - ne;
    const int64_t f = e / P;
    int p = (int)(e % P), j = 0;
    while (p >= K - j) { p -= K - j; ++j; }
    feat_slot[e] = (int32_t)find_key(u, nnz, pkey(fidx[(int64_t)j * nf + f], fidx[(int64_t)(j + p) * nf + f], sb));
  }
}

// contributions of the chunk records: (key = BSR slot or node, value = chunk * W + position)
__global__ void k_contrib(int64_t nchunk, const int4* chunks, const int32_t* table, int W, int32_t* key,
                          int32_t* val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nchunk * W) return;
  const int64_t c = t / W;
  const int p = (int)(t % W);
  key[t] = table[(int64_t)chunks[c].x * W + p];
  val[t] = (int32_t)t;
}

// CSR row pointers over nbins from sorted keys
__global__ void k_csr_ptr(int64_t n, const int32_t* key, const int64_t* nbins_dev, int nbins_host, int32_t* ptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nbins = nbins_dev ? (int)*nbins_dev : nbins_host;
  const int k = key[i];
  const int kp = (i == 0) ? -1 : key[i - 1];
  for (int b = kp + 1; b <= k; ++b) ptr[b] = (int32_t)i;
  if (i == n - 1)
    for (int b = k + 1; b <= nbins; ++b) ptr[b] = (int32_t)n;
}

// nbins: upper bound (host); nbins_dev: exact count on the device (or null: nbins is exact)
static cudaError_t build_contrib(Ctx* c, const int32_t* table, int W, int nbins, const int64_t* nbins_dev, DBuf& ptr,
                                 DBuf& src) {
  const int64_t n = c->nchunk * W;
  CK(ensure(c, ptr, (size_t)(nbins + 1) * 4));
  CK(ensure(c, src, (size_t)n * 4 + 16));
  if (n == 0) return cudaMemsetAsync(ptr.p, 0, (size_t)(nbins + 1) * 4, c->st);
  CK(ensure(c, c->ck_key, n * 4)); CK(ensure(c, c->ck_val, n * 4));
  CK(ensure(c, c->ck_key2, n * 4));
  const int b = (int)((n + 255) / 256);
  k_contrib<<<b, 256, 0, c->st>>>(c->nchunk, c->chunks.as<int4>(), table, W, c->ck_key.as<int32_t>(),
                                  c->ck_val.as<int32_t>());
  int bits = 1;
  while ((1ll << bits) <= (int64_t)nbins) ++bits;
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceRadixSort::SortPairs(t, s, c->ck_key.as<int32_t>(), c->ck_key2.as<int32_t>(),
                                           c->ck_val.as<int32_t>(), src.as<int32_t>(), (int)n, 0, bits, c->st);
  }));
  k_csr_ptr<<<b, 256, 0, c->st>>>(n, c->ck_key2.as<int32_t>(), nbins_dev, nbins, ptr.as<int32_t>());
  return cudaGetLastError();
}

cudaError_t build_pattern(Ctx* c) {
  const int K = c->K, P = K * (K + 1) / 2;
  const int64_t total = c->nseg * P + (int64_t)c->m * c->prm.n_nbr + (int64_t)c->nf * P + c->m;
  const int64_t nk = 2 * total;
  const int sb = bits_for(c->m);
  CK(ensure(c, c->ckeys, nk * 8)); CK(ensure(c, c->ckeys2, nk * 8));
  CK(ensure(c, c->uflag, nk * 4)); CK(ensure(c, c->upos, nk * 4));
  CK(ensure(c, c->nnz_dev, 64));
  const int bt = (int)((total + 255) / 256), bk = (int)((nk + 255) / 256);
  k_candidates<<<bt, 256, 0, c->st>>>(c->nseg, c->seg_nodes.as<int32_t>(), K, c->m, c->prm.n_nbr,
                                      c->nbr.as<int32_t>(), c->nf, c->fidx.as<int32_t>(), c->ckeys.as<uint64_t>(), total, sb);
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceRadixSort::SortKeys(t, s, c->ckeys.as<uint64_t>(), c->ckeys2.as<uint64_t>(), (int)nk, 0, 2 * sb + 1, c->st);
  }));
  k_unique_flags<<<bk, 256, 0, c->st>>>(nk, c->ckeys2.as<uint64_t>(), c->uflag.as<int32_t>());
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceScan::InclusiveSum(t, s, c->uflag.as<int32_t>(), c->upos.as<int32_t>(), (int)nk, c->st);
  }));
  CK(ensure(c, c->ukeys, nk * 8));
  k_unique_write<<<bk, 256, 0, c->st>>>(nk, c->ckeys2.as<uint64_t>(), c->uflag.as<int32_t>(), c->upos.as<int32_t>(),
                                        c->ukeys.as<uint64_t>(), c->nnz_dev.as<int64_t>());
  int64_t nnz = nk;   // upper bound until the single readback below
  if (c->world > 1) {
    // union of the ranks' patterns: every rank ends with the same sorted unique keys
    CK(cudaMemcpyAsync(&nnz, c->nnz_dev.p, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    int64_t mx = nnz;
    int64_t* dmx = c->nnz_dev.as<int64_t>() + 1;
    CK(cudaMemcpyAsync(dmx, &mx, 8, cudaMemcpyHostToDevice, c->st));
    CK(nccl_allreduce_max_i64(c, dmx, 1));
    CK(cudaMemcpyAsync(&mx, dmx, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    const int64_t all = mx * c->world;
    // send buffer: local unique keys padded to mx with kNoKey (ckeys2 is free now)
    CK(ensure(c, c->ckeys2, mx * 8));
    CK(cudaMemcpyAsync(c->ckeys2.p, c->ukeys.p, nnz * 8, cudaMemcpyDeviceToDevice, c->st));
    if (mx > nnz) CK(cudaMemsetAsync(c->ckeys2.as<uint64_t>() + nnz, 0xff, (mx - nnz) * 8, c->st));
    CK(ensure(c, c->ckeys, all * 8));
    CK(nccl_allgather_u64(c, c->ckeys2.as<uint64_t>(), c->ckeys.as<uint64_t>(), (size_t)mx));
    CK(ensure(c, c->ckeys2, all * 8));
    CK(ensure(c, c->uflag, all * 4)); CK(ensure(c, c->upos, all * 4)); CK(ensure(c, c->ukeys, all * 8));
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceRadixSort::SortKeys(t, s, c->ckeys.as<uint64_t>(), c->ckeys2.as<uint64_t>(), (int)all, 0, 2 * sb + 1, c->st);
    }));
    const int ba = (int)((all + 255) / 256);
    k_unique_flags<<<ba, 256, 0, c->st>>>(all, c->ckeys2.as<uint64_t>(), c->uflag.as<int32_t>());
    CK(cub_call(c, [&](void* t, size_t& s) {
      return cub::DeviceScan::InclusiveSum(t, s, c->uflag.as<int32_t>(), c->upos.as<int32_t>(), (int)all, c->st);
    }));
    k_unique_write<<<ba, 256, 0, c->st>>>(all, c->ckeys2.as<uint64_t>(), c->uflag.as<int32_t>(),
                                          c->upos.as<int32_t>(), c->ukeys.as<uint64_t>(), c->nnz_dev.as<int64_t>());
    nnz = all;
  }
  const int64_t cap = nnz;   // upper bound of the unique count
  CK(ensure(c, c->row_ptr, (c->m + 1) * 4));
  CK(ensure(c, c->col, cap * 4)); CK(ensure(c, c->upper_of, cap * 4)); CK(ensure(c, c->lower_of, cap * 4));
  CK(ensure(c, c->diag_pos, c->m * 4));
  CK(ensure(c, c->part, 32 * 4));
  PlanOut* plan = reinterpret_cast<PlanOut*>(c->nnz_dev.as<int64_t>() + 2);
  const int bn = (int)((cap + 255) / 256);
  k_rows<<<bn, 256, 0, c->st>>>(cap, c->nnz_dev.as<int64_t>(), c->ukeys.as<uint64_t>(), c->m, c->row_ptr.as<int32_t>(),
                                c->col.as<int32_t>(), c->upper_of.as<int32_t>(), c->lower_of.as<int32_t>(),
                                c->diag_pos.as<int32_t>(), sb);
  launch_plan_cluster(c->row_ptr.as<int32_t>(), c->m, 16, plan, c->part.as<int32_t>(), c->st);
  CK(ensure(c, c->seg_slot, (c->nseg * P + 1) * 4));
  CK(ensure(c, c->edge_slot, ((int64_t)c->m * c->prm.n_nbr + 1) * 4));
  CK(ensure(c, c->feat_slot, ((int64_t)c->nf * P + 1) * 4));
  k_slots<<<bt, 256, 0, c->st>>>(c->nseg, c->seg_nodes.as<int32_t>(), K, c->m, c->prm.n_nbr, c->nbr.as<int32_t>(),
                                 c->nf, c->fidx.as<int32_t>(), c->ukeys.as<uint64_t>(), c->nnz_dev.as<int64_t>(),
                                 c->seg_slot.as<int32_t>(), c->edge_slot.as<int32_t>(), c->feat_slot.as<int32_t>(), total,
                                 sb);
  CK(cudaGetLastError());
  // chunk records and their (deterministic, sorted) contribution lists
  CK(ensure(c, c->records, (size_t)c->nchunk * rec_stride(K) * 4 + 16));
  CK(build_contrib(c, c->seg_slot.as<int32_t>(), P, (int)cap, c->nnz_dev.as<int64_t>(), c->slot_ptr, c->slot_src));
  CK(build_contrib(c, c->seg_nodes.as<int32_t>(), K, c->m, nullptr, c->node_ptr, c->node_src));
  // the single host readback of the pattern build: nnz and the cluster plan
  struct { int64_t nnz, pad; PlanOut plan; } info;
  CK(cudaMemcpyAsync(&info, c->nnz_dev.p, sizeof(info), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  nnz = info.nnz;
  c->nnzb = nnz;
  c->cl_size = info.plan.cl_size;
  c->cl_max_rows = info.plan.max_rows;
  c->cl_max_nnz = info.plan.max_nnz;
  c->cl_smem = (size_t)info.plan.smem;
  // accumulators and solver buffers
  const size_t m6 = 6 * (size_t)c->m;
  c->acc_floats = (size_t)nnz * (36 + 16 + 36) + m6 + 12 * (size_t)c->m + m6;
  CK(ensure(c, c->acc, c->acc_floats * 4));
  CK(ensure(c, c->energy, 8 * 8));
  CK(ensure(c, c->Hval, (size_t)nnz * 36 * 4));
  CK(ensure(c, c->rhs, m6 * 4)); CK(ensure(c, c->Minv, (size_t)c->m * 36 * 4));
  CK(ensure(c, c->x, m6 * 4)); CK(ensure(c, c->r, m6 * 4)); CK(ensure(c, c->z, m6 * 4));
  CK(ensure(c, c->p, m6 * 4)); CK(ensure(c, c->Ap, m6 * 4));
  CK(ensure(c, c->dots, (2 * (size_t)c->prm.pcg_iters + 8) * 8));
  c->pattern_valid = true;
  return cudaSuccess;
}

}  // namespace mis
