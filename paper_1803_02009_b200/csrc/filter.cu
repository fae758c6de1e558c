// filter.cu -- NEXT-1: Alg. 3 point filtering with the grid-box downsampling of P:597,
// readings A30-A34.  Per frame, after mis_fuse:
//
//   K14a k_cell_keys     one 63-bit key per point: (kx, ky, kz) = floor(v / s) (fp32 IEEE division, A30),
//                        21 bits per axis, x-major, plus the point's internal index
//   (CUB)                stable radix sort of (key, index): a cell's members become contiguous, in
//                        ascending internal index (the oracle's member order)
//   K14b k_cell_merge    one thread per sorted position; the cell's first position merges the cell
//                        (S:369 weighted averages, omega cap, max stamp, first member's id, A31) into the
//                        other model buffer set at that position and applies Alg. 3's deletion test (A32);
//                        keep flag 0 elsewhere
//   (CUB)                exclusive scan of the keep flags
//   K14c k_cell_compact  survivors -> the current buffer set in ascending cell-key order (A33)
//   K2   launch_skin     Eq. 2 skinning of the survivors against the current nodes (A34)
//
// HBM-bound: every pass is a streaming read / write of the point records (K14).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace mis {

namespace {

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return e_;          \
  } while (0)

constexpr int kAxisBits = 21;
constexpr int kAxisOff = 1 << (kAxisBits - 1);   // cell coordinates in [-2^20, 2^20)

__device__ __forceinline__ uint64_t axis_code(float v, float s, int* bad) {
  const float q = floorf(__fdiv_rn(v, s));   // fp32 IEEE division and floor: the oracle's decision (A30)
  if (!(q >= -(float)kAxisOff && q < (float)kAxisOff)) {   // out of range or non-finite
    atomicOr(bad, 1);
    return 0;
  }
  return (uint64_t)((int)q + kAxisOff);
}

__global__ void __launch_bounds__(256) k_cell_keys(ModelView md, float s, uint64_t* __restrict__ keys,
                                                   uint32_t* __restrict__ vals, int64_t* __restrict__ info) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= md.n) return;
  int* bad = reinterpret_cast<int*>(info + 3);
  const uint64_t kx = axis_code(md.px[i], s, bad), ky = axis_code(md.py[i], s, bad), kz = axis_code(md.pz[i], s, bad);
  keys[i] = (kx << (2 * kAxisBits)) | (ky << kAxisBits) | kz;
  vals[i] = (uint32_t)i;
}

struct MergeArgs {
  ModelView a;   // current model (read)
  ModelView b;   // other buffer set: merged cell at its first sorted position
  const uint64_t* keys;   // sorted
  const uint32_t* vals;   // sorted internal indices
  int32_t* keep;          // n: 1 at a surviving cell's first position, else 0
  int64_t* info;          // [0] survivors (K14c), [1] cells, [2] stable survivors, [3] bad-key flag
  int32_t frame, tau_time;
  float tau_weight, omega_max;
};

__global__ void __launch_bounds__(256) k_cell_merge(MergeArgs r) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = r.a.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool head = false, kept = false, stable = false;
  const bool bad = reinterpret_cast<const int*>(r.info + 3)[0] != 0;   // K14a flagged a key: keep nothing,
  if (i < n && bad) r.keep[i] = 0;                                     // the compaction then writes nothing
  if (i < n && !bad) {
    const uint64_t key = r.keys[i];
    head = (i == 0) || (r.keys[i - 1] != key);
    if (head) {
      int64_t e = i + 1;
      while (e < n && r.keys[e] == key) ++e;
      const ModelView& a = r.a;
      float wsum = 0.f;
      for (int64_t j = i; j < e; ++j) wsum += a.w[r.vals[j]];
      const bool weighted = wsum > 0.f;
      float vx = 0.f, vy = 0.f, vz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f, cr = 0.f, cg = 0.f, cb = 0.f, den = 0.f;
      int32_t t = INT_MIN;
      const uint32_t p0 = r.vals[i];
      for (int64_t j = i; j < e; ++j) {
        const uint32_t p = r.vals[j];
        const float wi = weighted ? a.w[p] : 1.f;
        vx = fmaf(wi, a.px[p], vx); vy = fmaf(wi, a.py[p], vy); vz = fmaf(wi, a.pz[p], vz);
        nx = fmaf(wi, a.nx[p], nx); ny = fmaf(wi, a.ny[p], ny); nz = fmaf(wi, a.nz[p], nz);
        cr = fmaf(wi, a.cr[p], cr); cg = fmaf(wi, a.cg[p], cg); cb = fmaf(wi, a.cb[p], cb);
        den += wi;
        t = max(t, a.stamp[p]);
      }
      const float om = fminf(wsum, r.omega_max);                                  // Eq. 15 cap
      // Alg. 3 line 3: delete iff t < frame - tau_time and omega < tau_weight (A32)
      const bool del = ((int64_t)t < (int64_t)r.frame - (int64_t)r.tau_time) && (om < r.tau_weight);
      kept = !del;
      stable = kept && om >= r.tau_weight;
      if (kept) {
        const float inv = 1.f / den;
        const float len2 = nx * nx + ny * ny + nz * nz;
        const ModelView& b = r.b;
        b.px[i] = vx * inv; b.py[i] = vy * inv; b.pz[i] = vz * inv;
        if (len2 > 0.f) {
          const float il = rsqrtf(len2);
          b.nx[i] = nx * il; b.ny[i] = ny * il; b.nz[i] = nz * il;
        } else {
          b.nx[i] = a.nx[p0]; b.ny[i] = a.ny[p0]; b.nz[i] = a.nz[p0];
        }
        b.cr[i] = cr * inv; b.cg[i] = cg * inv; b.cb[i] = cb * inv;
        b.w[i] = om;
        b.stamp[i] = t;
        b.ids[i] = a.ids[p0];
      }
    }
    r.keep[i] = kept ? 1 : 0;
  }
  // cells and stable survivors: one atomic per warp
  const unsigned hb = __ballot_sync(0xffffffffu, head), sb = __ballot_sync(0xffffffffu, stable);
  if ((threadIdx.x & 31) == 0) {
    if (hb) atomicAdd(reinterpret_cast<unsigned long long*>(r.info + 1), (unsigned long long)__popc(hb));
    if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(r.info + 2), (unsigned long long)__popc(sb));
  }
}

__global__ void __launch_bounds__(256) k_cell_compact(ModelView b, ModelView a, const int32_t* __restrict__ keep,
                                                      const int32_t* __restrict__ pos, int64_t* __restrict__ info) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = b.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) info[0] = (int64_t)pos[i] + keep[i];
  if (!keep[i]) return;
  const int64_t o = pos[i];
  a.px[o] = b.px[i]; a.py[o] = b.py[i]; a.pz[o] = b.pz[i];
  a.nx[o] = b.nx[i]; a.ny[o] = b.ny[i]; a.nz[o] = b.nz[i];
  a.cr[o] = b.cr[i]; a.cg[o] = b.cg[i]; a.cb[o] = b.cb[i];
  a.w[o] = b.w[i];
  a.stamp[o] = b.stamp[i];
  a.ids[o] = b.ids[i];
}

template <class F>
cudaError_t cub_call(Ctx* c, F f) {
  size_t need = 0;
  CK(f(nullptr, need));
  CK(ensure(c, c->cub_tmp, need + 256));
  size_t have = c->cub_tmp.bytes;
  return f(c->cub_tmp.p, have);
}

}  // namespace

// Enqueues K14a-c (3 launches; the caller's ProfScope counts them) and the two CUB passes on the
// context stream; info (4 x int64, zeroed here) receives [survivors, cells, stable, bad key].  With a
// bad key nothing is kept or written (the model is unchanged).  The caller reads info back, sets the
// model size and then skins the survivors (run_filter_skin).
cudaError_t run_filter(Ctx* c, float grid, int32_t frame, int32_t tau_time, float tau_weight, int64_t* info) {
  const int64_t n = c->n;
  CK(cudaMemsetAsync(info, 0, 32, c->st));
  if (n == 0) return cudaSuccess;
  CK(ensure(c, c->keys, n * 8)); CK(ensure(c, c->keys2, n * 8));
  CK(ensure(c, c->vals, n * 4)); CK(ensure(c, c->vals2, n * 4));
  CK(ensure(c, c->flags, n * 4)); CK(ensure(c, c->scan, n * 4));
  const int b = (int)((n + 255) / 256);
  ModelView A = model_view(c);
  ModelView B = model_view_of(c, c->mb[1 - c->cur]);
  B.n = n;
  launch_pdl(k_cell_keys, dim3(b), dim3(256), 0, c->st, A, grid, c->keys.as<uint64_t>(), c->vals.as<uint32_t>(), info);
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceRadixSort::SortPairs(t, s, c->keys.as<uint64_t>(), c->keys2.as<uint64_t>(), c->vals.as<uint32_t>(),
                                           c->vals2.as<uint32_t>(), (int)n, 0, 3 * kAxisBits, c->st);
  }));
  MergeArgs r{A, B, c->keys2.as<uint64_t>(), c->vals2.as<uint32_t>(), c->flags.as<int32_t>(), info, frame, tau_time,
              tau_weight, c->prm.omega_max};
  launch_pdl(k_cell_merge, dim3(b), dim3(256), 0, c->st, r);
  CK(cub_call(c, [&](void* t, size_t& s) {
    return cub::DeviceScan::ExclusiveSum(t, s, c->flags.as<int32_t>(), c->scan.as<int32_t>(), (int)n, c->st);
  }));
  launch_pdl(k_cell_compact, dim3(b), dim3(256), 0, c->st, B, A, c->flags.as<int32_t>(), c->scan.as<int32_t>(), info);
  return cudaGetLastError();
}

// Eq. 2 skinning of the first ns model points (the survivors) against the current nodes (A34).
void run_filter_skin(Ctx* c, int64_t ns) {
  ModelView A = model_view(c);
  launch_skin(ns, A.px, A.py, A.pz, 1, c->g.as<float>(), c->m, c->K, A.kidx, A.kw, c->cap, c->st);
}

}  // namespace mis
