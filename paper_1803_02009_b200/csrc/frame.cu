// frame.cu -- K1 frame prep and K2 Eq. 2 skinning.
#include "common.cuh"

namespace mis {

__device__ __forceinline__ bool depth_ok(float d) { return isfinite(d) && d > 0.0f; }

// K1: per pixel the back-projection Pi and the central-difference
// normal (reading A11), in fp64 -- the precision the association decisions are
// taken in (K3a) --:
//   N = normalize((q(x+1,y) - q(x-1,y)) x (q(x,y+1) - q(x,y-1))), flipped so N.q < 0;
// invalid (N = 0) on the border or next to an invalid depth.  Writes nmapd
// (N in fp64, D) and nmap (N rounded to fp32, D; D = 0 for an invalid depth).
// HBM-bound: 4 B read (+ neighbours from L1/L2), 48 B written per pixel.
__global__ void __launch_bounds__(256) k_frame_prep(FrameView f, float4* __restrict__ nmap, double4* __restrict__ nmapd) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= f.W || y >= f.H) return;
  const int W = f.W;
  const float* D = f.depth;
  const float c = __ldg(D + y * W + x);
  double N[3] = {0.0, 0.0, 0.0};
  bool dv = depth_ok(c), nv = false;
  if (dv && x > 0 && y > 0 && x < W - 1 && y < f.H - 1) {
    const float l = __ldg(D + y * W + x - 1), r = __ldg(D + y * W + x + 1);
    const float u = __ldg(D + (y - 1) * W + x), d = __ldg(D + (y + 1) * W + x);
    if (depth_ok(l) && depth_ok(r) && depth_ok(u) && depth_ok(d)) {
      const double ax = ((x + 1) - f.cxd) * r / f.fxd - ((x - 1) - f.cxd) * l / f.fxd;
      const double ay = (y - f.cyd) * (double)r / f.fyd - (y - f.cyd) * (double)l / f.fyd;
      const double az = (double)r - (double)l;
      const double bx = (x - f.cxd) * (double)d / f.fxd - (x - f.cxd) * (double)u / f.fxd;
      const double by = ((y + 1) - f.cyd) * d / f.fyd - ((y - 1) - f.cyd) * u / f.fyd;
      const double bz = (double)d - (double)u;
      N[0] = ay * bz - az * by; N[1] = az * bx - ax * bz; N[2] = ax * by - ay * bx;
      const double len = sqrt(N[0] * N[0] + N[1] * N[1] + N[2] * N[2]);
      if (len >= 1e-12) {
        nv = true;
        for (int k = 0; k < 3; ++k) N[k] /= len;
        const double q[3] = {(x - f.cxd) * c / f.fxd, (y - f.cyd) * c / f.fyd, (double)c};
        if (N[0] * q[0] + N[1] * q[1] + N[2] * q[2] > 0) for (int k = 0; k < 3; ++k) N[k] = -N[k];
      } else {
        N[0] = N[1] = N[2] = 0.0;
      }
    }
  }
  const int p = y * W + x;
  nmap[p] = make_float4((float)N[0], (float)N[1], (float)N[2], dv ? c : 0.f);
  nmapd[p] = make_double4(N[0], N[1], N[2], dv ? (double)c : 0.0);
  (void)nv;
}

void launch_frame_prep(const FrameView& f, float4* nmap, double4* nmapd, cudaStream_t s) {
  dim3 blk(32, 8), grd((f.W + 31) / 32, (f.H + 7) / 8);
  launch_pdl(k_frame_prep, dim3(grd), dim3(blk), 0, s, f, nmap, nmapd);
}

// K2: Eq. 2 -- the k+1 nearest nodes of each query (ties to the
// lower id), w_j = 1 - |v - g_j| / d_max with d_max the distance to the
// (k+1)-th, normalised (d_max = 0 -> 1/k).  Output ids
// ascending (the canonical tuple order used by the K13 sort).  Brute force
// over all nodes staged through shared memory.
//
// A team of S lanes (S | 32) serves one query: lane l scans nodes l, l+S, ...
// (ascending, so its strict-< insertion keeps the lower id on equal distance),
// then the team merges its S sorted lists in k+1 rounds of a butterfly
// (d, id)-lexicographic min -- the same k+1 nodes the sequential scan picks.
// S is chosen so that nq * S fills the GPU: feature points (nq ~ 500) and lifted
// points (nq ~ 10^4) get 32 / 16 lanes, the full model (nq ~ 10^5+) one.
template <int K, int S>
__global__ void __launch_bounds__(256) k_skin(int64_t nq, const float* __restrict__ px, const float* __restrict__ py,
                                              const float* __restrict__ pz, int64_t sxyz, const float* __restrict__ g,
                                              int m, int32_t* __restrict__ idx, float* __restrict__ w, int64_t os) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ float4 sg[1024];
  const int tl = threadIdx.x % S;   // lane within the team
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / S;
  const bool act = i < nq;
  float vx = 0, vy = 0, vz = 0;
  if (act) { vx = px[i * sxyz]; vy = py[i * sxyz]; vz = pz[i * sxyz]; }
  float bd[K + 1];
  int bi[K + 1];
#pragma unroll
  for (int s = 0; s <= K; ++s) { bd[s] = INFINITY; bi[s] = 0x7fffffff; }
  for (int base = 0; base < m; base += 1024) {
    const int cnt = min(1024, m - base);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x)
      sg[t] = make_float4(g[3 * (base + t)], g[3 * (base + t) + 1], g[3 * (base + t) + 2], 0.f);
    __syncthreads();
    if (act) {
#pragma unroll 8
      for (int t = tl; t < cnt; t += S) {
        const float4 q = sg[t];
        const float dx = vx - q.x, dy = vy - q.y, dz = vz - q.z;
        const float d2 = dx * dx + dy * dy + dz * dz;
        const int id = base + t;
        if (d2 < bd[K]) {   // ids arrive ascending: equal distance keeps the lower id
          float cd = d2;
          int ci = id;
#pragma unroll
          for (int s = 0; s <= K; ++s) {
            if (cd < bd[s]) { float td = bd[s]; int ti = bi[s]; bd[s] = cd; bi[s] = ci; cd = td; ci = ti; }
          }
        }
      }
    }
  }
  if (S > 1) {   // merge the team's sorted lists: k+1 rounds of (d, id) min + pop
    float od[K + 1];
    int oi[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      float d = bd[0];
      int id = bi[0];
#pragma unroll
      for (int o = S / 2; o > 0; o >>= 1) {
        const float d2 = __shfl_xor_sync(0xffffffffu, d, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, id, o);
        if (d2 < d || (d2 == d && i2 < id)) { d = d2; id = i2; }
      }
      od[r] = d;
      oi[r] = id;
      const bool pop = bi[0] == id && bd[0] == d;
#pragma unroll
      for (int s = 0; s < K; ++s) { bd[s] = pop ? bd[s + 1] : bd[s]; bi[s] = pop ? bi[s + 1] : bi[s]; }
      if (pop) { bd[K] = INFINITY; bi[K] = 0x7fffffff; }
    }
#pragma unroll
    for (int s = 0; s <= K; ++s) { bd[s] = od[s]; bi[s] = oi[s]; }
  }
  if (!act || tl != 0) return;
  const float dmax = sqrtf(bd[K]);
  float ww[K];
  float sum = 0.f;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    ww[s] = dmax > 0.f ? 1.0f - sqrtf(bd[s]) / dmax : 1.0f / K;
    sum += ww[s];
  }
#pragma unroll
  for (int s = 0; s < K; ++s) ww[s] = sum > 0.f ? ww[s] / sum : 1.0f / K;
  // canonical order: ids ascending (insertion sort of K pairs)
#pragma unroll
  for (int a = 1; a < K; ++a)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (bi[b] < bi[b - 1]) {
        int ti = bi[b]; bi[b] = bi[b - 1]; bi[b - 1] = ti;
        float tw = ww[b]; ww[b] = ww[b - 1]; ww[b - 1] = tw;
      }
#pragma unroll
  for (int s = 0; s < K; ++s) { idx[s * os + i] = bi[s]; w[s * os + i] = ww[s]; }
}

// K2 over spatially coherent blocks of queries (the points of a sorted cell order: node regeneration,
// merged filter boxes): per 256-query block, the (k+1)-th smallest farthest-corner distance U from
// the block's bounding box to the nodes bounds every query's (k+1)-th nearest distance, so only the
// nodes whose distance to the box is <= U are candidates -- exact Eq. 2 (the same (d^2, id) order as
// k_skin) at a small fraction of the brute-force distances.  Falls back to all nodes when the
// candidate list overflows.  order (nullable): query q = order[i]; its output goes to q (out_at_q) or i.
constexpr int kBoxCand = 2048;
template <int K>
__global__ void __launch_bounds__(256) k_skin_boxed(int64_t nq, const uint32_t* __restrict__ order, int out_at_q,
                                                    const float* __restrict__ px, const float* __restrict__ py,
                                                    const float* __restrict__ pz, int64_t sxyz,
                                                    const float* __restrict__ g, int m, int32_t* __restrict__ idx,
                                                    float* __restrict__ w, int64_t os) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 cand[kBoxCand];
  __shared__ float red[6][8];
  __shared__ float sel[8][K + 1];
  __shared__ int ncand;
  __shared__ float U2s;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t i = (int64_t)blockIdx.x * 256 + t;
  const bool act = i < nq;
  const int64_t q = act ? (order ? (int64_t)order[i] : i) : 0;
  float v[3] = {0.f, 0.f, 0.f};
  if (act) { v[0] = px[q * sxyz]; v[1] = py[q * sxyz]; v[2] = pz[q * sxyz]; }
  float lo[3], hi[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = act ? v[c] : INFINITY;
    hi[c] = act ? v[c] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  }
  if (t == 0) ncand = 0;
  if (lane == 0) for (int c = 0; c < 3; ++c) { red[c][wid] = lo[c]; red[3 + c][wid] = hi[c]; }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = red[c][0]; hi[c] = red[3 + c][0];
    for (int ww = 1; ww < 8; ++ww) { lo[c] = fminf(lo[c], red[c][ww]); hi[c] = fmaxf(hi[c], red[3 + c][ww]); }
  }
  // U^2: the (k+1)-th smallest farthest-corner squared distance (thread, warp, block)
  float ub[K + 1];
#pragma unroll
  for (int s = 0; s <= K; ++s) ub[s] = INFINITY;
  for (int j = t; j < m; j += 256) {
    float u2 = 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float gc = g[3 * j + c], e = fmaxf(fabsf(gc - lo[c]), fabsf(gc - hi[c]));
      u2 += e * e;
    }
    if (u2 < ub[K]) {
      float cu = u2;
#pragma unroll
      for (int s = 0; s <= K; ++s) if (cu < ub[s]) { const float tt = ub[s]; ub[s] = cu; cu = tt; }
    }
  }
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    float mn = ub[0];
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) sel[wid][r] = mn;
    const unsigned who = __ballot_sync(0xffffffffu, ub[0] == mn);
    if (lane == __ffs(who) - 1) {
#pragma unroll
      for (int s = 0; s < K; ++s) ub[s] = ub[s + 1];
      ub[K] = INFINITY;
    }
  }
  __syncthreads();
  if (wid == 0) {   // the (k+1)-th smallest of the 8 warps' k+1 smallest
    constexpr int NV = 8 * (K + 1);
    float vv[3];
#pragma unroll
    for (int z = 0; z < 3; ++z) {
      const int qq = lane + 32 * z;
      vv[z] = qq < NV ? sel[qq / (K + 1)][qq % (K + 1)] : INFINITY;
    }
    float kth = INFINITY;
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      float mn = fminf(vv[0], fminf(vv[1], vv[2]));
      for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      kth = mn;
      bool popped = false;
#pragma unroll
      for (int z = 0; z < 3; ++z) {
        const unsigned hz = __ballot_sync(0xffffffffu, vv[z] == mn);
        if (!popped && hz) {
          if (lane == __ffs(hz) - 1) vv[z] = INFINITY;
          popped = true;
        }
      }
    }
    if (lane == 0) U2s = kth * (1.0f + 1e-5f) + 1e-6f;   // conservative against rounding
  }
  __syncthreads();
  const float U2 = U2s;
  for (int j = t; j < m; j += 256) {
    float l2 = 0.f, gj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gj[c] = g[3 * j + c];
      const float e = fmaxf(0.f, fmaxf(lo[c] - gj[c], gj[c] - hi[c]));
      l2 += e * e;
    }
    if (l2 <= U2) {   // appended in any order: the scan below sorts ties by id
      const int slot = atomicAdd(&ncand, 1);
      if (slot < kBoxCand) cand[slot] = make_float4(gj[0], gj[1], gj[2], __int_as_float(j));
    }
  }
  __syncthreads();
  if (!act) return;
  const int nc = ncand;
  float bd[K + 1];
  int bi[K + 1];
#pragma unroll
  for (int s = 0; s <= K; ++s) { bd[s] = INFINITY; bi[s] = 0x7fffffff; }
  auto ins = [&](float d2, int id) {
    if (d2 > bd[K] || (d2 == bd[K] && id >= bi[K])) return;
    float cd = d2;
    int ci = id;
#pragma unroll
    for (int s = 0; s <= K; ++s)
      if (cd < bd[s] || (cd == bd[s] && ci < bi[s])) {
        const float td = bd[s];
        const int ti = bi[s];
        bd[s] = cd; bi[s] = ci; cd = td; ci = ti;
      }
  };
  if (nc <= kBoxCand) {
    for (int qq = 0; qq < nc; ++qq) {
      const float4 c4 = cand[qq];
      const float dx = v[0] - c4.x, dy = v[1] - c4.y, dz = v[2] - c4.z;
      ins(dx * dx + dy * dy + dz * dz, __float_as_int(c4.w));
    }
  } else {
    for (int j = 0; j < m; ++j) {
      const float dx = v[0] - g[3 * j], dy = v[1] - g[3 * j + 1], dz = v[2] - g[3 * j + 2];
      ins(dx * dx + dy * dy + dz * dz, j);
    }
  }
  const float dmax = sqrtf(bd[K]);
  float ww[K];
  float sum = 0.f;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    ww[s] = dmax > 0.f ? 1.0f - sqrtf(bd[s]) / dmax : 1.0f / K;
    sum += ww[s];
  }
#pragma unroll
  for (int s = 0; s < K; ++s) ww[s] = sum > 0.f ? ww[s] / sum : 1.0f / K;
#pragma unroll
  for (int a = 1; a < K; ++a)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (bi[b] < bi[b - 1]) {
        int ti = bi[b]; bi[b] = bi[b - 1]; bi[b - 1] = ti;
        float tw = ww[b]; ww[b] = ww[b - 1]; ww[b - 1] = tw;
      }
  const int64_t o = out_at_q ? q : i;
#pragma unroll
  for (int s = 0; s < K; ++s) { idx[s * os + o] = bi[s]; w[s * os + o] = ww[s]; }
}

void launch_skin_boxed(int64_t nq, const uint32_t* order, int out_at_q, const float* px, const float* py,
                       const float* pz, int64_t sxyz, const float* g, int m, int K, int32_t* idx, float* w, int64_t os,
                       cudaStream_t s) {
  if (nq <= 0) return;
  const unsigned blocks = (unsigned)((nq + 255) / 256);
  switch (K) {
#define SB(KK) case KK: launch_pdl(k_skin_boxed<KK>, dim3(blocks), dim3(256), 0, s, nq, order, out_at_q, px, py, pz, \
                                   sxyz, g, m, idx, w, os); break;
    SB(1) SB(2) SB(3) SB(4) SB(5) SB(6) SB(7) SB(8)
#undef SB
    default: break;
  }
}

template <int K>
static void skin_k(int64_t nq, const float* px, const float* py, const float* pz, int64_t sxyz, const float* g, int m,
                   int32_t* idx, float* w, int64_t os, cudaStream_t s) {
  static int fill = 0;   // threads that fill the device (SMs x 2048)
  if (!fill) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    fill = sms * 2048;
  }
  int S = 1;
  while (S < 32 && nq * S < fill && S * 8 <= m) S *= 2;
  const int blocks = (int)((nq * S + 255) / 256);
  switch (S) {
#define SK(SS) case SS: launch_pdl(k_skin<K, SS>, dim3(blocks), dim3(256), 0, s, nq, px, py, pz, sxyz, g, m, idx, w, os); break;
    SK(1) SK(2) SK(4) SK(8) SK(16) SK(32)
#undef SK
    default: break;
  }
}

void launch_skin(int64_t nq, const float* px, const float* py, const float* pz, int64_t sxyz, const float* g, int m,
                 int K, int32_t* idx, float* w, int64_t os, cudaStream_t s) {
  if (nq <= 0) return;
  switch (K) {
#define SK(KK) case KK: skin_k<KK>(nq, px, py, pz, sxyz, g, m, idx, w, os, s); break;
    SK(1) SK(2) SK(3) SK(4) SK(5) SK(6) SK(7) SK(8)
#undef SK
    default: break;
  }
}

}  // namespace mis
