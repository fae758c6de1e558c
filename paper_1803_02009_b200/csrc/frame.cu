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
