// fuse.cu -- K9 final warp (Alg. 2 Step 2), K10/K11 point-to-depth registration
// and weighted-average fusion (Alg. 1, Eq. 12-15), K12 Group-2 lift (Alg. 2 Step 3).
// All per-point / per-pixel, HBM-bound; decisions in fp64 (cheap here) so the
// exclusive per-pixel winner matches the oracle outside 1e-8 mm key ties.
#include "common.cuh"

namespace mis {

__device__ __forceinline__ bool dok(float d) { return isfinite(d) && d > 0.0f; }

// K9: x_hat = sum_j w_j (R_j (v - g_j) + g_j + t_j), n = normalize(sum_j w_j R_j n) (Eq. 1, A_j = R_j)
// AFF (NEXT-4, A43): the node matrices are general A_j, normals warp by A_j^-T (A_j if |det| < 1e-9)
template <int K, bool AFF = false>
__global__ void __launch_bounds__(256) k_warp_model(ModelView md, NodeView nd, FrameView fr, float* xyz_cam,
                                                   float* nrm_cam) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= md.n) return;
  float v[3] = {md.px[i], md.py[i], md.pz[i]}, n[3] = {md.nx[i], md.ny[i], md.nz[i]};
  float w[K], W = 0.f;
#pragma unroll
  for (int s = 0; s < K; ++s) { w[s] = md.kw[s * md.cap + i]; W += w[s]; }
  if (W > 0.f) {
    float xh[3] = {0, 0, 0}, mh[3] = {0, 0, 0};
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const float* N = nd.node32 + 16 * md.kidx[s * md.cap + i];
      const float wn = w[s] / W;
      const float d[3] = {v[0] - N[12], v[1] - N[13], v[2] - N[14]};
#pragma unroll
      for (int r = 0; r < 3; ++r)
        xh[r] += wn * (N[3 * r] * d[0] + N[3 * r + 1] * d[1] + N[3 * r + 2] * d[2] + N[12 + r] + N[9 + r]);
      float C[9];
      if constexpr (AFF) {   // cofactors / det
        C[0] = N[4] * N[8] - N[5] * N[7]; C[1] = N[5] * N[6] - N[3] * N[8]; C[2] = N[3] * N[7] - N[4] * N[6];
        C[3] = N[2] * N[7] - N[1] * N[8]; C[4] = N[0] * N[8] - N[2] * N[6]; C[5] = N[1] * N[6] - N[0] * N[7];
        C[6] = N[1] * N[5] - N[2] * N[4]; C[7] = N[2] * N[3] - N[0] * N[5]; C[8] = N[0] * N[4] - N[1] * N[3];
        const float det = N[0] * C[0] + N[1] * C[1] + N[2] * C[2];
        if (fabsf(det) < 1e-9f) {
#pragma unroll
          for (int q = 0; q < 9; ++q) C[q] = N[q];
        } else {
#pragma unroll
          for (int q = 0; q < 9; ++q) C[q] /= det;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 9; ++q) C[q] = N[q];
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) mh[r] += wn * (C[3 * r] * n[0] + C[3 * r + 1] * n[1] + C[3 * r + 2] * n[2]);
    }
    const float ml = sqrtf(mh[0] * mh[0] + mh[1] * mh[1] + mh[2] * mh[2]);
    if (ml >= 1e-12f) {
      for (int r = 0; r < 3; ++r) { v[r] = xh[r]; n[r] = mh[r] / ml; }
      md.px[i] = v[0]; md.py[i] = v[1]; md.pz[i] = v[2];
      md.nx[i] = n[0]; md.ny[i] = n[1]; md.nz[i] = n[2];
    }
  }
  if (xyz_cam || nrm_cam) {
    double Rd[9], Td[3];
    frame_pose(fr, Rd, Td);   // the refined pose after a joint registration (NEXT-2)
    float R[9], T[3];
    for (int q = 0; q < 9; ++q) R[q] = (float)Rd[q];
    for (int q = 0; q < 3; ++q) T[q] = (float)Td[q];
    if (xyz_cam)
      for (int r = 0; r < 3; ++r) xyz_cam[3 * i + r] = R[3 * r] * v[0] + R[3 * r + 1] * v[1] + R[3 * r + 2] * v[2] + T[r];
    if (nrm_cam)
      for (int r = 0; r < 3; ++r) nrm_cam[3 * i + r] = R[3 * r] * n[0] + R[3 * r + 1] * n[1] + R[3 * r + 2] * n[2];
  }
}

void launch_warp_model(int K, const ModelView& md, const NodeView& nd, const FrameView& fr, float* xyz_cam,
                       float* nrm_cam, cudaStream_t s, bool affine) {
  if (md.n <= 0) return;
  const int b = (int)((md.n + 255) / 256);
  if (affine) {
    switch (K) {
#define WA(KK) case KK: launch_pdl(k_warp_model<KK, true>, dim3(b), dim3(256), 0, s, md, nd, fr, xyz_cam, nrm_cam); break;
      WA(1) WA(2) WA(3) WA(4)
#undef WA
      default: break;
    }
    return;
  }
  switch (K) {
#define WK(KK) case KK: launch_pdl(k_warp_model<KK>, dim3(b), dim3(256), 0, s, md, nd, fr, xyz_cam, nrm_cam); break;
    WK(1) WK(2) WK(3) WK(4) WK(5) WK(6) WK(7) WK(8)
#undef WK
    default: break;
  }
}

// Reading A26: g_j += t_j, then R_j = I, t_j = 0.
__global__ void k_advance_nodes(NodeView nd, float* g) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nd.m) return;
  double* Rt = nd.Rt64 + 12 * j;
  float* n32 = nd.node32 + 16 * j;
  for (int c = 0; c < 3; ++c) {
    const float gn = (float)((double)g[3 * j + c] + Rt[9 + c]);
    g[3 * j + c] = gn;
    n32[12 + c] = gn;
  }
  for (int i = 0; i < 12; ++i) Rt[i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
  for (int i = 0; i < 12; ++i) n32[i] = (float)Rt[i];
}

void launch_advance_nodes(const NodeView& nd, float* g, cudaStream_t s) {
  if (nd.m <= 0) return;
  launch_pdl(k_advance_nodes, dim3((nd.m + 255) / 256), dim3(256), 0, s, nd, g);
}

// fp64 normal at a pixel from the five depths (reading A11); false if invalid
// (N, q) at pixel (px, py) from the fp64 normal map of K1 (central differences, reading A11)
__device__ __forceinline__ bool normal_map64(const FrameView& f, int px, int py, double* N, double* q) {
  const double4 nm = f.nmapd[py * f.W + px];
  if (!(nm.w > 0)) return false;
  q[0] = (px - f.cxd) * nm.w / f.fxd; q[1] = (py - f.cyd) * nm.w / f.fyd; q[2] = nm.w;
  if (nm.x == 0 && nm.y == 0 && nm.z == 0) return false;
  N[0] = nm.x; N[1] = nm.y; N[2] = nm.z;
  return true;
}


// K10: Alg. 1 gates + exclusive registration by 64-bit atomicMin
// of ((|dz| / tz quantised to 32 bits) << 32 | point index) per pixel (reading A19).  The
// quantum is tz / 2^32 (2.3e-9 mm at tz = 10 mm) for every gate width, no overflow since |dz| < tz.
__global__ void __launch_bounds__(256) k_fuse_register(FuseArgs a) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && a.n_reg) *a.n_reg = 0;   // counted later by the lift count
  if (i >= a.md.n) return;
  const FrameView& f = a.fr;
  double Rd[9], Td[3];
  frame_pose(f, Rd, Td);   // the refined pose after a joint registration (NEXT-2)
  const double v[3] = {a.md.px[i], a.md.py[i], a.md.pz[i]}, n[3] = {a.md.nx[i], a.md.ny[i], a.md.nz[i]};
  double vt[3], nt[3];
  for (int r = 0; r < 3; ++r) {
    vt[r] = Rd[3 * r] * v[0] + Rd[3 * r + 1] * v[1] + Rd[3 * r + 2] * v[2] + Td[r];
    nt[r] = Rd[3 * r] * n[0] + Rd[3 * r + 1] * n[1] + Rd[3 * r + 2] * n[2];
  }
  uint8_t why = 0;
  int32_t pix = -1;
  if (vt[2] > 0) {
    why |= 1;
    const double fu = floor(f.fxd * vt[0] / vt[2] + f.cxd + 0.5), fv = floor(f.fyd * vt[1] / vt[2] + f.cyd + 0.5);
    if (fu >= 0 && fv >= 0 && fu < f.W && fv < f.H) {
      why |= 2;
      const int px = (int)fu, py = (int)fv;
      const double D = f.nmapd[py * f.W + px].w;   // the depth (0: invalid), from K1
      double N[3], q[3];
      if (D > 0) {
        why |= 4;
        if (normal_map64(f, px, py, N, q)) {
          why |= 8;
          const double dz = fabs(vt[2] - D);
          if (dz < a.tz) {
            why |= 16;
            if (nt[0] * N[0] + nt[1] * N[1] + nt[2] * N[2] > a.cos_delta) {
              why |= 32;
              pix = py * f.W + px;
              const unsigned long long key =
                  ((unsigned long long)(dz * a.key_scale) << 32) | (unsigned long long)(a.rank_tag | (uint32_t)i);
              atomicMin(a.pixkey + pix, key);
            }
          }
        }
      }
    }
  }
  a.pix[i] = pix;
  if (a.why) a.why[i] = why;
}

void launch_fuse_register(const FuseArgs& a, cudaStream_t s) {
  if (a.md.n <= 0) return;
  launch_pdl(k_fuse_register, dim3((int)((a.md.n + 255) / 256)), dim3(256), 0, s, a);
}

// K11: Eq. 12-15 on each pixel's winner; 3-D weighted average (reading A21)
__global__ void __launch_bounds__(256) k_fuse_apply(FuseArgs a) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.md.n) return;
  if (a.fits && !*a.fits) return;   // the lift would exceed the capacity: the model stays unchanged
  const int32_t pix = a.pix[i];
  if (pix < 0) return;
  if ((uint32_t)(a.pixkey[pix] & 0xffffffffull) != (a.rank_tag | (uint32_t)i)) return;
  const FrameView& f = a.fr;
  double Rd[9], Td[3];
  frame_pose(f, Rd, Td);   // the refined pose after a joint registration (NEXT-2)
  const int px = pix % f.W, py = pix / f.W;
  double N[3], q[3];
  normal_map64(f, px, py, N, q);
  const double v[3] = {a.md.px[i], a.md.py[i], a.md.pz[i]}, n[3] = {a.md.nx[i], a.md.ny[i], a.md.nz[i]};
  const double om = a.md.w[i];
  double pf[3], nf[3];
  for (int r = 0; r < 3; ++r) {
    const double vt = Rd[3 * r] * v[0] + Rd[3 * r + 1] * v[1] + Rd[3 * r + 2] * v[2] + Td[r];
    const double nt = Rd[3 * r] * n[0] + Rd[3 * r + 1] * n[1] + Rd[3 * r + 2] * n[2];
    pf[r] = (om * vt + q[r]) / (om + 1.0);      // Eq. 12 (its z) lifted to 3-D
    nf[r] = (om * nt + N[r]) / (om + 1.0);      // Eq. 14
  }
  const double nl = sqrt(nf[0] * nf[0] + nf[1] * nf[1] + nf[2] * nf[2]);
  for (int r = 0; r < 3; ++r) { nf[r] /= nl; pf[r] -= Td[r]; }
  float vo[3], no[3];
  for (int c = 0; c < 3; ++c) {   // back to world: R^T (p - T), R^T n
    vo[c] = (float)(Rd[c] * pf[0] + Rd[3 + c] * pf[1] + Rd[6 + c] * pf[2]);
    no[c] = (float)(Rd[c] * nf[0] + Rd[3 + c] * nf[1] + Rd[6 + c] * nf[2]);
  }
  a.md.px[i] = vo[0]; a.md.py[i] = vo[1]; a.md.pz[i] = vo[2];
  a.md.nx[i] = no[0]; a.md.ny[i] = no[1]; a.md.nz[i] = no[2];
  if (a.rgb_obs) {   // Eq. 13
    const float* c = a.rgb_obs + 3 * (int64_t)pix;
    a.md.cr[i] = (float)((om * a.md.cr[i] + c[0]) / (om + 1.0));
    a.md.cg[i] = (float)((om * a.md.cg[i] + c[1]) / (om + 1.0));
    a.md.cb[i] = (float)((om * a.md.cb[i] + c[2]) / (om + 1.0));
  }
  a.md.w[i] = (float)fmin(om + 1.0, a.omega_max);   // Eq. 15
  a.md.stamp[i] = a.frame_index;
}

void launch_fuse_apply(const FuseArgs& a, cudaStream_t s) {
  if (a.md.n <= 0) return;
  launch_pdl(k_fuse_apply, dim3((int)((a.md.n + 255) / 256)), dim3(256), 0, s, a);
}

// K12: valid (depth and normal), unregistered pixels -> new points, row-major.
constexpr int kLiftBlock = 256;
int lift_blocks(int W, int H) { return (W * H + kLiftBlock - 1) / kLiftBlock; }

__device__ __forceinline__ bool lift_pixel(const FuseArgs& a, int p) {
  const FrameView& f = a.fr;
  double Rd[9], Td[3];
  frame_pose(f, Rd, Td);   // the refined pose after a joint registration (NEXT-2)
  if (p >= f.W * f.H) return false;
  const float4 nm = f.nmap[p];
  return nm.w > 0.f && (nm.x != 0.f || nm.y != 0.f || nm.z != 0.f) && a.pixkey[p] == ~0ull;
}

// per block: lifted pixels (scanned next) and registered pixels (the fusion count)
__global__ void __launch_bounds__(kLiftBlock) k_lift_count(FuseArgs a, int32_t* counts, unsigned long long* n_reg,
                                                           int do_lift) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int p = blockIdx.x * kLiftBlock + threadIdx.x;
  const int c = __syncthreads_count(do_lift && lift_pixel(a, p));
  const int r = __syncthreads_count(p < a.fr.W * a.fr.H && a.pixkey[p] != ~0ull);
  if (threadIdx.x == 0) {
    counts[blockIdx.x] = c;
    if (r) atomicAdd(n_reg, (unsigned long long)r);
  }
}

// exclusive scan of the per-block counts (single block; offs[nb] = total);
// ids_dev[2] = lifted points that fit the capacity
__global__ void __launch_bounds__(1024) k_scan_counts(const int32_t* counts, int32_t* offs, int nb,
                                                      long long* ids_dev, int64_t base, int64_t cap) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ int32_t wtot[32];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t s = 0;
  for (int b = b0; b < min(nb, b0 + per); ++b) s += counts[b];
  int32_t inc = s;   // warp inclusive scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wtot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int32_t t = wtot[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += v;
    }
    wtot[lane] = ti - t;   // exclusive warp offsets
    if (lane == 31) {
      offs[nb] = ti;
      const bool fits = (int64_t)ti <= cap - base;
      ids_dev[1] = ids_dev[0];   // ids of the lifted points: ids_dev[1] + rank
      if (fits) ids_dev[0] += ti;   // an exceeded capacity consumes no ids (MIS_E_CAPACITY: unchanged)
      ids_dev[2] = ti < cap - base ? ti : cap - base;
      ids_dev[3] = fits ? 1 : 0;  // read by K11 and the lift write: nothing is applied unless it fits
    }
  }
  __syncthreads();
  int32_t run = wtot[wid] + inc - s;
  for (int b = b0; b < min(nb, b0 + per); ++b) { offs[b] = run; run += counts[b]; }
}

__global__ void __launch_bounds__(kLiftBlock) k_lift_write(FuseArgs a, const int32_t* offs, int64_t base,
                                                           int64_t cap, const long long* ids_dev, int32_t* lift_pos) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ int wsum[kLiftBlock / 32];
  const int p = blockIdx.x * kLiftBlock + threadIdx.x;
  const bool on = lift_pixel(a, p);
  if (p < a.fr.W * a.fr.H) {
    a.pixkey[p] = ~0ull;   // the next fusion finds the keys reset (no memset)
    lift_pos[p] = -1;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, on);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int i = 0; i < w; ++i) before += wsum[i];
  if (!on || !ids_dev[3]) return;   // over capacity: nothing written, reported by mis_fuse (MIS_E_CAPACITY)
  const int64_t o = base + offs[blockIdx.x] + before + __popc(bal & ((1u << lane) - 1u));
  lift_pos[p] = (int32_t)o;
  const FrameView& f = a.fr;
  double Rd[9], Td[3];
  frame_pose(f, Rd, Td);   // the refined pose after a joint registration (NEXT-2)
  const int px = p % f.W, py = p / f.W;
  double N[3], q[3];
  normal_map64(f, px, py, N, q);
  for (int c = 0; c < 3; ++c) q[c] -= Td[c];
  float vo[3], no[3];
  for (int c = 0; c < 3; ++c) {
    vo[c] = (float)(Rd[c] * q[0] + Rd[3 + c] * q[1] + Rd[6 + c] * q[2]);
    no[c] = (float)(Rd[c] * N[0] + Rd[3 + c] * N[1] + Rd[6 + c] * N[2]);
  }
  ModelView md = a.md;
  md.px[o] = vo[0]; md.py[o] = vo[1]; md.pz[o] = vo[2];
  md.nx[o] = no[0]; md.ny[o] = no[1]; md.nz[o] = no[2];
  if (a.rgb_obs) {
    md.cr[o] = a.rgb_obs[3 * (int64_t)p]; md.cg[o] = a.rgb_obs[3 * (int64_t)p + 1]; md.cb[o] = a.rgb_obs[3 * (int64_t)p + 2];
  } else {
    md.cr[o] = md.cg[o] = md.cb[o] = 0.f;
  }
  md.w[o] = 1.0f;
  md.stamp[o] = a.frame_index;
  md.ids[o] = ids_dev[1] + (o - base);
}

void launch_lift_count(const FuseArgs& a, int32_t* counts, int nblocks, long long* ids_dev, unsigned long long* n_reg,
                       int do_lift, int64_t base, int64_t cap, cudaStream_t s) {
  launch_pdl(k_lift_count, dim3(nblocks), dim3(kLiftBlock), 0, s, a, counts, n_reg, do_lift);
  launch_pdl(k_scan_counts, dim3(1), dim3(1024), 0, s, counts, counts + nblocks + 1, nblocks, ids_dev, base, cap);
}

void launch_lift_write(const FuseArgs& a, const int32_t* offs, int nblocks, int64_t base, int64_t cap,
                       const long long* ids_dev, int32_t* lift_pos, cudaStream_t s) {
  launch_pdl(k_lift_write, dim3(nblocks), dim3(kLiftBlock), 0, s, a, offs, base, cap, ids_dev, lift_pos);
}

// K2 for the lifted points, per 16 x 16 pixel tile (the lifted points of a tile are close in 3-D):
// the tile's candidate nodes are those whose distance to the points' bounding box can be <= U, U
// the (k+1)-th smallest farthest-corner distance -- every point of the box has k+1 nodes within U,
// so every node of its k+1 nearest is a candidate; the points then scan only the candidates, keeping
// (d^2, id) in lexicographic order (ties to the lower id).  Exact Eq. 2, ~20x fewer distances than
// scanning all m nodes per point.
constexpr int kTile = 16, kMaxCand = 2048;

template <int K>
__device__ __forceinline__ void knn_insert(float (&bd)[K + 1], int (&bi)[K + 1], float d2, int id) {
  if (d2 > bd[K] || (d2 == bd[K] && id >= bi[K])) return;
  float cd = d2;
  int ci = id;
#pragma unroll
  for (int s = 0; s <= K; ++s) {
    if (cd < bd[s] || (cd == bd[s] && ci < bi[s])) {
      const float td = bd[s];
      const int ti = bi[s];
      bd[s] = cd; bi[s] = ci; cd = td; ci = ti;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kTile * kTile) k_skin_tiles(int W, int H, const int32_t* __restrict__ lift_pos,
                                                              ModelView md, const float* __restrict__ g, int m) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ float4 cand[kMaxCand];
  __shared__ float red[6][8];
  __shared__ float sel[kTile * kTile / 32][K + 1];
  __shared__ int ncand, any;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int x = blockIdx.x * kTile + (t % kTile), y = blockIdx.y * kTile + (t / kTile);
  const int o = (x < W && y < H) ? lift_pos[y * W + x] : -1;
  float v[3] = {0.f, 0.f, 0.f};
  if (o >= 0) { v[0] = md.px[o]; v[1] = md.py[o]; v[2] = md.pz[o]; }
  // bounding box of the tile's lifted points
  float lo[3], hi[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) { lo[c] = o >= 0 ? v[c] : INFINITY; hi[c] = o >= 0 ? v[c] : -INFINITY; }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int s = 16; s > 0; s >>= 1) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], s));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], s));
    }
  if (t == 0) { ncand = 0; any = 0; }
  if (lane == 0) for (int c = 0; c < 3; ++c) { red[c][wid] = lo[c]; red[3 + c][wid] = hi[c]; }
  __syncthreads();
  if (o >= 0) any = 1;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = red[c][0]; hi[c] = red[3 + c][0];
    for (int w = 1; w < 8; ++w) { lo[c] = fminf(lo[c], red[c][w]); hi[c] = fmaxf(hi[c], red[3 + c][w]); }
  }
  __syncthreads();
  if (!any) return;
  // U^2: the (k+1)-th smallest farthest-corner squared distance (per thread, per warp, per block)
  float ub[K + 1];
#pragma unroll
  for (int s = 0; s <= K; ++s) ub[s] = INFINITY;
  for (int j = t; j < m; j += blockDim.x) {
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
  // warp merge: k+1 rounds of (min, pop) over the lanes' sorted lists
  float wsel[K + 1];
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    float mn = ub[0];
    for (int s = 16; s > 0; s >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, s));
    wsel[r] = mn;
    const unsigned who = __ballot_sync(0xffffffffu, ub[0] == mn);
    if (lane == __ffs(who) - 1) {
#pragma unroll
      for (int s = 0; s < K; ++s) ub[s] = ub[s + 1];
      ub[K] = INFINITY;
    }
  }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r <= K; ++r) sel[wid][r] = wsel[r];
  __syncthreads();
  __shared__ float U2s;
  if (wid == 0) {   // block: the (k+1)-th smallest of the 8 warps' k+1 smallest, k+1 rounds of (min, pop)
    constexpr int NV = (kTile * kTile / 32) * (K + 1);   // 8 (k+1) values, <= 3 per lane (k <= 8)
    static_assert(NV <= 96, "skin tile merge");
    float v[3];
#pragma unroll
    for (int z = 0; z < 3; ++z) {
      const int q = lane + 32 * z;
      v[z] = q < NV ? sel[q / (K + 1)][q % (K + 1)] : INFINITY;
    }
    float kth = INFINITY;
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      float mn = fminf(v[0], fminf(v[1], v[2]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      kth = mn;
      // pop exactly one copy of the minimum (lowest slot, then lowest lane holding it)
      bool popped = false;
#pragma unroll
      for (int z = 0; z < 3; ++z) {
        const unsigned hz = __ballot_sync(0xffffffffu, v[z] == mn);
        if (!popped && hz) {
          if (lane == __ffs(hz) - 1) v[z] = INFINITY;
          popped = true;
        }
      }
    }
    if (lane == 0) U2s = kth * (1.0f + 1e-5f) + 1e-6f;   // conservative against rounding
  }
  __syncthreads();
  const float U2 = U2s;
  // candidates: nodes whose squared distance to the box can be <= U^2
  for (int j = t; j < m; j += blockDim.x) {
    float l2 = 0.f;
    float gj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gj[c] = g[3 * j + c];
      const float e = fmaxf(0.f, fmaxf(lo[c] - gj[c], gj[c] - hi[c]));
      l2 += e * e;
    }
    if (l2 <= U2) {
      const int q = atomicAdd(&ncand, 1);
      if (q < kMaxCand) cand[q] = make_float4(gj[0], gj[1], gj[2], __int_as_float(j));
    }
  }
  __syncthreads();
  if (o < 0) return;
  const int nc = ncand;
  float bd[K + 1];
  int bi[K + 1];
#pragma unroll
  for (int s = 0; s <= K; ++s) { bd[s] = INFINITY; bi[s] = 0x7fffffff; }
  if (nc <= kMaxCand) {
    for (int q = 0; q < nc; ++q) {
      const float4 c4 = cand[q];
      const float dx = v[0] - c4.x, dy = v[1] - c4.y, dz = v[2] - c4.z;
      knn_insert<K>(bd, bi, dx * dx + dy * dy + dz * dz, __float_as_int(c4.w));
    }
  } else {   // candidate overflow (a very spread-out tile): all nodes
    for (int j = 0; j < m; ++j) {
      const float dx = v[0] - g[3 * j], dy = v[1] - g[3 * j + 1], dz = v[2] - g[3 * j + 2];
      knn_insert<K>(bd, bi, dx * dx + dy * dy + dz * dz, j);
    }
  }
  // Eq. 2 weights (as K2), ids ascending
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
#pragma unroll
  for (int s = 0; s < K; ++s) { md.kidx[s * md.cap + o] = bi[s]; md.kw[s * md.cap + o] = ww[s]; }
}

void launch_skin_lifted(int K, int W, int H, const int32_t* lift_pos, const ModelView& md, const float* g, int m,
                        cudaStream_t s) {
  dim3 grd((W + kTile - 1) / kTile, (H + kTile - 1) / kTile);
  switch (K) {
#define SK(KK) case KK: launch_pdl(k_skin_tiles<KK>, dim3(grd), dim3(kTile * kTile), 0, s, W, H, lift_pos, md, g, m); break;
    SK(1) SK(2) SK(3) SK(4) SK(5) SK(6) SK(7) SK(8)
#undef SK
    default: break;
  }
}

}  // namespace mis
