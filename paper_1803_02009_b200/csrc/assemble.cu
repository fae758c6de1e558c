// assemble.cu -- K3 (per-point warp + association + residuals + J^T J) and
// K4/K5 (regulariser and feature terms) of one Gauss-Newton iteration.
//
// K3 design: points are sorted by their canonical kNN tuple
// (K13), so a "chunk" (<= 256 consecutive points of one tuple segment) shares
// all K nodes.  One warp owns a chunk: each lane warps one point (Eq. 1),
// associates it (Eq. 7, with an fp64 guard band at every decision boundary)
// and writes one row f of per-point factors to shared memory:
//   c' = [w_1 u_1, ..., w_K u_K, r_pl]      u_j = [a_j x n', n'] (Eq. 8 Jacobian row / w_j)
//   e' = [w_1 a_1, w_1, ..., w_K a_K, w_K, r']   (point-to-point moments, r' = R^T (v~ - q))
// Every per-chunk sum the normal equations need is an entry of sum_i c'c'^T or
// sum_i e'e'^T (upper triangles), i.e. two tiny SYRKs.  Lanes own 4x4 tiles of
// those triangles and accumulate them from shared memory in registers over the
// chunk's points (16 FFMA per 2 LDS.128), then commit each entry once per
// chunk with a global atomic add.  K_finalize (solve.cu) turns the moments
// into 6x6 point-to-point blocks: sum of w_j w_l [-[a_j]x[a_l]x, [a_j]x; -[a_l]x, I].
#include <cuda_runtime.h>

#include "solve_common.cuh"

namespace mis {

#ifndef MIS_K3_SPLIT
#define MIS_K3_SPLIT 2   // 2: split each tile's batch into halves across lanes (measured best at K=4)
#endif

template <int K>
struct Lay {
  static constexpr int CD = 6 * K + 1;
  static constexpr int CDP = (CD + 3) & ~3;
  static constexpr int CE = 4 * K + 3;
  static constexpr int CEP = (CE + 3) & ~3;
  static constexpr int FS = CDP + CEP;
  static constexpr int FSP = FS + 4;                 // padded smem row stride (bank spread)
  static constexpr int ND = CDP / 4, NE = CEP / 4;   // tile grid sizes
  static constexpr int TD = ND * (ND + 1) / 2;
  static constexpr int TE = NE * (NE + 1) / 2;
  static constexpr int NT = TD + TE;
  static constexpr int R = (NT + 31) / 32;           // tiles per lane
  static constexpr int P = K * (K + 1) / 2;
  // work items = (tile, batch half): 2 NT items over 32 lanes balance better than NT
  // (K=4: 86 items = 3 rounds of 16 points instead of 2 rounds of 32); needs 2 NT tile
  // dumps to fit the warp's row buffer at commit
  static constexpr int SPLIT = (MIS_K3_SPLIT == 2 && 2 * NT * 16 <= 32 * FSP) ? 2 : 1;
  static constexpr int NI = NT * SPLIT;
  static constexpr int RI = (NI + 31) / 32;          // items per lane
  static constexpr int PS = 32 / SPLIT;              // points per item per batch
};

constexpr int kWarps = 8;
#ifndef MIS_K3_MINB
#define MIS_K3_MINB 2   // resident blocks per SM the register budget is sized for
#endif
#ifndef MIS_GUARD_SCALE
#define MIS_GUARD_SCALE 1.0f
#endif
// Guard bands around every fp32 decision, each >=3x the fp32
// error bound: u, v <= ~1.5e-4 px (x_hat = v + small correction, then R x_hat + T
// and one division); |v~ - q| <= ~3e-5 mm; n~.N <= ~1e-6.
constexpr float kGuardPx = 5e-4f * MIS_GUARD_SCALE;     // rounding of u, v (pixels)
constexpr float kGuardRel = 2e-5f * MIS_GUARD_SCALE;    // distance gate (relative to eps_d)
constexpr float kGuardCos = 1e-5f * MIS_GUARD_SCALE;    // angle gate (cosine)

__device__ __forceinline__ bool depth_ok_d(float d) { return isfinite(d) && d > 0.0f; }

// fp64 re-evaluation of one point's warp and Eq. 7 gates (the oracle's
// arithmetic order is irrelevant here; only decisions within ~1e-12 of a
// threshold can differ).  Used for the rare points whose fp32 quantities lie
// inside a guard band.
// Arguments by value / pointer-to-global only: a reference to the kernel's
// parameter struct would force an addressable (local-memory) copy of it.
struct Fp64Args {
  const float *px, *py, *pz, *nx, *ny, *nz, *kw;
  int64_t cap;
  const double* Rt64;
  const float* g;
  const float* depth;
  int W, H;
  double fxd, fyd, cxd, cyd;
  double Rd[9], Td[3];
  double eps_dd, cos_eps_nd;
};

template <int K>
__device__ __noinline__ void assoc_fp64(const Fp64Args* __restrict__ pa, int64_t i, const int32_t* nodes, float* vt_out,
                                        float* q_out, float* N_out, int* pix_out, uint8_t* why_out) {
  const Fp64Args& a = *pa;
  struct MV { const float *px, *py, *pz, *nx, *ny, *nz, *kw; int64_t cap; } md = {a.px, a.py, a.pz, a.nx, a.ny, a.nz,
                                                                                 a.kw, a.cap};
  struct FV { int W, H; double fxd, fyd, cxd, cyd; const double *Rd, *Td; const float* depth; } f = {
      a.W, a.H, a.fxd, a.fyd, a.cxd, a.cyd, a.Rd, a.Td, a.depth};
  struct ND { const double* Rt64; const float* g; } ndv = {a.Rt64, a.g};
  double v[3] = {md.px[i], md.py[i], md.pz[i]}, n[3] = {md.nx[i], md.ny[i], md.nz[i]};
  double W = 0, wr[K];
  for (int s = 0; s < K; ++s) { wr[s] = md.kw[s * md.cap + i]; W += wr[s]; }
  *pix_out = -1;
  *why_out = 0;
  if (!(W > 0)) return;
  double xh[3] = {0, 0, 0}, mh[3] = {0, 0, 0};
  for (int s = 0; s < K; ++s) {
    const double* Rt = ndv.Rt64 + 12 * nodes[s];
    const float* g = ndv.g + 3 * nodes[s];
    const double wn = wr[s] / W;
    double d[3] = {v[0] - g[0], v[1] - g[1], v[2] - g[2]};
    for (int r = 0; r < 3; ++r) {
      double ar = Rt[3 * r] * d[0] + Rt[3 * r + 1] * d[1] + Rt[3 * r + 2] * d[2];
      xh[r] += wn * (ar + (double)g[r] + Rt[9 + r]);
      mh[r] += wn * (Rt[3 * r] * n[0] + Rt[3 * r + 1] * n[1] + Rt[3 * r + 2] * n[2]);
    }
  }
  double vt[3], nt[3];
  for (int r = 0; r < 3; ++r) {
    vt[r] = f.Rd[3 * r] * xh[0] + f.Rd[3 * r + 1] * xh[1] + f.Rd[3 * r + 2] * xh[2] + f.Td[r];
    nt[r] = f.Rd[3 * r] * mh[0] + f.Rd[3 * r + 1] * mh[1] + f.Rd[3 * r + 2] * mh[2];
  }
  const double ml = sqrt(mh[0] * mh[0] + mh[1] * mh[1] + mh[2] * mh[2]);
  if (ml < 1e-12) return;
  for (int r = 0; r < 3; ++r) { nt[r] /= ml; vt_out[r] = (float)vt[r]; }
  uint8_t why = 0;
  if (!(vt[2] > 0)) { *why_out = why; return; }
  why |= 1;
  const double u = f.fxd * vt[0] / vt[2] + f.cxd, vv = f.fyd * vt[1] / vt[2] + f.cyd;
  const double fu = floor(u + 0.5), fv = floor(vv + 0.5);
  if (fu < 0 || fv < 0 || fu >= f.W || fv >= f.H) { *why_out = why; return; }
  why |= 2;
  const int px = (int)fu, py = (int)fv, W_ = f.W;
  const float D = f.depth[py * W_ + px];
  if (!depth_ok_d(D)) { *why_out = why; return; }
  why |= 4;
  // normal in fp64 from the five depths (reading A11)
  if (px <= 0 || py <= 0 || px >= W_ - 1 || py >= f.H - 1) { *why_out = why; return; }
  const float l = f.depth[py * W_ + px - 1], r = f.depth[py * W_ + px + 1];
  const float up = f.depth[(py - 1) * W_ + px], dn = f.depth[(py + 1) * W_ + px];
  if (!depth_ok_d(l) || !depth_ok_d(r) || !depth_ok_d(up) || !depth_ok_d(dn)) { *why_out = why; return; }
  const double ax = ((px + 1) - f.cxd) * r / f.fxd - ((px - 1) - f.cxd) * l / f.fxd;
  const double ay = (py - f.cyd) * (double)r / f.fyd - (py - f.cyd) * (double)l / f.fyd;
  const double az = (double)r - (double)l;
  const double bx = (px - f.cxd) * (double)dn / f.fxd - (px - f.cxd) * (double)up / f.fxd;
  const double by = ((py + 1) - f.cyd) * dn / f.fyd - ((py - 1) - f.cyd) * up / f.fyd;
  const double bz = (double)dn - (double)up;
  double N[3] = {ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bx};
  const double len = sqrt(N[0] * N[0] + N[1] * N[1] + N[2] * N[2]);
  if (len < 1e-12) { *why_out = why; return; }
  const double q[3] = {(px - f.cxd) * D / f.fxd, (py - f.cyd) * D / f.fyd, (double)D};
  for (int c = 0; c < 3; ++c) N[c] /= len;
  if (N[0] * q[0] + N[1] * q[1] + N[2] * q[2] > 0) for (int c = 0; c < 3; ++c) N[c] = -N[c];
  why |= 8;
  const double dd = sqrt((vt[0] - q[0]) * (vt[0] - q[0]) + (vt[1] - q[1]) * (vt[1] - q[1]) + (vt[2] - q[2]) * (vt[2] - q[2]));
  for (int c = 0; c < 3; ++c) { q_out[c] = (float)q[c]; N_out[c] = (float)N[c]; }
  if (!(dd < a.eps_dd)) { *why_out = why; return; }
  why |= 16;
  const double cs = nt[0] * N[0] + nt[1] * N[1] + nt[2] * N[2];
  if (!(cs > a.cos_eps_nd)) { *why_out = why; return; }
  why |= 32;
  *why_out = why;
  *pix_out = py * W_ + px;
}

// A point's inputs, loaded one batch ahead (software prefetch: the global loads
// of batch b+1 are in flight while batch b is warped and accumulated).
template <int K>
struct PointIn {
  float v[3], n[3], w[K];
};

template <int K>
__device__ __forceinline__ void load_point(const ModelView& md, int64_t i, bool act, PointIn<K>& p) {
  if (!act) return;
  p.v[0] = md.px[i]; p.v[1] = md.py[i]; p.v[2] = md.pz[i];
  p.n[0] = md.nx[i]; p.n[1] = md.ny[i]; p.n[2] = md.nz[i];
#pragma unroll
  for (int s = 0; s < K; ++s) p.w[s] = md.kw[s * md.cap + i];
}

// One lane, one point: warp, associate, write the factor row (zeros if not associated).
template <int K, bool DBG>
__device__ __forceinline__ bool point_row(const AsmPointsArgs& a, int64_t i, bool act, const PointIn<K>& pin,
                                          const float* __restrict__ ND, const int32_t* nodes,
                                          float* __restrict__ row) {
  using L = Lay<K>;
  bool assoc = false;
  int pix = -1;
  uint8_t why = 0;
  if (act) {
    const ModelView& md = a.md;
    const FrameView& fr = a.fr;
    const float v0 = pin.v[0], v1 = pin.v[1], v2 = pin.v[2];
    const float n0 = pin.n[0], n1 = pin.n[1], n2 = pin.n[2];
    float wn[K], ax[K], ay[K], az[K];
    float W = 0.f;
#pragma unroll
    for (int s = 0; s < K; ++s) { wn[s] = pin.w[s]; W += wn[s]; }
    if (W > 0.f) {
      const float iW = 1.0f / W;
      float x0 = 0, x1 = 0, x2 = 0, m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const float* nd = ND + 16 * s;   // R(9) t(3) g(3)
        wn[s] *= iW;
        const float d0 = v0 - nd[12], d1 = v1 - nd[13], d2 = v2 - nd[14];
        ax[s] = nd[0] * d0 + nd[1] * d1 + nd[2] * d2;
        ay[s] = nd[3] * d0 + nd[4] * d1 + nd[5] * d2;
        az[s] = nd[6] * d0 + nd[7] * d1 + nd[8] * d2;
        // x_hat = sum w (a + g + t) = v + sum w ((R - I) d + t)  (sum w = 1): the correction is
        // small, so its fp32 rounding is ~100x below that of summing ~60 mm terms
        x0 += wn[s] * ((ax[s] - d0) + nd[9]);
        x1 += wn[s] * ((ay[s] - d1) + nd[10]);
        x2 += wn[s] * ((az[s] - d2) + nd[11]);
        m0 += wn[s] * (nd[0] * n0 + nd[1] * n1 + nd[2] * n2);
        m1 += wn[s] * (nd[3] * n0 + nd[4] * n1 + nd[5] * n2);
        m2 += wn[s] * (nd[6] * n0 + nd[7] * n1 + nd[8] * n2);
      }
      x0 += v0;
      x1 += v1;
      x2 += v2;
      const float* R = fr.R;
      float vt[3] = {R[0] * x0 + R[1] * x1 + R[2] * x2 + fr.T[0], R[3] * x0 + R[4] * x1 + R[5] * x2 + fr.T[1],
                     R[6] * x0 + R[7] * x1 + R[8] * x2 + fr.T[2]};
      const float ml = sqrtf(m0 * m0 + m1 * m1 + m2 * m2);
      float q[3] = {0, 0, 0}, N[3] = {0, 0, 0};
      bool guard = !(ml > 1e-6f) || fabsf(vt[2]) < 1e-3f;
      if (!guard && vt[2] > 0.f) {
        why = 1;
        const float iz = 1.0f / vt[2];
        const float uu = fr.fx * vt[0] * iz + fr.cx + 0.5f, vv = fr.fy * vt[1] * iz + fr.cy + 0.5f;
        const float fu = floorf(uu), fv = floorf(vv);
        if (fminf(uu - fu, fu + 1.f - uu) < kGuardPx || fminf(vv - fv, fv + 1.f - vv) < kGuardPx) {
          guard = true;
        } else if (fu >= 0.f && fv >= 0.f && fu < (float)fr.W && fv < (float)fr.H) {
          why |= 2;
          const int px = (int)fu, py = (int)fv;
          const float4 nm = fr.nmap[py * fr.W + px];
          if (nm.w > 0.f) {
            why |= 4;
            if (nm.x != 0.f || nm.y != 0.f || nm.z != 0.f) {
              why |= 8;
              N[0] = nm.x; N[1] = nm.y; N[2] = nm.z;
              q[0] = (px - fr.cx) * nm.w / fr.fx;
              q[1] = (py - fr.cy) * nm.w / fr.fy;
              q[2] = nm.w;
              const float e0 = vt[0] - q[0], e1 = vt[1] - q[1], e2 = vt[2] - q[2];
              const float dd = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
              if (fabsf(dd - a.eps_d) < kGuardRel * a.eps_d) {
                guard = true;
              } else if (dd < a.eps_d) {
                why |= 16;
                const float im = 1.0f / ml;
                const float nt0 = (R[0] * m0 + R[1] * m1 + R[2] * m2) * im;
                const float nt1 = (R[3] * m0 + R[4] * m1 + R[5] * m2) * im;
                const float nt2 = (R[6] * m0 + R[7] * m1 + R[8] * m2) * im;
                const float cs = nt0 * N[0] + nt1 * N[1] + nt2 * N[2];
                if (fabsf(cs - a.cos_eps_n) < kGuardCos) guard = true;
                else if (cs > a.cos_eps_n) { why |= 32; pix = py * fr.W + px; }
              }
            }
          }
        }
      }
      if (guard) {
        atomicAdd(a.guard_counter, 1.0);
        Fp64Args fa;
        fa.px = md.px; fa.py = md.py; fa.pz = md.pz; fa.nx = md.nx; fa.ny = md.ny; fa.nz = md.nz; fa.kw = md.kw;
        fa.cap = md.cap;
        fa.Rt64 = a.nd.Rt64;
        fa.g = a.nd.g;
        fa.depth = fr.depth;
        fa.W = fr.W; fa.H = fr.H;
        fa.fxd = fr.fxd; fa.fyd = fr.fyd; fa.cxd = fr.cxd; fa.cyd = fr.cyd;
#pragma unroll
        for (int k = 0; k < 9; ++k) fa.Rd[k] = fr.Rd[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) fa.Td[k] = fr.Td[k];
        fa.eps_dd = a.eps_dd;
        fa.cos_eps_nd = a.cos_eps_nd;
        assoc_fp64<K>(&fa, i, nodes, vt, q, N, &pix, &why);
      }
      assoc = (pix >= 0);
      if (assoc) {
        const float e0 = vt[0] - q[0], e1 = vt[1] - q[1], e2 = vt[2] - q[2];
        const float rpl = N[0] * e0 + N[1] * e1 + N[2] * e2;                 // Eq. 8
        const float np0 = R[0] * N[0] + R[3] * N[1] + R[6] * N[2];         // n' = R^T N
        const float np1 = R[1] * N[0] + R[4] * N[1] + R[7] * N[2];
        const float np2 = R[2] * N[0] + R[5] * N[1] + R[8] * N[2];
        const float rp0 = R[0] * e0 + R[3] * e1 + R[6] * e2;               // r' = R^T (v~ - q)
        const float rp1 = R[1] * e0 + R[4] * e1 + R[7] * e2;
        const float rp2 = R[2] * e0 + R[5] * e1 + R[8] * e2;
        // the factor row, straight to shared memory (8-byte / 16-byte stores)
#pragma unroll
        for (int s = 0; s < K; ++s) {
          float2* c2 = reinterpret_cast<float2*>(row + 6 * s);
          c2[0] = make_float2(wn[s] * (ay[s] * np2 - az[s] * np1), wn[s] * (az[s] * np0 - ax[s] * np2));  // w_j (a_j x n')
          c2[1] = make_float2(wn[s] * (ax[s] * np1 - ay[s] * np0), wn[s] * np0);
          c2[2] = make_float2(wn[s] * np1, wn[s] * np2);
          *reinterpret_cast<float4*>(row + L::CDP + 4 * s) = make_float4(wn[s] * ax[s], wn[s] * ay[s], wn[s] * az[s], wn[s]);
        }
        row[6 * K] = rpl;
#pragma unroll
        for (int c = 6 * K + 1; c < L::CDP; ++c) row[c] = 0.f;
        row[L::CDP + 4 * K + 0] = rp0;
        row[L::CDP + 4 * K + 1] = rp1;
        row[L::CDP + 4 * K + 2] = rp2;
#pragma unroll
        for (int c = L::CDP + 4 * K + 3; c < L::FS; ++c) row[c] = 0.f;
      }
    }
    if (DBG) { a.dbg_pix[i] = pix; a.dbg_why[i] = why; }
  }
  if (!assoc) {
    float4* r4 = reinterpret_cast<float4*>(row);
#pragma unroll
    for (int c = 0; c < L::FS / 4; ++c) r4[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  return assoc;
}

template <int K, bool DBG>
__global__ void __launch_bounds__(kWarps * 32, MIS_K3_MINB) k_assemble_points(AsmPointsArgs a) {
  using L = Lay<K>;
  constexpr int P = L::P;
  constexpr int RS = (52 * P + 18 * K + 5 + 3) & ~3;   // == rec_stride(K)
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* F = reinterpret_cast<float*>(smem4) + warp * (32 * L::FSP + 16 * K);
  float* ND = F + 32 * L::FSP;

  // tile table of the two upper triangles: (I, J) in units of 4 entries
  __shared__ uint8_t tabI[L::NT], tabJ[L::NT];
  // record permutation: perm[d] = tile-dump index feeding record float d (-1: zero)
  __shared__ int16_t perm[RS];
  for (int t = threadIdx.x; t < L::NT; t += blockDim.x) {
    const bool e = t >= L::TD;
    const int nb = e ? L::NE : L::ND;
    int u = e ? t - L::TD : t, I = 0;
    while (u >= nb - I) { u -= nb - I; ++I; }
    tabI[t] = (uint8_t)I;
    tabJ[t] = (uint8_t)(I + u);
  }
  for (int d = threadIdx.x; d < RS; d += blockDim.x) perm[d] = -1;
  __syncthreads();
  for (int q = threadIdx.x; q < 16 * L::NT; q += blockDim.x) {
    const int t = q >> 4, A = 4 * tabI[t] + ((q >> 2) & 3), B = 4 * tabJ[t] + (q & 3);
    if (A > B) continue;
    int d = -1;
    if (t < L::TD) {             // c' = [w_j u_j ..., r_pl]
      if (B < 6 * K) d = 52 * pair_index(A / 6, B / 6, K) + 6 * (A % 6) + (B % 6);
      else if (B == 6 * K && A < 6 * K) d = 52 * P + 18 * (A / 6) + (A % 6);
      else if (B == 6 * K && A == 6 * K) d = 52 * P + 18 * K;
    } else {                     // e' = [w_j a_j, w_j ..., r']
      if (B < 4 * K) d = 52 * pair_index(A / 4, B / 4, K) + 36 + 4 * (A % 4) + (B % 4);
      else if (B < 4 * K + 3 && A < 4 * K) d = 52 * P + 18 * (A / 4) + 6 + 3 * (A % 4) + (B - 4 * K);
      else if (B < 4 * K + 3 && A == B) d = 52 * P + 18 * K + 1 + (A - 4 * K);
    }
    if (d >= 0) perm[d] = (int16_t)q;
  }
  __syncthreads();
  // static ownership: lane owns items lane, lane + 32, ...; item = tile + NT * half
  int offA[L::RI], offB[L::RI], p0[L::RI];
  bool tV[L::RI];
#pragma unroll
  for (int r = 0; r < L::RI; ++r) {
    const int it = lane + 32 * r;
    tV[r] = it < L::NI;
    const int t = it % L::NT;
    const int base = (t >= L::TD) ? L::CDP : 0;
    offA[r] = tV[r] ? base + 4 * tabI[t] : 0;
    offB[r] = tV[r] ? base + 4 * tabJ[t] : 0;
    p0[r] = (it / L::NT) * L::PS;
  }

  double e_data = 0.0, e_pt = 0.0;   // per-lane energy partials (fp64 across chunks)
  unsigned long long n_tot = 0;      // associations of this warp's chunks
  // dynamic chunk scheduling (segments are uneven): one atomic fetch per chunk per warp
  int64_t c = 0;
  if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
  c = __shfl_sync(0xffffffffu, c, 0);
  for (; c < a.nchunk;) {
    const int4 ch = a.chunks[c];
    const int seg = ch.x;
    const int32_t* nodes = a.seg_nodes + (int64_t)seg * K;
    __syncwarp();
    for (int t = lane; t < 16 * K; t += 32) ND[t] = a.nd.node32[16 * nodes[t >> 4] + (t & 15)];
    __syncwarp();
    float acc[L::RI][16];
#pragma unroll
    for (int r = 0; r < L::RI; ++r)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[r][e] = 0.f;
    unsigned n_assoc = 0;
    for (int base = ch.y; base < ch.z; base += 32) {
      const int64_t i = base + lane;
      PointIn<K> cur;
      load_point<K>(a.md, i, i < ch.z, cur);
      const bool as = point_row<K, DBG>(a, i, i < ch.z, cur, ND, nodes, F + lane * L::FSP);
      n_assoc += __popc(__ballot_sync(0xffffffffu, as));
      __syncwarp();
      const int np = min(32, ch.z - base);
#pragma unroll
      for (int r = 0; r < L::RI; ++r) {
        if (!tV[r]) continue;
        const float* pa = F + offA[r];
        const float* pb = F + offB[r];
        const int pe = min(np, p0[r] + L::PS);
#pragma unroll 4
        for (int p = p0[r]; p < pe; ++p) {
          const float4 A = *reinterpret_cast<const float4*>(pa + p * L::FSP);
          const float4 B = *reinterpret_cast<const float4*>(pb + p * L::FSP);
          const float Av[4] = {A.x, A.y, A.z, A.w}, Bv[4] = {B.x, B.y, B.z, B.w};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[r][4 * x + y] = fmaf(Av[x], Bv[y], acc[r][4 * x + y]);
        }
      }
      __syncwarp();
    }
    // ---- commit: tiles -> shared memory -> atomic adds into the BSR accumulators
#pragma unroll
    for (int r = 0; r < L::RI; ++r) {
      if (!tV[r]) continue;
      float4* d4 = reinterpret_cast<float4*>(F + 16 * (lane + 32 * r));
#pragma unroll
      for (int x = 0; x < 4; ++x) d4[x] = make_float4(acc[r][4 * x], acc[r][4 * x + 1], acc[r][4 * x + 2], acc[r][4 * x + 3]);
    }
    __syncwarp();
    int64_t next_chunk = 0;
    if (lane == 0) next_chunk = (int64_t)atomicAdd(a.work_counter, 1ull);   // prefetch the next chunk id
    // vector atomic adds (sm_90+ float4 / float2 RED) into the accumulators: per pair
    // 9 x 4 data + 4 x 4 moments of its BSR slot, per node slot 3 x 2 rhs + 3 x 4
    // moments; all-zero vectors (no association) are skipped.  Energies stay in registers.
    const int32_t* slots = a.seg_slot + (int64_t)seg * P;
    auto rv = [&](int d) -> float {
      const int q = perm[d];
      if (q < 0) return 0.f;
      float v = F[q];
      if (L::SPLIT == 2) v += F[q + 16 * L::NT];   // the second half's partial tile
      return v;
    };
    for (int it = lane; it < 13 * P + 6 * K; it += 32) {
      if (it < 13 * P) {
        const int pr = it / 13, q = it - 13 * pr;
        const int d0 = 52 * pr + 4 * q;   // data (q < 9) then moments: contiguous in the record
        const float4 v = make_float4(rv(d0), rv(d0 + 1), rv(d0 + 2), rv(d0 + 3));
        if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
        const int64_t u = slots[pr];
        float* dst = q < 9 ? a.acc.data + 36 * u + 4 * q : a.acc.mom + 16 * u + 4 * (q - 9);
        atomicAdd(reinterpret_cast<float4*>(dst), v);
      } else {
        const int t2 = it - 13 * P, sl = t2 / 6, q = t2 - 6 * sl;
        const int64_t nd = nodes[sl];
        if (q < 3) {
          const int d0 = 52 * P + 18 * sl + 2 * q;
          const float2 v = make_float2(rv(d0), rv(d0 + 1));
          if (v.x != 0.f || v.y != 0.f) atomicAdd(reinterpret_cast<float2*>(a.acc.rhs_data + 6 * nd + 2 * q), v);
        } else {
          const int d0 = 52 * P + 18 * sl + 6 + 4 * (q - 3);
          const float4 v = make_float4(rv(d0), rv(d0 + 1), rv(d0 + 2), rv(d0 + 3));
          if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)
            atomicAdd(reinterpret_cast<float4*>(a.acc.node_mom + 12 * nd + 4 * (q - 3)), v);
        }
      }
    }
    if (lane == 0) {
      const int de = 52 * P + 18 * K;
      e_data += rv(de);
      e_pt += (double)rv(de + 1) + rv(de + 2) + rv(de + 3);
    }
    n_tot += n_assoc;
    c = __shfl_sync(0xffffffffu, next_chunk, 0);
  }
  // energies and association count: warp, then block, then one fp64 atomic per block
  __shared__ double red_e[3][kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e_data += __shfl_xor_sync(0xffffffffu, e_data, o);
    e_pt += __shfl_xor_sync(0xffffffffu, e_pt, o);
  }
  if (lane == 0) { red_e[0][warp] = e_data; red_e[1][warp] = e_pt; red_e[2][warp] = (double)n_tot; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += red_e[threadIdx.x][w];
    if (t != 0.0) atomicAdd(a.acc.energy + (threadIdx.x == 2 ? 4 : threadIdx.x), t);
  }
}

// Finalisation of the normal equations from the accumulators (so the
// latency-bound solver only streams its rows): warps [0, m) the diagonal blocks
// -- first, so their block-Jacobi inverses (K7) overlap the rest --, then one
// warp per off-diagonal upper entry, then one per node, then one for the
// energies (report slot).  Every accumulator is re-zeroed after it is read, so
// the next assembly needs no memset:
//   H(j,l) = w_data sum c c^T + w_pt PT(moments) + graph  (and its mirror H(l,j)),
//   b_j = -(w_data sum c r_pl + w_pt sum w_j [a_j x r'; r']) + graph rhs.
__global__ void __launch_bounds__(256) k_finalize(FinalArgs r) {
  __shared__ float stage[8][124];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* st = stage[wib];
  int64_t e = -1;
  if (gw < r.m) {
    e = r.diag_pos[gw];
  } else if (gw < r.m + r.nnzb) {
    e = gw - r.m;
    if (r.upper_of[e] != e || r.lower_of[e] < 0) return;   // mirrors and diagonals are written elsewhere
  }
  if (e >= 0) {
    st[lane] = r.acc.data[36 * e + lane];                  // D (36) | Mo (16) | G (36)
    if (lane < 4) st[32 + lane] = r.acc.data[36 * e + 32 + lane];
    if (lane < 16) st[36 + lane] = r.acc.mom[16 * e + lane];
    st[52 + lane] = r.acc.graph[36 * e + lane];
    if (lane < 4) st[84 + lane] = r.acc.graph[36 * e + 32 + lane];
    r.acc.data[36 * e + lane] = 0.f;                       // ready for the next assembly
    if (lane < 4) r.acc.data[36 * e + 32 + lane] = 0.f;
    if (lane < 16) r.acc.mom[16 * e + lane] = 0.f;
    r.acc.graph[36 * e + lane] = 0.f;
    if (lane < 4) r.acc.graph[36 * e + 32 + lane] = 0.f;
    __syncwarp();
    const int lo = r.lower_of[e];
    const bool diag = lo < 0;
    for (int l = lane; l < 36; l += 32) {
      const int i = l / 6, j = l - 6 * (l / 6);
      const float h = block_entry(st, st + 36, st + 52, diag, i, j, r.w_data, r.w_pt);
      r.Hval[36 * e + l] = h;
      if (!diag) r.Hval[36 * (int64_t)lo + 6 * j + i] = h;
      st[88 + l] = h;
    }
    if (diag && r.Minv) {   // block-Jacobi inverse of this node (K7), off the solver's critical path:
      __syncwarp();         // fp64 Gauss-Jordan, lane rr < 6 holds row rr of [H + (lambda + mu) I | I]
      const int64_t row_j = gw;
      const int rr = lane < 6 ? lane : 0;
      double trc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) trc += (double)st[88 + 7 * q];
      const double mu = 1e-9 * trc / 6.0;
      double row[12];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        row[q] = (double)st[88 + 6 * rr + q] + (q == rr ? (double)r.lambda + mu : 0.0);
        row[6 + q] = q == rr ? 1.0 : 0.0;
      }
      bool pd = true;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const double pv = __shfl_sync(0xffffffffu, row[p], p);
        if (!(pv > 0.0)) pd = false;
        const double ipv = 1.0 / pv, f = row[p] * ipv;
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const double pq = __shfl_sync(0xffffffffu, row[q], p);
          row[q] = rr == p ? pq * ipv : row[q] - f * pq;
        }
      }
      if (lane < 6)
#pragma unroll
        for (int q = 0; q < 6; ++q) r.Minv[36 * row_j + 6 * rr + q] = pd ? (float)row[6 + q] : 0.f;
    }
    return;
  }
  const int64_t n = gw - r.m - r.nnzb;
  if (n == r.m) {   // energies -> report slot; zeroed (with K3's work counter) for the next assembly
    if (lane == 0) {
      double* E = r.acc.energy;
      if (r.slot >= 0) {
        double* rep = r.rep_energy + 5 * r.slot;
        rep[0] = E[0]; rep[1] = E[1]; rep[2] = E[2]; rep[3] = E[3];
        rep[4] = (double)r.w_data * E[0] + (double)r.w_pt * E[1] + (double)r.w_reg * E[2] + (double)r.w_corr * E[3];
        r.rep_nassoc[r.slot] = E[4];
        r.rep_nassoc[MIS_MAX_GN + 1 + r.slot] = E[5];   // fp64 guard-band re-evaluations
      }
      for (int q = 0; q < 7; ++q) E[q] = 0.0;
    }
    return;
  }
  if (n > r.m) return;
  if (lane < 6) st[lane] = r.acc.rhs_data[6 * n + lane];   // 6 rhs_data | 12 node moments
  else if (lane < 18) st[lane] = r.acc.node_mom[12 * n + lane - 6];
  if (lane < 6) { r.acc.rhs_data[6 * n + lane] = 0.f; }
  else if (lane < 18) r.acc.node_mom[12 * n + lane - 6] = 0.f;
  __syncwarp();
  if (lane < 6) {
    const float* Nm = st + 6;
    float pt;
    if (lane < 3) {
      const int c1 = (lane + 1) % 3, c2 = (lane + 2) % 3;
      pt = Nm[3 * c1 + c2] - Nm[3 * c2 + c1];
    } else {
      pt = Nm[9 + (lane - 3)];
    }
    r.rhs[6 * n + lane] = -r.w_data * st[lane] - r.w_pt * pt + r.acc.rhs_graph[6 * n + lane];
    r.acc.rhs_graph[6 * n + lane] = 0.f;
  }
}

void launch_finalize(const FinalArgs& r, cudaStream_t s) {
  const int64_t warps = 2 * (int64_t)r.m + r.nnzb + 1;
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > 0) k_finalize<<<(unsigned)blocks, 256, 0, s>>>(r);
}

template <int K>
static void launch_points_k(const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  using L = Lay<K>;
  const size_t smem = sizeof(float) * kWarps * (32 * L::FSP + 16 * K);
  const bool dbg = a.dbg_pix != nullptr;
  auto kern = dbg ? k_assemble_points<K, true> : k_assemble_points<K, false>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[dbg]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set[dbg] = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = (a.nchunk + kWarps - 1) / kWarps;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, kWarps * 32, smem, s>>>(a);
}

void launch_assemble_points(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  if (a.nchunk <= 0) return;
  switch (K) {
    case 1: launch_points_k<1>(a, num_sms, s); break;
    case 2: launch_points_k<2>(a, num_sms, s); break;
    case 3: launch_points_k<3>(a, num_sms, s); break;
    case 4: launch_points_k<4>(a, num_sms, s); break;
    case 5: launch_points_k<5>(a, num_sms, s); break;
    case 6: launch_points_k<6>(a, num_sms, s); break;
    case 7: launch_points_k<7>(a, num_sms, s); break;
    case 8: launch_points_k<8>(a, num_sms, s); break;
    default: break;
  }
}

// ---------------------------------------------------------------- K4 / K5
// One thread per (edge, block row), (feature, node pair, block row) and
// (feature, node): ~50k independent items at C3 instead of 4.5k serial
// atomic chains (the regulariser and feature blocks are few: latency-bound).
__device__ __forceinline__ void feature_warp(const AsmGraphArgs& a, int fi, float (*am)[3], float* wn, float* e,
                                             float* rp, bool* ok) {
  const int K = a.K;
  const float V[3] = {a.fsrc[3 * fi], a.fsrc[3 * fi + 1], a.fsrc[3 * fi + 2]};
  float W = 0.f;
  for (int s = 0; s < K; ++s) W += a.fw[(int64_t)s * a.nf + fi];
  *ok = W > 0.f;
  if (!*ok) return;
  float xh[3] = {0, 0, 0};
  for (int s = 0; s < K; ++s) {
    const float* Nd = a.nd.node32 + 16 * a.fidx[(int64_t)s * a.nf + fi];
    wn[s] = a.fw[(int64_t)s * a.nf + fi] / W;
    const float d[3] = {V[0] - Nd[12], V[1] - Nd[13], V[2] - Nd[14]};
    for (int r = 0; r < 3; ++r) {
      am[s][r] = Nd[3 * r] * d[0] + Nd[3 * r + 1] * d[1] + Nd[3 * r + 2] * d[2];
      xh[r] += wn[s] * (am[s][r] + Nd[12 + r] + Nd[9 + r]);
    }
  }
  const float* R = a.fr.R;
  for (int r = 0; r < 3; ++r)
    e[r] = R[3 * r] * xh[0] + R[3 * r + 1] * xh[1] + R[3 * r + 2] * xh[2] + a.fr.T[r] - a.fdst[3 * fi + r];
  for (int r = 0; r < 3; ++r) rp[r] = R[r] * e[0] + R[3 + r] * e[1] + R[6 + r] * e[2];
}

// row r of [ (a.b) I - b a^T , [a]x ; -[b]x , I ]
__device__ __forceinline__ void pt_row(const float* a, const float* b, int r, float* row) {
  const float Ax[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
  const float Bx[9] = {0, -b[2], b[1], b[2], 0, -b[0], -b[1], b[0], 0};
  if (r < 3) {
    const float ab = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
    for (int c = 0; c < 3; ++c) {
      row[c] = (r == c ? ab : 0.f) - b[r] * a[c];
      row[3 + c] = Ax[3 * r + c];
    }
  } else {
    const int rr = r - 3;
    for (int c = 0; c < 3; ++c) {
      row[c] = -Bx[3 * rr + c];
      row[3 + c] = (rr == c) ? 1.f : 0.f;
    }
  }
}

__device__ __forceinline__ void add_row(float* B, int r, const float* row, float w) {
  for (int c = 0; c < 6; ++c)
    if (row[c] != 0.f) atomicAdd(B + 6 * r + c, w * row[c]);
}

__global__ void __launch_bounds__(256) k_assemble_graph(AsmGraphArgs a) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int K = a.K, P = K * (K + 1) / 2;
  const int64_t n_edge = (int64_t)a.nd.m * a.n_nbr * 6, n_fp = (int64_t)a.nf * P * 6, n_fr = (int64_t)a.nf * K;
  float eR = 0.f, eC = 0.f;
  if (tid < n_edge) {
    // Eq. 6, alpha = 1, directed edge j -> l (reading A14):
    // J_j = [-[b]x, I], J_l = [0, -I], b = R_j (g_l - g_j)
    const int64_t ei = tid / 6;
    const int r = (int)(tid % 6);
    const int j = (int)(ei / a.n_nbr), l = a.nbr[ei];
    if (l >= 0) {
      const float* Nj = a.nd.node32 + 16 * j;
      const float* Nl = a.nd.node32 + 16 * l;
      const float d[3] = {Nl[12] - Nj[12], Nl[13] - Nj[13], Nl[14] - Nj[14]};
      float b[3], e[3], row[6];
      for (int q = 0; q < 3; ++q) b[q] = Nj[3 * q] * d[0] + Nj[3 * q + 1] * d[1] + Nj[3 * q + 2] * d[2];
      for (int q = 0; q < 3; ++q) e[q] = b[q] + Nj[12 + q] + Nj[9 + q] - Nl[12 + q] - Nl[9 + q];
      if (r == 0) eR = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
      pt_row(b, b, r, row);                                           // J_j^T J_j
      add_row(a.acc.graph + 36 * (int64_t)a.diag_slot[j], r, row, a.w_reg);
      if (r >= 3) atomicAdd(a.acc.graph + 36 * (int64_t)a.diag_slot[l] + 7 * r, a.w_reg);   // J_l^T J_l
      const float Bx[9] = {0, -b[2], b[1], b[2], 0, -b[0], -b[1], b[0], 0};
      for (int c = 0; c < 6; ++c) row[c] = 0.f;
      if (j < l) {                                                    // J_j^T J_l = [0, -[b]x ; 0, -I]
        if (r < 3) for (int c = 0; c < 3; ++c) row[3 + c] = -Bx[3 * r + c];
        else row[r] = -1.f;
      } else if (r >= 3) {                                            // its transpose [0, 0 ; -[b]x^T, -I]
        for (int c = 0; c < 3; ++c) row[c] = -Bx[3 * c + (r - 3)];
        row[r] = -1.f;
      }
      add_row(a.acc.graph + 36 * (int64_t)a.edge_slot[ei], r, row, a.w_reg);
      if (r < 3) {                                                    // rhs = -J^T e
        const float bxe = b[(r + 1) % 3] * e[(r + 2) % 3] - b[(r + 2) % 3] * e[(r + 1) % 3];
        atomicAdd(a.acc.rhs_graph + 6 * j + r, -a.w_reg * bxe);
      } else {
        atomicAdd(a.acc.rhs_graph + 6 * j + r, -a.w_reg * e[r - 3]);
        atomicAdd(a.acc.rhs_graph + 6 * l + r, a.w_reg * e[r - 3]);
      }
    }
  } else if (tid < n_edge + n_fp + n_fr) {
    // Eq. 9, squared 3-vector residual (reading A12): J_j = w_j R [-[a_j]x, I]
    const bool is_rhs = tid >= n_edge + n_fp;
    const int64_t t2 = is_rhs ? tid - n_edge - n_fp : tid - n_edge;
    const int fi = is_rhs ? (int)(t2 / K) : (int)(t2 / (6 * P));
    float am[MIS_MAX_K][3], wn[MIS_MAX_K], e[3], rp[3];
    bool ok;
    feature_warp(a, fi, am, wn, e, rp, &ok);
    if (ok) {
      if (!is_rhs) {
        const int pr = (int)((t2 / 6) % P), r = (int)(t2 % 6);
        int s = 0, q = pr;
        while (q >= K - s) { q -= K - s; ++s; }
        const int s2 = s + q;
        float row[6];
        pt_row(am[s], am[s2], r, row);
        add_row(a.acc.graph + 36 * (int64_t)a.feat_slot[(int64_t)fi * P + pr], r, row, a.w_corr * wn[s] * wn[s2]);
      } else {
        const int s = (int)(t2 % K);
        if (s == 0) eC = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
        const int node = a.fidx[(int64_t)s * a.nf + fi];
        const float axr[3] = {am[s][1] * rp[2] - am[s][2] * rp[1], am[s][2] * rp[0] - am[s][0] * rp[2],
                              am[s][0] * rp[1] - am[s][1] * rp[0]};
        for (int q = 0; q < 3; ++q) {
          atomicAdd(a.acc.rhs_graph + 6 * node + q, -a.w_corr * wn[s] * axr[q]);
          atomicAdd(a.acc.rhs_graph + 6 * node + 3 + q, -a.w_corr * wn[s] * rp[q]);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    eR += __shfl_xor_sync(0xffffffffu, eR, o);
    eC += __shfl_xor_sync(0xffffffffu, eC, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (eR != 0.f) atomicAdd(a.acc.energy + 2, (double)eR);
    if (eC != 0.f) atomicAdd(a.acc.energy + 3, (double)eC);
  }
}

void launch_assemble_graph(const AsmGraphArgs& a, cudaStream_t s) {
  const int P = a.K * (a.K + 1) / 2;
  const int64_t n = (int64_t)a.nd.m * a.n_nbr * 6 + (int64_t)a.nf * P * 6 + (int64_t)a.nf * a.K;
  if (n <= 0) return;
  k_assemble_graph<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
}


}  // namespace mis
