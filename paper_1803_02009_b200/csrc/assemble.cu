// assemble.cu -- K3 (per-point warp + association + residuals + J^T J) and
// K4/K5 (regulariser and feature terms) of one Gauss-Newton iteration.
//
// K3 design, two kernels per Gauss-Newton iteration:
//  K3a, one thread per point: warp (Eq. 1), projective association (Eq. 7) and
//   residuals in fp64 (the oracle's arithmetic: decisions agree up to rounding
//   order), writing a compact per-point factor state;
//  K3b, one warp per chunk (<= kChunk consecutive points of one kNN-tuple
//   segment, so all points share the K nodes): lanes rebuild the factor rows
//     c' = [w_1 u_1, ..., w_K u_K, r_pl]      u_j = [a_j x n', n'] (Eq. 8 Jacobian row / w_j)
//     e' = [w_1 a_1, w_1, ..., w_K a_K, w_K, r']   (point-to-point moments, r' = R^T (v~ - q))
//   in shared memory.  Every per-chunk sum the normal equations need is an entry
//   of sum_i c'c'^T or sum_i e'e'^T (upper triangles), i.e. two tiny SYRKs: lanes
//   own 4x4 tiles and accumulate them in registers (16 FFMA per 2 LDS.128), then
//   commit each chunk's sums with float4 / float2 atomic adds.  K_finalize turns
//   the moments into 6x6 point-to-point blocks:
//   sum of w_j w_l [-[a_j]x[a_l]x, [a_j]x; -[a_l]x, I].
// Splitting the latency-bound per-point pass (light threads, many warps in
// flight) from the register-heavy SYRK pass doubled the K3 throughput over a
// fused kernel that could keep only 16 warps per SM resident.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "solve_common.cuh"

namespace mis {

#ifndef MIS_K3_SPLIT
#define MIS_K3_SPLIT 1   // 2: split each tile batch into halves across lanes (K3b measured best with 1)
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
#ifndef MIS_K3_STATIC
#define MIS_K3_STATIC 0   // 1: static round-robin chunk schedule (measured ~1.5% slower at C3: tail imbalance)
#endif
#ifndef MIS_K3_MINB
#define MIS_K3_MINB 2   // resident blocks per SM the register budget is sized for
#endif
// ---------------------------------------------------------------- K3a
// One thread per point (points in tuple order, so neighbouring threads read the
// same node states from L1): warp (Eq. 1), projective association (Eq. 7) and
// residuals (Eq. 8, point to point), all in fp64 from the fp64 node state --
// the same arithmetic as the oracle, so every association decision agrees with
// it up to fp64 rounding order (B200 runs fp64 at half the fp32 rate; this pass
// is bound by its loads).  Writes the point's compact factor state, K + 2 float4
// planes
//   s < K: (w_s a_s, w_s)     K: (r', r_pl)     K + 1: (n', 0)
// (zeros when not associated) from which K3b rebuilds the factor rows, and
// accumulates E_data = sum r_pl^2, E_pt = sum |r'|^2 and the association count.
#ifndef MIS_K3A_MINB
#define MIS_K3A_MINB 2
#endif
template <int K>
struct PState {   // a point's compact factor state (zeros: not associated)
  float4 wa[K];   // (w_s a_s, w_s)
  float4 rr;      // (r', r_pl)
  float4 nn;      // (n', 0)
};

// JOINT (NEXT-2, A37): the pose comes from a.pose_cur and is written as factor slot K: (x_hat, 1),
// the form of a node of weight 1 with a = x_hat (Jacobian R [-[x_hat]x, I])
// AFF (NEXT-4, A41-A43): the node matrices are general A_j (same R9 t3 layout); normals warp by
// A_j^-T (cofactors / det; A_j itself if |det| < 1e-9) and the state's slot s holds (w_s d_s, w_s),
// d_s = v - g_s, the factor of the 12-unknown Jacobian rows
// Where a point's K node states come from: the per-point skinning ids (K3a), or the chunk's
// tuple staged in shared memory (the fused K3, every point of a chunk shares its K nodes)
struct NodesGlobal {
  __device__ __forceinline__ int id(const AsmPointsArgs& a, int64_t i, int s) const {
    return a.md.kidx[s * a.md.cap + i];
  }
  __device__ __forceinline__ void get(const AsmPointsArgs& a, int id, int, double2 (&r)[6], const float*& g) const {
    const double2* p = reinterpret_cast<const double2*>(a.nd.Rt64 + 12 * (int64_t)id);   // R (9), t (3)
#pragma unroll
    for (int q = 0; q < 6; ++q) r[q] = __ldg(p + q);
    g = a.nd.g + 3 * (int64_t)id;
  }
};
struct NodesChunk {
  const double2* rt;   // K x 6 double2 (R, t) of the chunk's nodes, shared memory
  const float* g;      // K x 4 (g, pad)
  __device__ __forceinline__ int id(const AsmPointsArgs&, int64_t, int) const { return 0; }
  __device__ __forceinline__ void get(const AsmPointsArgs&, int, int s, double2 (&r)[6], const float*& gp) const {
#pragma unroll
    for (int q = 0; q < 6; ++q) r[q] = rt[6 * s + q];
    gp = g + 4 * s;
  }
};

template <int K, bool DBG, bool JOINT, bool AFF = false, class NS = NodesGlobal>
__device__ __forceinline__ void assoc_point(const AsmPointsArgs& a, int64_t i, PState<K + (JOINT ? 1 : 0)>& st,
                                            double& ed, double& ep, int& as, const NS& ns = NS()) {
  const ModelView& md = a.md;
  const FrameView& fr = a.fr;
  const double v[3] = {md.px[i], md.py[i], md.pz[i]}, n[3] = {md.nx[i], md.ny[i], md.nz[i]};
  double wn[K], W = 0.0;
  int nid[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    wn[s] = md.kw[s * md.cap + i];
    nid[s] = ns.id(a, i, s);
    W += wn[s];
  }
  int pix = -1;
  uint8_t why = 0;
  double vt[3] = {0, 0, 0}, q[3] = {0, 0, 0}, N[3] = {0, 0, 0};
  double xh[3] = {0, 0, 0};
  const double* Rd = JOINT ? a.pose_cur : fr.Rd;
  const double* Td = JOINT ? a.pose_cur + 9 : fr.Td;
  float af[K][3];
#pragma unroll
  for (int s = 0; s < K; ++s) af[s][0] = af[s][1] = af[s][2] = 0.f;
  if (W > 0.0) {
    // divisions and square roots (slow fp64 sequences) are replaced by one reciprocal
    // each and squared comparisons: the results differ from the oracle's only in the
    // last bits, so only exact ties could decide differently
    const double iW = 1.0 / W;
    double mh[3] = {0, 0, 0};
#pragma unroll
    for (int s = 0; s < K; ++s) {
      double2 rq[6];
      const float* g;
      ns.get(a, nid[s], s, rq, g);
      const double2 R01 = rq[0], R23 = rq[1], R45 = rq[2], R67 = rq[3], R8t0 = rq[4], t12 = rq[5];
      wn[s] *= iW;
      const double d0 = v[0] - g[0], d1 = v[1] - g[1], d2 = v[2] - g[2];
      const double a0 = R01.x * d0 + R01.y * d1 + R23.x * d2;
      const double a1 = R23.y * d0 + R45.x * d1 + R45.y * d2;
      const double a2 = R67.x * d0 + R67.y * d1 + R8t0.x * d2;
      if constexpr (AFF) {
        af[s][0] = (float)d0; af[s][1] = (float)d1; af[s][2] = (float)d2;
      } else {
        af[s][0] = (float)a0; af[s][1] = (float)a1; af[s][2] = (float)a2;
      }
      xh[0] += wn[s] * (a0 + (double)g[0] + R8t0.y);
      xh[1] += wn[s] * (a1 + (double)g[1] + t12.x);
      xh[2] += wn[s] * (a2 + (double)g[2] + t12.y);
      if constexpr (AFF) {   // A^-T = cof(A) / det(A)
        const double A0 = R01.x, A1 = R01.y, A2 = R23.x, A3 = R23.y, A4 = R45.x, A5 = R45.y, A6 = R67.x,
                     A7 = R67.y, A8 = R8t0.x;
        double C[9] = {A4 * A8 - A5 * A7, A5 * A6 - A3 * A8, A3 * A7 - A4 * A6,
                       A2 * A7 - A1 * A8, A0 * A8 - A2 * A6, A1 * A6 - A0 * A7,
                       A1 * A5 - A2 * A4, A2 * A3 - A0 * A5, A0 * A4 - A1 * A3};
        const double det = A0 * C[0] + A1 * C[1] + A2 * C[2];
        if (fabs(det) < 1e-9) {
          C[0] = A0; C[1] = A1; C[2] = A2; C[3] = A3; C[4] = A4; C[5] = A5; C[6] = A6; C[7] = A7; C[8] = A8;
        } else {
          const double id = 1.0 / det;
#pragma unroll
          for (int q = 0; q < 9; ++q) C[q] *= id;
        }
        mh[0] += wn[s] * (C[0] * n[0] + C[1] * n[1] + C[2] * n[2]);
        mh[1] += wn[s] * (C[3] * n[0] + C[4] * n[1] + C[5] * n[2]);
        mh[2] += wn[s] * (C[6] * n[0] + C[7] * n[1] + C[8] * n[2]);
      } else {
        mh[0] += wn[s] * (R01.x * n[0] + R01.y * n[1] + R23.x * n[2]);
        mh[1] += wn[s] * (R23.y * n[0] + R45.x * n[1] + R45.y * n[2]);
        mh[2] += wn[s] * (R67.x * n[0] + R67.y * n[1] + R8t0.x * n[2]);
      }
    }
    double nt[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      vt[r] = Rd[3 * r] * xh[0] + Rd[3 * r + 1] * xh[1] + Rd[3 * r + 2] * xh[2] + Td[r];
      nt[r] = Rd[3 * r] * mh[0] + Rd[3 * r + 1] * mh[1] + Rd[3 * r + 2] * mh[2];
    }
    const double ml2 = mh[0] * mh[0] + mh[1] * mh[1] + mh[2] * mh[2];
    if (ml2 >= 1e-24 && vt[2] > 0) {
      why = 1;
      const double iz = 1.0 / vt[2];
      const double fu = floor(fr.fxd * vt[0] * iz + fr.cxd + 0.5), fv = floor(fr.fyd * vt[1] * iz + fr.cyd + 0.5);
      if (fu >= 0 && fv >= 0 && fu < fr.W && fv < fr.H) {
        why |= 2;
        const int px = (int)fu, py = (int)fv;
        const double4 nm = fr.nmapd[py * fr.W + px];   // (N, D) in fp64 (K1)
        if (nm.w > 0) {
          why |= 4;
          if (nm.x != 0 || nm.y != 0 || nm.z != 0) {
            why |= 8;
            N[0] = nm.x; N[1] = nm.y; N[2] = nm.z;
            q[0] = (px - fr.cxd) * nm.w * fr.ifxd;
            q[1] = (py - fr.cyd) * nm.w * fr.ifyd;
            q[2] = nm.w;
            const double e0 = vt[0] - q[0], e1 = vt[1] - q[1], e2 = vt[2] - q[2];
            if (e0 * e0 + e1 * e1 + e2 * e2 < a.eps_dd * a.eps_dd) {   // |v~ - q| < eps_d
              why |= 16;
              const double dot = nt[0] * N[0] + nt[1] * N[1] + nt[2] * N[2];   // n~.N = dot / |m|
              const double ce = a.cos_eps_nd;
              const bool pass = ce >= 0 ? (dot > 0 && dot * dot > ce * ce * ml2) : (dot > 0 || dot * dot < ce * ce * ml2);
              if (pass) { why |= 32; pix = py * fr.W + px; }
            }
          }
        }
      }
    }
  }
  if (DBG) { a.dbg_pix[i] = pix; a.dbg_why[i] = why; }
  if (pix >= 0) {
    as = 1;
    const double e0 = vt[0] - q[0], e1 = vt[1] - q[1], e2 = vt[2] - q[2];
    const double rpl = N[0] * e0 + N[1] * e1 + N[2] * e2;                        // Eq. 8
    const float np0 = (float)(Rd[0] * N[0] + Rd[3] * N[1] + Rd[6] * N[2]);      // n' = R^T N
    const float np1 = (float)(Rd[1] * N[0] + Rd[4] * N[1] + Rd[7] * N[2]);
    const float np2 = (float)(Rd[2] * N[0] + Rd[5] * N[1] + Rd[8] * N[2]);
    const double rp0 = Rd[0] * e0 + Rd[3] * e1 + Rd[6] * e2;                     // r' = R^T (v~ - q)
    const double rp1 = Rd[1] * e0 + Rd[4] * e1 + Rd[7] * e2;
    const double rp2 = Rd[2] * e0 + Rd[5] * e1 + Rd[8] * e2;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const float w = (float)wn[s];
      st.wa[s] = make_float4(w * af[s][0], w * af[s][1], w * af[s][2], w);
    }
    if constexpr (JOINT) st.wa[K] = make_float4((float)xh[0], (float)xh[1], (float)xh[2], 1.f);
    st.rr = make_float4((float)rp0, (float)rp1, (float)rp2, (float)rpl);
    st.nn = make_float4(np0, np1, np2, 0.f);
    ed += rpl * rpl;
    ep += rp0 * rp0 + rp1 * rp1 + rp2 * rp2;
  } else {
#pragma unroll
    for (int s = 0; s < K + (JOINT ? 1 : 0); ++s) st.wa[s] = make_float4(0.f, 0.f, 0.f, 0.f);
    st.rr = st.nn = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// energies and association count: warp sums, one striped fp64 atomic each per warp
__device__ __forceinline__ void commit_point_energies(const AsmPointsArgs& a, double ed, double ep, int as) {
  double ca = as;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ed += __shfl_xor_sync(0xffffffffu, ed, o);
    ep += __shfl_xor_sync(0xffffffffu, ep, o);
    ca += __shfl_xor_sync(0xffffffffu, ca, o);
  }
  if ((threadIdx.x & 31) == 0) {
    energy_add(a.acc.energy, 0, ed);
    energy_add(a.acc.energy, 1, ep);
    energy_add(a.acc.energy, 4, ca);
  }
}

__device__ __forceinline__ void graph_item(const AsmGraphArgs& a, int64_t tid);

// K3a; the blocks after the points' run the K4/K5 items (independent of K3a, same launch)
// SP (sparse state, read by the tcgen05 K3b only): plane K + 1 = (n', associated ? 1 : 0) for every point,
// the other planes only for associated points (~47 % of the points at C5 are not: their planes are
// never read -- K3b builds rows for associated points only)
template <int K, bool DBG, bool JOINT, bool AFF = false, bool SP = false>
__global__ void __launch_bounds__(256, MIS_K3A_MINB) k_assoc_points(AsmPointsArgs a, AsmGraphArgs ga,
                                                                   unsigned point_blocks) {
  pdl_wait();   // node states from the previous solve
  pdl_trigger();   // K3b's CTAs may start their table prologue on the SMs this grid's tail frees
  if (blockIdx.x >= point_blocks) {
    if constexpr (!AFF) graph_item(ga, (int64_t)(blockIdx.x - point_blocks) * blockDim.x + threadIdx.x);
    return;
  }
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double ed = 0.0, ep = 0.0;
  int as = 0;
  if (i < a.md.n) {
    constexpr int KS = K + (JOINT ? 1 : 0);   // factor slots (the pose last, NEXT-2)
    PState<KS> st;
    assoc_point<K, DBG, JOINT, AFF>(a, i, st, ed, ep, as);
    float4* ps = a.pstate;
    const int64_t S = a.pstride;
    if (!SP || as) {
#pragma unroll
      for (int s = 0; s < KS; ++s) ps[s * S + i] = st.wa[s];
      ps[KS * S + i] = st.rr;
    }
    ps[(KS + 1) * S + i] = SP ? make_float4(st.nn.x, st.nn.y, st.nn.z, as ? 1.f : 0.f) : st.nn;
  }
  commit_point_energies(a, ed, ep, as);
}

// factor row of one point from its compact state (K3b: shared memory, FSP floats)
template <int K>
__device__ __forceinline__ void build_row(const PState<K>& st, float* row) {
  using L = Lay<K>;
  const float4 nn = st.nn;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const float4 wa = st.wa[s];   // (w a, w)
    float2* c2 = reinterpret_cast<float2*>(row + 6 * s);
    c2[0] = make_float2(wa.y * nn.z - wa.z * nn.y, wa.z * nn.x - wa.x * nn.z);   // w_j (a_j x n')
    c2[1] = make_float2(wa.x * nn.y - wa.y * nn.x, wa.w * nn.x);                 // w_j n'
    c2[2] = make_float2(wa.w * nn.y, wa.w * nn.z);
    *reinterpret_cast<float4*>(row + L::CDP + 4 * s) = wa;
  }
  row[6 * K] = st.rr.w;
#pragma unroll
  for (int q = 6 * K + 1; q < L::CDP; ++q) row[q] = 0.f;
  row[L::CDP + 4 * K + 0] = st.rr.x;
  row[L::CDP + 4 * K + 1] = st.rr.y;
  row[L::CDP + 4 * K + 2] = st.rr.z;
#pragma unroll
  for (int q = L::CDP + 4 * K + 3; q < L::FS; ++q) row[q] = 0.f;
}

// ---------------------------------------------------------------- K3b
// One warp per chunk (<= kChunk consecutive points of one tuple segment, dynamic
// scheduling): each lane rebuilds its point's factor row from the K3a state
//   c' = [w_1 u_1, ..., w_K u_K, r_pl]      u_j = [a_j x n', n'] (Eq. 8 Jacobian row / w_j)
//   e' = [w_1 a_1, w_1, ..., w_K a_K, w_K, r']   (point-to-point moments)
// in shared memory; lanes own 4x4 tiles of the upper triangles of sum c'c'^T and
// sum e'e'^T and accumulate them in registers (16 FFMA per 2 LDS.128); the
// chunk's sums are committed with float4 / float2 atomic adds into its BSR slots.
// FUSED (k > 4: C5): K3a's association computed per lane into the factor row, the chunk's node
// states staged in shared memory (as k_accum_points_tc<K, true>); the CTAs past point_grid run the
// K4 / K5 items.  Saves the 16 (k + 2) B per point factor-state round trip through HBM.
__device__ __forceinline__ void commit_point_energies(const AsmPointsArgs& a, double ed, double ep, int as);
template <int K, bool FUSED = false>
__global__ void __launch_bounds__(kWarps * 32, MIS_K3_MINB) k_accum_points(AsmPointsArgs a, AsmGraphArgs ga,
                                                                           unsigned point_grid) {
  if constexpr (FUSED) {
    if (blockIdx.x >= point_grid) {
      pdl_wait();
      pdl_trigger();
      graph_item(ga, (int64_t)(blockIdx.x - point_grid) * blockDim.x + threadIdx.x);
      return;
    }
  }
  using L = Lay<K>;
  constexpr int P = L::P;
  constexpr int RT = 52 * P + 20 * K;   // commit record (aliases the warp's row buffer at commit)
  constexpr int NIT = (13 * P + 6 * K + 31) / 32;
  static_assert(RT <= 32 * L::FSP, "record must fit the row buffer");
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* F = reinterpret_cast<float*>(smem4) + warp * (32 * L::FSP);
  float* Rec = F;
  __shared__ int32_t slot_sm[kWarps][P + K];   // the chunk's BSR slots, then its K node ids
  int32_t* slots = slot_sm[warp];
  __shared__ double2 nrt_sm[FUSED ? kWarps : 1][6 * K];   // FUSED: the chunk's node states (R, t)
  __shared__ float4 ng_sm[FUSED ? kWarps : 1][K];          // and positions
  double ed = 0.0, ep = 0.0;
  int n_as = 0;

  // tile table of the two upper triangles: (I, J) in units of 4 entries
  __shared__ uint8_t tabI[L::NT], tabJ[L::NT];
  // per lane: record index of each of its items' 16 tile entries (-1: not part of the system)
  __shared__ int16_t dm[L::RI * 16][32];
  __shared__ uint32_t cdesc[NIT][32];   // commit items, as in k_accum_points_tc
  // tiles in blocks of 4 rows x 8 columns of the tile grid (each triangle separately), so the 32
  // lanes of one round read <= 4 distinct A and <= 8 distinct B float4 of a point's row: two
  // shared-memory wavefronts per point and round instead of three (row-major order: up to 13 B's)
  if (threadIdx.x == 0) {
    int t = 0;
#pragma unroll 1
    for (int e = 0; e < 2; ++e) {
      const int nb = e ? L::NE : L::ND;
      for (int I0 = 0; I0 < nb; I0 += 4)
        for (int J0 = I0; J0 < nb; J0 += 8)
          for (int dI = 0; dI < 4; ++dI)
            for (int dJ = 0; dJ < 8; ++dJ) {
              const int I = I0 + dI, J = J0 + dJ;
              if (I < nb && J < nb && I <= J) {
                tabI[t] = (uint8_t)I;
                tabJ[t] = (uint8_t)J;
                ++t;
              }
            }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < L::RI * 16 * 32; q += blockDim.x) {
    const int ln = q & 31, rv = q >> 5, r = rv >> 4, v = rv & 15, it = ln + 32 * r;
    int d = -1;
    if (it < L::NI) {
      const int t = it % L::NT, A = 4 * tabI[t] + (v >> 2), B = 4 * tabJ[t] + (v & 3);
      if (A <= B) {
        if (t < L::TD) {             // c' = [w_j u_j ..., r_pl]
          if (B < 6 * K) d = 52 * pair_index(A / 6, B / 6, K) + 6 * (A % 6) + (B % 6);
          else if (B == 6 * K && A < 6 * K) d = 52 * P + 20 * (A / 6) + (A % 6);
        } else {                     // e' = [w_j a_j, w_j ..., r']
          if (B < 4 * K) d = 52 * pair_index(A / 4, B / 4, K) + 36 + 4 * (A % 4) + (B % 4);
          else if (B < 4 * K + 3 && A < 4 * K) d = 52 * P + 20 * (A / 4) + 8 + 3 * (A % 4) + (B - 4 * K);
        }
      }
    }
    dm[rv][ln] = (int16_t)d;
  }
  for (int q = threadIdx.x; q < NIT * 32; q += blockDim.x) {
    const int it = q;
    uint32_t d = ~0u;
    if (it < 13 * P) {
      const int pr = it / 13, qq = it - 13 * pr;
      d = (qq < 9 ? 0u : 1u) | ((uint32_t)pr << 2) | ((uint32_t)(qq < 9 ? 4 * qq : 4 * (qq - 9)) << 10) |
          ((uint32_t)(4 * it) << 18);
    } else if (it < 13 * P + 6 * K) {
      const int t2 = it - 13 * P, sl = t2 / 6, qq = t2 - 6 * sl;
      d = qq < 3 ? (2u | ((uint32_t)sl << 2) | ((uint32_t)(2 * qq) << 10) | ((uint32_t)(52 * P + 20 * sl + 2 * qq) << 18))
                 : (3u | ((uint32_t)sl << 2) | ((uint32_t)(4 * (qq - 3)) << 10) |
                    ((uint32_t)(52 * P + 20 * sl + 8 + 4 * (qq - 3)) << 18));
    }
    cdesc[q / 32][q % 32] = d;
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

  pdl_wait();   // K3a's factor state (the tables above are independent of it)
  pdl_trigger();   // the finalisation may launch early (it waits for this grid's completion)
  // dynamic chunk scheduling (segments are uneven): one atomic fetch per chunk per warp
  int64_t c = 0;
  if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
  c = __shfl_sync(0xffffffffu, c, 0);
  const float4* ps = a.pstate;
  const int64_t S = a.pstride;
  for (; c < a.nchunk;) {
    const int4 ch = a.chunks[c];
    const int seg = ch.x;
    const int32_t* nodes = a.seg_nodes + (int64_t)seg * K;
    __syncwarp();
    for (int q = lane; q < P + K; q += 32) slots[q] = q < P ? a.seg_slot[(int64_t)seg * P + q] : nodes[q - P];
    if constexpr (FUSED) {   // stage the chunk's node states (fp64 master) and positions
      for (int q = lane; q < 7 * K; q += 32) {
        if (q < 6 * K) {
          nrt_sm[warp][q] = __ldg(reinterpret_cast<const double2*>(a.nd.Rt64 + 12 * (int64_t)nodes[q / 6]) + q % 6);
        } else {
          const float* g = a.nd.g + 3 * (int64_t)nodes[q - 6 * K];
          ng_sm[warp][q - 6 * K] = make_float4(g[0], g[1], g[2], 0.f);
        }
      }
      __syncwarp();
    }
    float acc[L::RI][16];
#pragma unroll
    for (int r = 0; r < L::RI; ++r)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[r][e] = 0.f;
    // the Gram sums over the rows F[0, np)
    auto gram = [&](int np) {
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
    };
    // Only associated points enter the sums (an unassociated point's state is all zeros, its rows
    // add nothing): their rows are compacted into F across the chunk's 32-point loads and the Gram
    // pass runs once per 32 rows (C5: ~53% of the points are associated)
    int fill = 0, nlive = 0;
    for (int base = ch.y; base < ch.z || fill > 0; base += 32) {
      const int64_t i = base + lane;
      PState<K> st;
      bool live = false;
      if (i < ch.z) {
        if constexpr (FUSED) {
          int as1 = 0;
          const NodesChunk nc{nrt_sm[warp], reinterpret_cast<const float*>(ng_sm[warp])};
          assoc_point<K, false, false, false, NodesChunk>(a, i, st, ed, ep, as1, nc);
          n_as += as1;
        } else {
#pragma unroll
          for (int s = 0; s < K; ++s) st.wa[s] = ps[s * S + i];
          st.rr = ps[K * S + i];
          st.nn = ps[(K + 1) * S + i];
        }
#pragma unroll
        for (int s = 0; s < K; ++s) live |= st.wa[s].w != 0.f;   // sum w = 1 when associated
      }
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      const int slot = live ? fill + __popc(bal & ((1u << lane) - 1u)) : -1;   // compacted row
      if (slot >= 0 && slot < 32) build_row<K>(st, F + slot * L::FSP);
      fill += __popc(bal);
      nlive += __popc(bal);
      if (fill >= 32 || (base + 32 >= ch.z && fill > 0)) {   // one call site of the pass
        const int np = min(fill, 32);
        __syncwarp();
        gram(np);
        __syncwarp();
        fill -= np;
        if (slot >= 32) {
          if constexpr (!FUSED) {   // reload (L1) rather than keep the state live across the pass
            const int64_t i2 = base + lane;
#pragma unroll
            for (int s = 0; s < K; ++s) st.wa[s] = ps[s * S + i2];
            st.rr = ps[K * S + i2];
            st.nn = ps[(K + 1) * S + i2];
          }
          build_row<K>(st, F + (slot - 32) * L::FSP);   // (an overflowing last load: one more trip)
        }
      }
    }
    if (nlive == 0) {   // no associated point in the chunk (e.g. outside the view): nothing to commit
      if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
      c = __shfl_sync(0xffffffffu, c, 0);
      continue;
    }
    // ---- commit: tiles scattered into the warp's record (aliasing the row buffer; a second batch
    // half adds to the first's entries), then one aligned shared load + vector atomic per item
    for (int q = lane; q < RT / 4; q += 32) reinterpret_cast<float4*>(Rec)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < L::SPLIT; ++h) {
#pragma unroll
      for (int r = 0; r < L::RI; ++r) {
        if (!tV[r] || (lane + 32 * r) / L::NT != h) continue;
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const int d = dm[16 * r + v][lane];
          if (d >= 0) Rec[d] = h == 0 ? acc[r][v] : Rec[d] + acc[r][v];
        }
      }
      __syncwarp();
    }
    int64_t next_chunk = 0;
    if (lane == 0) next_chunk = (int64_t)atomicAdd(a.work_counter, 1ull);   // prefetch the next chunk id
#pragma unroll 1
    for (int k = 0; k < NIT; ++k) {
      const uint32_t d = cdesc[k][lane];
      if (d == ~0u) continue;
      const uint32_t kind = d & 3u, idx = (d >> 2) & 255u, off = (d >> 10) & 255u;
      const float* src = Rec + (d >> 18);
      if (kind == 2u) {
        const float2 v = *reinterpret_cast<const float2*>(src);
        if (v.x != 0.f || v.y != 0.f)
          atomicAdd(reinterpret_cast<float2*>(a.acc.rhs_data + 6 * (int64_t)slots[P + idx] + off), v);
      } else {
        const float4 v = *reinterpret_cast<const float4*>(src);
        if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
        float* dst = kind == 0u ? a.acc.data + 36 * (int64_t)slots[idx]
                   : kind == 1u ? a.acc.mom + 16 * (int64_t)slots[idx] : a.acc.node_mom + 12 * (int64_t)slots[P + idx];
        atomicAdd(reinterpret_cast<float4*>(dst + off), v);
      }
    }
    __syncwarp();
    c = __shfl_sync(0xffffffffu, next_chunk, 0);
  }
  if constexpr (FUSED) commit_point_energies(a, ed, ep, n_as);
}

// ---------------------------------------------------------------- K3b on tensor cores (k <= 4)
// The same per-chunk sums as k_accum_points, as two small GEMMs per 8-point step on the tensor
// cores: C_c += F_c^T F_c (c' block, 32 x 32 padded) and C_e += F_e^T F_e (e' block, 32 x 24),
// mma.sync m16n8k8 TF32 with the 3xTF32 split (a = a_hi + a_lo; a_hi b_hi + a_hi b_lo + a_lo b_hi,
// FP32 accumulation): products to ~2^-21 relative, as accurate as the FP32 FMA path for these
// sums, at a fraction of its issue slots.  Only the upper-triangle tiles are computed (10 of 14).
constexpr int kTcFSP = 72;   // row stride: c' [0, 32) | e' [32, 64) | pad; 72 = 8 (mod 32): conflict-free
// per-warp commit record of the tensor-core K3b: P pair records of 52 (36 data | 16 moments),
// then K node records of 20 (6 rhs | 2 pad | 12 node moments), so every commit item is one
// aligned float2 / float4 shared load
__host__ __device__ constexpr int tc_rec_floats(int K) { return 52 * (K * (K + 1) / 2) + 20 * K; }

template <int K>
__device__ __forceinline__ void build_row_tc(const PState<K>& st, float* row) {
  const float4 nn = st.nn;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const float4 wa = st.wa[s];   // (w a, w)
    row[6 * s + 0] = wa.y * nn.z - wa.z * nn.y;   // w_j (a_j x n')
    row[6 * s + 1] = wa.z * nn.x - wa.x * nn.z;
    row[6 * s + 2] = wa.x * nn.y - wa.y * nn.x;
    row[6 * s + 3] = wa.w * nn.x;                 // w_j n'
    row[6 * s + 4] = wa.w * nn.y;
    row[6 * s + 5] = wa.w * nn.z;
    *reinterpret_cast<float4*>(row + 32 + 4 * s) = wa;
  }
  row[6 * K] = st.rr.w;
#pragma unroll
  for (int q = 6 * K + 1; q < 32; ++q) row[q] = 0.f;
  row[32 + 4 * K + 0] = st.rr.x;
  row[32 + 4 * K + 1] = st.rr.y;
  row[32 + 4 * K + 2] = st.rr.z;
#pragma unroll
  for (int q = 32 + 4 * K + 3; q < 64; ++q) row[q] = 0.f;
}

// 3xTF32 split by truncation: hi = x with the 13 low mantissa bits cleared (what the
// tensor core reads of a TF32 operand), lo = x - hi exactly (the tensor core truncates
// lo in turn).  Two integer/FP ops per element; cvt.rna.tf32.f32 costs ~6 on sm_100.
// Dropped terms: lo lo' and the truncation of lo, both < 2^-20 relative per product.
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A fragments (hi, lo) of F^T for the two 16-row tiles of one block (column base cb), k-step k0,
// and the B fragments of the four n8 tiles (pairs (a0, a2) / (a1, a3) of the A quads, kept as
// their own registers so each mma reads aligned pairs without per-tile moves)
struct FragT {
  uint32_t h[2][4], l[2][4];
  uint32_t bh[4][2], bl[4][2];
};
__device__ __forceinline__ void load_frag(const float* F, int k0, int cb, int g, int tig, FragT& f) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const float x[4] = {F[(k0 + tig) * kTcFSP + cb + 16 * mi + g], F[(k0 + tig) * kTcFSP + cb + 16 * mi + g + 8],
                        F[(k0 + tig + 4) * kTcFSP + cb + 16 * mi + g],
                        F[(k0 + tig + 4) * kTcFSP + cb + 16 * mi + g + 8]};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      f.h[mi][q] = tf32_hi(x[q]);
      f.l[mi][q] = __float_as_uint(x[q] - __uint_as_float(f.h[mi][q]));
    }
#pragma unroll
    for (int bq = 0; bq < 2; ++bq) {
      f.bh[2 * mi + bq][0] = f.h[mi][bq];
      f.bh[2 * mi + bq][1] = f.h[mi][bq + 2];
      f.bl[2 * mi + bq][0] = f.l[mi][bq];
      f.bl[2 * mi + bq][1] = f.l[mi][bq + 2];
    }
  }
}

// tile (mi, ni): the B fragment of n8-tile ni is part of the A fragment of m16-tile ni / 2
__device__ __forceinline__ void mma3(float (&d)[4], const FragT& f, int mi, int ni) {
  mma_tf32(d, f.h[mi][0], f.h[mi][1], f.h[mi][2], f.h[mi][3], f.bh[ni][0], f.bh[ni][1]);
  mma_tf32(d, f.h[mi][0], f.h[mi][1], f.h[mi][2], f.h[mi][3], f.bl[ni][0], f.bl[ni][1]);
  mma_tf32(d, f.l[mi][0], f.l[mi][1], f.l[mi][2], f.l[mi][3], f.bh[ni][0], f.bh[ni][1]);
}

// FUSED: K3a and K3b in one kernel -- every point of a chunk shares the chunk's k nodes, so the
// warp stages their fp64 states in shared memory once per chunk and each lane computes its
// point's association, residuals and factor state (assoc_point, the K3a arithmetic) straight
// into its factor row: no per-point node loads, no factor-state round trip through memory.
// The CTAs past point_grid run the K4 / K5 items (as K3a's extra blocks do).
template <int K, bool FUSED = false>
__global__ void __launch_bounds__(kWarps * 32, MIS_K3_MINB) k_accum_points_tc(AsmPointsArgs a, AsmGraphArgs ga,
                                                                              unsigned point_grid) {
  static_assert(6 * K + 1 <= 32 && 4 * K + 3 <= 24, "tensor-core K3b: k <= 4");
  if constexpr (FUSED) {
    if (blockIdx.x >= point_grid) {
      pdl_wait();   // node states of the previous solve
      pdl_trigger();
      graph_item(ga, (int64_t)(blockIdx.x - point_grid) * blockDim.x + threadIdx.x);
      return;
    }
  }
  constexpr int P = K * (K + 1) / 2;
  constexpr int RT = tc_rec_floats(K);
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  float* F = reinterpret_cast<float*>(smem4) + warp * (32 * kTcFSP);
  float* Rec = reinterpret_cast<float*>(smem4) + kWarps * 32 * kTcFSP + warp * RT;
  __shared__ int32_t slot_sm[kWarps][P + K];   // the chunk's BSR slots, then its K node ids
  int32_t* slots = slot_sm[warp];
  __shared__ double2 nrt_sm[FUSED ? kWarps : 1][6 * K];   // FUSED: the chunk's node states (R, t)
  __shared__ float4 ng_sm[FUSED ? kWarps : 1][K];          // and positions
  double ed = 0.0, ep = 0.0;
  int n_as = 0;
  // where each summed entry goes: inv[q] = record index of position q of the dumped sums
  // (c' 32 x 32 at 0, e' 24 x 24 at 1024; upper triangles), -1: not part of the system
  __shared__ int16_t inv[32 * 32 + 24 * 24];
  for (int q = threadIdx.x; q < 32 * 32 + 24 * 24; q += blockDim.x) {
    const bool e = q >= 1024;
    const int A = e ? (q - 1024) / 24 : q / 32, B = e ? (q - 1024) % 24 : q % 32;
    int d = -1;
    if (A <= B) {
      if (!e) {                    // c' = [w_j u_j ..., r_pl]
        if (B < 6 * K) d = 52 * pair_index(A / 6, B / 6, K) + 6 * (A % 6) + (B % 6);
        else if (B == 6 * K && A < 6 * K) d = 52 * P + 20 * (A / 6) + (A % 6);
      } else {                     // e' = [w_j a_j, w_j ..., r']
        if (B < 4 * K) d = 52 * pair_index(A / 4, B / 4, K) + 36 + 4 * (A % 4) + (B % 4);
        else if (B < 4 * K + 3 && A < 4 * K) d = 52 * P + 20 * (A / 4) + 8 + 3 * (A % 4) + (B - 4 * K);
      }
    }
    inv[q] = (int16_t)d;
  }
  for (int q = lane; q < RT; q += 32) Rec[q] = 0.f;   // entries no fragment maps to stay zero
  // commit items of each lane (item it = lane + 32 k), decoded once: kind (0 data, 1 moments,
  // 2 node rhs, 3 node moments) | record index (pair or node slot) << 2 | offset in the
  // destination record << 10 | offset in Rec (floats) << 18; ~0u: no item
  constexpr int NIT = (13 * P + 6 * K + 31) / 32;
  __shared__ uint32_t cdesc[NIT][32];
  for (int q = threadIdx.x; q < NIT * 32; q += blockDim.x) {
    const int it = q;   // = lane + 32 k with k = q / 32
    uint32_t d = ~0u;
    if (it < 13 * P) {
      const int pr = it / 13, qq = it - 13 * pr;
      d = (qq < 9 ? 0u : 1u) | ((uint32_t)pr << 2) | ((uint32_t)(qq < 9 ? 4 * qq : 4 * (qq - 9)) << 10) |
          ((uint32_t)(4 * it) << 18);
    } else if (it < 13 * P + 6 * K) {
      const int t2 = it - 13 * P, sl = t2 / 6, qq = t2 - 6 * sl;
      d = qq < 3 ? (2u | ((uint32_t)sl << 2) | ((uint32_t)(2 * qq) << 10) | ((uint32_t)(52 * P + 20 * sl + 2 * qq) << 18))
                 : (3u | ((uint32_t)sl << 2) | ((uint32_t)(4 * (qq - 3)) << 10) |
                    ((uint32_t)(52 * P + 20 * sl + 8 + 4 * (qq - 3)) << 18));
    }
    cdesc[q / 32][q % 32] = d;
  }
  __syncthreads();
  // this lane's 36 fragment positions -> record indices, packed in pairs (0xffff: dropped)
  // (in shared memory, the same for every warp, read once per chunk at the commit: 18 registers fewer
  // live across the chunk loop, whose spills sat on the per-chunk path)
  __shared__ uint32_t dmap_sm[18][32];
  if (warp == 0) {
    const int tmi[6] = {0, 0, 0, 0, 1, 1}, tni[6] = {0, 1, 2, 3, 2, 3};
    const int emi[3] = {0, 0, 0}, eni[3] = {0, 1, 2};
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const bool e = t >= 6;
      const int r0 = 16 * (e ? emi[t - 6] : tmi[t]) + g, c0 = 8 * (e ? eni[t - 6] : tni[t]) + 2 * tig;
      int d4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int rr = r0 + 8 * (h >> 1), cc = c0 + (h & 1);
        d4[h] = e ? (rr < 24 ? inv[1024 + rr * 24 + cc] : -1) : inv[rr * 32 + cc];
      }
      dmap_sm[2 * t][lane] = (uint32_t)(d4[0] & 0xffff) | ((uint32_t)(d4[1] & 0xffff) << 16);
      dmap_sm[2 * t + 1][lane] = (uint32_t)(d4[2] & 0xffff) | ((uint32_t)(d4[3] & 0xffff) << 16);
    }
  }
  __syncthreads();

  pdl_wait();   // K3a's factor state (the tables above are independent of it)
  pdl_trigger();   // the finalisation may launch early (it waits for this grid's completion)
  // chunk schedule: dynamic through one global counter (default), or static round robin over the
  // grid's warps with the next chunk's header loaded one chunk ahead (MIS_K3_STATIC=1): ~12% of
  // the fused kernel's stall samples sit on the counter's atomics, but the static schedule's tail
  // imbalance costs more (C3: 0.647 vs 0.637 ms/step)
  const int64_t cstride = (int64_t)point_grid * kWarps;
  int64_t c = 0;
  if (MIS_K3_STATIC) {
    c = (int64_t)blockIdx.x * kWarps + warp;
  } else {
    if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
  }
  const float4* ps = a.pstate;
  const int64_t S = a.pstride;
  int4 ch_next = c < a.nchunk ? a.chunks[c] : make_int4(0, 0, 0, 0);
  for (; c < a.nchunk;) {
    const int4 ch = ch_next;
    if (MIS_K3_STATIC && c + cstride < a.nchunk) ch_next = a.chunks[c + cstride];   // in flight meanwhile
    const int seg = ch.x;
    const int32_t* nodes = a.seg_nodes + (int64_t)seg * K;
    __syncwarp();
    if (lane < P) slots[lane] = a.seg_slot[(int64_t)seg * P + lane];
    else if (lane < P + K) slots[lane] = nodes[lane - P];
    if constexpr (FUSED) {   // stage the chunk's node states (fp64 master) and positions
      if (lane < 6 * K) {
        const int nid = nodes[lane / 6];
        nrt_sm[warp][lane] = __ldg(reinterpret_cast<const double2*>(a.nd.Rt64 + 12 * (int64_t)nid) + lane % 6);
      } else if (lane < 7 * K) {
        const int nid = nodes[lane - 6 * K];
        const float* g = a.nd.g + 3 * (int64_t)nid;
        ng_sm[warp][lane - 6 * K] = make_float4(g[0], g[1], g[2], 0.f);
      }
      __syncwarp();
    }
    // c' tiles (0,0..3),(1,2),(1,3); e' tiles (0,0..2) -- the e' rows >= 4k (r') pair only with
    // each other there, which the system does not use
    float dc[6][4], de[3][4];
#pragma unroll
    for (int t = 0; t < 6; ++t) dc[t][0] = dc[t][1] = dc[t][2] = dc[t][3] = 0.f;
#pragma unroll
    for (int t = 0; t < 3; ++t) de[t][0] = de[t][1] = de[t][2] = de[t][3] = 0.f;
    auto gram = [&](int np) {   // rows F[0, np), np rounded up to the k-step (the rows past np are zero)
      for (int k0 = 0; k0 < np; k0 += 8) {
        FragT f;
        load_frag(F, k0, 0, g, tig, f);   // c'
        mma3(dc[0], f, 0, 0);
        mma3(dc[1], f, 0, 1);
        mma3(dc[2], f, 0, 2);
        mma3(dc[3], f, 0, 3);
        mma3(dc[4], f, 1, 2);
        mma3(dc[5], f, 1, 3);
        load_frag(F, k0, 32, g, tig, f);   // e'
        mma3(de[0], f, 0, 0);
        mma3(de[1], f, 0, 1);
        mma3(de[2], f, 0, 2);
      }
    };
    // associated points' rows compacted across the chunk's loads (as in k_accum_points): the
    // mma passes skip the unassociated points' zero rows
    int fill = 0, nlive = 0;
    for (int base = ch.y; base < ch.z; base += 32) {
      const int64_t i = base + lane;
      PState<K> st;
      bool live = false;
      if (i < ch.z) {
        if constexpr (FUSED) {
          int as1 = 0;
          const NodesChunk nc{nrt_sm[warp], reinterpret_cast<const float*>(ng_sm[warp])};
          assoc_point<K, false, false, false, NodesChunk>(a, i, st, ed, ep, as1, nc);
          n_as += as1;
        } else {
#pragma unroll
          for (int s = 0; s < K; ++s) st.wa[s] = ps[s * S + i];
          st.rr = ps[K * S + i];
          st.nn = ps[(K + 1) * S + i];
        }
#pragma unroll
        for (int s = 0; s < K; ++s) live |= st.wa[s].w != 0.f;   // sum w = 1 when associated
      }
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      const int pos = fill + __popc(bal & ((1u << lane) - 1u));
      if (live && pos < 32) build_row_tc<K>(st, F + pos * kTcFSP);
      fill += __popc(bal);
      nlive += __popc(bal);
      if (fill >= 32) {
        __syncwarp();
        gram(32);
        __syncwarp();
        fill -= 32;
        if (live && pos >= 32) build_row_tc<K>(st, F + (pos - 32) * kTcFSP);
      }
    }
    if (fill > 0) {   // zero rows up to the next k-step, then the last pass
      const int np = (fill + 7) & ~7;
      if (lane >= fill && lane < np) {
        float4* z = reinterpret_cast<float4*>(F + lane * kTcFSP);
#pragma unroll
        for (int q = 0; q < 16; ++q) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncwarp();
      gram(np);
    }
    __syncwarp();
    if (nlive == 0) {   // no associated point in the chunk: nothing to commit
      if (!MIS_K3_STATIC && lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
      c = MIS_K3_STATIC ? c + cstride : __shfl_sync(0xffffffffu, c, 0);
      if (!MIS_K3_STATIC && c < a.nchunk) ch_next = a.chunks[c];
      continue;
    }
    // ---- commit: fragments -> the warp's record (scattered by the per-lane map) -> atomic adds
    {
      auto put = [&](uint32_t pk, float v0, float v1) {
        const uint32_t d0 = pk & 0xffffu, d1 = pk >> 16;
        if (d0 != 0xffffu) Rec[d0] = v0;
        if (d1 != 0xffffu) Rec[d1] = v1;
      };
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        put(dmap_sm[2 * t][lane], dc[t][0], dc[t][1]);
        put(dmap_sm[2 * t + 1][lane], dc[t][2], dc[t][3]);
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        put(dmap_sm[12 + 2 * t][lane], de[t][0], de[t][1]);
        put(dmap_sm[12 + 2 * t + 1][lane], de[t][2], de[t][3]);
      }
    }
    __syncwarp();
    int64_t next_chunk = c + cstride;
    if (!MIS_K3_STATIC && lane == 0) next_chunk = (int64_t)atomicAdd(a.work_counter, 1ull);   // prefetch the next id
#pragma unroll
    for (int k = 0; k < NIT; ++k) {
      const uint32_t d = cdesc[k][lane];
      if (d == ~0u) continue;
      const uint32_t kind = d & 3u, idx = (d >> 2) & 255u, off = (d >> 10) & 255u;
      const float* src = Rec + (d >> 18);
      if (kind == 2u) {
        const float2 v = *reinterpret_cast<const float2*>(src);
        if (v.x != 0.f || v.y != 0.f)
          atomicAdd(reinterpret_cast<float2*>(a.acc.rhs_data + 6 * (int64_t)slots[P + idx] + off), v);
      } else {
        const float4 v = *reinterpret_cast<const float4*>(src);
        if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
        float* dst = kind == 0u ? a.acc.data + 36 * (int64_t)slots[idx]
                   : kind == 1u ? a.acc.mom + 16 * (int64_t)slots[idx] : a.acc.node_mom + 12 * (int64_t)slots[P + idx];
        atomicAdd(reinterpret_cast<float4*>(dst + off), v);
      }
    }
    __syncwarp();
    c = __shfl_sync(0xffffffffu, next_chunk, 0);
    if (!MIS_K3_STATIC && c < a.nchunk) ch_next = a.chunks[c];
  }
  if constexpr (FUSED) commit_point_energies(a, ed, ep, n_as);
}

// ---- tensor-core K3b for 5 <= k <= 8 (C5): the same per-chunk Gram sums as k_accum_points_tc with
// c' padded to 64 columns and e' to 40, upper-triangle 16x8 tiles restricted to the entries the
// system uses (c' rows < 6k, columns <= 6k; e' rows < 4k, columns < 4k + 3): 15 + 8 tiles at k = 8.
// 92 accumulator registers, so one 8-warp CTA per SM; the fragment -> record map and the commit
// items are tables in shared memory.
#ifndef MIS_K3B_TCW
#define MIS_K3B_TCW 0
#endif
template <int K>
struct TcW {
  static constexpr int CW = 64, EW = 40, S = 104;   // row: c' [0, 64) | e' [64, 104); 104 = 8 (mod 32)
  static constexpr int CMT = (6 * K + 15) / 16, CNT = (6 * K) / 8 + 1;
  static constexpr int EMT = (4 * K + 15) / 16, ENT = (4 * K + 2) / 8 + 1;
  static constexpr int CQ = (CMT > (CNT + 1) / 2 ? CMT : (CNT + 1) / 2);   // A quads loaded for c'
  static constexpr int EQ = (EMT > (ENT + 1) / 2 ? EMT : (ENT + 1) / 2);
  static constexpr int NC = CMT * CNT - CMT * (CMT - 1), NE = EMT * ENT - EMT * (EMT - 1);
  static constexpr int NT = NC + NE;
  static constexpr int P = K * (K + 1) / 2;
  static constexpr int RT = 52 * P + 20 * K;
  static constexpr int NIT = (13 * P + 6 * K + 31) / 32;
  __host__ __device__ static constexpr int cidx(int mi, int ni) { return mi * CNT - mi * (mi - 1) + (ni - 2 * mi); }
  __host__ __device__ static constexpr int eidx(int mi, int ni) { return NC + mi * ENT - mi * (mi - 1) + (ni - 2 * mi); }
};

template <int QM, int NB>
struct FragW {
  uint32_t h[QM][4], l[QM][4];
  uint32_t bh[NB][2], bl[NB][2];
};
template <int QM, int NB, int S>
__device__ __forceinline__ void load_frag_w(const float* F, int k0, int cb, int g, int tig, FragW<QM, NB>& f) {
#pragma unroll
  for (int mi = 0; mi < QM; ++mi) {
    const float x[4] = {F[(k0 + tig) * S + cb + 16 * mi + g], F[(k0 + tig) * S + cb + 16 * mi + g + 8],
                        F[(k0 + tig + 4) * S + cb + 16 * mi + g], F[(k0 + tig + 4) * S + cb + 16 * mi + g + 8]};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      f.h[mi][q] = tf32_hi(x[q]);
      f.l[mi][q] = __float_as_uint(x[q] - __uint_as_float(f.h[mi][q]));
    }
#pragma unroll
    for (int bq = 0; bq < 2; ++bq)
      if (2 * mi + bq < NB) {
        f.bh[2 * mi + bq][0] = f.h[mi][bq];
        f.bh[2 * mi + bq][1] = f.h[mi][bq + 2];
        f.bl[2 * mi + bq][0] = f.l[mi][bq];
        f.bl[2 * mi + bq][1] = f.l[mi][bq + 2];
      }
  }
}
template <int QM, int NB>
__device__ __forceinline__ void mma3w(float (&d)[4], const FragW<QM, NB>& f, int mi, int ni) {
  mma_tf32(d, f.h[mi][0], f.h[mi][1], f.h[mi][2], f.h[mi][3], f.bh[ni][0], f.bh[ni][1]);
  mma_tf32(d, f.h[mi][0], f.h[mi][1], f.h[mi][2], f.h[mi][3], f.bl[ni][0], f.bl[ni][1]);
  mma_tf32(d, f.l[mi][0], f.l[mi][1], f.l[mi][2], f.l[mi][3], f.bh[ni][0], f.bh[ni][1]);
}

template <int K>
__device__ __forceinline__ void build_row_w(const PState<K>& st, float* row) {
  using T = TcW<K>;
  const float4 nn = st.nn;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const float4 wa = st.wa[s];
    row[6 * s + 0] = wa.y * nn.z - wa.z * nn.y;
    row[6 * s + 1] = wa.z * nn.x - wa.x * nn.z;
    row[6 * s + 2] = wa.x * nn.y - wa.y * nn.x;
    row[6 * s + 3] = wa.w * nn.x;
    row[6 * s + 4] = wa.w * nn.y;
    row[6 * s + 5] = wa.w * nn.z;
    *reinterpret_cast<float4*>(row + T::CW + 4 * s) = wa;
  }
  row[6 * K] = st.rr.w;
#pragma unroll
  for (int q = 6 * K + 1; q < T::CW; ++q) row[q] = 0.f;
  row[T::CW + 4 * K + 0] = st.rr.x;
  row[T::CW + 4 * K + 1] = st.rr.y;
  row[T::CW + 4 * K + 2] = st.rr.z;
#pragma unroll
  for (int q = T::CW + 4 * K + 3; q < T::CW + T::EW; ++q) row[q] = 0.f;
}

template <int K>
__global__ void __launch_bounds__(kWarps * 32, 1) k_accum_points_tcw(AsmPointsArgs a) {
  using T = TcW<K>;
  constexpr int P = T::P, RT = T::RT, NIT = T::NIT, S = T::S;
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  float* F = reinterpret_cast<float*>(smem4) + warp * (32 * S);
  float* Rec = reinterpret_cast<float*>(smem4) + kWarps * 32 * S + warp * RT;
  int16_t* dmap = reinterpret_cast<int16_t*>(reinterpret_cast<float*>(smem4) + kWarps * (32 * S + RT));  // [4 NT][32]
  __shared__ int32_t slot_sm[kWarps][P + K];
  __shared__ uint32_t cdesc[NIT][32];
  int32_t* slots = slot_sm[warp];
  // fragment position (row A, column B of the c' or e' Gram matrix) -> record index, -1: unused
  auto rec_of = [&](bool e, int A, int B) -> int {
    if (A > B) return -1;
    if (!e) {
      if (B < 6 * K) return 52 * pair_index(A / 6, B / 6, K) + 6 * (A % 6) + (B % 6);
      if (B == 6 * K && A < 6 * K) return 52 * P + 20 * (A / 6) + (A % 6);
      return -1;
    }
    if (B < 4 * K) return 52 * pair_index(A / 4, B / 4, K) + 36 + 4 * (A % 4) + (B % 4);
    if (B < 4 * K + 3 && A < 4 * K) return 52 * P + 20 * (A / 4) + 8 + 3 * (A % 4) + (B - 4 * K);
    return -1;
  };
  for (int q = threadIdx.x; q < 4 * T::NT * 32; q += blockDim.x) {   // dmap[4 t + h][lane]
    const int ln = q & 31, th = q >> 5, t = th >> 2, h = th & 3, gg = ln >> 2, tg = ln & 3;
    int mi = 0, ni = 0;
    bool e = t >= T::NC;
    {
      int r = e ? t - T::NC : t;
      const int MT = e ? T::EMT : T::CMT, NTL = e ? T::ENT : T::CNT;
      for (int m = 0; m < MT; ++m) {
        const int cnt = NTL - 2 * m;
        if (r < cnt) { mi = m; ni = 2 * m + r; break; }
        r -= cnt;
      }
    }
    const int A = 16 * mi + gg + 8 * (h >> 1), B = 8 * ni + 2 * tg + (h & 1);
    const int lim = e ? T::EW : T::CW;
    dmap[q] = (int16_t)(A < lim && B < lim ? rec_of(e, A, B) : -1);
  }
  for (int q = threadIdx.x; q < NIT * 32; q += blockDim.x) {   // commit items, as in k_accum_points_tc
    const int it = q;
    uint32_t d = ~0u;
    if (it < 13 * P) {
      const int pr = it / 13, qq = it - 13 * pr;
      d = (qq < 9 ? 0u : 1u) | ((uint32_t)pr << 2) | ((uint32_t)(qq < 9 ? 4 * qq : 4 * (qq - 9)) << 10) |
          ((uint32_t)(4 * it) << 18);
    } else if (it < 13 * P + 6 * K) {
      const int t2 = it - 13 * P, sl = t2 / 6, qq = t2 - 6 * sl;
      d = qq < 3 ? (2u | ((uint32_t)sl << 2) | ((uint32_t)(2 * qq) << 10) | ((uint32_t)(52 * P + 20 * sl + 2 * qq) << 18))
                 : (3u | ((uint32_t)sl << 2) | ((uint32_t)(4 * (qq - 3)) << 10) |
                    ((uint32_t)(52 * P + 20 * sl + 8 + 4 * (qq - 3)) << 18));
    }
    cdesc[q / 32][q % 32] = d;
  }
  for (int q = lane; q < RT; q += 32) Rec[q] = 0.f;
  __syncthreads();

  pdl_wait();   // K3a's factor state
  int64_t c = 0;
  if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
  c = __shfl_sync(0xffffffffu, c, 0);
  const float4* ps = a.pstate;
  const int64_t SS = a.pstride;
  for (; c < a.nchunk;) {
    const int4 ch = a.chunks[c];
    const int seg = ch.x;
    const int32_t* nodes = a.seg_nodes + (int64_t)seg * K;
    __syncwarp();
    for (int q = lane; q < P + K; q += 32) slots[q] = q < P ? a.seg_slot[(int64_t)seg * P + q] : nodes[q - P];
    float acc[T::NT][4];
#pragma unroll
    for (int t = 0; t < T::NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
    for (int base = ch.y; base < ch.z; base += 32) {
      const int64_t i = base + lane;
      PState<K> st;
      if (i < ch.z) {
#pragma unroll
        for (int s = 0; s < K; ++s) st.wa[s] = ps[s * SS + i];
        st.rr = ps[K * SS + i];
        st.nn = ps[(K + 1) * SS + i];
      } else {
#pragma unroll
        for (int s = 0; s < K; ++s) st.wa[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        st.rr = st.nn = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      build_row_w<K>(st, F + lane * S);
      __syncwarp();
      const int np = min(32, ch.z - base);
      for (int k0 = 0; k0 < np; k0 += 8) {
        {
          FragW<T::CQ, T::CNT> f;
          load_frag_w<T::CQ, T::CNT, S>(F, k0, 0, g, tig, f);   // c'
#pragma unroll
          for (int mi = 0; mi < T::CMT; ++mi)
#pragma unroll
            for (int ni = 2 * mi; ni < T::CNT; ++ni) mma3w(acc[T::cidx(mi, ni)], f, mi, ni);
        }
        {
          FragW<T::EQ, T::ENT> f;
          load_frag_w<T::EQ, T::ENT, S>(F, k0, T::CW, g, tig, f);   // e'
#pragma unroll
          for (int mi = 0; mi < T::EMT; ++mi)
#pragma unroll
            for (int ni = 2 * mi; ni < T::ENT; ++ni) mma3w(acc[T::eidx(mi, ni)], f, mi, ni);
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < T::NT; ++t)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int d = dmap[(4 * t + h) * 32 + lane];
        if (d >= 0) Rec[d] = acc[t][h];
      }
    __syncwarp();
    int64_t next_chunk = 0;
    if (lane == 0) next_chunk = (int64_t)atomicAdd(a.work_counter, 1ull);
#pragma unroll 1
    for (int k = 0; k < NIT; ++k) {
      const uint32_t d = cdesc[k][lane];
      if (d == ~0u) continue;
      const uint32_t kind = d & 3u, idx = (d >> 2) & 255u, off = (d >> 10) & 255u;
      const float* src = Rec + (d >> 18);
      if (kind == 2u) {
        const float2 v = *reinterpret_cast<const float2*>(src);
        if (v.x != 0.f || v.y != 0.f)
          atomicAdd(reinterpret_cast<float2*>(a.acc.rhs_data + 6 * (int64_t)slots[P + idx] + off), v);
      } else {
        const float4 v = *reinterpret_cast<const float4*>(src);
        if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
        float* dst = kind == 0u ? a.acc.data + 36 * (int64_t)slots[idx]
                   : kind == 1u ? a.acc.mom + 16 * (int64_t)slots[idx] : a.acc.node_mom + 12 * (int64_t)slots[P + idx];
        atomicAdd(reinterpret_cast<float4*>(dst + off), v);
      }
    }
    __syncwarp();
    c = __shfl_sync(0xffffffffu, next_chunk, 0);
  }
  pdl_trigger();
}
__host__ inline size_t tcw_smem(int K) {
  const int P = K * (K + 1) / 2, RT = 52 * P + 20 * K;
  const int CMT = (6 * K + 15) / 16, CNT = (6 * K) / 8 + 1, EMT = (4 * K + 15) / 16, ENT = (4 * K + 2) / 8 + 1;
  const int NT = CMT * CNT - CMT * (CMT - 1) + EMT * ENT - EMT * (EMT - 1);
  return sizeof(float) * kWarps * (32 * 104 + RT) + sizeof(int16_t) * 4 * NT * 32;
}

// Finalisation of the normal equations from the accumulators (so the
// latency-bound solver only streams its rows): warps [0, m) the diagonal blocks
// -- first, so their block-Jacobi inverses (K7) overlap the rest --, then one
// warp per kFB off-diagonal upper entries, then one per kFB nodes, then one for the
// energies (report slot).  Every accumulator is re-zeroed after it is read, so
// the next assembly needs no memset:
//   H(j,l) = w_data sum c c^T + w_pt PT(moments) + graph  (and its mirror H(l,j)),
//   b_j = -(w_data sum c r_pl + w_pt sum w_j [a_j x r'; r']) + graph rhs.
#ifndef MIS_KFB
#define MIS_KFB 4
#endif
constexpr int kFB = MIS_KFB;   // off-diagonal entries / nodes per warp (their loads overlap)

// Entry l = 6 i + j of a block as a branch-free recipe over the staged D | Mo | G:
//   h = w_data D[d] + G[l] + w_pt sum_k coef_k Mo[idx_k]
// (the same terms as block_entry: tr(S) I - S^T, [s_j]x, -[s_l]x, s0 I), built once per lane.
struct Recipe {
  int d, tr;          // D index (upper triangle on the diagonal), mirror position 6 j + i
  uint32_t idx;       // four Mo indices, one per byte
  float4 coef;        // their coefficients (0, +-1)
};
__device__ inline Recipe make_recipe(int l, bool diag) {
  const int i = l / 6, j = l - 6 * (l / 6);
  Recipe rc;
  rc.d = diag ? 6 * min(i, j) + max(i, j) : l;
  rc.tr = 6 * j + i;
  int id[4] = {0, 0, 0, 0};
  float cf[4] = {0.f, 0.f, 0.f, 0.f};
  if (i < 3 && j < 3) {   // tr(S) I - S^T
    if (i == j) { id[0] = 0; id[1] = 5; id[2] = 10; cf[0] = cf[1] = cf[2] = 1.f; }
    id[3] = diag ? 4 * min(i, j) + max(i, j) : 4 * j + i;
    cf[3] = -1.f;
  } else if (i < 3) {     // [s_j]x (i, j-3), s_j = Mo[p][3]
    const int c = j - 3;
    if (i != c) {
      if (c == (i + 1) % 3) { id[0] = 4 * ((i + 2) % 3) + 3; cf[0] = -1.f; }
      else { id[0] = 4 * ((i + 1) % 3) + 3; cf[0] = 1.f; }
    }
  } else if (j < 3) {     // -[s_l]x (i-3, j), s_l = Mo[3][q] (= Mo[q][3] on the diagonal)
    const int rr = i - 3, q1 = (rr + 2) % 3, q2 = (rr + 1) % 3;
    if (rr != j) {
      if (j == (rr + 1) % 3) { id[0] = diag ? 4 * q1 + 3 : 12 + q1; cf[0] = 1.f; }
      else { id[0] = diag ? 4 * q2 + 3 : 12 + q2; cf[0] = -1.f; }
    }
  } else if (i == j) {
    id[0] = 15;
    cf[0] = 1.f;
  }
  rc.idx = (uint32_t)id[0] | ((uint32_t)id[1] << 8) | ((uint32_t)id[2] << 16) | ((uint32_t)id[3] << 24);
  rc.coef = make_float4(cf[0], cf[1], cf[2], cf[3]);
  return rc;
}
__device__ __forceinline__ float apply_recipe(const Recipe& rc, const float* st, int l, float w_data, float w_pt) {
  const float* Mo = st + 36;
  const float pt = rc.coef.x * Mo[rc.idx & 0xff] + rc.coef.y * Mo[(rc.idx >> 8) & 0xff] +
                   rc.coef.z * Mo[(rc.idx >> 16) & 0xff] + rc.coef.w * Mo[rc.idx >> 24];
  return fmaf(w_data, st[rc.d], st[52 + l]) + w_pt * pt;
}

// one 6x6 block from its staged D | Mo | G (88 floats): H entries (and the mirror's);
// lane owns entries lane and lane + 32 (< 36) with their recipes rc[0], rc[1]
__device__ __forceinline__ void final_block(const FinalArgs& r, const float* st, float* hst, int64_t e, int lo, int lane,
                                            const Recipe (&rc)[2]) {
  const bool diag = lo < 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int l = lane + 32 * k;
    if (l < 36) {
      const float h = r.pre_weighted ? apply_recipe(rc[k], st, l, 1.f, 0.f) : apply_recipe(rc[k], st, l, r.w_data, r.w_pt);
      r.Hval[36 * e + l] = h;
      if (!diag) r.Hval[36 * (int64_t)lo + rc[k].tr] = h;
      if (hst) hst[l] = h;
    }
  }
}

__global__ void __launch_bounds__(256, 3) k_finalize(FinalArgs r) {   // 3 CTAs / SM: C5 1.23 -> 0.97 ms per step
  __shared__ float stage[8][kFB][124];
  __shared__ Recipe rtab[2][36];   // [diagonal?][entry], built before the dependency wait
  if (threadIdx.x < 72) rtab[threadIdx.x / 36][threadIdx.x % 36] = make_recipe(threadIdx.x % 36, threadIdx.x < 36);
  __syncthreads();
  pdl_wait();      // K3a/K3b/K4 accumulators
  if (r.lm && r.lm->acc_buf == 0) {   // LM: keep the accepted system, write the trial's into the other buffer
    r.Hval = r.Hval_alt;
    r.rhs = r.rhs_alt;
  }
  pdl_trigger();   // the solver may launch (it waits for this grid's completion before reading)
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n_off = (r.nup + kFB - 1) / kFB, n_nod = (r.m + kFB - 1) / kFB;
  if (gw < r.m) {   // diagonal block of node gw, then its block-Jacobi inverse
    float* st = stage[wib][0];
    const int64_t e = r.diag_pos[gw];
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
    if (gw == r.pose_node) {   // NEXT-2: + w_r J_r^T J_r + w_p J_p^T J_p of Eq. 10 (A38-A39), into G
      double pr[6], pJ[36];
      pose_prior_dev(r.pose_prior, r.pose_cur, pr, pJ);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int l = lane + 32 * k, i = l / 6, j = l - 6 * (l / 6);
        if (l < 36) {
          double h = 0.0;
          for (int q = 0; q < 6; ++q) h += (q < 3 ? (double)r.w_r : (double)r.w_p) * pJ[6 * q + i] * pJ[6 * q + j];
          st[52 + l] += (float)h;
        }
      }
      __syncwarp();
    }
    const Recipe rc[2] = {rtab[0][lane], rtab[0][lane < 4 ? lane + 32 : 0]};
    final_block(r, st, st + 88, e, -1, lane, rc);
    if (r.Minv) {   // block-Jacobi inverse of this node (K7), off the solver's critical path:
      __syncwarp();   // fp64 Gauss-Jordan, lane rr < 6 holds row rr of [H + (lambda + mu) I | I]
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
  int64_t g2 = gw - r.m;
  if (g2 < n_off) {   // kFB off-diagonal upper entries from the per-frame work list, loads first
    int64_t e[kFB];
    int lo[kFB];
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      const int64_t idx = g2 * kFB + q;
      e[q] = -1;
      lo[q] = -1;
      if (idx < r.nup) {
        const int2 ul = r.ulist[idx];
        e[q] = ul.x;
        lo[q] = ul.y;
      }
    }
    float v[kFB][5];
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      if (e[q] < 0) continue;
      const int64_t E = e[q];
      v[q][0] = r.acc.data[36 * E + lane];
      v[q][1] = lane < 4 ? r.acc.data[36 * E + 32 + lane] : 0.f;
      v[q][2] = lane < 16 ? r.acc.mom[16 * E + lane] : 0.f;
      v[q][3] = r.acc.graph[36 * E + lane];
      v[q][4] = lane < 4 ? r.acc.graph[36 * E + 32 + lane] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      if (e[q] < 0) continue;
      const int64_t E = e[q];
      float* st = stage[wib][q];
      st[lane] = v[q][0];
      if (lane < 4) st[32 + lane] = v[q][1];
      if (lane < 16) st[36 + lane] = v[q][2];
      st[52 + lane] = v[q][3];
      if (lane < 4) st[84 + lane] = v[q][4];
      r.acc.data[36 * E + lane] = 0.f;
      if (lane < 4) r.acc.data[36 * E + 32 + lane] = 0.f;
      if (lane < 16) r.acc.mom[16 * E + lane] = 0.f;
      r.acc.graph[36 * E + lane] = 0.f;
      if (lane < 4) r.acc.graph[36 * E + 32 + lane] = 0.f;
    }
    __syncwarp();
    const Recipe rc[2] = {rtab[1][lane], rtab[1][lane < 4 ? lane + 32 : 0]};
#pragma unroll
    for (int q = 0; q < kFB; ++q)
      if (e[q] >= 0) final_block(r, stage[wib][q], nullptr, e[q], lo[q], lane, rc);
    return;
  }
  g2 -= n_off;
  if (g2 < n_nod) {   // kFB nodes: b = -(w_data sum c r_pl + w_pt sum w_j [a_j x r'; r']) + graph rhs
    float v[kFB], gv[kFB];
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      const int64_t n = g2 * kFB + q;
      v[q] = 0.f;
      gv[q] = 0.f;
      if (n >= r.m) continue;
      if (lane < 6) { v[q] = r.acc.rhs_data[6 * n + lane]; gv[q] = r.acc.rhs_graph[6 * n + lane]; }
      else if (lane < 18) v[q] = r.acc.node_mom[12 * n + lane - 6];
    }
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      const int64_t n = g2 * kFB + q;
      if (n >= r.m) continue;
      float* st = stage[wib][q];
      if (lane < 18) st[lane] = v[q];
      if (lane < 6) { r.acc.rhs_data[6 * n + lane] = 0.f; r.acc.rhs_graph[6 * n + lane] = 0.f; }
      else if (lane < 18) r.acc.node_mom[12 * n + lane - 6] = 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kFB; ++q) {
      const int64_t n = g2 * kFB + q;
      if (n >= r.m || lane >= 6) continue;
      const float* st = stage[wib][q];
      const float* Nm = st + 6;
      float pt;
      if (lane < 3) {
        const int c1 = (lane + 1) % 3, c2 = (lane + 2) % 3;
        pt = Nm[3 * c1 + c2] - Nm[3 * c2 + c1];
      } else {
        pt = Nm[9 + (lane - 3)];
      }
      float prior = 0.f;
      if (n == r.pose_node) {   // NEXT-2: -(w_r J_r^T r_r + w_p J_p^T r_p)
        double pr[6], pJ[36], b = 0.0;
        pose_prior_dev(r.pose_prior, r.pose_cur, pr, pJ);
        for (int k = 0; k < 6; ++k) b += (k < 3 ? (double)r.w_r : (double)r.w_p) * pJ[6 * k + lane] * pr[k];
        prior = (float)(-b);
      }
      r.rhs[6 * n + lane] = (r.pre_weighted ? -st[lane] : -r.w_data * st[lane] - r.w_pt * pt) + gv[q] + prior;
    }
    return;
  }
  if (g2 == n_nod) {   // energies -> report slot; zeroed (with K3's work counter) for the next assembly
    double* E = r.acc.energy;
    double tot[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {   // striped partials: lane l sums stripes l, l + 32
      double* st_q = E + 8 + kEnergyStripes * q;
      double vv = st_q[lane] + st_q[lane + 32];
      st_q[lane] = 0.0;
      st_q[lane + 32] = 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) vv += __shfl_xor_sync(0xffffffffu, vv, o);
      tot[q] = E[q] + vv;
    }
    if (lane == 0) {
      if (r.slot >= 0) {
        double* rep = r.rep_energy + 5 * r.slot;
        double Er = 0.0, Ep = 0.0;
        if (r.pose_node >= 0) {   // NEXT-2: E_r, E_p (Eq. 10) at the assembled pose
          double pr[6], pJ[36];
          pose_prior_dev(r.pose_prior, r.pose_cur, pr, pJ);
          Er = pr[0] * pr[0] + pr[1] * pr[1] + pr[2] * pr[2];
          Ep = pr[3] * pr[3] + pr[4] * pr[4] + pr[5] * pr[5];
          if (r.rep_pose) { r.rep_pose[2 * r.slot] = Er; r.rep_pose[2 * r.slot + 1] = Ep; }
        }
        rep[0] = tot[0]; rep[1] = tot[1]; rep[2] = tot[2]; rep[3] = tot[3];
        rep[4] = (double)r.w_data * tot[0] + (double)r.w_pt * tot[1] + (double)r.w_reg * tot[2] +
                 (double)r.w_corr * tot[3] + (double)r.w_r * Er + (double)r.w_p * Ep;
        r.rep_nassoc[r.slot] = tot[4];
        r.rep_nassoc[MIS_MAX_GN + 1 + r.slot] = 0.0;   // (no fp32 guard band: the association runs in fp64)
      }
      for (int q = 0; q < 8; ++q) E[q] = 0.0;
    }
  }
}

void launch_finalize(const FinalArgs& r, cudaStream_t s) {
  const int64_t warps = (int64_t)r.m + (r.nup + kFB - 1) / kFB + (r.m + kFB - 1) / kFB + 1;
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > 0) launch_pdl(k_finalize, dim3((unsigned)blocks), dim3(256), 0, s, r);
}

// ---- multi-GPU reduction payload: before the cross-rank sum, each rank turns its point
// accumulators (data | mom per upper block, rhs_data | node_mom per node) into the point part of the
// final system -- the 6x6 upper blocks (36 floats) and the 6-vector b per node -- so the all-reduce moves
// 36 (m + nup) + 6 m floats (C5: ~39 MB per GN iteration) instead of the raw accumulators (52 floats per
// BSR entry, both triangles).  H is linear in the accumulators, so this commutes with the sum.  After the
// reduce k_shard_scatter puts the point part back as "data" (mom = 0, rhs_data = -b) and the regular
// finalisation runs with w_data = 1, w_pt = 0, adding each rank's own (identical) graph terms.
// HU: [m diagonal blocks | nup off-diagonal upper blocks in the finalisation's list order] x 36, RU: 6 m.
__global__ void __launch_bounds__(256) k_shard_partial(FinalArgs r, float* HU, float* RU) {
  __shared__ float stage[8][52];
  __shared__ Recipe rtab[2][36];
  if (threadIdx.x < 72) rtab[threadIdx.x / 36][threadIdx.x % 36] = make_recipe(threadIdx.x % 36, threadIdx.x < 36);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nblk = r.m + r.nup;
  float* st = stage[wib];
  if (gw < nblk) {
    const bool diag = gw < r.m;
    const int64_t e = diag ? (int64_t)r.diag_pos[gw] : (int64_t)r.ulist[gw - r.m].x;
    st[lane] = r.acc.data[36 * e + lane];
    if (lane < 4) st[32 + lane] = r.acc.data[36 * e + 32 + lane];
    if (lane < 16) st[36 + lane] = r.acc.mom[16 * e + lane];
    __syncwarp();
    float g0[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {   // the recipes read G at st[52 + l]: evaluate with G = 0 by hand
      const int l = lane + 32 * k;
      g0[k] = 0.f;
      if (l < 36) {
        const Recipe rc = rtab[diag ? 0 : 1][l];
        const float* Mo = st + 36;
        const float pt = rc.coef.x * Mo[rc.idx & 0xff] + rc.coef.y * Mo[(rc.idx >> 8) & 0xff] +
                         rc.coef.z * Mo[(rc.idx >> 16) & 0xff] + rc.coef.w * Mo[rc.idx >> 24];
        g0[k] = r.w_data * st[rc.d] + r.w_pt * pt;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int l = lane + 32 * k;
      if (l < 36) HU[36 * gw + l] = g0[k];
    }
    r.acc.data[36 * e + lane] = 0.f;
    if (lane < 4) r.acc.data[36 * e + 32 + lane] = 0.f;
    if (lane < 16) r.acc.mom[16 * e + lane] = 0.f;
    return;
  }
  const int64_t n = gw - nblk;
  if (n < r.m && lane < 6) {   // b's point part of node n (as k_finalize, without the graph rhs)
    const float* Nm = r.acc.node_mom + 12 * n;
    float pt;
    if (lane < 3) {
      const int c1 = (lane + 1) % 3, c2 = (lane + 2) % 3;
      pt = Nm[3 * c1 + c2] - Nm[3 * c2 + c1];
    } else {
      pt = Nm[9 + (lane - 3)];
    }
    RU[6 * n + lane] = -r.w_data * r.acc.rhs_data[6 * n + lane] - r.w_pt * pt;
    __syncwarp(0x3fu);
    r.acc.rhs_data[6 * n + lane] = 0.f;
    r.acc.node_mom[12 * n + lane] = 0.f;
    r.acc.node_mom[12 * n + 6 + lane] = 0.f;
  }
}

__global__ void __launch_bounds__(256) k_shard_scatter(FinalArgs r, const float* HU, const float* RU) {
  pdl_wait();
  pdl_trigger();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nblk = r.m + r.nup;
  if (gw < nblk) {
    const int64_t e = gw < r.m ? (int64_t)r.diag_pos[gw] : (int64_t)r.ulist[gw - r.m].x;
    r.acc.data[36 * e + lane] = HU[36 * gw + lane];   // mom stays zero (zeroed by k_shard_partial)
    if (lane < 4) r.acc.data[36 * e + 32 + lane] = HU[36 * gw + 32 + lane];
    return;
  }
  const int64_t n = gw - nblk;
  if (n < r.m && lane < 6) r.acc.rhs_data[6 * n + lane] = -RU[6 * n + lane];
}

void launch_shard_partial(const FinalArgs& r, float* HU, float* RU, cudaStream_t s) {
  const int64_t warps = (int64_t)r.m + r.nup + r.m;
  launch_pdl(k_shard_partial, dim3((unsigned)((warps * 32 + 255) / 256)), dim3(256), 0, s, r, HU, RU);
}
void launch_shard_scatter(const FinalArgs& r, const float* HU, const float* RU, cudaStream_t s) {
  const int64_t warps = (int64_t)r.m + r.nup + r.m;
  launch_pdl(k_shard_scatter, dim3((unsigned)((warps * 32 + 255) / 256)), dim3(256), 0, s, r, HU, RU);
}

// K3a by chunk (k > 4 with the tcgen05 K3b; MIS_K3A_CHUNKED=0 selects the per-point K3a): one warp per
// chunk (dynamic schedule), the chunk's k fp64 node states staged in shared memory once (as the fused
// k <= 4 kernel), so a point reads neither its k node ids nor 6k node-state vectors from memory; the
// sparse state out.  C5: 8.8 -> 6.6 ms per step.
template <int K, bool JOINT = false>
__global__ void __launch_bounds__(256, MIS_K3A_MINB) k_assoc_chunks(AsmPointsArgs a, AsmGraphArgs ga,
                                                                   unsigned point_grid) {
  constexpr int KS = K + (JOINT ? 1 : 0);   // NEXT-2: the pose as the last factor slot (not staged)
  if (blockIdx.x >= point_grid) {
    pdl_wait();
    pdl_trigger();
    graph_item(ga, (int64_t)(blockIdx.x - point_grid) * blockDim.x + threadIdx.x);
    return;
  }
  __shared__ double2 nrt_sm[kWarps][6 * K];
  __shared__ float4 ng_sm[kWarps][K];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  double ed = 0.0, ep = 0.0;
  int n_as = 0;
  float4* ps = a.pstate;
  const int64_t S = a.pstride;
  int64_t c = 0;
  if (lane == 0) c = (int64_t)atomicAdd(a.work_counter, 1ull);
  c = __shfl_sync(0xffffffffu, c, 0);
  while (c < a.nchunk) {
    const int4 ch = a.chunks[c];
    const int32_t* nodes = a.seg_nodes + (int64_t)ch.x * KS;
    __syncwarp();
    for (int q = lane; q < 7 * K; q += 32) {
      if (q < 6 * K) {
        nrt_sm[warp][q] = __ldg(reinterpret_cast<const double2*>(a.nd.Rt64 + 12 * (int64_t)nodes[q / 6]) + q % 6);
      } else {
        const float* g = a.nd.g + 3 * (int64_t)nodes[q - 6 * K];
        ng_sm[warp][q - 6 * K] = make_float4(g[0], g[1], g[2], 0.f);
      }
    }
    int64_t nc = 0;
    if (lane == 0) nc = (int64_t)atomicAdd(a.work_counter, 1ull);   // the next chunk id in flight
    __syncwarp();
    const NodesChunk nch{nrt_sm[warp], reinterpret_cast<const float*>(ng_sm[warp])};
    int anylive = 0;
    for (int base = ch.y; base < ch.z; base += 32) {
      const int64_t i = base + lane;
      if (i < ch.z) {
        PState<KS> st;
        int as1 = 0;
        assoc_point<K, false, JOINT, false, NodesChunk>(a, i, st, ed, ep, as1, nch);
        n_as += as1;
        if (as1) {
#pragma unroll
          for (int q = 0; q < KS; ++q) ps[q * S + i] = st.wa[q];
          ps[KS * S + i] = st.rr;
        }
        ps[(KS + 1) * S + i] = make_float4(st.nn.x, st.nn.y, st.nn.z, as1 ? 1.f : 0.f);
        anylive |= as1;
      }
    }
    anylive = __any_sync(0xffffffffu, anylive);
    if (lane == 0) a.chunk_live[c] = anylive;
    c = __shfl_sync(0xffffffffu, nc, 0);
  }
  commit_point_energies(a, ed, ep, n_as);
}

template <int K>
static void launch_assoc_k(const AsmPointsArgs& a, const AsmGraphArgs* ga, cudaStream_t s) {
  const int64_t n = a.md.n;
  const unsigned g = (unsigned)((n + 255) / 256);
  AsmGraphArgs gz{};
  int64_t ng = 0;
  if (ga) {
    gz = *ga;
    const int PS = gz.KS * (gz.KS + 1) / 2;
    ng = (int64_t)gz.nd.m * gz.n_nbr * 6 + (int64_t)gz.nf * PS * 6 + (int64_t)gz.nf * gz.KS;
  }
  const unsigned gg = (unsigned)((ng + 255) / 256);
  if (g + gg == 0) return;
  const bool joint = a.pose_cur != nullptr;
  if constexpr (K <= 4) {
    if (a.affine) {   // NEXT-4: the graph terms run in their own kernel (affine.cu)
      if (g == 0) return;
      if (a.dbg_pix != nullptr) launch_pdl(k_assoc_points<K, true, false, true>, dim3(g), dim3(256), 0, s, a, gz, g);
      else launch_pdl(k_assoc_points<K, false, false, true>, dim3(g), dim3(256), 0, s, a, gz, g);
      return;
    }
  }
  // k > 4 (or the joint pose's k + 1 > 4 slots) with the tcgen05 K3b: K3a by chunk (api.cu decides)
  if (a.chunk_live != nullptr) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned pg = (unsigned)std::min<int64_t>((a.nchunk + kWarps - 1) / kWarps, 2 * (int64_t)sms);
    if (joint) {
      if constexpr (K < MIS_MAX_K) launch_pdl(k_assoc_chunks<K, true>, dim3(pg + gg), dim3(256), 0, s, a, gz, pg);
    } else {
      if constexpr (K > 4) launch_pdl(k_assoc_chunks<K, false>, dim3(pg + gg), dim3(256), 0, s, a, gz, pg);
    }
    return;
  }
  if constexpr (K < MIS_MAX_K) {
    if (joint) {
      if (a.sparse_state) {   // the joint slots K + 1 >= 5 run through the tcgen05 K3b
        if (a.dbg_pix != nullptr) launch_pdl(k_assoc_points<K, true, true, false, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
        else launch_pdl(k_assoc_points<K, false, true, false, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
        return;
      }
      if (a.dbg_pix != nullptr) launch_pdl(k_assoc_points<K, true, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
      else launch_pdl(k_assoc_points<K, false, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
      return;
    }
  }
  if constexpr (K > 4) {
    if (a.sparse_state) {
      if (a.dbg_pix != nullptr) launch_pdl(k_assoc_points<K, true, false, false, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
      else launch_pdl(k_assoc_points<K, false, false, false, true>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
      return;
    }
  }
  if (a.dbg_pix != nullptr) launch_pdl(k_assoc_points<K, true, false>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
  else launch_pdl(k_assoc_points<K, false, false>, dim3(g + gg), dim3(256), 0, s, a, gz, g);
}

#ifndef MIS_K3B_TC
#define MIS_K3B_TC 1   // 0: the FP32 FMA path for every k
#endif
template <int K>
static void launch_accum_k(const AsmPointsArgs& a, int num_sms, cudaStream_t s, bool fused, const AsmGraphArgs* ga) {
  using L = Lay<K>;
  constexpr bool tc = MIS_K3B_TC && K <= 4;   // tensor-core SYRK: k <= 4 (8 warps x 2 CTAs / SM),
  // 5 <= k <= 8 on tensor cores (one 8-warp CTA / SM at 167 registers) measured slower than the FP32
  // tiles at 16 warps / SM (C5: 2.9 vs 2.5 ms per launch, latency-bound), so it is opt-in
  constexpr bool tcw = MIS_K3B_TCW && K > 4;
  const size_t smem = tc    ? sizeof(float) * kWarps * (32 * kTcFSP + tc_rec_floats(K <= 4 ? K : 4))
                      : tcw ? tcw_smem(K)
                            : sizeof(float) * kWarps * 32 * L::FSP;
  if constexpr (tc) {   // K3b, or K3a + K3b fused (with the K4 / K5 items in extra CTAs)
    auto kern = fused ? k_accum_points_tc<(K <= 4 ? K : 4), true> : k_accum_points_tc<(K <= 4 ? K : 4), false>;
    static bool attr_set[2] = {false, false};
    if (!attr_set[fused]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set[fused] = true;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t want = (a.nchunk + kWarps - 1) / kWarps;
    int64_t grid = (int64_t)num_sms * per_sm;
    if (want < grid) grid = want;
    if (grid < 1) grid = 1;
    AsmGraphArgs gz{};
    int64_t gg = 0;
    if (fused && ga) {
      gz = *ga;
      const int PS = gz.KS * (gz.KS + 1) / 2;
      const int64_t ng = (int64_t)gz.nd.m * gz.n_nbr * 6 + (int64_t)gz.nf * PS * 6 + (int64_t)gz.nf * gz.KS;
      gg = (ng + kWarps * 32 - 1) / (kWarps * 32);
    }
    if (a.nchunk <= 0) grid = 0;
    if (grid + gg == 0) return;
    launch_pdl(kern, dim3((unsigned)(grid + gg)), dim3(kWarps * 32), smem, s, a, gz, (unsigned)grid);
    return;
  }
  if constexpr (tcw) {
    if (a.nchunk <= 0) return;
    void (*kern)(AsmPointsArgs) = k_accum_points_tcw<(K > 4 ? K : 5)>;
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set = true;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t want = (a.nchunk + kWarps - 1) / kWarps;
    int64_t grid = (int64_t)num_sms * per_sm;
    if (want < grid) grid = want;
    if (grid < 1) grid = 1;
    launch_pdl(kern, dim3((unsigned)grid), dim3(kWarps * 32), smem, s, a);
    return;
  }
  // FP32 register-tile SYRK (k > 4), K3a fused into it when `fused`
  auto kern = fused ? k_accum_points<K, true> : k_accum_points<K, false>;
  static bool attr_set2[2] = {false, false};
  if (!attr_set2[fused]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set2[fused] = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = (a.nchunk + kWarps - 1) / kWarps;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (want < grid) grid = want;
  if (a.nchunk <= 0) grid = 0;
  AsmGraphArgs gz{};
  int64_t gg = 0;
  if (fused && ga) {
    gz = *ga;
    const int PS = gz.KS * (gz.KS + 1) / 2;
    const int64_t ng = (int64_t)gz.nd.m * gz.n_nbr * 6 + (int64_t)gz.nf * PS * 6 + (int64_t)gz.nf * gz.KS;
    gg = (ng + kWarps * 32 - 1) / (kWarps * 32);
  }
  if (grid + gg == 0) return;
  launch_pdl(kern, dim3((unsigned)(grid + gg)), dim3(kWarps * 32), smem, s, a, gz, (unsigned)grid);
}

void launch_assoc_points(int K, const AsmPointsArgs& a, const AsmGraphArgs* ga, cudaStream_t s) {
  switch (K) {
#define LP(KK) case KK: launch_assoc_k<KK>(a, ga, s); break;
    LP(1) LP(2) LP(3) LP(4) LP(5) LP(6) LP(7) LP(8)
#undef LP
    default: break;
  }
}

void launch_accum_points(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s, bool fused,
                         const AsmGraphArgs* ga) {
  switch (K) {
#define LP(KK) case KK: launch_accum_k<KK>(a, num_sms, s, fused, ga); break;
    LP(1) LP(2) LP(3) LP(4) LP(5) LP(6) LP(7) LP(8)
#undef LP
    default: break;
  }
}

// ---------------------------------------------------------------- K4 / K5
// One thread per (edge, block row), (feature, node pair, block row) and
// (feature, node): ~50k independent items at C3 instead of 4.5k serial
// atomic chains (the regulariser and feature blocks are few: latency-bound).
__device__ __forceinline__ void feature_warp(const AsmGraphArgs& a, int fi, float (*am)[3], float* wn, double* e,
                                             float* rp, bool* ok) {
  // the residual in fp64 from the fp64 master node state (the feature term is O(n_f k): free), so
  // E_corr carries no fp32 cancellation of ~50 mm positions; the Jacobian rows are fp32
  const int K = a.K;
  const double V[3] = {a.fsrc[3 * fi], a.fsrc[3 * fi + 1], a.fsrc[3 * fi + 2]};
  double W = 0.0;
  for (int s = 0; s < K; ++s) W += a.fw[(int64_t)s * a.nf + fi];
  *ok = W > 0.0;
  if (!*ok) return;
  double xh[3] = {0, 0, 0};
  for (int s = 0; s < K; ++s) {
    const int j = a.fidx[(int64_t)s * a.nf + fi];
    const double* Rt = a.nd.Rt64 + 12 * j;
    const float* g = a.nd.g + 3 * j;
    const double w = a.fw[(int64_t)s * a.nf + fi] / W;
    wn[s] = (float)w;
    const double d[3] = {V[0] - g[0], V[1] - g[1], V[2] - g[2]};
    for (int r = 0; r < 3; ++r) {
      const double ar = Rt[3 * r] * d[0] + Rt[3 * r + 1] * d[1] + Rt[3 * r + 2] * d[2];
      am[s][r] = (float)ar;
      xh[r] += w * (ar + g[r] + Rt[9 + r]);
    }
  }
  const double* R = a.pose_cur ? a.pose_cur : a.fr.Rd;
  const double* T = a.pose_cur ? a.pose_cur + 9 : a.fr.Td;
  if (a.KS > K) {   // NEXT-2: the pose as slot K, a = x_hat, weight 1 (A37)
    for (int r = 0; r < 3; ++r) am[K][r] = (float)xh[r];
    wn[K] = 1.f;
  }
  for (int r = 0; r < 3; ++r)
    e[r] = R[3 * r] * xh[0] + R[3 * r + 1] * xh[1] + R[3 * r + 2] * xh[2] + T[r] - a.fdst[3 * fi + r];
  for (int r = 0; r < 3; ++r) rp[r] = (float)(R[r] * e[0] + R[3 + r] * e[1] + R[6 + r] * e[2]);
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

__device__ __forceinline__ int64_t graph_items(const AsmGraphArgs& a) {
  const int P = a.KS * (a.KS + 1) / 2;
  return (int64_t)a.nd.m * a.n_nbr * 6 + (int64_t)a.nf * P * 6 + (int64_t)a.nf * a.KS;
}

// one K4/K5 item per thread (whole warps call this; tid >= graph_items: no work)
__device__ __forceinline__ void graph_item(const AsmGraphArgs& a, int64_t tid) {
  const int K = a.KS, P = K * (K + 1) / 2;   // feature slots (incl. the pose, NEXT-2)
  const int64_t n_edge = (int64_t)a.nd.m * a.n_nbr * 6, n_fp = (int64_t)a.nf * P * 6, n_fr = (int64_t)a.nf * K;
  double eR = 0.0, eC = 0.0;
  if (tid < n_edge) {
    // Eq. 6, alpha = 1, directed edge j -> l (reading A14):
    // J_j = [-[b]x, I], J_l = [0, -I], b = R_j (g_l - g_j)
    const int64_t ei = tid / 6;
    const int r = (int)(tid % 6);
    const int j = (int)(ei / a.n_nbr), l = a.nbr[ei];
    if (l >= 0) {
      // residual in fp64 from the master state: e = R_j d - d + t_j - t_l with d = g_l - g_j exact,
      // so a rigid-consistent field gives E_reg = 0 like the oracle (no fp32 cancellation of g)
      const double* Rj = a.nd.Rt64 + 12 * j;
      const double* Rl = a.nd.Rt64 + 12 * l;
      const float* gj = a.nd.g + 3 * j;
      const float* gl = a.nd.g + 3 * l;
      const double d[3] = {(double)gl[0] - gj[0], (double)gl[1] - gj[1], (double)gl[2] - gj[2]};
      double bd[3], ed[3];
      for (int q = 0; q < 3; ++q) bd[q] = Rj[3 * q] * d[0] + Rj[3 * q + 1] * d[1] + Rj[3 * q + 2] * d[2];
      for (int q = 0; q < 3; ++q) ed[q] = (bd[q] - d[q]) + (Rj[9 + q] - Rl[9 + q]);
      if (r == 0) eR = ed[0] * ed[0] + ed[1] * ed[1] + ed[2] * ed[2];
      float b[3], e[3], row[6];
      for (int q = 0; q < 3; ++q) { b[q] = (float)bd[q]; e[q] = (float)ed[q]; }
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
    float am[MIS_MAX_K][3], wn[MIS_MAX_K], rp[3];
    double e[3];
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
    energy_add(a.acc.energy, 2, eR);
    energy_add(a.acc.energy, 3, eC);
  }
}

__global__ void __launch_bounds__(256) k_assemble_graph(AsmGraphArgs a) {
  graph_item(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}

void launch_assemble_graph(const AsmGraphArgs& a, cudaStream_t s) {
  const int P = a.KS * (a.KS + 1) / 2;
  const int64_t n = (int64_t)a.nd.m * a.n_nbr * 6 + (int64_t)a.nf * P * 6 + (int64_t)a.nf * a.KS;
  if (n <= 0) return;
  k_assemble_graph<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
}


}  // namespace mis
