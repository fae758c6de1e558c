// affine.cu -- NEXT-4 (MIS_F_AFFINE): the assembly of the affine-node model (Eq. 1 with a
// general A_j, Eq. 4-5 E_rot, Eq. 6 with A_j; readings A41-A45) in 12-unknown node
// blocks [dA_j row-major, dt_j]:
//   K3b_aff  per chunk (points sharing their k nodes): two small SYRKs of the factor rows
//              c' = [w_s (n' (x) d_s) (9), w_s n' (3) ..., r_pl]     (Eq. 8 Jacobian row / R)
//              e' = [w_s d_s, w_s ..., r']                           (point-to-point moments)
//            d_s = v - g_s, n' = R^T N, r' = R^T (v~ - q), committed with float4 atomics;
//   K4/K5/E_rot  regulariser edges, ORB features and the Eq. 5 terms (one thread per item, fp64
//            residuals, fp32 atomics into the graph accumulators);
//   finalise 12 x 12 blocks (both triangles), b, fp64 block-Jacobi inverses, energies.
// The k-tuple grouping, the BSR pattern and the slot tables are the SE(3) path's (the pattern is
// a node-pair pattern, independent of the block size).
#include <cuda_runtime.h>

#include "solve_common.cuh"

namespace mis {

constexpr int kAW = 8;   // warps per CTA

template <int K>
struct LayA {
  static constexpr int CD = 12 * K + 1, CDP = (CD + 3) & ~3;
  static constexpr int CE = 4 * K + 3, CEP = (CE + 3) & ~3;
  static constexpr int FSP = CDP + CEP + 4;           // smem row stride (floats)
  static constexpr int ND = CDP / 4, NE = CEP / 4;
  static constexpr int TD = ND * (ND + 1) / 2, TE = NE * (NE + 1) / 2, NT = TD + TE;
  static constexpr int R = (NT + 31) / 32;            // tiles per lane
  static constexpr int P = K * (K + 1) / 2;
  static constexpr int RT = 160 * P + 24 * K;         // record: P x (144 data | 16 moments), K x (12 rhs | 12 moments)
};

// K3b for the affine model: one warp per chunk (dynamic scheduling), lanes own 4 x 4 tiles of the
// upper triangles of sum c'c'^T and sum e'e'^T
template <int K>
__global__ void __launch_bounds__(kAW * 32, 1) k_accum_points_aff(AsmPointsArgs a) {
  using L = LayA<K>;
  constexpr int P = L::P;
  static_assert(L::RT <= 32 * L::FSP, "record must fit the row buffer");
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* F = reinterpret_cast<float*>(smem4) + warp * (32 * L::FSP);
  float* Rec = F;   // aliases the row buffer at commit
  __shared__ int32_t slot_sm[kAW][P + K];
  int32_t* slots = slot_sm[warp];
  __shared__ uint8_t tabI[L::NT], tabJ[L::NT];
  __shared__ int16_t dm[L::R * 16][32];
  for (int t = threadIdx.x; t < L::NT; t += blockDim.x) {
    const bool e = t >= L::TD;
    const int nb = e ? L::NE : L::ND;
    int u = e ? t - L::TD : t, I = 0;
    while (u >= nb - I) { u -= nb - I; ++I; }
    tabI[t] = (uint8_t)I;
    tabJ[t] = (uint8_t)(I + u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < L::R * 16 * 32; q += blockDim.x) {
    const int ln = q & 31, rv = q >> 5, r = rv >> 4, v = rv & 15, t = ln + 32 * r;
    int d = -1;
    if (t < L::NT) {
      const bool isd = t < L::TD;
      const int A = 4 * tabI[t] + (v >> 2), B = 4 * tabJ[t] + (v & 3);
      if (A <= B) {
        if (isd) {        // c'
          if (B < 12 * K) d = 160 * pair_index(A / 12, B / 12, K) + 12 * (A % 12) + (B % 12);
          else if (B == 12 * K && A < 12 * K) d = 160 * P + 24 * (A / 12) + (A % 12);
        } else {          // e'
          if (B < 4 * K) d = 160 * pair_index(A / 4, B / 4, K) + 144 + 4 * (A % 4) + (B % 4);
          else if (B < 4 * K + 3 && A < 4 * K) {
            const int p = A % 4, qq = B - 4 * K;   // sum (w d)_p r'_q (p < 3) or sum w r'_q (p = 3)
            d = 160 * P + 24 * (A / 4) + 12 + (p < 3 ? 3 * p + qq : 9 + qq);
          }
        }
      }
    }
    dm[rv][ln] = (int16_t)d;
  }
  __syncthreads();
  int offA[L::R], offB[L::R];
  bool tV[L::R];
#pragma unroll
  for (int r = 0; r < L::R; ++r) {
    const int t = lane + 32 * r;
    tV[r] = t < L::NT;
    const int base = (tV[r] && t >= L::TD) ? L::CDP : 0;
    offA[r] = tV[r] ? base + 4 * tabI[t] : 0;
    offB[r] = tV[r] ? base + 4 * tabJ[t] : 0;
  }
  pdl_wait();
  pdl_trigger();
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
    float acc[L::R][16];
#pragma unroll
    for (int r = 0; r < L::R; ++r)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[r][e] = 0.f;
    for (int base = ch.y; base < ch.z; base += 32) {
      const int64_t i = base + lane;
      float* row = F + lane * L::FSP;
      if (i < ch.z) {   // factor row of the point (zeros when not associated)
        const float4 rr = ps[K * S + i], nn = ps[(K + 1) * S + i];
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const float4 wd = ps[s * S + i];   // (w d, w)
          const float n3[3] = {nn.x, nn.y, nn.z}, d3[3] = {wd.x, wd.y, wd.z};
#pragma unroll
          for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) row[12 * s + 3 * r3 + cc] = n3[r3] * d3[cc];
          row[12 * s + 9] = wd.w * nn.x;
          row[12 * s + 10] = wd.w * nn.y;
          row[12 * s + 11] = wd.w * nn.z;
          *reinterpret_cast<float4*>(row + L::CDP + 4 * s) = wd;
        }
        row[12 * K] = rr.w;
#pragma unroll
        for (int q = 12 * K + 1; q < L::CDP; ++q) row[q] = 0.f;
        row[L::CDP + 4 * K + 0] = rr.x;
        row[L::CDP + 4 * K + 1] = rr.y;
        row[L::CDP + 4 * K + 2] = rr.z;
#pragma unroll
        for (int q = L::CDP + 4 * K + 3; q < L::CDP + L::CEP; ++q) row[q] = 0.f;
      }
      __syncwarp();
      const int np = min(32, ch.z - base);
#pragma unroll
      for (int r = 0; r < L::R; ++r) {
        if (!tV[r]) continue;
        const float* pa = F + offA[r];
        const float* pb = F + offB[r];
#pragma unroll 4
        for (int p = 0; p < np; ++p) {
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
    // commit: tiles -> the warp's record (aliasing the row buffer), then float4 atomics
    for (int q = lane; q < L::RT / 4; q += 32) reinterpret_cast<float4*>(Rec)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < L::R; ++r) {
      if (!tV[r]) continue;
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const int d = dm[16 * r + v][lane];
        if (d >= 0) Rec[d] = acc[r][v];
      }
    }
    __syncwarp();
    int64_t next_chunk = 0;
    if (lane == 0) next_chunk = (int64_t)atomicAdd(a.work_counter, 1ull);
    for (int q = lane; q < L::RT / 4; q += 32) {
      const float4 v = reinterpret_cast<const float4*>(Rec)[q];
      if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
      const int f = 4 * q;
      float* dst;
      if (f < 160 * P) {
        const int pr = f / 160, o = f - 160 * pr;
        dst = o < 144 ? a.acc.data + 144 * (int64_t)slots[pr] + o : a.acc.mom + 16 * (int64_t)slots[pr] + (o - 144);
      } else {
        const int g = f - 160 * P, sl = g / 24, o = g - 24 * sl;
        dst = o < 12 ? a.acc.rhs_data + 12 * (int64_t)slots[P + sl] + o
                     : a.acc.node_mom + 12 * (int64_t)slots[P + sl] + (o - 12);
      }
      atomicAdd(reinterpret_cast<float4*>(dst), v);
    }
    __syncwarp();
    c = __shfl_sync(0xffffffffu, next_chunk, 0);
  }
}

template <int K>
static void launch_aff_k(const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  using L = LayA<K>;
  if (a.nchunk <= 0) return;
  const size_t smem = sizeof(float) * kAW * 32 * L::FSP;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_accum_points_aff<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_accum_points_aff<K>, kAW * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm, want = (a.nchunk + kAW - 1) / kAW;
  if (want < grid) grid = want;
  launch_pdl(k_accum_points_aff<K>, dim3((unsigned)grid), dim3(kAW * 32), smem, s, a);
}

void launch_accum_points_aff(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  switch (K) {
    case 1: launch_aff_k<1>(a, num_sms, s); break;
    case 2: launch_aff_k<2>(a, num_sms, s); break;
    case 3: launch_aff_k<3>(a, num_sms, s); break;
    case 4: launch_aff_k<4>(a, num_sms, s); break;
    default: break;
  }
}

// ---------------------------------------------------------------- K4 / K5 / E_rot
// 12 x 12 block entry (i, j) += v at the upper entry `e` of (a, b): when a > b the entry is
// stored transposed
__device__ __forceinline__ void add_e(float* G, int64_t e, bool transposed, int i, int j, float v) {
  if (v == 0.f) return;
  atomicAdd(G + 144 * e + (transposed ? 12 * j + i : 12 * i + j), v);
}

// entry (i, j) of J_s^T J_s' for two point-like 3 x 12 Jacobians J = w R [(d_c e_r) columns, I]
// (R^T R = I):  (r,c),(r',c') -> w w' delta_rr' d_c d'_c';  (r,c), 9+r' -> w w' delta_rr' d_c;
//               9+r, (r',c') -> w w' delta_rr' d'_c';     9+r, 9+r' -> w w' delta_rr'
__device__ __forceinline__ float pt_entry(const double* d, const double* d2, double ww, int i, int j) {
  const int ri = i < 9 ? i / 3 : i - 9, rj = j < 9 ? j / 3 : j - 9;
  if (ri != rj) return 0.f;
  const double fi = i < 9 ? d[i % 3] : 1.0, fj = j < 9 ? d2[j % 3] : 1.0;
  return (float)(ww * fi * fj);
}

__global__ void __launch_bounds__(256) k_assemble_graph_aff(AsmGraphArgs a) {
  pdl_wait();
  pdl_trigger();
  const int m = a.nd.m, K = a.K;
  const int64_t n_edge = (int64_t)m * a.n_nbr, P = K * (K + 1) / 2, n_fp = (int64_t)a.nf * P;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double eR = 0.0, eC = 0.0, eO = 0.0;
  if (tid < n_edge) {
    // Eq. 6 with A_j (A44): e = A_j d + g_j + t_j - g_l - t_l, d = g_l - g_j
    const int j = (int)(tid / a.n_nbr), l = a.nbr[tid];
    if (l >= 0) {
      const double* Aj = a.nd.Rt64 + 12 * j;
      const double* Al = a.nd.Rt64 + 12 * l;
      const float* gj = a.nd.g + 3 * j;
      const float* gl = a.nd.g + 3 * l;
      const double d[3] = {(double)gl[0] - gj[0], (double)gl[1] - gj[1], (double)gl[2] - gj[2]};
      double e[3];
      for (int q = 0; q < 3; ++q)
        e[q] = (Aj[3 * q] * d[0] + Aj[3 * q + 1] * d[1] + Aj[3 * q + 2] * d[2] - d[q]) + (Aj[9 + q] - Al[9 + q]);
      eR = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
      const float w = a.w_reg;
      float* G = a.acc.graph;
      const int64_t dj = a.diag_slot[j], dl = a.diag_slot[l], ej = a.edge_slot[tid];
      const bool tr = j > l;   // the (min, max) entry holds the (l, j) block
      // J_j = [d_c at (q, 3q + c), I], J_l = [0, -I]
      for (int q = 0; q < 3; ++q) {
        for (int c = 0; c < 3; ++c) {
          for (int c2 = 0; c2 < 3; ++c2) add_e(G, dj, false, 3 * q + c, 3 * q + c2, (float)(w * d[c] * d[c2]));
          add_e(G, dj, false, 3 * q + c, 9 + q, (float)(w * d[c]));
          add_e(G, dj, false, 9 + q, 3 * q + c, (float)(w * d[c]));
          add_e(G, ej, tr, 3 * q + c, 9 + q, (float)(-w * d[c]));   // J_j^T J_l
        }
        add_e(G, dj, false, 9 + q, 9 + q, w);
        add_e(G, dl, false, 9 + q, 9 + q, w);
        add_e(G, ej, tr, 9 + q, 9 + q, -w);
        for (int c = 0; c < 3; ++c) atomicAdd(a.acc.rhs_graph + 12 * j + 3 * q + c, (float)(-w * e[q] * d[c]));
        atomicAdd(a.acc.rhs_graph + 12 * j + 9 + q, (float)(-w * e[q]));
        atomicAdd(a.acc.rhs_graph + 12 * l + 9 + q, (float)(w * e[q]));
      }
    }
  } else if (tid < n_edge + n_fp) {
    // Eq. 9 (A12) with affine nodes: one thread per (feature, slot pair)
    const int64_t t2 = tid - n_edge;
    const int fi = (int)(t2 / P), pr = (int)(t2 % P);
    int s = 0, q = pr;
    while (q >= K - s) { q -= K - s; ++s; }
    const int s2 = s + q;
    const double V[3] = {a.fsrc[3 * fi], a.fsrc[3 * fi + 1], a.fsrc[3 * fi + 2]};
    double W = 0.0;
    for (int u = 0; u < K; ++u) W += a.fw[(int64_t)u * a.nf + fi];
    if (W > 0.0) {
      double xh[3] = {0, 0, 0}, dd[MIS_MAX_K][3], wn[MIS_MAX_K];
      for (int u = 0; u < K; ++u) {
        const int j = a.fidx[(int64_t)u * a.nf + fi];
        const double* A = a.nd.Rt64 + 12 * j;
        const float* g = a.nd.g + 3 * j;
        wn[u] = a.fw[(int64_t)u * a.nf + fi] / W;
        for (int r = 0; r < 3; ++r) dd[u][r] = V[r] - g[r];
        for (int r = 0; r < 3; ++r)
          xh[r] += wn[u] * (A[3 * r] * dd[u][0] + A[3 * r + 1] * dd[u][1] + A[3 * r + 2] * dd[u][2] + g[r] + A[9 + r]);
      }
      const double* R = a.fr.Rd;
      double e[3], rp[3];
      for (int r = 0; r < 3; ++r)
        e[r] = R[3 * r] * xh[0] + R[3 * r + 1] * xh[1] + R[3 * r + 2] * xh[2] + a.fr.Td[r] - a.fdst[3 * fi + r];
      for (int r = 0; r < 3; ++r) rp[r] = R[r] * e[0] + R[3 + r] * e[1] + R[6 + r] * e[2];   // r' = R^T e
      const int ja = a.fidx[(int64_t)s * a.nf + fi], jb = a.fidx[(int64_t)s2 * a.nf + fi];
      const int64_t ef = a.feat_slot[t2];
      const bool tr = ja > jb;
      const double ww = a.w_corr * wn[s] * wn[s2];
      for (int i = 0; i < 12; ++i)
        for (int jj = 0; jj < 12; ++jj) add_e(a.acc.graph, ef, tr, i, jj, pt_entry(dd[s], dd[s2], ww, i, jj));
      if (s == s2) {   // the slot's rhs (once per slot) and the energy (once per feature)
        if (s == 0) eC = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
        const double wc = a.w_corr * wn[s];
        for (int r = 0; r < 3; ++r) {
          for (int cc = 0; cc < 3; ++cc)
            atomicAdd(a.acc.rhs_graph + 12 * ja + 3 * r + cc, (float)(-wc * dd[s][cc] * rp[r]));
          atomicAdd(a.acc.rhs_graph + 12 * ja + 9 + r, (float)(-wc * rp[r]));
        }
      }
    }
  } else if (tid < n_edge + n_fp + m) {
    // Eq. 4-5 (A42): r = [c1.c2, c1.c3, c2.c3, |c1|^2 - 1, |c2|^2 - 1, |c3|^2 - 1], A row-major
    const int j = (int)(tid - n_edge - n_fp);
    const double* A = a.nd.Rt64 + 12 * j;
    const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {1, 2, 2, 0, 1, 2};
    double r[6], J[6][9];
    for (int q = 0; q < 6; ++q) {
      const int ca = pa[q], cb = pb[q];
      r[q] = A[ca] * A[cb] + A[3 + ca] * A[3 + cb] + A[6 + ca] * A[6 + cb] - (ca == cb ? 1.0 : 0.0);
      for (int e = 0; e < 9; ++e) J[q][e] = 0.0;
      for (int row = 0; row < 3; ++row) {
        J[q][3 * row + ca] += A[3 * row + cb];
        J[q][3 * row + cb] += A[3 * row + ca];
      }
      eO += r[q] * r[q];
    }
    const int64_t dj = a.diag_slot[j];
    const double w = a.w_rot;
    for (int i = 0; i < 9; ++i) {
      for (int jj = 0; jj < 9; ++jj) {
        double h = 0.0;
        for (int q = 0; q < 6; ++q) h += J[q][i] * J[q][jj];
        add_e(a.acc.graph, dj, false, i, jj, (float)(w * h));
      }
      double b = 0.0;
      for (int q = 0; q < 6; ++q) b += J[q][i] * r[q];
      atomicAdd(a.acc.rhs_graph + 12 * j + i, (float)(-w * b));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    eR += __shfl_xor_sync(0xffffffffu, eR, o);
    eC += __shfl_xor_sync(0xffffffffu, eC, o);
    eO += __shfl_xor_sync(0xffffffffu, eO, o);
  }
  if ((threadIdx.x & 31) == 0) {
    energy_add(a.acc.energy, 2, eR);
    energy_add(a.acc.energy, 3, eC);
    energy_add(a.acc.energy, 5, eO);
  }
}

void launch_assemble_graph_aff(const AsmGraphArgs& a, cudaStream_t s) {
  const int64_t P = a.K * (a.K + 1) / 2;
  const int64_t n = (int64_t)a.nd.m * a.n_nbr + (int64_t)a.nf * P + a.nd.m;
  if (n <= 0) return;
  launch_pdl(k_assemble_graph_aff, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, a);
}

// ---------------------------------------------------------------- finalisation (12 x 12)
// One warp per upper BSR entry (diagonals first, then the off-diagonal work list), entries
// l = lane, lane + 32, ... < 144:
//   H = w_data D + w_pt PT(moments) + G, PT[(r,c),(r',c')] = delta_rr' S[c][c'],
//   PT[(r,c), 9+r'] = delta_rr' s_j[c], PT[9+r, (r',c')] = delta_rr' s_l[c'], PT[9+r, 9+r'] = delta s0
// (S = Mo[4p+q], s_j = Mo[4p+3], s_l = Mo[12+q] -- symmetric / upper-only on the diagonal);
// the mirror gets the transpose; every accumulator read is re-zeroed.  Diagonal warps then build
// the fp64 block-Jacobi inverse of (H_jj + lambda I + mu_j I), mu_j = 1e-9 tr / 12 (A17).
__device__ __forceinline__ float pt_aff(const float* Mo, bool diag, int i, int j) {
  const int ri = i < 9 ? i / 3 : i - 9, rj = j < 9 ? j / 3 : j - 9;
  if (ri != rj) return 0.f;
  if (i < 9 && j < 9) {
    const int p = i % 3, q = j % 3;
    return diag ? Mo[4 * min(p, q) + max(p, q)] : Mo[4 * p + q];
  }
  if (i < 9) return Mo[4 * (i % 3) + 3];
  if (j < 9) return diag ? Mo[4 * (j % 3) + 3] : Mo[12 + (j % 3)];
  return Mo[15];
}

__global__ void __launch_bounds__(256) k_finalize_aff(FinalArgs r) {
  __shared__ float hst[8][144];
  pdl_wait();
  if (r.lm && r.lm->acc_buf == 0) {   // LM: keep the accepted system, write the trial's into the other buffer
    r.Hval = r.Hval_alt;
    r.rhs = r.rhs_alt;
  }
  pdl_trigger();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n_blk = r.m + r.nup;
  if (gw < n_blk) {
    const bool diag = gw < r.m;
    int64_t e;
    int lo = -1;
    if (diag) {
      e = r.diag_pos[gw];
    } else {
      const int2 ul = r.ulist[gw - r.m];
      e = ul.x;
      lo = ul.y;
    }
    float Mo[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) Mo[q] = r.acc.mom[16 * e + q];
    __syncwarp();
    if (lane < 16) r.acc.mom[16 * e + lane] = 0.f;
    for (int l = lane; l < 144; l += 32) {
      const int i = l / 12, j = l - 12 * (l / 12);
      const float D = diag ? r.acc.data[144 * e + 12 * min(i, j) + max(i, j)] : r.acc.data[144 * e + l];
      hst[wib][l] = r.w_data * D + r.w_pt * pt_aff(Mo, diag, i, j) + r.acc.graph[144 * e + l];
    }
    __syncwarp();
    for (int l = lane; l < 144; l += 32) {
      const float h = hst[wib][l];
      r.Hval[144 * e + l] = h;
      if (!diag) {
        const int i = l / 12, j = l - 12 * (l / 12);
        r.Hval[144 * (int64_t)lo + 12 * j + i] = h;
      }
      r.acc.data[144 * e + l] = 0.f;
      r.acc.graph[144 * e + l] = 0.f;
    }
    if (!diag || !r.Minv) return;
    __syncwarp();
    // Gauss-Jordan on [H + (lambda + mu) I | I] in fp64, lane rr < 12 holds row rr
    double trc = 0.0;
    for (int q = 0; q < 12; ++q) trc += (double)hst[wib][13 * q];
    const double mu = 1e-9 * trc / 12.0;
    const int rr = lane < 12 ? lane : 0;
    double row[24];
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      row[q] = (double)hst[wib][12 * rr + q] + (q == rr ? (double)r.lambda + mu : 0.0);
      row[12 + q] = q == rr ? 1.0 : 0.0;
    }
    bool pd = true;
#pragma unroll
    for (int p = 0; p < 12; ++p) {
      const double pv = __shfl_sync(0xffffffffu, row[p], p);
      if (!(pv > 0.0)) pd = false;
      const double ipv = 1.0 / pv, f = row[p] * ipv;
#pragma unroll
      for (int q = 0; q < 24; ++q) {
        const double pq = __shfl_sync(0xffffffffu, row[q], p);
        row[q] = rr == p ? pq * ipv : row[q] - f * pq;
      }
    }
    if (lane < 12)
#pragma unroll
      for (int q = 0; q < 12; ++q) r.Minv[144 * gw + 12 * rr + q] = pd ? (float)row[12 + q] : 0.f;
    return;
  }
  const int64_t g2 = gw - n_blk;
  if (g2 < r.m) {   // node rhs: b = -(w_data sum c r_pl + w_pt sum_pt) + graph, 12 entries
    const int64_t n = g2;
    if (lane < 12) {
      const float* Nm = r.acc.node_mom + 12 * n;   // [3p + q] = sum (w d)_p r'_q, [9 + q] = sum w r'_q
      const float pt = lane < 9 ? Nm[3 * (lane % 3) + lane / 3] : Nm[lane];
      const float v = -r.w_data * r.acc.rhs_data[12 * n + lane] - r.w_pt * pt + r.acc.rhs_graph[12 * n + lane];
      __syncwarp(0x00000fffu);
      r.rhs[12 * n + lane] = v;
      r.acc.rhs_data[12 * n + lane] = 0.f;
      r.acc.rhs_graph[12 * n + lane] = 0.f;
      r.acc.node_mom[12 * n + lane] = 0.f;
    }
    return;
  }
  if (g2 == r.m) {   // energies -> report slot; zeroed for the next assembly
    double* E = r.acc.energy;
    double tot[kEnergyQ];
#pragma unroll
    for (int q = 0; q < kEnergyQ; ++q) {
      double* st_q = E + 8 + kEnergyStripes * q;
      double vv = st_q[lane] + st_q[lane + 32];
      st_q[lane] = 0.0;
      st_q[lane + 32] = 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) vv += __shfl_xor_sync(0xffffffffu, vv, o);
      tot[q] = (q < 5 ? E[q] : 0.0) + vv;
    }
    if (lane == 0) {
      if (r.slot >= 0) {
        double* rep = r.rep_energy + 5 * r.slot;
        rep[0] = tot[0]; rep[1] = tot[1]; rep[2] = tot[2]; rep[3] = tot[3];
        rep[4] = (double)r.w_data * tot[0] + (double)r.w_pt * tot[1] + (double)r.w_reg * tot[2] +
                 (double)r.w_corr * tot[3] + (double)r.w_rot * tot[5];
        r.rep_nassoc[r.slot] = tot[4];
        r.rep_nassoc[MIS_MAX_GN + 1 + r.slot] = 0.0;
        if (r.rep_rot) r.rep_rot[r.slot] = tot[5];
      }
      for (int q = 0; q < 8; ++q) E[q] = 0.0;
    }
  }
}

void launch_finalize_aff(const FinalArgs& r, cudaStream_t s) {
  const int64_t warps = (int64_t)r.m + r.nup + r.m + 1;
  launch_pdl(k_finalize_aff, dim3((unsigned)((warps * 32 + 255) / 256)), dim3(256), 0, s, r);
}

}  // namespace mis
