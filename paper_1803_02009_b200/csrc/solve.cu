// solve.cu -- K6-K8: finalise the 6x6 block system, block-Jacobi PCG and the
// node update, as ONE persistent cooperative kernel per Gauss-Newton
// iteration (grid-wide barriers between the PCG phases instead of ~40 kernel
// launches).
//
//   H = w_data * sum c c^T  +  w_pt * PT(moments)  +  graph blocks (K4/K5)
//   b = -(w_data sum c r_pl + w_pt sum w_j [a_j x r'; r']) + graph rhs
//   (H + lambda I) dx = b  by PCG from x0 = 0, M_j = (H_jj + lambda I + mu_j I)^-1,
//   mu_j = 1e-9 tr(H_jj) / 6 (reading A17), P fixed iterations (early stop if
//   r.z == 0 or p.Ap <= 0, exactly like the oracle's MIRROR mode)
//   R_j <- Exp(dtheta_j) R_j, t_j += dt_j (fp64 master state, reading A18).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mis {

__device__ __forceinline__ void skew_into(float* M, int r0, int c0, const float* v, float s) {
  // M[r0.., c0..] += s [v]x   (6x6 row-major)
  M[6 * (r0 + 0) + c0 + 1] += -s * v[2];
  M[6 * (r0 + 0) + c0 + 2] += s * v[1];
  M[6 * (r0 + 1) + c0 + 0] += s * v[2];
  M[6 * (r0 + 1) + c0 + 2] += -s * v[0];
  M[6 * (r0 + 2) + c0 + 0] += -s * v[1];
  M[6 * (r0 + 2) + c0 + 1] += s * v[0];
}

// Block (j, l), j <= l, from the accumulators of upper slot u.
__device__ void upper_block(const SolveArgs& a, int64_t u, bool diag, float* B) {
  const float* D = a.acc.data + 36 * u;
  const float* Mo = a.acc.mom + 16 * u;
  const float* G = a.acc.graph + 36 * u;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      float d = diag ? D[6 * min(r, c) + max(r, c)] : D[6 * r + c];
      B[6 * r + c] = a.w_data * d + G[6 * r + c];
    }
  // point-to-point from moments: S = sum s a_j a_l^T, sj = sum s a_j, sl = sum s a_l, s0 = sum s
  float S[9], sj[3], sl[3];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) S[3 * p + q] = diag ? Mo[4 * min(p, q) + max(p, q)] : Mo[4 * p + q];
  for (int p = 0; p < 3; ++p) { sj[p] = Mo[4 * p + 3]; sl[p] = diag ? Mo[4 * p + 3] : Mo[12 + p]; }
  const float s0 = Mo[15];
  const float tr = S[0] + S[4] + S[8];
  const float w = a.w_pt;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) B[6 * r + c] += w * ((r == c ? tr : 0.f) - S[3 * c + r]);   // tr(S) I - S^T
  skew_into(B, 0, 3, sj, w);     //  [sum s a_j]x
  skew_into(B, 3, 0, sl, -w);    // -[sum s a_l]x
  for (int r = 0; r < 3; ++r) B[6 * (3 + r) + 3 + r] += w * s0;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;   // valid on thread 0
}

// 6x6 SPD inverse in fp64 via Cholesky; false if not positive definite
__device__ bool inv6(const double* A, double* Ai) {
  double L[36];
  for (int i = 0; i < 36; ++i) L[i] = A[i];
  for (int j = 0; j < 6; ++j) {
    double s = L[6 * j + j];
    for (int k = 0; k < j; ++k) s -= L[6 * j + k] * L[6 * j + k];
    if (!(s > 0)) return false;
    const double d = sqrt(s);
    L[6 * j + j] = d;
    for (int i = j + 1; i < 6; ++i) {
      double t = L[6 * i + j];
      for (int k = 0; k < j; ++k) t -= L[6 * i + k] * L[6 * j + k];
      L[6 * i + j] = t / d;
    }
  }
  for (int c = 0; c < 6; ++c) {
    double y[6], x[6];
    for (int i = 0; i < 6; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[6 * i + k] * y[k];
      y[i] = s / L[6 * i + i];
    }
    for (int i = 5; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < 6; ++k) s -= L[6 * k + i] * x[k];
      x[i] = s / L[6 * i + i];
    }
    for (int r = 0; r < 6; ++r) Ai[6 * r + c] = x[r];
  }
  return true;
}

__global__ void __launch_bounds__(256) k_solve(SolveArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int m = a.m, n6 = 6 * m;

  // ---- phase 0: finalise H (both triangles) and b; report energies
  for (int64_t e = tid; e < a.nnzb; e += nth) {
    const int64_t u = a.upper_of[e];
    const bool tr = (u != e);
    // diagonal entries are their own upper entry; row index needed only for diag test
    float B[36];
    // an entry is diagonal iff its column equals its row; find row cheaply: diag iff u==e and col==row
    // (upper_of == e for diagonal and strictly-upper entries; diag test via diag_pos of its column)
    const int c = a.col[e];
    const bool diag = (a.diag_pos[c] == e);
    upper_block(a, u, diag, B);
    float* out = a.Hval + 36 * e;
    if (!tr) {
      for (int i = 0; i < 36; ++i) out[i] = B[i];
    } else {
      for (int r = 0; r < 6; ++r)
        for (int cc = 0; cc < 6; ++cc) out[6 * r + cc] = B[6 * cc + r];
    }
  }
  for (int64_t i = tid; i < n6; i += nth) {
    const int j = (int)(i / 6), c = (int)(i % 6);
    const float* Nm = a.acc.node_mom + 12 * j;
    float pt;
    if (c < 3) {
      const int c1 = (c + 1) % 3, c2 = (c + 2) % 3;   // (sum w a x r')_c = Nm[c1][c2] - Nm[c2][c1]
      pt = Nm[3 * c1 + c2] - Nm[3 * c2 + c1];
    } else {
      pt = Nm[9 + (c - 3)];
    }
    a.rhs[i] = -a.w_data * a.acc.rhs_data[i] - a.w_pt * pt + a.acc.rhs_graph[i];
  }
  if (tid < 2 * a.pcg_iters + 4) a.dots[tid] = 0.0;
  grid.sync();
  if (a.pcg_iters <= 0 && !a.do_update) return;

  // ---- phase 1: preconditioner, x = 0, r = b, z = M r, p = z
  double my = 0.0;
  for (int64_t j = tid; j < m; j += nth) {
    const float* Hd = a.Hval + 36 * (int64_t)a.diag_pos[j];
    double A[36], Ai[36];
    double tr = 0;
    for (int i = 0; i < 36; ++i) A[i] = Hd[i];
    for (int i = 0; i < 6; ++i) tr += A[7 * i];
    const double mu = 1e-9 * tr / 6.0;
    for (int i = 0; i < 6; ++i) A[7 * i] += (double)a.lambda + mu;
    if (!inv6(A, Ai))
      for (int i = 0; i < 36; ++i) Ai[i] = 0.0;
    float* Mi = a.Minv + 36 * j;
    for (int i = 0; i < 36; ++i) Mi[i] = (float)Ai[i];
    for (int r = 0; r < 6; ++r) {
      double z = 0;
      for (int c = 0; c < 6; ++c) z += (double)Mi[6 * r + c] * a.rhs[6 * j + c];
      a.x[6 * j + r] = 0.f;
      a.r[6 * j + r] = a.rhs[6 * j + r];
      a.z[6 * j + r] = (float)z;
      a.p[6 * j + r] = (float)z;
      my += (double)a.rhs[6 * j + r] * (double)(float)z;
    }
  }
  double s = block_sum(my, sh);
  if (threadIdx.x == 0) atomicAdd(a.dots + 0, s);
  grid.sync();
  double rz = a.dots[0];
  const double rz0 = rz;
  for (int it = 0; it < a.pcg_iters; ++it) {
    if (rz == 0.0) break;
    // Ap = (H + lambda I) p ; p.Ap
    my = 0.0;
    for (int64_t q = tid; q < n6; q += nth) {
      const int row = (int)(q / 6), c = (int)(q % 6);
      float acc = a.lambda * a.p[q];
      for (int e = a.row_ptr[row]; e < a.row_ptr[row + 1]; ++e) {
        const float* Hb = a.Hval + 36 * (int64_t)e + 6 * c;
        const float* pp = a.p + 6 * a.col[e];
#pragma unroll
        for (int b = 0; b < 6; ++b) acc = fmaf(Hb[b], pp[b], acc);
      }
      a.Ap[q] = acc;
      my += (double)a.p[q] * (double)acc;
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 1 + 2 * it, s);
    grid.sync();
    const double pAp = a.dots[1 + 2 * it];
    if (!(pAp > 0.0)) break;
    const float alpha = (float)(rz / pAp);
    my = 0.0;
    for (int64_t j = tid; j < m; j += nth) {
      float rr[6];
      for (int c = 0; c < 6; ++c) {
        const int64_t q = 6 * j + c;
        a.x[q] = fmaf(alpha, a.p[q], a.x[q]);
        rr[c] = fmaf(-alpha, a.Ap[q], a.r[q]);
        a.r[q] = rr[c];
      }
      const float* Mi = a.Minv + 36 * j;
      for (int r = 0; r < 6; ++r) {
        float z = 0.f;
        for (int c = 0; c < 6; ++c) z = fmaf(Mi[6 * r + c], rr[c], z);
        a.z[6 * j + r] = z;
        my += (double)rr[r] * (double)z;
      }
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 2 + 2 * it, s);
    grid.sync();
    const double rzn = a.dots[2 + 2 * it];
    const float beta = (float)(rzn / rz);
    rz = rzn;
    for (int64_t q = tid; q < n6; q += nth) a.p[q] = fmaf(beta, a.p[q], a.z[q]);
    grid.sync();
  }
  if (tid == 0) a.rep_res[a.gn_it] = (float)(rz0 > 0 ? sqrt(fabs(rz / rz0)) : 0.0);
  if (!a.do_update) return;

  // ---- node update (fp64 master), rolled back as a whole on a non-finite step
  for (int64_t j = tid; j < m; j += nth)
    for (int c = 0; c < 6; ++c)
      if (!isfinite(a.x[6 * j + c])) atomicOr(a.numeric_flag, 1);
  grid.sync();
  if (*a.numeric_flag) return;
  for (int64_t j = tid; j < m; j += nth) {
    const double w0 = a.x[6 * j], w1 = a.x[6 * j + 1], w2 = a.x[6 * j + 2];
    const double th = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
    double K2[9];
    for (int i = 0; i < 3; ++i)
      for (int jj = 0; jj < 3; ++jj) K2[3 * i + jj] = K[3 * i] * K[jj] + K[3 * i + 1] * K[3 + jj] + K[3 * i + 2] * K[6 + jj];
    double A, Bc;
    if (th < 1e-12) { A = 1.0; Bc = 0.0; }
    else { A = sin(th) / th; Bc = (1.0 - cos(th)) / (th * th); }
    double E[9];
    for (int i = 0; i < 9; ++i) E[i] = ((i % 4) == 0 ? 1.0 : 0.0) + A * K[i] + Bc * K2[i];
    double* Rt = a.nd.Rt64 + 12 * j;
    double Rn[9];
    for (int i = 0; i < 3; ++i)
      for (int jj = 0; jj < 3; ++jj) Rn[3 * i + jj] = E[3 * i] * Rt[jj] + E[3 * i + 1] * Rt[3 + jj] + E[3 * i + 2] * Rt[6 + jj];
    float* n32 = a.nd.node32 + 16 * j;
    for (int i = 0; i < 9; ++i) { Rt[i] = Rn[i]; n32[i] = (float)Rn[i]; }
    for (int c = 0; c < 3; ++c) {
      Rt[9 + c] += (double)a.x[6 * j + 3 + c];
      n32[9 + c] = (float)Rt[9 + c];
    }
  }
}

cudaError_t launch_solve(const SolveArgs& a, int num_sms, cudaStream_t s) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, 256, 0);
  int64_t work = 6 * (int64_t)a.m;
  if (a.nnzb > work) work = a.nnzb;
  int64_t grid = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > num_sms) grid = num_sms;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  SolveArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)k_solve, dim3((unsigned)grid), dim3(256), params, 0, s);
}

__global__ void k_energy_report(AccView acc, float w_data, float w_pt, float w_reg, float w_corr, int slot,
                                double* rep_energy, double* rep_nassoc) {
  const double* E = acc.energy;
  double* rep = rep_energy + 5 * slot;
  rep[0] = E[0]; rep[1] = E[1]; rep[2] = E[2]; rep[3] = E[3];
  rep[4] = (double)w_data * E[0] + (double)w_pt * E[1] + (double)w_reg * E[2] + (double)w_corr * E[3];
  rep_nassoc[slot] = E[4];
}

void launch_energy_report(const AccView& acc, float w_data, float w_pt, float w_reg, float w_corr, int slot,
                          double* rep_energy, double* rep_nassoc, cudaStream_t s) {
  k_energy_report<<<1, 1, 0, s>>>(acc, w_data, w_pt, w_reg, w_corr, slot, rep_energy, rep_nassoc);
}

}  // namespace mis
