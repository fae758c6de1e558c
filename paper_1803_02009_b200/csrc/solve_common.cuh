// solve_common.cuh -- device helpers shared by the two PCG kernels (solve.cu:
// grid-wide cooperative variant; pcg_cluster.cu: thread-block-cluster variant
// with the system resident in shared memory).
#pragma once
#include "common.cuh"

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

// Block (j, l), j <= l, of H from the accumulators of upper slot u:
//   H = w_data sum c c^T + w_pt PT(moments) + graph (K4/K5, already weighted),
//   PT = [tr(S) I - S^T, [s_j]x ; -[s_l]x, s0 I]  with S = sum s a_j a_l^T,
//   s_j = sum s a_j, s_l = sum s a_l, s0 = sum s, s = w_j w_l (point-to-point).
__device__ __forceinline__ void upper_block(const AccView& acc, float w_data, float w_pt, int64_t u, bool diag,
                                            float* B) {
  const float* D = acc.data + 36 * u;
  const float* Mo = acc.mom + 16 * u;
  const float* G = acc.graph + 36 * u;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      const float d = diag ? D[6 * min(r, c) + max(r, c)] : D[6 * r + c];
      B[6 * r + c] = w_data * d + G[6 * r + c];
    }
  float S[9], sj[3], sl[3];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) S[3 * p + q] = diag ? Mo[4 * min(p, q) + max(p, q)] : Mo[4 * p + q];
  for (int p = 0; p < 3; ++p) { sj[p] = Mo[4 * p + 3]; sl[p] = diag ? Mo[4 * p + 3] : Mo[12 + p]; }
  const float s0 = Mo[15];
  const float tr = S[0] + S[4] + S[8];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) B[6 * r + c] += w_pt * ((r == c ? tr : 0.f) - S[3 * c + r]);
  skew_into(B, 0, 3, sj, w_pt);
  skew_into(B, 3, 0, sl, -w_pt);
  for (int r = 0; r < 3; ++r) B[6 * (3 + r) + 3 + r] += w_pt * s0;
}

// Entry (i, j) of the block B(j, l), j <= l, from its summed data D (36; upper
// triangle only when diag), moments Mo (16) and graph part G (36).
__device__ __forceinline__ float block_entry(const float* D, const float* Mo, const float* G, bool diag, int i, int j,
                                             float w_data, float w_pt) {
  const float d = diag ? D[6 * min(i, j) + max(i, j)] : D[6 * i + j];
  float pt;
  if (i < 3 && j < 3) {   // tr(S) I - S^T, S = sum s a_j a_l^T
    const float trS = diag ? Mo[0] + Mo[5] + Mo[10] : Mo[0] + Mo[5] + Mo[10];
    const float Sji = diag ? Mo[4 * min(i, j) + max(i, j)] : Mo[4 * j + i];
    pt = (i == j ? trS : 0.f) - Sji;
  } else if (i < 3) {     // [s_j]x (i, j-3), s_j = Mo[p][3]
    const int c = j - 3;
    pt = (i == c) ? 0.f : ((c == (i + 1) % 3) ? -Mo[4 * ((i + 2) % 3) + 3] : Mo[4 * ((i + 1) % 3) + 3]);
  } else if (j < 3) {     // -[s_l]x (i-3, j), s_l = Mo[3][q] (= Mo[q][3] on the diagonal)
    const int rr = i - 3;
    const int q1 = (rr + 2) % 3, q2 = (rr + 1) % 3;
    const float sl1 = diag ? Mo[4 * q1 + 3] : Mo[12 + q1], sl2 = diag ? Mo[4 * q2 + 3] : Mo[12 + q2];
    pt = (rr == j) ? 0.f : ((j == (rr + 1) % 3) ? sl1 : -sl2);
  } else {
    pt = (i == j) ? Mo[15] : 0.f;
  }
  return w_data * d + G[6 * i + j] + w_pt * pt;
}

// Row r of the block B(j,l) of upper slot u (tr: row r of B^T), same formula as
// upper_block; one thread per (entry, row) keeps the loads parallel.
__device__ __forceinline__ void block_row(const AccView& acc, float w_data, float w_pt, int64_t u, bool diag, bool tr,
                                          int r, float* out) {
  const float* D = acc.data + 36 * u;
  const float* G = acc.graph + 36 * u;
  float Mo[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) Mo[q] = acc.mom[16 * u + q];
  float S[9], sj[3], sl[3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) S[3 * p + q] = diag ? Mo[4 * min(p, q) + max(p, q)] : Mo[4 * p + q];
#pragma unroll
  for (int p = 0; p < 3; ++p) { sj[p] = Mo[4 * p + 3]; sl[p] = diag ? Mo[4 * p + 3] : Mo[12 + p]; }
  const float s0 = Mo[15], trS = S[0] + S[4] + S[8];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int i = tr ? k : r, j = tr ? r : k;   // entry (i, j) of B
    const float d = diag ? D[6 * min(i, j) + max(i, j)] : D[6 * i + j];
    float pt;
    if (i < 3 && j < 3) {
      pt = (i == j ? trS : 0.f) - S[3 * j + i];
    } else if (i < 3) {            // [s_j]x (i, j-3)
      const int c = j - 3;
      pt = (i == c) ? 0.f : ((c == (i + 1) % 3) ? -sj[(i + 2) % 3] : sj[(i + 1) % 3]);
    } else if (j < 3) {            // -[s_l]x (i-3, j)
      const int rr = i - 3;
      pt = (rr == j) ? 0.f : ((j == (rr + 1) % 3) ? sl[(rr + 2) % 3] : -sl[(rr + 1) % 3]);
    } else {
      pt = (i == j) ? s0 : 0.f;
    }
    out[k] = w_data * d + G[6 * i + j] + w_pt * pt;
  }
}

// b_i = -(w_data sum c r_pl + w_pt sum w_j [a_j x r'; r']) + graph rhs
__device__ __forceinline__ float rhs_entry(const AccView& acc, float w_data, float w_pt, int64_t i) {
  const int64_t j = i / 6;
  const int c = (int)(i % 6);
  const float* Nm = acc.node_mom + 12 * j;
  float pt;
  if (c < 3) {
    const int c1 = (c + 1) % 3, c2 = (c + 2) % 3;   // (sum w a x r')_c = Nm[c1][c2] - Nm[c2][c1]
    pt = Nm[3 * c1 + c2] - Nm[3 * c2 + c1];
  } else {
    pt = Nm[9 + (c - 3)];
  }
  return -w_data * acc.rhs_data[i] - w_pt * pt + acc.rhs_graph[i];
}

// 6x6 SPD inverse in fp64 via Cholesky; false if not positive definite
__device__ inline bool inv6(const double* A, double* Ai) {
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

// M_j = (H_jj + lambda I + mu_j I)^-1, mu_j = 1e-9 tr(H_jj)/6 (reading A17); 0 if not PD
__device__ inline void precond_block(const float* Hjj, float lambda, float* Mi) {
  double A[36], Ai[36], tr = 0;
  for (int i = 0; i < 36; ++i) A[i] = Hjj[i];
  for (int i = 0; i < 6; ++i) tr += A[7 * i];
  const double mu = 1e-9 * tr / 6.0;
  for (int i = 0; i < 6; ++i) A[7 * i] += (double)lambda + mu;
  if (!inv6(A, Ai))
    for (int i = 0; i < 36; ++i) Ai[i] = 0.0;
  for (int i = 0; i < 36; ++i) Mi[i] = (float)Ai[i];
}

// Row r of R_j <- Exp(dtheta) R_j and t_j[r] += dt[r] (the update split over 3 threads per node);
// Rt: the node's current fp64 state (R row-major, t), out to the fp64 master and the fp32 copy
__device__ inline void node_update_row(const float* dx, const double* Rt, int r, double* Rt_out, float* n32) {
  const double w0 = dx[0], w1 = dx[1], w2 = dx[2];
  const double t2 = w0 * w0 + w1 * w1 + w2 * w2, th = sqrt(t2);
  double A, Bc;
  if (th < 0.05) {   // Taylor series of sin(th)/th and (1 - cos th)/th^2: truncation < 1e-20 here
    A = 1.0 + t2 * (-1.0 / 6 + t2 * (1.0 / 120 + t2 * (-1.0 / 5040 + t2 * (1.0 / 362880))));
    Bc = 0.5 + t2 * (-1.0 / 24 + t2 * (1.0 / 720 + t2 * (-1.0 / 40320 + t2 * (1.0 / 3628800))));
  } else {
    A = sin(th) / th;
    Bc = (1.0 - cos(th)) / t2;
  }
  const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
  double E[3];
  for (int jj = 0; jj < 3; ++jj) {
    const double k2 = K[3 * r] * K[jj] + K[3 * r + 1] * K[3 + jj] + K[3 * r + 2] * K[6 + jj];
    E[jj] = (r == jj ? 1.0 : 0.0) + A * K[3 * r + jj] + Bc * k2;
  }
  for (int jj = 0; jj < 3; ++jj) {
    const double v = E[0] * Rt[jj] + E[1] * Rt[3 + jj] + E[2] * Rt[6 + jj];
    Rt_out[3 * r + jj] = v;
    n32[3 * r + jj] = (float)v;
  }
  const double tv = Rt[9 + r] + (double)dx[3 + r];
  Rt_out[9 + r] = tv;
  n32[9 + r] = (float)tv;
}

// R_j <- Exp(dtheta) R_j (Rodrigues; series coefficients for small theta), t_j += dt (reading A18)
__device__ inline void node_update(const float* dx, double* Rt, float* n32) {
  const double w0 = dx[0], w1 = dx[1], w2 = dx[2];
  const double th = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int jj = 0; jj < 3; ++jj) K2[3 * i + jj] = K[3 * i] * K[jj] + K[3 * i + 1] * K[3 + jj] + K[3 * i + 2] * K[6 + jj];
  double A, Bc;
  if (th < 0.05) {   // Taylor series of sin(th)/th and (1 - cos th)/th^2: truncation < 1e-20 here
    const double t2 = th * th;
    A = 1.0 + t2 * (-1.0 / 6 + t2 * (1.0 / 120 + t2 * (-1.0 / 5040 + t2 * (1.0 / 362880))));
    Bc = 0.5 + t2 * (-1.0 / 24 + t2 * (1.0 / 720 + t2 * (-1.0 / 40320 + t2 * (1.0 / 3628800))));
  } else {
    A = sin(th) / th;
    Bc = (1.0 - cos(th)) / (th * th);
  }
  double E[9];
  for (int i = 0; i < 9; ++i) E[i] = ((i % 4) == 0 ? 1.0 : 0.0) + A * K[i] + Bc * K2[i];
  double Rn[9];
  for (int i = 0; i < 3; ++i)
    for (int jj = 0; jj < 3; ++jj) Rn[3 * i + jj] = E[3 * i] * Rt[jj] + E[3 * i + 1] * Rt[3 + jj] + E[3 * i + 2] * Rt[6 + jj];
  for (int i = 0; i < 9; ++i) { Rt[i] = Rn[i]; n32[i] = (float)Rn[i]; }
  for (int c = 0; c < 3; ++c) {
    Rt[9 + c] += (double)dx[3 + c];
    n32[9 + c] = (float)Rt[9 + c];
  }
}

// ---- NEXT-2 (MIS_F_JOINT_POSE, readings A37-A40)
// A37: R <- R Exp(dphi), T <- T + R dtau (fp64, in place; dx = [dphi, dtau])
__device__ inline void pose_update(const float* dx, double* P) {
  const double w0 = dx[0], w1 = dx[1], w2 = dx[2];
  const double t2 = w0 * w0 + w1 * w1 + w2 * w2, th = sqrt(t2);
  double A, Bc;
  if (th < 0.05) {
    A = 1.0 + t2 * (-1.0 / 6 + t2 * (1.0 / 120 + t2 * (-1.0 / 5040 + t2 * (1.0 / 362880))));
    Bc = 0.5 + t2 * (-1.0 / 24 + t2 * (1.0 / 720 + t2 * (-1.0 / 40320 + t2 * (1.0 / 3628800))));
  } else {
    A = sin(th) / th;
    Bc = (1.0 - cos(th)) / t2;
  }
  const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
  double E[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double k2 = K[3 * i] * K[j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
      E[3 * i + j] = (i == j ? 1.0 : 0.0) + A * K[3 * i + j] + Bc * k2;
    }
  double Rn[9], dT[3];
  for (int i = 0; i < 3; ++i) {
    dT[i] = P[3 * i] * dx[3] + P[3 * i + 1] * dx[4] + P[3 * i + 2] * dx[5];
    for (int j = 0; j < 3; ++j) Rn[3 * i + j] = P[3 * i] * E[j] + P[3 * i + 1] * E[3 + j] + P[3 * i + 2] * E[6 + j];
  }
  for (int i = 0; i < 9; ++i) P[i] = Rn[i];
  for (int i = 0; i < 3; ++i) P[9 + i] += dT[i];
}

// Eq. 10 at the current pose P against the prior P0 (R row-major 9, T 3, world -> camera):
//  r[0..3) = wrap(e(O) - e(O0)), e = ZYX Euler angles (yaw, pitch, roll) of the scope orientation
//  O = R^T (A38); r[3..6) = c - c0, c = -R^T T the scope position (A39); J = dr/d[dphi, dtau]
//  under A37's increment: O' = Exp(-dphi) O, so the Euler rows are -E_s^-1 with E_s^-1 written out
//  row by row (yaw: [tan(th) cos(psi), tan(th) sin(psi), 1], pitch: [-sin(psi), cos(psi), 0],
//  roll: [cos(psi), sin(psi), 0] / cos(th)); c' = c - dtau + [c]x dphi.  Returns false at gimbal
//  lock (|cos th| < 1e-6), where the orientation rows are zero.
__device__ inline bool pose_prior_dev(const double* P0, const double* P, double* r, double* J) {
  // O = R^T: O[i][j] = R[j][i]; yaw = atan2(O10, O00), pitch = asin(-O20), roll = atan2(O21, O22)
  const double yaw = atan2(P[1], P[0]), pitch = asin(fmin(1.0, fmax(-1.0, -P[2]))), roll = atan2(P[5], P[8]);
  const double yaw0 = atan2(P0[1], P0[0]), pitch0 = asin(fmin(1.0, fmax(-1.0, -P0[2]))), roll0 = atan2(P0[5], P0[8]);
  const double d[3] = {yaw - yaw0, pitch - pitch0, roll - roll0};
  for (int q = 0; q < 3; ++q) {
    double v = d[q];
    while (v > M_PI) v -= 2.0 * M_PI;
    while (v <= -M_PI) v += 2.0 * M_PI;
    r[q] = v;
  }
  double c[3], c0[3];
  for (int q = 0; q < 3; ++q) {
    c[q] = -(P[q] * P[9] + P[3 + q] * P[10] + P[6 + q] * P[11]);
    c0[q] = -(P0[q] * P0[9] + P0[3 + q] * P0[10] + P0[6 + q] * P0[11]);
    r[3 + q] = c[q] - c0[q];
  }
  for (int q = 0; q < 36; ++q) J[q] = 0.0;
  J[18 + 1] = -c[2]; J[18 + 2] = c[1];     // [c]x
  J[24 + 0] = c[2];  J[24 + 2] = -c[0];
  J[30 + 0] = -c[1]; J[30 + 1] = c[0];
  J[18 + 3] = J[24 + 4] = J[30 + 5] = -1.0;
  const double cp = cos(yaw), sp = sin(yaw), ct = cos(pitch), st = sin(pitch);
  if (fabs(ct) < 1e-6) { r[0] = r[1] = r[2] = 0.0; return false; }
  const double tt = st / ct;
  J[0] = -tt * cp; J[1] = -tt * sp; J[2] = -1.0;
  J[6] = sp;       J[7] = -cp;      J[8] = 0.0;
  J[12] = -cp / ct; J[13] = -sp / ct; J[14] = 0.0;
  return true;
}

}  // namespace mis
