// solve.cu -- K6-K8, grid-wide variant: finalise the 6x6 block system,
// block-Jacobi PCG and the node update as ONE persistent cooperative kernel per
// Gauss-Newton iteration, for systems too large for the cluster-resident
// variant (pcg_cluster.cu).  Two grid barriers per PCG iteration: the search
// direction is advanced with the recurrence A p_{k+1} = A z_{k+1} + beta A p_k,
// so the SpMV reads z (complete after the r.z barrier) and the p / Ap updates
// fuse into the same phase.
//
//   (H + lambda I) dx = b from x0 = 0, M_j = (H_jj + lambda I + mu_j I)^-1,
//   P fixed iterations, early stop if r.z == 0 or p.Ap <= 0 (the oracle's
//   MIRROR mode); R_j <- Exp(dtheta_j) R_j, t_j += dt_j in fp64.
#include <cooperative_groups.h>

#include <cstdlib>

#include "solve_common.cuh"

namespace cg = cooperative_groups;

namespace mis {

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

// B: unknowns per node block -- 6 (SE(3) nodes) or 12 (NEXT-4 affine nodes, additive update)
template <int B>
__global__ void __launch_bounds__(256) k_solve(SolveArgs a) {
  constexpr int BB = B * B;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int m = a.m, n6 = B * m;
  // NEXT-2 (arrowhead): the dense pose row (unknown pose_node = m - 1, ~m blocks) is not a row of
  // the row loop: its blocks are spread over all threads, each warp's partial H_pose,j z_j sums
  // go to per-iteration slots pose_y (fp64 atomics), and after the dot's grid barrier every
  // thread finishes the pose's 6 components from them identically (its p.Ap share included)
  const int64_t n6s = a.pose_node >= 0 ? B * (int64_t)a.pose_node : n6;
  const int lane = threadIdx.x & 31;
  double* pose_y = a.dots + 2 * a.pcg_iters + 8;   // 6 per iteration

  // ---- phase 0: H (both triangles) and b are final (record reduction); clear the dot slots
  if (tid < 8 * a.pcg_iters + 16) a.dots[tid] = 0.0;
  grid.sync();
  if (a.pcg_iters <= 0 && !a.do_update) return;

  // ---- phase 1: preconditioner, x = 0, r = b, z = M r, p = Ap = 0
  double my = 0.0;
  for (int64_t j = tid; j < m; j += nth) {
    float* Mi = a.Minv + BB * j;
    if constexpr (B == 6) {
      if (!a.minv_ready) precond_block(a.Hval + 36 * (int64_t)a.diag_pos[j], a.lambda, Mi);
    }
    for (int r = 0; r < B; ++r) {
      float z = 0.f;
      for (int c = 0; c < B; ++c) z = fmaf(Mi[B * r + c], a.rhs[B * j + c], z);
      const int64_t q = B * j + r;
      a.x[q] = 0.f; a.r[q] = a.rhs[q]; a.z[q] = z; a.p[q] = 0.f; a.Ap[q] = 0.f;
      my += (double)a.rhs[q] * (double)z;
    }
  }
  double s = block_sum(my, sh);
  if (threadIdx.x == 0) atomicAdd(a.dots + 0, s);
  grid.sync();
  double rz = a.dots[0], rz_prev = 1.0;
  bool nonfin = false;
  const double rz0 = rz;
  // NEXT-2: every thread keeps the pose's p, Ap, r, z, x in registers (computed identically from
  // the same inputs), so no thread reads a pose value another thread is about to overwrite; the
  // pose's z (read by the other rows' SpMV) and x are published by thread 0
  const bool has_pose = B == 6 && a.pose_node >= 0;
  float pp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, pAp_[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float pr[6], pz[6], px[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (has_pose)
    for (int c = 0; c < 6; ++c) {
      pr[c] = a.r[6 * (int64_t)a.pose_node + c];
      pz[c] = a.z[6 * (int64_t)a.pose_node + c];
    }
  for (int it = 0; it < a.pcg_iters; ++it) {
    if (rz == 0.0) break;
    const float beta = it == 0 ? 0.f : (float)(rz / rz_prev);
    // Az, p = z + beta p, Ap = Az + beta Ap, p.Ap: kG lanes per block row, each lane a strided
    // subset of the row's blocks (a block = B float4-aligned rows of H, loaded as float4), the
    // B partial outputs summed over the kG lanes by shuffles, lane c < B finishing component c
    my = 0.0;
    {
      constexpr int kG = 8;
      const int lg = threadIdx.x & (kG - 1);
      const unsigned gmask = (kG == 32 ? 0xffffffffu : ((1u << kG) - 1u) << (threadIdx.x & 31 & ~(kG - 1)));
      const int64_t nrows = n6s / B;
      for (int64_t rb = tid / kG; rb < nrows; rb += nth / kG) {   // uniform within a lane group
        const bool on = true;
        const int row = (int)rb;
        float y[B];
#pragma unroll
        for (int i = 0; i < B; ++i) y[i] = 0.f;
        if (on) {
          for (int e = a.row_ptr[row] + lg; e < a.row_ptr[row + 1]; e += kG) {
            const float4* H4 = reinterpret_cast<const float4*>(a.Hval + BB * (int64_t)e);
            const float* zz = a.z + B * a.col[e];
            float zv[B];
#pragma unroll
            for (int b = 0; b < B; b += 2) {
              const float2 t = *reinterpret_cast<const float2*>(zz + b);
              zv[b] = t.x;
              zv[b + 1] = t.y;
            }
#pragma unroll
            for (int f = 0; f < BB / 4; ++f) {
              const float4 h = __ldg(H4 + f);
              const int i0 = (4 * f) / B, c0 = (4 * f) % B;   // B % 2 == 0: a float4 spans <= 2 rows
              const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + (c0 + u) / B, c = (c0 + u) % B;
                y[i] = fmaf(hv[u], zv[c], y[i]);
              }
            }
          }
        }
#pragma unroll
        for (int o = kG / 2; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < B; ++i) y[i] += __shfl_xor_sync(gmask, y[i], o, kG);
#pragma unroll
        for (int c0 = 0; c0 < B; c0 += kG) {   // lane lg finishes components lg, lg + kG, ... (B = 12 > kG)
          const int cc = c0 + lg;
          if (!on || cc >= B) continue;
          float yc = 0.f;
#pragma unroll
          for (int i = 0; i < B; ++i) yc = (i == cc) ? y[i] : yc;
          const int64_t q = B * (int64_t)row + cc;
          const float az = fmaf(a.lambda, a.z[q], yc);
          const float pn = fmaf(beta, a.p[q], a.z[q]);
          const float apn = fmaf(beta, a.Ap[q], az);
          a.p[q] = pn;
          a.Ap[q] = apn;
          my += (double)pn * (double)apn;
        }
      }
    }
    if (B == 6 && a.pose_node >= 0) {   // the pose row's blocks, one per thread, warp sums -> pose_y
      const int prow = a.pose_node, e0 = a.row_ptr[prow], e1 = a.row_ptr[prow + 1];
      float yp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int64_t e = e0 + tid; e < e1; e += nth) {
        const float4* H4 = reinterpret_cast<const float4*>(a.Hval + 36 * e);
        const float* zz = a.z + 6 * a.col[e];
        float zv[6];
#pragma unroll
        for (int b = 0; b < 6; b += 2) {
          const float2 t = *reinterpret_cast<const float2*>(zz + b);
          zv[b] = t.x;
          zv[b + 1] = t.y;
        }
#pragma unroll
        for (int f = 0; f < 9; ++f) {
          const float4 h = __ldg(H4 + f);
          const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) yp[(4 * f + u) / 6] = fmaf(hv[u], zv[(4 * f + u) % 6], yp[(4 * f + u) / 6]);
        }
      }
      if (e0 + (tid & ~31ll) < e1) {   // this warp holds pose blocks
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < 6; ++i) yp[i] += __shfl_xor_sync(0xffffffffu, yp[i], o);
        if (lane < 6) {
          float v = 0.f;
#pragma unroll
          for (int i = 0; i < 6; ++i) v = (i == lane) ? yp[i] : v;
          atomicAdd(pose_y + 6 * it + lane, (double)v);
        }
      }
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 1 + 2 * it, s);
    grid.sync();
    double pAp = a.dots[1 + 2 * it];
    if (has_pose) {   // the pose row: p = z + beta p, Ap = (H z)_pose + lambda z + beta Ap
      for (int c = 0; c < 6; ++c) {
        const float az = fmaf(a.lambda, pz[c], (float)pose_y[6 * it + c]);
        pp[c] = fmaf(beta, pp[c], pz[c]);
        pAp_[c] = fmaf(beta, pAp_[c], az);
        pAp += (double)pp[c] * (double)pAp_[c];
      }
    }
    if (!isfinite(pAp) || !isfinite(rz)) { nonfin = true; break; }   // MIS_E_NUMERIC below
    if (!(pAp > 0.0)) break;
    const float alpha = (float)(rz / pAp);
    my = 0.0;
    {   // x += alpha p, r -= alpha Ap, z = M r, r.z: kN lanes per node, lane lg owns components
        // lg, lg + kN (B = 12); the group's r is shared by shuffles for the 6x6 / 12x12 product
      constexpr int kN = 8;
      const int lg = threadIdx.x & (kN - 1);
      const unsigned gm = ((1u << kN) - 1u) << (threadIdx.x & 31 & ~(kN - 1));
      for (int64_t j = tid / kN; j < m; j += nth / kN) {   // uniform within a lane group
        if (has_pose && j == a.pose_node) continue;   // in registers (below)
        float rr[(B + kN - 1) / kN];
#pragma unroll
        for (int h = 0; h < (B + kN - 1) / kN; ++h) {
          const int c = lg + kN * h;
          rr[h] = 0.f;
          if (c < B) {
            const int64_t q = B * j + c;
            a.x[q] = fmaf(alpha, a.p[q], a.x[q]);
            rr[h] = fmaf(-alpha, a.Ap[q], a.r[q]);
            a.r[q] = rr[h];
          }
        }
        float rv[B];   // the node's whole r in every lane of the group
#pragma unroll
        for (int c = 0; c < B; ++c) rv[c] = __shfl_sync(gm, rr[c / kN], c % kN, kN);
#pragma unroll
        for (int h = 0; h < (B + kN - 1) / kN; ++h) {
          const int r = lg + kN * h;
          if (r < B) {
            const float2* Mi = reinterpret_cast<const float2*>(a.Minv + BB * j + B * r);
            float z = 0.f;
#pragma unroll
            for (int c = 0; c < B; c += 2) {
              const float2 mv = __ldg(Mi + c / 2);
              z = fmaf(mv.x, rv[c], z);
              z = fmaf(mv.y, rv[c + 1], z);
            }
            a.z[B * j + r] = z;
            my += (double)rr[h] * (double)z;   // rr[h] is component r of this lane
          }
        }
      }
      if (has_pose) {   // the pose: x += alpha p, r -= alpha Ap, z = M r (every thread, same values)
        const float* Mp = a.Minv + 36 * (int64_t)a.pose_node;
        for (int c = 0; c < 6; ++c) {
          px[c] = fmaf(alpha, pp[c], px[c]);
          pr[c] = fmaf(-alpha, pAp_[c], pr[c]);
        }
        double rzp = 0.0;
        for (int r = 0; r < 6; ++r) {
          float z = 0.f;
          for (int c = 0; c < 6; ++c) z = fmaf(__ldg(Mp + 6 * r + c), pr[c], z);
          pz[r] = z;
          rzp += (double)pr[r] * (double)z;
        }
        if (tid == 0) {
          for (int c = 0; c < 6; ++c) a.z[6 * (int64_t)a.pose_node + c] = pz[c];   // read after the barrier
          my += rzp;
        }
      }
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 2 + 2 * it, s);
    grid.sync();
    rz_prev = rz;
    rz = a.dots[2 + 2 * it];
  }
  if (tid == 0) a.rep_res[a.gn_it] = (float)(rz0 > 0 ? sqrt(fabs(rz / rz0)) : 0.0);
  if (has_pose && tid == 0)   // the pose's step (its finiteness checked here: others may read it stale)
    for (int c = 0; c < 6; ++c) {
      a.x[6 * (int64_t)a.pose_node + c] = px[c];
      if (a.do_update && !isfinite(px[c])) atomicOr(a.numeric_flag, 1);
    }
  if (!a.do_update) return;

  // ---- node update (fp64 master), rolled back as a whole on a non-finite step
  if (nonfin && tid == 0) atomicOr(a.numeric_flag, 1);
  for (int64_t j = tid; j < m; j += nth)
    for (int c = 0; c < B; ++c)
      if (!isfinite(a.x[B * j + c])) atomicOr(a.numeric_flag, 1);
  grid.sync();
  if (*a.numeric_flag) return;
  for (int64_t j = tid; j < m; j += nth) {
    if constexpr (B == 12) {   // NEXT-4 (A41): A_j += dA_j, t_j += dt_j
      for (int c = 0; c < 12; ++c) {
        const double v = a.nd.Rt64[12 * j + c] + (double)a.x[12 * j + c];
        a.nd.Rt64[12 * j + c] = v;
        a.nd.node32[16 * j + c] = (float)v;
      }
    } else {
      if (j == a.pose_node) pose_update(a.x + 6 * j, a.pose);   // A37
      else node_update(a.x + 6 * j, a.nd.Rt64 + 12 * j, a.nd.node32 + 16 * j);
    }
  }
}

// LM (MIS_F_LM) block-Jacobi inverse of the damped diagonal block: (H_jj with its diagonal times
// (1 + mu) + (lambda + guard) I)^-1, guard = 1e-9 tr / B of the damped block (A17), fp64 Gauss-Jordan
// (one thread per node; zeros if not positive definite)
template <int B>
__device__ void precond_block_lm(const float* Hjj, float lambda, double mu, float* Mi) {
  double A[B][2 * B];
  double tr = 0.0;
  for (int i = 0; i < B; ++i) tr += (double)Hjj[(B + 1) * i] * (1.0 + mu);
  const double guard = 1e-9 * tr / B;
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < B; ++j) {
      const double h = (double)Hjj[B * i + j];
      A[i][j] = i == j ? h * (1.0 + mu) + (double)lambda + guard : h;
      A[i][B + j] = i == j ? 1.0 : 0.0;
    }
  bool pd = true;
  for (int p = 0; p < B; ++p) {
    const double pv = A[p][p];
    if (!(pv > 0.0)) { pd = false; break; }
    const double ipv = 1.0 / pv;
    for (int q = 0; q < 2 * B; ++q) A[p][q] *= ipv;
    for (int i = 0; i < B; ++i) {
      if (i == p) continue;
      const double f = A[i][p];
      for (int q = 0; q < 2 * B; ++q) A[i][q] -= f * A[p][q];
    }
  }
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < B; ++j) Mi[B * i + j] = pd ? (float)A[i][B + j] : 0.f;
}

// ---- pipelined grid PCG (Ghysels & Vanroose 2014, as the cluster kernel): ONE grid barrier per
// iteration.  Per iteration every lane group of kG lanes owns a block row j: n_j = (A m)_j, then
//   z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p,
//   x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z,
// then m'_j = M_j w_j (the node's whole block in the group) and the partials of the next dots
// gamma = (r, u), delta = (w, u); the barrier completes the dots (fp64 atomics), alpha and beta follow
// on every thread (same values everywhere).  m is double-buffered by iteration parity.  The same
// Krylov iterates as the standard recurrence in exact arithmetic; the MIRROR early stops are
// gamma == r.z == 0 and delta - beta gamma / alpha_prev == p.A p <= 0.
// NEXT-2: the dense pose row (unknown pose_node) as an arrowhead: every thread keeps the pose's
// vector entries in registers and uses them for the pose column of every block row; the pose row's
// products n_pose are partial sums over all threads (fp64 slots per iteration), finished after
// the barrier identically by every thread.
// Planes of a.pv (B m floats each): 0 r, 1 u, 2 w, 3 z, 4 q, 5 s, 6 p, 7 m (even), 8 m (odd).
// POSE: compiled with the NEXT-2 arrowhead (its ~90 registers of replicated pose state are not
// carried by the plain kernel).  MINB: resident 256-thread CTAs per SM the registers are sized for --
// 2 (128 registers, a few spills, twice the loads in flight) for HBM-bound systems (C5: 3.4 vs
// 3.9 ms of PCG per step), else 1 (C4: 0.42 vs 0.51 ms)
template <int B, bool POSE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_solve_pipe(SolveArgs a) {
  constexpr int BB = B * B, kG = 8, H2 = (B + kG - 1) / kG;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int m = a.m;
  constexpr bool has_pose = B == 6 && POSE;
  const int pose = has_pose ? a.pose_node : -1;
  const int64_t nrows = has_pose ? pose : m;   // block rows of the row loop
  const int64_t BM = (int64_t)B * m;
  float* const R = a.pv;
  float* const U = a.pv + BM;
  float* const Wv = a.pv + 2 * BM;
  float* const Z = a.pv + 3 * BM;
  float* const Q = a.pv + 4 * BM;
  float* const S = a.pv + 5 * BM;
  float* const P = a.pv + 6 * BM;
  float* const Mb[2] = {a.pv + 7 * BM, a.pv + 8 * BM};
  double* const dots = a.dots;                        // [0, 2]: init gamma, delta; 2 + 2 it (+1): iteration it
  double* const pose_y = a.dots + 2 * a.pcg_iters + 8;   // 6 per pass (init: slot 0, iteration it: slot it + 1)
  const int lg = threadIdx.x & (kG - 1);
  const unsigned gm = ((1u << kG) - 1u) << (threadIdx.x & 31 & ~(kG - 1));
  const int lane = threadIdx.x & 31;

  // ---- Levenberg-Marquardt (MIS_F_LM, reading A29): every thread takes the same decision on the
  // trial whose energy the finalisation reported -- accept if first or strictly lower than the last
  // accepted -- then solves the trial's (accept) or the kept (reject) system, damped by mu H_cc on
  // every diagonal entry, from the trial or the restored kept state (the pose included, NEXT-2)
  const bool lm = a.lm != nullptr;
  bool lm_accept = true;
  double lm_mu = 0.0, lm_E = 0.0;
  int lm_src = 0;
  if (lm) {
    const double Et = a.rep_energy[5 * a.gn_it + 4];
    const LmDev st = *a.lm;
    lm_accept = a.gn_it == 0 || Et < st.E_acc;
    lm_mu = a.gn_it == 0 ? (double)a.lm_mu0 : (lm_accept ? 0.5 * st.mu : 10.0 * st.mu);
    lm_E = lm_accept ? Et : st.E_acc;
    lm_src = lm_accept ? 1 - st.acc_buf : st.acc_buf;
  }
  const float* const Hs = lm && lm_src == 1 ? a.Hval_alt : a.Hval;
  const float* const bs = lm && lm_src == 1 ? a.rhs_alt : a.rhs;
  if (tid < 8 * a.pcg_iters + 16) dots[tid] = 0.0;
  if (lm) {
    for (int64_t q = tid; q < 12 * (int64_t)m; q += nth) {   // the step's base state; Rt_acc: the kept one
      const int64_t j = q / 12;
      if (j == pose) {   // the pose (A37) is kept after the nodes' rows of Rt_acc
        const int c = (int)(q % 12);
        if (lm_accept) a.Rt_acc[12 * (int64_t)pose + c] = a.pose[c];
        else a.pose[c] = a.Rt_acc[12 * (int64_t)pose + c];
        continue;
      }
      if (lm_accept) {
        a.Rt_acc[q] = a.nd.Rt64[q];
      } else {
        const double v = a.Rt_acc[q];
        a.nd.Rt64[q] = v;
        a.nd.node32[16 * j + q % 12] = (float)v;
      }
    }
    for (int64_t j = tid; j < m; j += nth)
      precond_block_lm<B>(Hs + BB * (int64_t)a.diag_pos[j], a.lambda, lm_mu, a.Minv + BB * j);
  }
  grid.sync();
  if (lm && tid == 0) {   // every thread has read the LM state
    a.lm->mu = lm_mu;
    a.lm->E_acc = lm_E;
    a.lm->acc_buf = lm_src;
    a.rep_flags[a.gn_it] = lm_accept ? 1.0 : 0.0;
  }
  if (a.pcg_iters <= 0 && !a.do_update) return;
  const float mu_f = (float)lm_mu;   // the Marquardt term of element (j, c): mu H_jj[c][c] (0 without LM)

  // pose registers (NEXT-2)
  float xp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, rp[6], up[6], wp[6], zp[6], qp[6], sp[6], pp[6], mp[6];
  float Mp[36];
  float lamp[6] = {a.lambda, a.lambda, a.lambda, a.lambda, a.lambda, a.lambda};   // LM: lambda + mu H_pp[c][c]
  if (has_pose) {
    for (int q = 0; q < 36; ++q) Mp[q] = a.Minv[36 * (int64_t)pose + q];
    for (int c = 0; c < 6; ++c) rp[c] = bs[6 * (int64_t)pose + c];
    if (lm)
      for (int c = 0; c < 6; ++c)
        lamp[c] = (float)((double)a.lambda + lm_mu * (double)Hs[36 * (int64_t)a.diag_pos[pose] + 7 * c]);
    for (int r = 0; r < 6; ++r) {
      float v = 0.f;
      for (int c = 0; c < 6; ++c) v = fmaf(Mp[6 * r + c], rp[c], v);
      up[r] = v;
      zp[r] = qp[r] = sp[r] = pp[r] = 0.f;
    }
  }

  // ---- init 1: x = 0, r = b, u = M r (lane groups per node)
  for (int64_t j = tid / kG; j < nrows; j += nth / kG) {
    float rr[H2];
#pragma unroll
    for (int h = 0; h < H2; ++h) {
      const int c = lg + kG * h;
      rr[h] = 0.f;
      if (c < B) {
        const int64_t q = B * j + c;
        rr[h] = bs[q];
        a.x[q] = 0.f;
        R[q] = rr[h];
        Z[q] = 0.f; Q[q] = 0.f; S[q] = 0.f; P[q] = 0.f;
      }
    }
    float rv[B];
#pragma unroll
    for (int c = 0; c < B; ++c) rv[c] = __shfl_sync(gm, rr[c / kG], c % kG, kG);
#pragma unroll
    for (int h = 0; h < H2; ++h) {
      const int r = lg + kG * h;
      if (r < B) {
        const float2* Mi = reinterpret_cast<const float2*>(a.Minv + BB * j + B * r);
        float v = 0.f;
#pragma unroll
        for (int c = 0; c < B; c += 2) {
          const float2 mv = Mi[c / 2];
          v = fmaf(mv.x, rv[c], v);
          v = fmaf(mv.y, rv[c + 1], v);
        }
        U[B * j + r] = v;
      }
    }
  }
  grid.sync();

  // block row j of (A v): the kG lanes' strided blocks, summed by shuffles (all lanes get all B);
  // the pose column from the registers pv_pose
  auto block_fma = [&](const float4 (&hb)[BB / 4], const float (&zv)[B], float (&y)[B]) {
#pragma unroll
    for (int f = 0; f < BB / 4; ++f) {
      const int i0 = (4 * f) / B, c0 = (4 * f) % B;
      const float hv[4] = {hb[f].x, hb[f].y, hb[f].z, hb[f].w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + (c0 + u) / B, c = (c0 + u) % B;
        y[i] = fmaf(hv[u], zv[c], y[i]);
      }
    }
  };
  auto load_z = [&](const float* vsrc, const float* pv_pose, int cl, float (&zv)[B]) {
    if (B == 6 && cl == pose) {
#pragma unroll
      for (int b = 0; b < B; ++b) zv[b] = pv_pose[b % 6];
    } else {
      const float* zz = vsrc + B * (int64_t)cl;
#pragma unroll
      for (int b = 0; b < B; b += 2) {
        const float2 t = *reinterpret_cast<const float2*>(zz + b);
        zv[b] = t.x;
        zv[b + 1] = t.y;
      }
    }
  };
  auto row_product = [&](int64_t j, const float* vsrc, const float* pv_pose, float (&y)[B]) {
#pragma unroll
    for (int i = 0; i < B; ++i) y[i] = 0.f;
    int e = a.row_ptr[j] + lg;
    const int e_end = a.row_ptr[j + 1];
    if constexpr (B == 6) {   // two blocks per step: 18 float4 of H in flight per lane (HBM-bound sizes)
      for (; e + kG < e_end; e += 2 * kG) {
        const int c0 = a.col[e], c1 = a.col[e + kG];
        float4 h0[9], h1[9];
        const float4* H0 = reinterpret_cast<const float4*>(Hs + 36 * (int64_t)e);
        const float4* H1 = reinterpret_cast<const float4*>(Hs + 36 * (int64_t)(e + kG));
#pragma unroll
        for (int f = 0; f < 9; ++f) { h0[f] = __ldg(H0 + f); h1[f] = __ldg(H1 + f); }
        float z0[B], z1[B];
        load_z(vsrc, pv_pose, c0, z0);
        load_z(vsrc, pv_pose, c1, z1);
        block_fma(h0, z0, y);
        block_fma(h1, z1, y);
      }
    }
    for (; e < e_end; e += kG) {
      const float4* H4 = reinterpret_cast<const float4*>(Hs + BB * (int64_t)e);
      const int cl = a.col[e];
      float zv[B];
      if (B == 6 && cl == pose) {
#pragma unroll
        for (int b = 0; b < B; ++b) zv[b] = pv_pose[b % 6];
      } else {
        const float* zz = vsrc + B * (int64_t)cl;
#pragma unroll
        for (int b = 0; b < B; b += 2) {
          const float2 t = *reinterpret_cast<const float2*>(zz + b);
          zv[b] = t.x;
          zv[b + 1] = t.y;
        }
      }
#pragma unroll
      for (int f = 0; f < BB / 4; ++f) {
        const float4 h = __ldg(H4 + f);
        const int i0 = (4 * f) / B, c0 = (4 * f) % B;
        const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + (c0 + u) / B, c = (c0 + u) % B;
          y[i] = fmaf(hv[u], zv[c], y[i]);
        }
      }
    }
#pragma unroll
    for (int o = kG / 2; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < B; ++i) y[i] += __shfl_xor_sync(gm, y[i], o, kG);
  };
  // the pose row's products over all threads -> slot (6 fp64)
  auto pose_row = [&](const float* vsrc, const float* pv_pose, double* slot) {
    if (!has_pose) return;
    const int e0 = a.row_ptr[pose], e1 = a.row_ptr[pose + 1];
    float yp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int64_t e = e0 + tid; e < e1; e += nth) {
      const float4* H4 = reinterpret_cast<const float4*>(Hs + 36 * e);
      const int cl = a.col[e];
      float zv[6];
      for (int b = 0; b < 6; ++b) zv[b] = cl == pose ? pv_pose[b] : vsrc[6 * (int64_t)cl + b];
#pragma unroll
      for (int f = 0; f < 9; ++f) {
        const float4 h = __ldg(H4 + f);
        const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) yp[(4 * f + u) / 6] = fmaf(hv[u], zv[(4 * f + u) % 6], yp[(4 * f + u) / 6]);
      }
    }
    if (e0 + (tid & ~31ll) < e1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 6; ++i) yp[i] += __shfl_xor_sync(0xffffffffu, yp[i], o);
      if (lane < 6) {
        float v = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) v = (i == lane) ? yp[i] : v;
        atomicAdd(slot + lane, (double)v);
      }
    }
  };
  // m'_j = M_j w_j for the group's node (w components wv[h] of this lane) -> dst; returns nothing
  auto precond_row = [&](int64_t j, const float (&wv)[H2], float* dst) {
    float wa[B];
#pragma unroll
    for (int c = 0; c < B; ++c) wa[c] = __shfl_sync(gm, wv[c / kG], c % kG, kG);
#pragma unroll
    for (int h = 0; h < H2; ++h) {
      const int r = lg + kG * h;
      if (r < B) {
        const float2* Mi = reinterpret_cast<const float2*>(a.Minv + BB * j + B * r);
        float v = 0.f;
#pragma unroll
        for (int c = 0; c < B; c += 2) {
          const float2 mv = Mi[c / 2];
          v = fmaf(mv.x, wa[c], v);
          v = fmaf(mv.y, wa[c + 1], v);
        }
        dst[B * j + r] = v;
      }
    }
  };

  // ---- init 2: w = A u, m = M w (parity 0), gamma0 = (r, u), delta0 = (w, u)
  double dg = 0.0, dd = 0.0;
  for (int64_t j = tid / kG; j < nrows; j += nth / kG) {
    float y[B];
    row_product(j, U, up, y);
    float wv[H2];
#pragma unroll
    for (int h = 0; h < H2; ++h) {
      const int c = lg + kG * h;
      wv[h] = 0.f;
      if (c < B) {
        float yc = 0.f;
#pragma unroll
        for (int i = 0; i < B; ++i) yc = (i == c) ? y[i] : yc;
        const int64_t q = B * j + c;
        const float uq = U[q];
        const float lamc = lm ? (float)((double)a.lambda + lm_mu * (double)Hs[BB * (int64_t)a.diag_pos[j] + (B + 1) * c])
                              : a.lambda;
        wv[h] = fmaf(lamc, uq, yc);
        Wv[q] = wv[h];
        dg += (double)R[q] * (double)uq;
        dd += (double)wv[h] * (double)uq;
      }
    }
    precond_row(j, wv, Mb[0]);
  }
  pose_row(U, up, pose_y);
  {
    const double s1 = block_sum(dg, sh), s2 = block_sum(dd, sh);
    if (threadIdx.x == 0) { atomicAdd(dots + 0, s1); atomicAdd(dots + 1, s2); }
  }
  grid.sync();
  double g = dots[0], d = dots[1];
  if (has_pose) {
    for (int c = 0; c < 6; ++c) wp[c] = fmaf(lamp[c], up[c], (float)pose_y[c]);
    for (int r = 0; r < 6; ++r) {
      float v = 0.f;
      for (int c = 0; c < 6; ++c) v = fmaf(Mp[6 * r + c], wp[c], v);
      mp[r] = v;
    }
    for (int c = 0; c < 6; ++c) {
      g += (double)rp[c] * (double)up[c];
      d += (double)wp[c] * (double)up[c];
    }
  }
  const double g0 = g;
  double gprev = 1.0, aprev_den = 1.0;
  bool nonfin = false;
  for (int it = 0; it < a.pcg_iters; ++it) {
    if (!isfinite(g) || !isfinite(d)) { nonfin = true; break; }   // MIS_E_NUMERIC below
    if (g == 0.0) break;
    const double beta = it == 0 ? 0.0 : g / gprev;
    const double den = it == 0 ? d : d - beta * g * (aprev_den / gprev);
    if (!(den > 0.0)) break;
    const float fa = (float)(g / den), fb = (float)beta;
    const float* Mc = Mb[it & 1];
    float* Mn = Mb[(it + 1) & 1];
    double* slot = pose_y + 6 * (it + 1);
    dg = 0.0;
    dd = 0.0;
    for (int64_t j = tid / kG; j < nrows; j += nth / kG) {
      float y[B];
      row_product(j, Mc, mp, y);
      float wv[H2];
#pragma unroll
      for (int h = 0; h < H2; ++h) {
        const int c = lg + kG * h;
        wv[h] = 0.f;
        if (c < B) {
          float yc = 0.f;
#pragma unroll
          for (int i = 0; i < B; ++i) yc = (i == c) ? y[i] : yc;
          const int64_t q = B * j + c;
          const float mq = Mc[q];
          const float lamc = lm ? (float)((double)a.lambda + lm_mu * (double)Hs[BB * (int64_t)a.diag_pos[j] + (B + 1) * c])
                                : a.lambda;
          const float n = fmaf(lamc, mq, yc);
          const float zn = fmaf(fb, Z[q], n), qn = fmaf(fb, Q[q], mq), sn = fmaf(fb, S[q], Wv[q]);
          const float pn = fmaf(fb, P[q], U[q]);
          const float xn = fmaf(fa, pn, a.x[q]), rn = fmaf(-fa, sn, R[q]), un = fmaf(-fa, qn, U[q]);
          const float wn = fmaf(-fa, zn, Wv[q]);
          Z[q] = zn; Q[q] = qn; S[q] = sn; P[q] = pn; a.x[q] = xn; R[q] = rn; U[q] = un; Wv[q] = wn;
          wv[h] = wn;
          dg += (double)rn * (double)un;
          dd += (double)wn * (double)un;
        }
      }
      precond_row(j, wv, Mn);
    }
    pose_row(Mc, mp, slot);
    {
      const double s1 = block_sum(dg, sh), s2 = block_sum(dd, sh);
      if (threadIdx.x == 0) { atomicAdd(dots + 2 + 2 * it, s1); atomicAdd(dots + 3 + 2 * it, s2); }
    }
    grid.sync();
    double gn = dots[2 + 2 * it], dn = dots[3 + 2 * it];
    if (has_pose) {   // the pose's entries, identically in every thread
      for (int c = 0; c < 6; ++c) {
        const float n = fmaf(lamp[c], mp[c], (float)slot[c]);
        zp[c] = fmaf(fb, zp[c], n);
        qp[c] = fmaf(fb, qp[c], mp[c]);
        sp[c] = fmaf(fb, sp[c], wp[c]);
        pp[c] = fmaf(fb, pp[c], up[c]);
        xp[c] = fmaf(fa, pp[c], xp[c]);
        rp[c] = fmaf(-fa, sp[c], rp[c]);
        up[c] = fmaf(-fa, qp[c], up[c]);
        wp[c] = fmaf(-fa, zp[c], wp[c]);
      }
      for (int r = 0; r < 6; ++r) {
        float v = 0.f;
        for (int c = 0; c < 6; ++c) v = fmaf(Mp[6 * r + c], wp[c], v);
        mp[r] = v;
      }
      for (int c = 0; c < 6; ++c) {
        gn += (double)rp[c] * (double)up[c];
        dn += (double)wp[c] * (double)up[c];
      }
    }
    gprev = g;
    aprev_den = den;
    g = gn;
    d = dn;
  }
  if (tid == 0) a.rep_res[a.gn_it] = (float)(g0 > 0 ? sqrt(fabs(g / g0)) : 0.0);
  if (has_pose && tid == 0)
    for (int c = 0; c < 6; ++c) {
      a.x[6 * (int64_t)pose + c] = xp[c];
      if (a.do_update && !isfinite(xp[c])) atomicOr(a.numeric_flag, 1);
    }
  if (!a.do_update) return;
  if (nonfin && tid == 0) atomicOr(a.numeric_flag, 1);
  for (int64_t j = tid; j < nrows; j += nth)
    for (int c = 0; c < B; ++c)
      if (!isfinite(a.x[B * j + c])) atomicOr(a.numeric_flag, 1);
  grid.sync();
  if (*a.numeric_flag) return;
  for (int64_t j = tid; j < m; j += nth) {
    if constexpr (B == 12) {   // NEXT-4 (A41): A_j += dA_j, t_j += dt_j
      for (int c = 0; c < 12; ++c) {
        const double v = a.nd.Rt64[12 * j + c] + (double)a.x[12 * j + c];
        a.nd.Rt64[12 * j + c] = v;
        a.nd.node32[16 * j + c] = (float)v;
      }
    } else {
      if (j == pose) pose_update(a.x + 6 * j, a.pose);   // A37
      else node_update(a.x + 6 * j, a.nd.Rt64 + 12 * j, a.nd.node32 + 16 * j);
    }
  }
}

cudaError_t launch_solve_grid(const SolveArgs& a, int num_sms, cudaStream_t s) {
  int per_sm = 1;
  // the pipelined recurrence (one grid barrier per iteration) unless MIS_F_STANDARD_PCG asks for
  // the textbook one (two barriers)
  const bool big = a.nnzb > 200000;   // H beyond ~30 MB: HBM-bound SpMV, more loads in flight pay
  const void* kern = a.pipelined ? (a.block == 12 ? (const void*)k_solve_pipe<12, false, 1>
                                    : a.pose_node >= 0 ? (const void*)k_solve_pipe<6, true, 1>
                                    : big ? (const void*)k_solve_pipe<6, false, 2>
                                          : (const void*)k_solve_pipe<6, false, 1>)
                                 : (a.block == 12 ? (const void*)k_solve<12> : (const void*)k_solve<6>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (void (*)(SolveArgs))kern, 256, 0);
  int64_t work = (int64_t)a.block * a.m;
  if (a.nnzb > work) work = a.nnzb;
  int64_t grid = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  static int per_sm_max = -1;   // CTAs per SM of the grid PCG (MIS_GRID_CTAS_PER_SM, default 2)
  if (per_sm_max < 0) {
    const char* e = getenv("MIS_GRID_CTAS_PER_SM");
    per_sm_max = e ? atoi(e) : 2;
    if (per_sm_max < 1) per_sm_max = 1;
  }
  if (grid > (int64_t)num_sms * per_sm_max) grid = (int64_t)num_sms * per_sm_max;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  SolveArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel(kern, dim3((unsigned)grid), dim3(256), params, 0, s);
}

cudaError_t launch_solve(const SolveArgs& a, int num_sms, cudaStream_t s) {
  if (a.cluster_size > 0) return launch_solve_cluster(a, s);
  return launch_solve_grid(a, num_sms, s);
}

}  // namespace mis
