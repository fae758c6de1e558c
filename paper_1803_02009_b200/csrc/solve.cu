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
  if (tid < 8 * a.pcg_iters + 8) a.dots[tid] = 0.0;
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

cudaError_t launch_solve_grid(const SolveArgs& a, int num_sms, cudaStream_t s) {
  int per_sm = 1;
  const void* kern = a.block == 12 ? (const void*)k_solve<12> : (const void*)k_solve<6>;
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
