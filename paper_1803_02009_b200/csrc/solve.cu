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
  // NEXT-2: the pose row (unknown pose_node = m - 1, ~m blocks) is summed by warps, not one thread
  const int64_t n6s = a.pose_node >= 0 ? B * (int64_t)a.pose_node : n6;
  const int64_t gwarp = tid >> 5;
  const int lane = threadIdx.x & 31;

  // ---- phase 0: H (both triangles) and b are final (record reduction); clear the dot slots
  if (tid < 2 * a.pcg_iters + 4) a.dots[tid] = 0.0;
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
  for (int it = 0; it < a.pcg_iters; ++it) {
    if (rz == 0.0) break;
    const float beta = it == 0 ? 0.f : (float)(rz / rz_prev);
    // Az, p = z + beta p, Ap = Az + beta Ap, p.Ap
    my = 0.0;
    for (int64_t q = tid; q < n6s; q += nth) {
      const int row = (int)(q / B), c = (int)(q % B);
      float az = a.lambda * a.z[q];
      for (int e = a.row_ptr[row]; e < a.row_ptr[row + 1]; ++e) {
        const float* Hb = a.Hval + BB * (int64_t)e + B * c;
        const float* zz = a.z + B * a.col[e];
#pragma unroll
        for (int b = 0; b < B; ++b) az = fmaf(Hb[b], zz[b], az);
      }
      const float pn = fmaf(beta, a.p[q], a.z[q]);
      const float apn = fmaf(beta, a.Ap[q], az);
      a.p[q] = pn;
      a.Ap[q] = apn;
      my += (double)pn * (double)apn;
    }
    if (B == 6 && a.pose_node >= 0 && gwarp < 6) {   // NEXT-2: the dense pose row, one warp per component
      const int row = a.pose_node, c = (int)gwarp;
      const int64_t q = 6 * (int64_t)row + c;
      float az = 0.f;
      for (int e = a.row_ptr[row] + lane; e < a.row_ptr[row + 1]; e += 32) {
        const float* Hb = a.Hval + 36 * (int64_t)e + 6 * c;
        const float* zz = a.z + 6 * a.col[e];
#pragma unroll
        for (int b = 0; b < 6; ++b) az = fmaf(Hb[b], zz[b], az);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) az += __shfl_xor_sync(0xffffffffu, az, o);
      if (lane == 0) {
        az = fmaf(a.lambda, a.z[q], az);
        const float pn = fmaf(beta, a.p[q], a.z[q]);
        const float apn = fmaf(beta, a.Ap[q], az);
        a.p[q] = pn;
        a.Ap[q] = apn;
        my += (double)pn * (double)apn;
      }
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 1 + 2 * it, s);
    grid.sync();
    const double pAp = a.dots[1 + 2 * it];
    if (!isfinite(pAp) || !isfinite(rz)) { nonfin = true; break; }   // MIS_E_NUMERIC below
    if (!(pAp > 0.0)) break;
    const float alpha = (float)(rz / pAp);
    my = 0.0;
    for (int64_t j = tid; j < m; j += nth) {
      float rr[B];
      for (int c = 0; c < B; ++c) {
        const int64_t q = B * j + c;
        a.x[q] = fmaf(alpha, a.p[q], a.x[q]);
        rr[c] = fmaf(-alpha, a.Ap[q], a.r[q]);
        a.r[q] = rr[c];
      }
      const float* Mi = a.Minv + BB * j;
      for (int r = 0; r < B; ++r) {
        float z = 0.f;
        for (int c = 0; c < B; ++c) z = fmaf(Mi[B * r + c], rr[c], z);
        a.z[B * j + r] = z;
        my += (double)rr[r] * (double)z;
      }
    }
    s = block_sum(my, sh);
    if (threadIdx.x == 0) atomicAdd(a.dots + 2 + 2 * it, s);
    grid.sync();
    rz_prev = rz;
    rz = a.dots[2 + 2 * it];
  }
  if (tid == 0) a.rep_res[a.gn_it] = (float)(rz0 > 0 ? sqrt(fabs(rz / rz0)) : 0.0);
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
  if (grid > num_sms) grid = num_sms;
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
