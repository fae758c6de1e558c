// pcg_cluster.cu -- K6-K8, cluster-resident variant.  One thread-block
// cluster (up to 16 CTAs, one per SM, 1024 threads each) owns the whole
// normal-equation system of a Gauss-Newton iteration: every CTA finalises the
// 6x6 blocks of its node rows straight from the K3/K4/K5 accumulators into its
// shared memory (the matrix never round-trips through global memory), builds
// its block-Jacobi preconditioner, and runs the P PCG iterations with
//   * the SpMV reading z of other CTAs through distributed shared memory,
//   * 2 cluster barriers per iteration (A p_{k+1} = A z_{k+1} + beta A p_k),
//   * dot products reduced per CTA and published to every CTA (DSMEM), summed
//     in rank order so every CTA sees bit-identical scalars,
// then updates its nodes (Exp(dtheta) R_j, t_j += dt, fp64).  Used whenever
// the system fits in the cluster's shared memory (C1-C3); the grid-wide
// cooperative kernel (solve.cu) handles larger ones.
#include <cooperative_groups.h>

#include <vector>

#include "solve_common.cuh"

namespace cg = cooperative_groups;

namespace mis {

constexpr int kCT = 1024;          // threads per CTA
constexpr int kMaxCluster = 16;

constexpr int kNVec = 10;         // local vectors (pipelined PCG needs 10, standard 6)

struct CLay {   // uniform shared-memory layout (identical offsets in every CTA)
  size_t dots, vec, zf, mi, col, own, h, total;
  __host__ __device__ CLay(int max_rows, int max_nnz, int m) {
    dots = 0;                                        // double partA..partE[16], red[32]
    vec = dots + sizeof(double) * (5 * kMaxCluster + 64);
    const size_t nv = (size_t)max_rows * 6;
    zf = vec + sizeof(float) * kNVec * nv;           // local vectors, then two replicated full vectors
    mi = zf + sizeof(float) * 2 * 6 * (size_t)m;
    col = mi + sizeof(float) * 36 * max_rows;
    own = col + sizeof(int) * max_nnz;
    h = (own + sizeof(int) * (max_nnz + 1) + 15) & ~(size_t)15;
    total = h + sizeof(float) * 36 * (size_t)max_nnz;
  }
};


// push this CTA's z slice into every CTA's full-length copy (remote stores,
// made visible by the following cluster barrier)
__device__ __forceinline__ void replicate(cg::cluster_group& cl, float* zf, const float* z, int r0, int nr, int cs) {
  const int n = 3 * nr;   // float2 units (6 r0 floats = 24 r0 bytes: 8-byte aligned)
  const float2* z2 = reinterpret_cast<const float2*>(z);
  for (int w = threadIdx.x; w < n * cs; w += kCT) {
    const int d = w / n, q = w - d * n;
    reinterpret_cast<float2*>(cl.map_shared_rank(zf, d) + 6 * r0)[q] = z2[q];
  }
}

// xor-butterfly sum: every lane ends with the bitwise-same value (IEEE + is commutative)
__device__ __forceinline__ double warp_sum_all(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA sum of v, published by warp 0 (lane c writes CTA c's slot[rank]); no serial loops
__device__ __forceinline__ void cta_publish(cg::cluster_group& cl, double v, double* red, double* slot, int rank,
                                            int cs) {
  v = warp_sum_all(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    const double x = warp_sum_all(red[l]);   // kCT / 32 == 32 warps
    if (l < cs) cl.map_shared_rank(slot, l)[rank] = x;
  }
}

// sum of the cs published partials, identical in every thread of every CTA
__device__ __forceinline__ double gather_sum(const double* slot, int cs) {
  const int l = threadIdx.x & 31;
  return warp_sum_all(l < cs ? slot[l] : 0.0);
}


// out = (H + lambda I) v for the CTA's rows; v read from the replicated full vector Z
__device__ __forceinline__ void spmv_local(const int* lrp, const int* col, const float* H, const float* Z,
                                           const float* v_local, float lambda, float* out, int nr) {
  const int n_items = 12 * nr;
  for (int base = 0; base < n_items; base += kCT) {
    const int item = base + threadIdx.x;
    const bool act = item < n_items;
    const int i = item / 12, c = (item % 12) >> 1, hf = item & 1;
    float v = 0.f;
    if (act)
      for (int k = lrp[i] + hf; k < lrp[i + 1]; k += 2) {
        const float* zr = Z + 6 * col[k];
        const float* h = H + 36 * (size_t)k + 6 * c;
#pragma unroll
        for (int b = 0; b < 6; ++b) v = fmaf(h[b], zr[b], v);
      }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    if (act && hf == 0) out[6 * i + c] = fmaf(lambda, v_local[6 * i + c], v);
  }
}

// Pipelined PCG (Ghysels & Vanroose 2014): the same Krylov iterates as PCG in
// exact arithmetic, with the two dot products of an iteration reduced together
// and overlapped with the preconditioner + replication of m = M w, so each
// iteration needs ONE cluster barrier:
//   gamma = (r, u), delta = (w, u), m = M w   [publish, replicate]   barrier
//   beta = gamma / gamma_prev, alpha = gamma / (delta - beta gamma / alpha_prev)
//   n = A m; z = n + beta z; q = m + beta q; s = w + beta s; p = u + beta p;
//   x += alpha p; r -= alpha s; u -= alpha q; w -= alpha z
// gamma == r.z and delta - beta gamma/alpha_prev == p.A p, so the oracle's
// MIRROR early stops (r.z == 0, p.Ap <= 0) are the same tests.
__device__ __forceinline__ void pcg_pipelined(const SolveArgs& a, cg::cluster_group& cl, unsigned char* sm,
                                              const CLay& L, int rank, int cs, int r0, int nr, const int* lrp,
                                              const int* col, const float* H, const float* Mi, double* g_last,
                                              double* g_first) {
  const int t = threadIdx.x, nv = a.max_rows * 6, n6 = 6 * nr;
  double* base = reinterpret_cast<double*>(sm + L.dots);
  double* gam[2] = {base, base + kMaxCluster};
  double* del[2] = {base + 3 * kMaxCluster, base + 4 * kMaxCluster};   // partF (= base + 2*16) stays free
  double* red = base + 5 * kMaxCluster;
  float* x = reinterpret_cast<float*>(sm + L.vec);
  float* r = x + nv;
  float* u = r + nv;
  float* w = u + nv;
  float* mm = w + nv;
  float* nn = mm + nv;
  float* zz = nn + nv;
  float* q = zz + nv;
  float* s = q + nv;
  float* p = s + nv;
  float* Z[2] = {reinterpret_cast<float*>(sm + L.zf), reinterpret_cast<float*>(sm + L.zf) + 6 * a.m};
  // u = M r; z = q = s = p = 0   (x = 0, r = b from phase 0)
  for (int e = t; e < n6; e += kCT) {
    const int i = e / 6, c = e - 6 * (e / 6);
    float v = 0.f;
    for (int b = 0; b < 6; ++b) v = fmaf(Mi[36 * i + 6 * c + b], r[6 * i + b], v);
    u[e] = v;
    zz[e] = 0.f; q[e] = 0.f; s[e] = 0.f; p[e] = 0.f;
  }
  __syncthreads();
  replicate(cl, Z[0], u, r0, nr, cs);
  cl.sync();
  spmv_local(lrp, col, H, Z[0], u, a.lambda, w, nr);   // w = A u
  __syncthreads();
  double gprev = 1.0, aprev = 1.0, g0 = 0.0, g = 0.0;
  for (int it = 0; it < a.pcg_iters; ++it) {
    double dg = 0.0, dd = 0.0;
    for (int e = t; e < n6; e += kCT) {
      const int i = e / 6, c = e - 6 * (e / 6);
      dg += (double)r[e] * (double)u[e];
      dd += (double)w[e] * (double)u[e];
      float v = 0.f;
      for (int b = 0; b < 6; ++b) v = fmaf(Mi[36 * i + 6 * c + b], w[6 * i + b], v);
      mm[e] = v;
    }
    __syncthreads();
    const int nb = (it + 1) & 1;
    replicate(cl, Z[nb], mm, r0, nr, cs);
    {   // both dots in one CTA reduction, published by warp 0 lanes (lane c -> CTA c)
      dg = warp_sum_all(dg);
      dd = warp_sum_all(dd);
      const int wi = t >> 5, l = t & 31;
      __syncthreads();
      if (l == 0) { red[wi] = dg; red[32 + wi] = dd; }
      __syncthreads();
      if (wi == 0) {
        const double sg = warp_sum_all(red[l]), sd = warp_sum_all(red[32 + l]);
        if (l < cs) {
          cl.map_shared_rank(gam[it & 1], l)[rank] = sg;
          cl.map_shared_rank(del[it & 1], l)[rank] = sd;
        }
      }
    }
    cl.sync();
    g = gather_sum(gam[it & 1], cs);
    const double d = gather_sum(del[it & 1], cs);
    if (it == 0) g0 = g;
    if (g == 0.0) break;
    const double beta = it == 0 ? 0.0 : g / gprev;
    const double den = it == 0 ? d : d - beta * g / aprev;
    if (!(den > 0.0)) break;
    const double alpha = g / den;
    spmv_local(lrp, col, H, Z[nb], mm, a.lambda, nn, nr);   // n = A m
    __syncthreads();
    const float fb = (float)beta, fa = (float)alpha;
    for (int e = t; e < n6; e += kCT) {
      zz[e] = fmaf(fb, zz[e], nn[e]);
      q[e] = fmaf(fb, q[e], mm[e]);
      s[e] = fmaf(fb, s[e], w[e]);
      p[e] = fmaf(fb, p[e], u[e]);
      x[e] = fmaf(fa, p[e], x[e]);
      r[e] = fmaf(-fa, s[e], r[e]);
      u[e] = fmaf(-fa, q[e], u[e]);
      w[e] = fmaf(-fa, zz[e], w[e]);
    }
    __syncthreads();
    gprev = g;
    aprev = alpha;
  }
  *g_last = g;
  *g_first = g0;
}

__global__ void __launch_bounds__(kCT, 1) k_pcg_cluster(SolveArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char sm[];
  const CLay L(a.max_rows, a.max_nnz, a.m);
  double* partA = reinterpret_cast<double*>(sm + L.dots);
  double* partB = partA + kMaxCluster;
  double* partF = partB + kMaxCluster;
  double* red = partF + 3 * kMaxCluster;   // partC, partD (pipelined PCG) sit between
  const int nv = a.max_rows * 6;
  float* x = reinterpret_cast<float*>(sm + L.vec);
  float* r = x + nv;
  float* z = r + nv;
  float* p = z + nv;
  float* Ap = p + nv;
  float* Az = Ap + nv;
  float* zf = reinterpret_cast<float*>(sm + L.zf);   // every CTA's copy of the full z
  float* Mi = reinterpret_cast<float*>(sm + L.mi);
  int* col = reinterpret_cast<int*>(sm + L.col);
  int* lrp = reinterpret_cast<int*>(sm + L.own);   // local row pointers (nr + 1)
  float* H = reinterpret_cast<float*>(sm + L.h);

  const int rank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  const int r0 = a.part[rank], r1 = a.part[rank + 1], nr = r1 - r0;
  const int e0 = a.row_ptr[r0], e1 = a.row_ptr[r1], ne = e1 - e0;
  const int t = threadIdx.x;
  const bool stamp = a.tstamp && t == 0;
  unsigned long long* ts = a.tstamp + 16 * rank;
  if (stamp) ts[0] = gtimer();

  // ---- phase 0: local rows of H (from the accumulators), b, column owners
  __shared__ int spart[kMaxCluster + 1];
  if (t <= cs) spart[t] = a.part[t];
  for (int i = t; i <= nr; i += kCT) lrp[i] = a.row_ptr[r0 + i] - e0;
  __syncthreads();
  {   // stream this CTA's rows of the final H (built by the record reduction) into shared memory
    const float4* src = reinterpret_cast<const float4*>(a.Hval + 36 * (int64_t)e0);
    float4* dst = reinterpret_cast<float4*>(H);
    for (int q = t; q < 9 * ne; q += kCT) dst[q] = src[q];
    for (int k = t; k < ne; k += kCT) col[k] = a.col[e0 + k];
  }
  for (int i = t; i < 6 * nr; i += kCT) {
    r[i] = a.rhs[6 * (int64_t)r0 + i];
    x[i] = 0.f;
    p[i] = 0.f;
    Ap[i] = 0.f;
  }
  __syncthreads();
  if (stamp) ts[1] = gtimer();
  if (a.pcg_iters <= 0 && !a.do_update) return;

  // ---- phase 1: block-Jacobi preconditioner, z = M r, r.z
  // M_j = (H_jj + (lambda + mu_j) I)^-1 in fp64 by Gauss-Jordan, 6 lanes per node
  // (one row each, pivot rows broadcast by shuffles), 5 nodes per warp.
  {
    const int wid = t >> 5, ln = t & 31, slot = ln / 6, rr = ln - 6 * slot;
    for (int base = 0; base < nr; base += 5 * (kCT / 32)) {
      const int i = base + 5 * wid + slot;
      const bool act = slot < 5 && i < nr;
      const float* Hd = H + 36 * (size_t)(act ? a.diag_pos[r0 + i] - e0 : 0);
      double row[12];
      double trc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) trc += act ? (double)Hd[7 * q] : 0.0;
      const double mu = 1e-9 * trc / 6.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        row[q] = act ? (double)Hd[6 * rr + q] + (q == rr ? (double)a.lambda + mu : 0.0) : (q == rr ? 1.0 : 0.0);
        row[6 + q] = (q == rr) ? 1.0 : 0.0;
      }
      bool pd = true;
      const int src0 = slot < 5 ? 6 * slot : 0;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const double pv = __shfl_sync(0xffffffffu, row[p], src0 + p);
        if (!(pv > 0.0)) pd = false;
        const double ipv = 1.0 / pv;
        const double f = row[p] * ipv;
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const double pq = __shfl_sync(0xffffffffu, row[q], src0 + p);
          row[q] = (rr == p) ? pq * ipv : row[q] - f * pq;
        }
      }
      if (act)
#pragma unroll
        for (int q = 0; q < 6; ++q) Mi[36 * i + 6 * rr + q] = pd ? (float)row[6 + q] : 0.f;
    }
  }
  __syncthreads();
  if (stamp) ts[2] = gtimer();
  double rz = 0.0, rz0 = 0.0;
  if (a.pipelined) {
    pcg_pipelined(a, cl, sm, L, rank, cs, r0, nr, lrp, col, H, Mi, &rz, &rz0);
    if (stamp) ts[3] = ts[2];
  } else {
  double my = 0.0;
  for (int q = t; q < 6 * nr; q += kCT) {
    const int i = q / 6, c = q % 6;
    float zz = 0.f;
    for (int b = 0; b < 6; ++b) zz = fmaf(Mi[36 * i + 6 * c + b], r[6 * i + b], zz);
    z[q] = zz;
    my += (double)r[q] * (double)zz;
  }
  __syncthreads();
  replicate(cl, zf, z, r0, nr, cs);
  if (stamp) ts[6] = gtimer();
  cta_publish(cl, my, red, partA, rank, cs);
  if (stamp) ts[7] = gtimer();
  cl.sync();
  rz = gather_sum(partA, cs);
  double rz_prev = 1.0;
  rz0 = rz;
  if (stamp) ts[3] = gtimer();
  int done = 0;
  const int n_items = 12 * nr, passes = (n_items + kCT - 1) / kCT;
  for (int it = 0; it < a.pcg_iters && !done; ++it) {
    if (rz == 0.0) break;
    const bool st1 = stamp && it == 1;
    if (st1) ts[8] = gtimer();
    const float beta = it == 0 ? 0.f : (float)(rz / rz_prev);
    // Az = (H + lambda I) z: two threads per (row, component) split the row's blocks,
    // reading the replicated z from local shared memory, pair-reduced by shuffle
    for (int ps = 0; ps < passes; ++ps) {
      const int item = t + ps * kCT;
      const bool act = item < n_items;
      const int i = item / 12, c = (item % 12) >> 1, hf = item & 1;
      float v = 0.f;
      if (act) {
        for (int k = lrp[i] + hf; k < lrp[i + 1]; k += 2) {
          const float* zr = zf + 6 * col[k];
          const float* h = H + 36 * (size_t)k + 6 * c;
#pragma unroll
          for (int b = 0; b < 6; ++b) v = fmaf(h[b], zr[b], v);
        }
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (act && hf == 0) Az[6 * i + c] = fmaf(a.lambda, z[6 * i + c], v);
    }
    __syncthreads();
    if (st1) ts[9] = gtimer();
    my = 0.0;
    for (int q = t; q < 6 * nr; q += kCT) {
      const float pn = fmaf(beta, p[q], z[q]);
      const float apn = fmaf(beta, Ap[q], Az[q]);
      p[q] = pn;
      Ap[q] = apn;
      my += (double)pn * (double)apn;
    }
    cta_publish(cl, my, red, partB, rank, cs);
    if (st1) ts[10] = gtimer();
    cl.sync();   // (B) p.Ap known everywhere; every CTA is done reading z
    if (st1) ts[11] = gtimer();
    const double pAp = gather_sum(partB, cs);
    if (!(pAp > 0.0)) { done = 1; break; }
    const float alpha = (float)(rz / pAp);
    for (int q = t; q < 6 * nr; q += kCT) {
      x[q] = fmaf(alpha, p[q], x[q]);
      r[q] = fmaf(-alpha, Ap[q], r[q]);
    }
    __syncthreads();
    my = 0.0;
    for (int q = t; q < 6 * nr; q += kCT) {
      const int i = q / 6, c = q % 6;
      float zz = 0.f;
      for (int b = 0; b < 6; ++b) zz = fmaf(Mi[36 * i + 6 * c + b], r[6 * i + b], zz);
      z[q] = zz;
      my += (double)r[q] * (double)zz;
    }
    __syncthreads();
    if (st1) ts[12] = gtimer();
    replicate(cl, zf, z, r0, nr, cs);
    cta_publish(cl, my, red, partA, rank, cs);
    if (st1) ts[13] = gtimer();
    cl.sync();   // (A) r.z known everywhere; z complete and replicated
    if (st1) ts[14] = gtimer();
    rz_prev = rz;
    rz = gather_sum(partA, cs);
  }
  }   // standard PCG
  if (stamp) ts[4] = gtimer();
  if (rank == 0 && t == 0) a.rep_res[a.gn_it] = (float)(rz0 > 0 ? sqrt(fabs(rz / rz0)) : 0.0);
  if (a.write_global)
    for (int q = t; q < 6 * nr; q += kCT) a.x[6 * (int64_t)r0 + q] = x[q];
  if (!a.do_update) {
    cl.sync();   // no CTA may exit while others still read its shared memory
    return;
  }
  // ---- node update; a non-finite step anywhere rolls the whole update back
  double bad = 0.0;
  for (int q = t; q < 6 * nr; q += kCT)
    if (!isfinite(x[q])) bad = 1.0;
  cta_publish(cl, bad, red, partF, rank, cs);
  cl.sync();
  if (gather_sum(partF, cs) != 0.0) {
    if (rank == 0 && t == 0) atomicOr(a.numeric_flag, 1);
    return;
  }
  if (*a.numeric_flag) return;   // sticky from an earlier iteration
  for (int i = t; i < nr; i += kCT) {
    const int j = r0 + i;
    node_update(x + 6 * i, a.nd.Rt64 + 12 * (int64_t)j, a.nd.node32 + 16 * (int64_t)j);
  }
  if (stamp) ts[5] = gtimer();
}

// The plan on the device (one warp; lane c binary-searches boundary c), so the
// host never reads the row structure back.  Same rule as plan_cluster.
__global__ void k_plan_cluster(const int32_t* row_ptr, int m, int max_cluster, PlanOut* out, int32_t* part) {
  __shared__ int32_t b[kMaxCluster + 1];
  int cs = max_cluster < m ? max_cluster : m;
  if (cs > kMaxCluster) cs = kMaxCluster;
  const int lane = threadIdx.x;
  const int64_t nnz = row_ptr[m];
  if (lane > 0 && lane < cs) {
    const int64_t target = (nnz * lane) / cs;
    int lo = 0, hi = m;   // first row with row_ptr[row] >= target
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (row_ptr[mid] < target) lo = mid + 1; else hi = mid;
    }
    b[lane] = lo;
  }
  __syncwarp();
  if (lane != 0) return;
  b[0] = 0;
  for (int c = 1; c < cs; ++c) {
    int row = b[c];
    if (row <= b[c - 1]) row = b[c - 1] + 1;
    if (row > m - (cs - c)) row = m - (cs - c);
    b[c] = row;
  }
  b[cs] = m;
  int mr = 0, mn = 0;
  for (int c = 0; c < cs; ++c) {
    const int nr = b[c + 1] - b[c];
    const int nz = row_ptr[b[c + 1]] - row_ptr[b[c]];
    mr = nr > mr ? nr : mr;
    mn = nz > mn ? nz : mn;
  }
  const CLay L(mr, mn, m);
  const bool fits = cs >= 1 && L.total <= 226 * 1024;   // 227 KB per CTA minus the static shared memory
  out->cl_size = fits ? cs : 0;
  out->max_rows = mr;
  out->max_nnz = mn;
  out->smem = (int64_t)L.total;
  for (int c = 0; c <= cs; ++c) part[c] = b[c];
}

void launch_plan_cluster(const int32_t* row_ptr, int m, int max_cluster, PlanOut* out, int32_t* part, cudaStream_t s) {
  k_plan_cluster<<<1, 32, 0, s>>>(row_ptr, m, max_cluster, out, part);
}

cudaError_t launch_solve_cluster(const SolveArgs& a, cudaStream_t s) {
  static size_t smem_set = 0;
  static bool nonportable = false;
  cudaError_t e;
  if (!nonportable) {
    if ((e = cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return e;
    nonportable = true;
  }
  if (a.smem_bytes > smem_set) {
    if ((e = cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem_bytes)) !=
        cudaSuccess)
      return e;
    smem_set = a.smem_bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.cluster_size);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = a.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)a.cluster_size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_pcg_cluster, a);
}

}  // namespace mis
