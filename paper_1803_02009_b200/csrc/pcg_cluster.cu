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

#ifndef MIS_PCG_THREADS
#define MIS_PCG_THREADS 512
#endif
constexpr int kCT = MIS_PCG_THREADS;   // threads per CTA
constexpr int kWarps = kCT / 32;
constexpr int kMaxCluster = 16;

constexpr int kNVec = 10;         // local vectors (pipelined PCG needs 10, standard 6)

constexpr int kPiece = 4;         // SpMV work unit: <= kPiece consecutive blocks of one row

__host__ __device__ inline int max_pieces(int max_rows, int max_nnz) { return max_nnz / kPiece + max_rows + 1; }

struct CLay {   // uniform shared-memory layout (identical offsets in every CTA)
  size_t dots, vec, zf, mi, col, own, pptr, pc, part, push, rt, h, total;
  __host__ __device__ CLay(int max_rows, int max_nnz, int m) {
    dots = 0;                                        // double partA..partE[16], red[64]
    vec = dots + sizeof(double) * (5 * kMaxCluster + 64);
    const size_t nv = (size_t)max_rows * 6;
    zf = vec + sizeof(float) * kNVec * nv;           // local vectors, then two replicated full vectors
    mi = zf + sizeof(float) * 2 * 6 * (size_t)m;
    col = mi + sizeof(float) * 36 * max_rows;
    own = col + sizeof(int) * max_nnz;               // local row pointers (nr + 1)
    pptr = own + sizeof(int) * (max_rows + 1);       // first SpMV piece of each local row (nr + 1)
    pc = pptr + sizeof(int) * (max_rows + 1);        // pieces: first block | count << 24
    part = pc + sizeof(int) * max_pieces(max_rows, max_nnz);   // 6 partial sums per piece
    push = part + sizeof(float) * 6 * max_pieces(max_rows, max_nnz);   // (destination CTA << 16 | local row)
    rt = (push + sizeof(int) * (size_t)max_rows * kMaxCluster + 15) & ~(size_t)15;   // own nodes' fp64 state
    h = rt + sizeof(double) * 12 * (size_t)max_rows;
    total = h + sizeof(float) * 36 * (size_t)max_nnz;
  }
};

// ---- per-frame preparation (the pattern and the partition are fixed for the
// frame's G Gauss-Newton iterations): SpMV pieces and halo push lists of every
// cluster rank, in global memory; each PCG launch only copies its rank's lists.
// Global layout (rank r): pptr [r * (max_rows + 1)], pieces [r * max_pieces],
// push [r * max_rows * 16], npush [r].
struct PcgLists {
  int32_t *pptr, *pc, *push, *npush;   // npush[16] | nin[16]: halo rows each rank receives from the others
  uint32_t* mask;   // m: ranks that read each row (zero outside the prep kernels)
};

// every rank marks the rows its blocks read in other ranks' ranges
__global__ void k_pcg_mark(const int32_t* row_ptr, const int32_t* col, const int32_t* part, PcgLists L) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int rank = blockIdx.x, r0 = part[rank], r1 = part[rank + 1];
  if (rank == 0 && threadIdx.x < kMaxCluster) L.npush[kMaxCluster + threadIdx.x] = 0;   // nin, summed by k_pcg_lists
  for (int k = row_ptr[r0] + threadIdx.x; k < row_ptr[r1]; k += blockDim.x) {
    const int j = col[k];
    if (j < r0 || j >= r1) atomicOr(L.mask + j, 1u << rank);
  }
}

// per rank: the pieces (<= kPiece blocks of one row, row order then block order) so the
// SpMV's work units are balanced whatever the row lengths; the push list ((destination,
// row) pairs grouped by destination, itself included); the rows' marks are cleared
__global__ void k_pcg_lists(const int32_t* row_ptr, const int32_t* part, int cs, int max_rows, int max_pc, PcgLists L) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int rank = blockIdx.x, r0 = part[rank], nr = part[rank + 1] - r0, l = threadIdx.x;
  const int e0 = row_ptr[r0];
  int32_t* pptr = L.pptr + (int64_t)rank * (max_rows + 1);
  int32_t* pc = L.pc + (int64_t)rank * max_pc;
  int32_t* push = L.push + (int64_t)rank * max_rows * kMaxCluster;
  {   // one warp: lane-chunked exclusive scan of the per-row piece counts
    const int per = (nr + 31) / 32, i0 = l * per, i1 = min(nr, i0 + per);
    int s = 0;
    for (int i = i0; i < i1; ++i) s += (row_ptr[r0 + i + 1] - row_ptr[r0 + i] + kPiece - 1) / kPiece;
    int inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (l >= o) inc += v;
    }
    int run = inc - s;
    for (int i = i0; i < i1; ++i) {
      pptr[i] = run;
      const int a = row_ptr[r0 + i] - e0, b = row_ptr[r0 + i + 1] - e0;
      for (int k = a; k < b; k += kPiece) pc[run++] = k | (min(kPiece, b - k) << 24);
    }
    if (l == 31) pptr[nr] = inc;
  }
  // the rows' reader masks, loaded once (registers for the first 128 rows): the d loop below
  // would otherwise issue a dependent global load per (destination, 32 rows)
  uint32_t mreg[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) mreg[q] = (32 * q + l < nr) ? L.mask[r0 + 32 * q + l] : 0u;
  int n = 0;
  for (int d = 0; d < cs; ++d)
    for (int b = 0; b < nr; b += 32) {
      const int i = b + l;
      const uint32_t mk = b < 128 ? (b == 0 ? mreg[0] : b == 32 ? mreg[1] : b == 64 ? mreg[2] : mreg[3])
                                  : (i < nr ? L.mask[r0 + i] : 0u);
      const bool on = i < nr && (d == rank || ((mk >> d) & 1u));
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) push[n + __popc(bal & ((1u << l) - 1u))] = (d << 16) | i;
      n += __popc(bal);
      if (l == 0 && d != rank && bal) atomicAdd(L.npush + kMaxCluster + d, __popc(bal));
    }
  __syncwarp();
  for (int i = l; i < nr; i += 32) L.mask[r0 + i] = 0u;
  if (l == 0) L.npush[rank] = n;
}

// push the CTA's slice of a vector into the full-length copies of the CTAs
// whose rows read it (the halo lists of build_push; itself included), as
// 8-byte remote stores made visible by the following cluster barrier.  The
// node graph is spatially local, so this moves ~1/7 of a full replication
// (c3: 2.2k of 15k rows) -- DSMEM bandwidth (~20 B/clk/SM) is what it costs.
__device__ __forceinline__ void replicate(cg::cluster_group& cl, float* zf, const float* z, int r0, const int* push,
                                          int npush) {
  for (int w = threadIdx.x; w < 3 * npush; w += kCT) {
    const int e = push[w / 3], q = w - 3 * (w / 3), d = e >> 16, i = e & 0xffff;
    const float2 v = reinterpret_cast<const float2*>(z + 6 * i)[q];
    reinterpret_cast<float2*>(cl.map_shared_rank(zf, d) + 6 * (r0 + i))[q] = v;
  }
}

// Halo lists (once per solve): every CTA marks, in the owner's mask, the rows
// its blocks read (DSMEM atomicOr), then lists (destination, row) pairs grouped
// by destination.  Returns the list length (all threads).
__device__ __forceinline__ int build_push(cg::cluster_group& cl, unsigned* mask, int* push, const int* col, int ne,
                                          const int32_t* part, int rank, int cs, int r0, int nr) {
  __shared__ int s_part[kMaxCluster + 1], s_npush;
  if (threadIdx.x <= cs) s_part[threadIdx.x] = part[threadIdx.x];
  for (int i = threadIdx.x; i < nr; i += kCT) mask[i] = 1u << rank;
  cl.sync();   // masks initialised in every CTA
  for (int k = threadIdx.x; k < ne; k += kCT) {
    const int j = col[k];
    if (j >= r0 && j < r0 + nr) continue;
    int o = 0;
    while (s_part[o + 1] <= j) ++o;
    atomicOr(cl.map_shared_rank(mask, o) + (j - s_part[o]), 1u << rank);
  }
  cl.sync();   // all marks landed
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    int n = 0;
    for (int d = 0; d < cs; ++d)
      for (int b = 0; b < nr; b += 32) {
        const int i = b + l;
        const bool on = i < nr && ((mask[i] >> d) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (on) push[n + __popc(bal & ((1u << l) - 1u))] = (d << 16) | i;
        n += __popc(bal);
      }
    if (l == 0) s_npush = n;
  }
  __syncthreads();
  return s_npush;
}

// ---- bulk (TMA) copies global -> shared memory completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: multiple of 16, both addresses 16-byte aligned; split in <= 32 KB copies
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  for (uint32_t o = 0; o < bytes; o += 32768u) {
    const uint32_t n = bytes - o < 32768u ? bytes - o : 32768u;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(static_cast<char*>(dst) + o)),
        "l"(static_cast<const char*>(src) + o), "r"(n), "r"(smem_u32(bar))
        : "memory");
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// remote (distributed shared memory) stores that complete_tx on the destination CTA's mbarrier
__device__ __forceinline__ uint32_t map_rank_u32(uint32_t local_smem, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_smem), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f2(uint32_t raddr, float2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
// bounded wait: a lost transfer traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (long long spin = 0; !ok; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (spin > (1ll << 26)) __trap();
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
    const double x = warp_sum_all(l < kWarps ? red[l] : 0.0);
    if (l < cs) cl.map_shared_rank(slot, l)[rank] = x;
  }
}

// sum of the 16 published partial slots (zero beyond the cluster size) in a fixed tree:
// identical in every thread of every CTA, no shuffles
__device__ __forceinline__ double gather_sum16(const double* slot) {
  const double2* s2 = reinterpret_cast<const double2*>(slot);
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = s2[k];
    a[k] = v.x + v.y;
  }
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// sum of the cs published partials, identical in every thread of every CTA
__device__ __forceinline__ double gather_sum(const double* slot, int cs) {
  const int l = threadIdx.x & 31;
  return warp_sum_all(l < cs ? slot[l] : 0.0);
}


// The SpMV's H operand lives in registers: thread t owns work units t, t + kCT,
// ..., t + (kU-1) kCT, each <= kPiece blocks x kCU block rows (half of each 6x6 block),
// loaded once per solve.  Streaming H from shared memory every iteration was
// bound by the shared-memory port (c3: 127 KB per CTA per SpMV at 128 B/clk);
// registers leave only the (broadcast) z loads, each shared by the unit's kCU rows.
// Units beyond kU kCT (larger systems) read H from shared memory.
#ifndef MIS_PCG_REG_UNITS
#define MIS_PCG_REG_UNITS 1
#endif
constexpr int kU = MIS_PCG_REG_UNITS;
constexpr int kCU = 3;   // block rows per unit: unit u = (piece u / 2, rows 3 (u % 2) .. + 2)
struct HReg {
  float h[kU][kPiece][kCU][6];
};

__device__ __forceinline__ void load_hreg(HReg& R, const int* pptr, const int* pc, const float* H, int nr) {
  const int units = 2 * pptr[nr];
#pragma unroll
  for (int j = 0; j < kU; ++j) {
    const int u = threadIdx.x + j * kCT;
    int k0 = 0, cnt = 0, c0 = 0;
    if (u < units) {
      const int w = pc[u >> 1];
      c0 = kCU * (u & 1);
      k0 = w & 0xffffff;
      cnt = w >> 24;
    }
#pragma unroll
    for (int b = 0; b < kPiece; ++b) {   // 8-byte loads: a block row is 6 contiguous floats at 24-byte offsets
#pragma unroll
      for (int r = 0; r < kCU; ++r) {
        const float2* h2 = reinterpret_cast<const float2*>(H + 36 * (size_t)(k0 + b) + 6 * (c0 + r));
        float2 v0 = make_float2(0.f, 0.f), v1 = v0, v2 = v0;
        if (b < cnt) { v0 = h2[0]; v1 = h2[1]; v2 = h2[2]; }
        R.h[j][b][r][0] = v0.x; R.h[j][b][r][1] = v0.y; R.h[j][b][r][2] = v1.x;
        R.h[j][b][r][3] = v1.y; R.h[j][b][r][4] = v2.x; R.h[j][b][r][5] = v2.y;
      }
    }
  }
}

// out = (H + lambda I) v for the CTA's rows; v read from the replicated full vector Z.
// Pass 1: one thread per (piece, half block row range) -- <= kPiece blocks, loads issued
// together (unrolled, predicated), each z row used by kCU rows; pass 2: per (row,
// component) the row's piece partials summed in piece order (deterministic).
__device__ __forceinline__ void spmv_local(const HReg& R, const int* pptr, const int* pc, float* part, const int* col,
                                           const float* H, const float* Z, const float* v_local, float lambda,
                                           float* out, int nr) {
  const int units = 2 * pptr[nr];
#pragma unroll
  for (int j = 0; j < kU; ++j) {
    const int u = threadIdx.x + j * kCT;
    if (u < units) {
      const int p = u >> 1, c0 = kCU * (u & 1), w = pc[p], k0 = w & 0xffffff, cnt = w >> 24;
      float v[kCU];
#pragma unroll
      for (int r = 0; r < kCU; ++r) v[r] = 0.f;
#pragma unroll
      for (int b = 0; b < kPiece; ++b) {
        if (b < cnt) {
          const float2* zr = reinterpret_cast<const float2*>(Z + 6 * col[k0 + b]);
          const float2 z0 = zr[0], z1 = zr[1], z2 = zr[2];
#pragma unroll
          for (int r = 0; r < kCU; ++r) {
            v[r] = fmaf(R.h[j][b][r][0], z0.x, v[r]);
            v[r] = fmaf(R.h[j][b][r][1], z0.y, v[r]);
            v[r] = fmaf(R.h[j][b][r][2], z1.x, v[r]);
            v[r] = fmaf(R.h[j][b][r][3], z1.y, v[r]);
            v[r] = fmaf(R.h[j][b][r][4], z2.x, v[r]);
            v[r] = fmaf(R.h[j][b][r][5], z2.y, v[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kCU; ++r) part[6 * p + c0 + r] = v[r];
    }
  }
  for (int u = threadIdx.x + kU * kCT; u < units; u += kCT) {
    const int p = u >> 1, c0 = kCU * (u & 1), w = pc[p], k0 = w & 0xffffff, cnt = w >> 24;
    float v[kCU];
#pragma unroll
    for (int r = 0; r < kCU; ++r) v[r] = 0.f;
#pragma unroll
    for (int b = 0; b < kPiece; ++b) {
      if (b < cnt) {
        const float2* zr = reinterpret_cast<const float2*>(Z + 6 * col[k0 + b]);
        const float2 z0 = zr[0], z1 = zr[1], z2 = zr[2];
#pragma unroll
        for (int r = 0; r < kCU; ++r) {
          const float2* h = reinterpret_cast<const float2*>(H + 36 * (size_t)(k0 + b) + 6 * (c0 + r));
          const float2 h0 = h[0], h1 = h[1], h2 = h[2];
          v[r] = fmaf(h0.x, z0.x, v[r]);
          v[r] = fmaf(h0.y, z0.y, v[r]);
          v[r] = fmaf(h1.x, z1.x, v[r]);
          v[r] = fmaf(h1.y, z1.y, v[r]);
          v[r] = fmaf(h2.x, z2.x, v[r]);
          v[r] = fmaf(h2.y, z2.y, v[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kCU; ++r) part[6 * p + c0 + r] = v[r];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 6 * nr; e += kCT) {
    const int i = e / 6, c = e - 6 * (e / 6);
    float v = 0.f;
    for (int p = pptr[i]; p < pptr[i + 1]; ++p) v += part[6 * p + c];
    out[e] = fmaf(lambda, v_local[e], v);
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
                                              double* g_first, unsigned long long* ts, const int* pptr,
                                              const int* pc, float* part, const int* push, int npush,
                                              const HReg& R) {
  const int t = threadIdx.x, nv = a.max_rows * 6, n6 = 6 * nr;
  double* base = reinterpret_cast<double*>(sm + L.dots);
  // double-buffered dot slots: gamma at base + (it & 1) * 16, delta at base + 48 + (it & 1) * 16
  // (partF = base + 32 stays free); selected arithmetically so they stay in shared space
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
  float* const Z0 = reinterpret_cast<float*>(sm + L.zf);   // two full-length buffers: Z0, Z0 + 6 m
  if (t < 5 * kMaxCluster) base[t] = 0.0;   // unused slots (>= cluster size) stay zero for gather_sum16
  // u = M r; z = q = s = p = 0   (x = 0, r = b from phase 0)
  for (int e = t; e < n6; e += kCT) {
    const int i = e / 6, c = e - 6 * (e / 6);
    float v = 0.f;
    for (int b = 0; b < 6; ++b) v = fmaf(Mi[36 * i + 6 * c + b], r[6 * i + b], v);
    u[e] = v;
    zz[e] = 0.f; q[e] = 0.f; s[e] = 0.f; p[e] = 0.f;
  }
  __syncthreads();
  replicate(cl, Z0, u, r0, push, npush);
  cl.sync();
  spmv_local(R, pptr, pc, part, col, H, Z0, u, a.lambda, w, nr);   // w = A u
  __syncthreads();
  double gprev = 1.0, aprev = 1.0, g0 = 0.0, g = 0.0;
  for (int it = 0; it < a.pcg_iters; ++it) {
    const bool st1 = ts && it == 1;   // sub-phase stamps of iteration 1 (slots 8-14, 15 = marker)
    if (st1) ts[8] = gtimer();
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
    if (st1) ts[9] = gtimer();
    float* const Zb = Z0 + ((it + 1) & 1) * 6 * a.m;
    double* const gam = base + (it & 1) * kMaxCluster;
    double* const del = base + 3 * kMaxCluster + (it & 1) * kMaxCluster;
    replicate(cl, Zb, mm, r0, push, npush);
    if (st1) ts[10] = gtimer();
    {   // both dots in one CTA reduction, published by warp 0 lanes (lane c -> CTA c)
      dg = warp_sum_all(dg);
      dd = warp_sum_all(dd);
      const int wi = t >> 5, l = t & 31;
      __syncthreads();
      if (l == 0) { red[wi] = dg; red[32 + wi] = dd; }
      __syncthreads();
      if (wi == 0) {
        const double sg = warp_sum_all(l < kWarps ? red[l] : 0.0), sd = warp_sum_all(l < kWarps ? red[32 + l] : 0.0);
        if (l < cs) {
          cl.map_shared_rank(gam, l)[rank] = sg;
          cl.map_shared_rank(del, l)[rank] = sd;
        }
      }
    }
    if (st1) ts[11] = gtimer();
    // split cluster barrier: the previous scalars' reciprocals are computed while it completes
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    double inv_gprev = 1.0 / gprev, inv_aprev = 1.0 / aprev;
    asm volatile("" : "+d"(inv_gprev), "+d"(inv_aprev));   // computed here, not after the wait
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (st1) ts[12] = gtimer();
    g = gather_sum16(gam);
    double d = gather_sum16(del);
    asm volatile("" : "+d"(g), "+d"(d));   // both sums before the early-exit test
    if (!isfinite(g) || !isfinite(d)) { g = NAN; break; }   // non-finite system: MIS_E_NUMERIC at the update
    if (it == 0) g0 = g;
    if (g == 0.0) break;
    const double beta = it == 0 ? 0.0 : g * inv_gprev;
    const double den = it == 0 ? d : d - beta * g * inv_aprev;
    if (!(den > 0.0)) break;
    const double alpha = g / den;
    if (st1) ts[6] = gtimer();
    spmv_local(R, pptr, pc, part, col, H, Zb, mm, a.lambda, nn, nr);   // n = A m
    __syncthreads();
    if (st1) ts[13] = gtimer();
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
    if (st1) { ts[14] = gtimer(); ts[15] = 1; }
    gprev = g;
    aprev = alpha;
  }
  *g_last = g;
  *g_first = g0;
}

// The same pipelined PCG with the CTA's vector slices in registers: thread t owns element t
// of its 6 nr rows (requires 6 max_rows <= kCT).  Only w (read by the 6x6 preconditioner
// products of its node), m (replicated / SpMV input) and n (SpMV output) pass through
// shared memory.
__device__ __forceinline__ void pcg_pipelined_reg(const SolveArgs& a, cg::cluster_group& cl, unsigned char* sm,
                                                  const CLay& L, int rank, int cs, int r0, int nr, const int* col,
                                                  const float* H, const float* Mi, double* g_last, double* g_first,
                                                  unsigned long long* ts, const int* pptr, const int* pc, float* part,
                                                  const int* push, int npush, const HReg& R, uint64_t* bars,
                                                  uint32_t in_bytes, float lam_t) {
  const int t = threadIdx.x, nv = a.max_rows * 6, n6 = 6 * nr;
  const bool own = t < n6;
  const int ti = t / 6, tc = t - 6 * (t / 6);
  double* base = reinterpret_cast<double*>(sm + L.dots);
  double* red = base + 5 * kMaxCluster;
  float* xs = reinterpret_cast<float*>(sm + L.vec);   // x (written back at the end), r (from phase 0)
  float* rs = xs + nv;
  float* us = rs + nv;
  float* ws = us + nv;
  float* ms = ws + nv;
  float* ns = ms + nv;
  float* const Z0 = reinterpret_cast<float*>(sm + L.zf);
  if (t < 5 * kMaxCluster) base[t] = 0.0;
  const float* Mrow = Mi + 36 * ti + 6 * tc;
  float x = 0.f, r = 0.f, u = 0.f, w = 0.f, zz = 0.f, q = 0.f, s = 0.f, p = 0.f;
  if (own) {   // u = M r
    r = rs[t];
    float v = 0.f;
#pragma unroll
    for (int b = 0; b < 6; ++b) v = fmaf(Mrow[b], rs[6 * ti + b], v);
    u = v;
    us[t] = v;
  }
  __syncthreads();
  replicate(cl, Z0, us, r0, push, npush);
  cl.sync();
  spmv_local(R, pptr, pc, part, col, H, Z0, us, lam_t, ws, nr);   // w = A u (own element: this thread's write)
  if (own) w = ws[t];
  __syncthreads();
  double gprev = 1.0, aprev_den = 1.0, g0 = 0.0, g = 0.0;
  for (int it = 0; it < a.pcg_iters; ++it) {
    const bool st1 = ts && it == 1;
    if (st1) ts[8] = gtimer();
    double dg = 0.0, dd = 0.0;
    if (own) {
      dg = (double)r * (double)u;
      dd = (double)w * (double)u;
      float v = 0.f;
#pragma unroll
      for (int b = 0; b < 6; ++b) v = fmaf(Mrow[b], ws[6 * ti + b], v);
      ms[t] = v;
    }
    __syncthreads();
    if (st1) ts[9] = gtimer();
    float* const Zb = Z0 + ((it + 1) & 1) * 6 * a.m;
    double* const gam = base + (it & 1) * kMaxCluster;
    double* const del = base + 3 * kMaxCluster + (it & 1) * kMaxCluster;
    // No cluster barrier in the loop: the halo rows of m and the dot partials travel as
    // st.async stores that complete_tx on the receiver's mbarrier of this iteration's parity,
    // whose expected byte count (incoming halo rows x 24 + 16 per other CTA) is armed by
    // the receiver itself.  Reuse of a buffer two iterations later is safe because every
    // CTA's next partials are sent only after it has finished reading that buffer.
    uint64_t* const bar = bars + (it & 1);
    const uint32_t bar_u = smem_u32(bar);
    if (t == 0) mbar_expect_tx(bar, in_bytes);
    {
      const uint32_t zb_u = smem_u32(Zb);
      for (int k = t; k < 3 * npush; k += kCT) {
        const int e = push[k / 3], qq = k - 3 * (k / 3), dst = e >> 16, i = e & 0xffff;
        const float2 v = reinterpret_cast<const float2*>(ms + 6 * i)[qq];
        // own rows too: every value read after the wait arrives through the mbarrier, so no
        // CTA barrier is needed after it
        st_async_f2(map_rank_u32(zb_u + 4u * (uint32_t)(6 * (r0 + i) + 2 * qq), dst), v, map_rank_u32(bar_u, dst));
      }
    }
    if (st1) ts[10] = gtimer();
    {
      dg = warp_sum_all(dg);
      dd = warp_sum_all(dd);
      const int wi = t >> 5, l = t & 31;
      if (l == 0) { red[wi] = dg; red[32 + wi] = dd; }
      __syncthreads();
      if (wi == 0) {
        const double sg = warp_sum_all(l < kWarps ? red[l] : 0.0), sd = warp_sum_all(l < kWarps ? red[32 + l] : 0.0);
        if (l < cs) {
          const uint32_t rb = map_rank_u32(bar_u, l);
          st_async_f64(map_rank_u32(smem_u32(gam + rank), l), sg, rb);
          st_async_f64(map_rank_u32(smem_u32(del + rank), l), sd, rb);
        }
      }
    }
    if (st1) ts[11] = gtimer();
    // reciprocals of the previous scalars (1 / alpha_prev = den_prev / g_prev) before the wait
    double inv_gprev = 1.0 / gprev, inv_aprev = aprev_den / gprev;
    asm volatile("" : "+d"(inv_gprev), "+d"(inv_aprev));
    mbar_wait_bounded(bar, (uint32_t)(it >> 1) & 1u);
    if (st1) ts[12] = gtimer();
    g = gather_sum16(gam);
    double d = gather_sum16(del);
    asm volatile("" : "+d"(g), "+d"(d));   // both sums before the early-exit test
    if (!isfinite(g) || !isfinite(d)) { g = NAN; break; }   // non-finite system: MIS_E_NUMERIC at the update
    if (it == 0) g0 = g;
    if (g == 0.0) break;
    const double beta = it == 0 ? 0.0 : g * inv_gprev;
    const double den = it == 0 ? d : d - beta * g * inv_aprev;
    if (!(den > 0.0)) break;
    // alpha only enters the fp32 vector updates: one fp32 division instead of an fp64 one
    const float fa = (float)g / (float)den;
    if (st1) ts[6] = gtimer();
    spmv_local(R, pptr, pc, part, col, H, Zb, ms, lam_t, ns, nr);   // n = A m (own element: this thread's write)
    if (st1) ts[13] = gtimer();
    const float fb = (float)beta;
    if (own) {
      const float n = ns[t], m = ms[t];
      zz = fmaf(fb, zz, n);
      q = fmaf(fb, q, m);
      s = fmaf(fb, s, w);
      p = fmaf(fb, p, u);
      x = fmaf(fa, p, x);
      r = fmaf(-fa, s, r);
      u = fmaf(-fa, q, u);
      w = fmaf(-fa, zz, w);
      ws[t] = w;
    }
    __syncthreads();
    if (st1) { ts[14] = gtimer(); ts[15] = 1; }
    gprev = g;
    aprev_den = den;
  }
  if (own) xs[t] = x;
  __syncthreads();
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
  int* pptr = reinterpret_cast<int*>(sm + L.pptr);
  int* pc = reinterpret_cast<int*>(sm + L.pc);
  float* part = reinterpret_cast<float*>(sm + L.part);
  int* push = reinterpret_cast<int*>(sm + L.push);
  float* H = reinterpret_cast<float*>(sm + L.h);
  __shared__ uint64_t tma_bar, pcg_bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&tma_bar, 1);
    mbar_init(pcg_bar, 1);       // the pipelined PCG's per-iteration exchanges (initialised before the
    mbar_init(pcg_bar + 1, 1);   // cluster barrier that precedes any remote arrival)
  }

  pdl_wait();      // H, b, M^-1 from the finalisation
  pdl_trigger();   // the next K3a may launch on the SMs this cluster leaves free (it waits for completion)
  const int rank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  const int r0 = a.part[rank], r1 = a.part[rank + 1], nr = r1 - r0;
  const int e0 = a.row_ptr[r0], e1 = a.row_ptr[r1], ne = e1 - e0;
  const int t = threadIdx.x;
  const bool stamp = a.tstamp && t == 0;
  unsigned long long* ts = a.tstamp + 16 * rank;
  if (stamp) ts[0] = gtimer();

  // ---- Levenberg-Marquardt (MIS_F_LM): every CTA takes the same decision on the trial whose
  // energy the finalisation just reported (accept if first or strictly lower than the last
  // accepted, reading A29) before rank 0 updates the state (after the PCG's first cluster
  // barrier): the system to solve is the trial's (accept) or the kept one (reject)
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
  const float* Hsys = lm && lm_src == 1 ? a.Hval_alt : a.Hval;
  const float* bsys = lm && lm_src == 1 ? a.rhs_alt : a.rhs;

  // ---- phase 0: the rank's rows of H, its block inverses and its nodes' fp64 states by bulk
  // copies (one thread issues them, completion on an mbarrier) while the other threads load
  // the lists of this rank (built once per frame), columns and b.  (LM: the inverses depend
  // on the damping decided here, so they are built below from the diagonal blocks.)
  const float* Hg = Hsys + 36 * (int64_t)e0;
  if (t == 0) {
    mbar_expect_tx(&tma_bar, (uint32_t)(144 * ne + (lm ? 0 : 144 * nr) + 96 * nr));
    bulk_g2s(H, Hg, (uint32_t)(144 * ne), &tma_bar);
    if (!lm) bulk_g2s(Mi, a.Minv + 36 * (int64_t)r0, (uint32_t)(144 * nr), &tma_bar);
    bulk_g2s(sm + L.rt, a.nd.Rt64 + 12 * (int64_t)r0, (uint32_t)(96 * nr), &tma_bar);
  }
  const int sticky = *a.numeric_flag;   // set by an earlier launch of this registration
  const int max_pc = max_pieces(a.max_rows, a.max_nnz);
  const int32_t* g_pptr = a.pptr + (int64_t)rank * (a.max_rows + 1);
  for (int i = t; i <= nr; i += kCT) pptr[i] = g_pptr[i];
  const int npush = a.npush[rank];
  const int32_t* g_push = a.push + (int64_t)rank * a.max_rows * kMaxCluster;
  for (int i = t; i < npush; i += kCT) push[i] = g_push[i];
  for (int k = t; k < ne; k += kCT) col[k] = a.col[e0 + k];
  for (int i = t; i < 6 * nr; i += kCT) {
    r[i] = bsys[6 * (int64_t)r0 + i];
    x[i] = 0.f;
    p[i] = 0.f;
    Ap[i] = 0.f;
  }
  __syncthreads();
  const int npc = pptr[nr];
  const int32_t* g_pc = a.pc + (int64_t)rank * max_pc;
  for (int i = t; i < npc; i += kCT) pc[i] = g_pc[i];
  __syncthreads();
  // H is staged in shared memory (the register units read 72-byte row groups that would
  // scatter global requests; units beyond the registers, for larger systems, read it there)
  mbar_wait(&tma_bar, 0);
  float lam_t = a.lambda;   // this thread's diagonal shift (register-resident variant: element t)
  if (lm) {
    double* rt = reinterpret_cast<double*>(sm + L.rt);
    // base state of the step: the trial (accepted: it becomes the kept state) or the kept one
    for (int q = t; q < 12 * nr; q += kCT) {
      if (lm_accept) a.Rt_acc[12 * (int64_t)r0 + q] = rt[q];
      else rt[q] = a.Rt_acc[12 * (int64_t)r0 + q];
    }
    // damped block-Jacobi inverses: (H_jj with its diagonal times (1 + mu) + (lambda + guard) I)^-1,
    // fp64 Gauss-Jordan, one 8-lane group per node (lane rr < 6 of the group holds row rr), so the
    // CTA's <= 64 nodes take one pass
    const int wi = t >> 5, l = t & 31, gl = l & 7, rr = gl < 6 ? gl : 0;
    for (int base = 4 * wi; base < nr; base += 4 * kWarps) {   // warp-uniform trip count (shuffles)
      const bool act = base + (l >> 3) < nr;
      const int i = act ? base + (l >> 3) : base;
      const int k0 = pc[pptr[i]] & 0xffffff, k1 = i + 1 < nr ? (pc[pptr[i + 1]] & 0xffffff) : ne;
      int kd = k0;
      for (int k = k0; k < k1; ++k)
        if (col[k] == r0 + i) kd = k;
      const float* B = H + 36 * kd;
      double row[12], trc = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) trc += (double)B[7 * q] * (1.0 + lm_mu);
      const double guard = 1e-9 * trc / 6.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double h = (double)B[6 * rr + q];
        row[q] = q == rr ? h * (1.0 + lm_mu) + (double)a.lambda + guard : h;
        row[6 + q] = q == rr ? 1.0 : 0.0;
      }
      bool pd = true;
#pragma unroll
      for (int pv_i = 0; pv_i < 6; ++pv_i) {
        const double pv = __shfl_sync(0xffffffffu, row[pv_i], pv_i, 8);
        if (!(pv > 0.0)) pd = false;
        const double ipv = 1.0 / pv, f = row[pv_i] * ipv;
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const double pq = __shfl_sync(0xffffffffu, row[q], pv_i, 8);
          row[q] = rr == pv_i ? pq * ipv : row[q] - f * pq;
        }
      }
      if (act && gl < 6)
#pragma unroll
        for (int q = 0; q < 6; ++q) Mi[36 * i + 6 * rr + q] = pd ? (float)row[6 + q] : 0.f;
    }
    if (t < 6 * nr) {   // the Marquardt term of element t: lambda + mu H_tt
      const int ti = t / 6, tc = t - 6 * ti;
      const int k0 = pc[pptr[ti]] & 0xffffff, k1 = ti + 1 < nr ? (pc[pptr[ti + 1]] & 0xffffff) : ne;
      int kd = k0;
      for (int k = k0; k < k1; ++k)
        if (col[k] == r0 + ti) kd = k;
      lam_t = (float)((double)a.lambda + lm_mu * (double)H[36 * kd + 7 * tc]);
    }
    __syncthreads();
  }
  if (stamp) ts[1] = gtimer();
  if (a.pcg_iters <= 0 && !a.do_update) return;
  HReg R;
  load_hreg(R, pptr, pc, H, nr);
  if (stamp) ts[2] = gtimer();
  double rz = 0.0, rz0 = 0.0;
  if (a.pipelined && 6 * a.max_rows <= kCT) {
    const uint32_t in_bytes = (uint32_t)(24 * (a.npush[kMaxCluster + rank] + nr) + 16 * cs);   // halo + own rows, dots
    pcg_pipelined_reg(a, cl, sm, L, rank, cs, r0, nr, col, H, Mi, &rz, &rz0, stamp ? ts : nullptr, pptr, pc, part, push,
                      npush, R, pcg_bar, in_bytes, lam_t);
    if (stamp) ts[3] = ts[2];
    if (lm && rank == 0 && t == 0) {   // every CTA has read the LM state (first cluster barrier passed)
      a.lm->mu = lm_mu;
      a.lm->E_acc = lm_E;
      a.lm->acc_buf = lm_src;
      a.rep_flags[a.gn_it] = lm_accept ? 1.0 : 0.0;
    }
  } else if (a.pipelined) {
    pcg_pipelined(a, cl, sm, L, rank, cs, r0, nr, lrp, col, H, Mi, &rz, &rz0, stamp ? ts : nullptr, pptr, pc, part, push,
                  npush, R);
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
  replicate(cl, zf, z, r0, push, npush);
  if (stamp) ts[6] = gtimer();
  cta_publish(cl, my, red, partA, rank, cs);
  if (stamp) ts[7] = gtimer();
  cl.sync();
  rz = gather_sum(partA, cs);
  double rz_prev = 1.0;
  rz0 = rz;
  if (stamp) ts[3] = gtimer();
  int done = 0;
  for (int it = 0; it < a.pcg_iters && !done; ++it) {
    if (rz == 0.0) break;
    const bool st1 = stamp && it == 1;
    if (st1) ts[8] = gtimer();
    const float beta = it == 0 ? 0.f : (float)(rz / rz_prev);
    spmv_local(R, pptr, pc, part, col, H, zf, z, a.lambda, Az, nr);   // Az = (H + lambda I) z
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
    if (!isfinite(pAp) || !isfinite(rz)) { rz = NAN; done = 1; break; }   // non-finite: MIS_E_NUMERIC below
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
    replicate(cl, zf, z, r0, push, npush);
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
  bool bad = !isfinite(rz);   // a PCG scalar went non-finite (identical in every CTA)
  for (int q = t; q < 6 * nr; q += kCT)
    if (!isfinite(x[q])) bad = true;
  const int bad_cta = __syncthreads_or(bad);
  int* bflag = reinterpret_cast<int*>(partF);   // one int per CTA
  if (t < cs) cl.map_shared_rank(bflag, t)[rank] = bad_cta;
  cl.sync();
  const bool any_bad = __any_sync(0xffffffffu, (t & 31) < cs && bflag[t & 31] != 0);
  if (any_bad) {
    if (rank == 0 && t == 0) atomicOr(a.numeric_flag, 1);
    return;
  }
  if (sticky) return;   // a numeric failure earlier in this registration
  const double* rt = reinterpret_cast<const double*>(sm + L.rt);
  for (int q = t; q < 3 * nr; q += kCT) {   // 3 threads per node, one row of R each
    const int i = q / 3, rw = q - 3 * i, j = r0 + i;
    node_update_row(x + 6 * i, rt + 12 * i, rw, a.nd.Rt64 + 12 * (int64_t)j, a.nd.node32 + 16 * (int64_t)j);
  }
  if (stamp) ts[5] = gtimer();
}

// The plan on the device (one warp; lane c binary-searches boundary c), so the
// host never reads the row structure back.  Same rule as plan_cluster.
__global__ void k_plan_cluster(const int32_t* row_ptr, int m, int max_cluster, PlanOut* out, int32_t* part,
                               int64_t* nnz_out) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ int32_t b[kMaxCluster + 1];
  int cs = max_cluster < m ? max_cluster : m;
  if (cs > kMaxCluster) cs = kMaxCluster;
  const int lane = threadIdx.x;
  const int64_t nnz = row_ptr[m];
  if (lane == 0 && nnz_out) *nnz_out = nnz;
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

void launch_pcg_prep(const int32_t* row_ptr, const int32_t* col, const int32_t* part, int cs, int max_rows, int max_nnz,
                     int32_t* pptr, int32_t* pc, int32_t* push, int32_t* npush, uint32_t* mask, cudaStream_t s,
                     bool marked) {
  PcgLists L{pptr, pc, push, npush, mask};
  if (!marked) launch_pdl(k_pcg_mark, dim3(cs), dim3(256), 0, s, row_ptr, col, part, L);
  launch_pdl(k_pcg_lists, dim3(cs), dim3(32), 0, s, row_ptr, part, cs, max_rows, max_pieces(max_rows, max_nnz), L);
}
int pcg_max_pieces(int max_rows, int max_nnz) { return max_pieces(max_rows, max_nnz); }

void launch_plan_cluster(const int32_t* row_ptr, int m, int max_cluster, PlanOut* out, int32_t* part, int64_t* nnz_out,
                         cudaStream_t s) {
  launch_pdl(k_plan_cluster, dim3(1), dim3(32), 0, s, row_ptr, m, max_cluster, out, part, nnz_out);
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
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)a.cluster_size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlaps the finalisation's tail
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_pcg_cluster, a);
}

// LM: the last trial (its energy in report slot `slot`) is kept only if accepted; otherwise
// the kept state is restored (fp64 master and its fp32 copy)
__global__ void k_lm_finish(int m, int slot, const LmDev* lm, const double* rep_energy, double* rep_flags,
                            double* Rt64, const double* Rt_acc, float* node32, double* pose) {
  pdl_wait();   // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const bool accept = rep_energy[5 * slot + 4] < lm->E_acc;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q == 0) rep_flags[slot] = accept ? 1.0 : 0.0;
  if (!accept && pose && q < 12) pose[q] = Rt_acc[12 * (int64_t)m + q];   // NEXT-2: the kept pose (after the nodes)
  if (accept || q >= 12 * (int64_t)m) return;
  const double v = Rt_acc[q];
  Rt64[q] = v;
  node32[16 * (q / 12) + q % 12] = (float)v;
}
void launch_lm_finish(int m, int slot, const LmDev* lm, const double* rep_energy, double* rep_flags, double* Rt64,
                      const double* Rt_acc, float* node32, cudaStream_t s, double* pose) {
  launch_pdl(k_lm_finish, dim3((unsigned)((12 * (int64_t)m + 255) / 256)), dim3(256), 0, s, m, slot, lm, rep_energy,
             rep_flags, Rt64, Rt_acc, node32, pose);
}

}  // namespace mis
