// k3b_umma.cu -- K3b for 5 <= k <= 8 (C5) on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// What it computes is K3b's (assemble.cu, k_accum_points): for every chunk (<= 128 consecutive
// points sharing one k-node tuple) the Gram sums of the factor rows
//   c' = [w_1 u_1, ..., w_k u_k, r_pl]          (6k + 1; Eq. 8 Jacobian rows)
//   e' = [w_1 a_1, w_1, ..., w_k a_k, w_k, r']   (4k + 3; point-to-point moments)
// over the chunk's associated points, committed with vector atomics into the BSR accumulators.
// Here the sums are tensor-core GEMMs over the chunk's associated points (rows), 8 per K-step:
// tcgen05.mma kind::tf32 with the 3xTF32 split x = hi + lo (hi = x with the 13 low mantissa bits
// cleared, what the tensor core reads of an fp32 operand; lo = x - hi) and three products accumulated
// in place in TMEM,  D_c = c_hi c_hi^T + c_hi c_lo^T + c_lo c_hi^T  (M = 64, N = 64; lo lo^T dropped:
// < 2^-20 relative per product, as in the k <= 4 mma.sync path), D_e likewise (N = 48).  D row i is
// TMEM lane 32 (i / 16) + i % 16 (the M = 64 data path), so every epilogue warp owns 16 Gram rows.
//
// Warp-specialised persistent kernel, two CTAs per SM (static round-robin chunk schedule):
//   warp 8  (issuer):  per chunk, TMA bulk copies (cp.async.bulk, mbarrier tx counts) of its K + 2
//                      factor-state planes and of 16-byte-aligned windows around its BSR slots and
//                      node ids into a 2-stage shared staging ring
//   warps 0-3 (build): compact the chunk's associated points (K3a's (n', associated) plane; K3a
//                      writes the other planes of associated points only), then write their hi / lo
//                      factor rows (lane = row, warp = every 4th feature group) into one of two
//                      32-row operand buffers, UMMA K-major layout
//   warp 9  (MMA):     one thread issues a round's tcgen05.mma into one of two TMEM stages (128
//                      columns each); tcgen05.commit frees the operand buffer and, at the chunk's
//                      last round, signals the epilogue
//   warps 4-7 (epi):   tcgen05.ld of the Gram rows; each upper-triangle entry (m, n) lands at a
//                      per-lane base + compile-time offset of the chunk record (k_accum_points' layout:
//                      P pair records of 52 = 36 data | 16 moments, K node records of 20); then one
//                      float4 / float2 atomic per record item, lanes on consecutive items (coalesced)
// Operand layout (bytes, per 8-point K-step block): group g of 8 features, row r = f % 8, point
// p8:  g * 288 + r * 16 + (p8 % 4) * 4 + (p8 / 4) * 144  (core matrices 8 x 16 B, LBO 144, SBO 288,
// block stride = 32 mod 128): the builders' scalar stores are bank-conflict free.  Groups:
// c_hi [0, GC), c_lo [GC, 2 GC), e_hi [2 GC, 2 GC + GE), e_lo [2 GC + GE, 2 GC + 2 GE).
// Measured at C5 (k = 8, 10M points, 171k segments): 1.39 ms per launch vs 1.63 ms for the FP32
// register-tile kernel (MIS_K3B_UMMA=0), parity as the other K3b paths (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace mis {
namespace {

#ifndef MIS_UMMA_ROWS
#define MIS_UMMA_ROWS 32   // operand rows per round (multiple of 8)
#endif
#ifndef MIS_UMMA_NS
#define MIS_UMMA_NS 2      // staging stages
#endif
template <int K>
struct UM {
  static constexpr int P = K * (K + 1) / 2;
  static constexpr int FC = 6 * K + 1, FE = 4 * K + 3;
  static constexpr int GC = (FC + 7) / 8, GE = (FE + 7) / 8;
  static constexpr int NG = 2 * (GC + GE);
  static constexpr int BLK = NG * 288 + (160 - (NG * 288) % 128) % 128;   // = 32 (mod 128)
  static constexpr int NC = 64, NE = 48;                                   // MMA N: the hi features
  static constexpr int NT = 2;                                             // TMEM stages of 128 columns
  static_assert(8 * GC <= NC && 8 * GE <= NE, "accumulator columns");
  static constexpr int ROWS = MIS_UMMA_ROWS, KSTEPS = ROWS / 8;
  // + slack after the last K-step block: an M = 64 A operand reads 8 groups from its start (at most
  // group 2 GC + GE), an N = 64 / 48 B operand 8 / 6: at most 2 GC + GE + 8 - NG groups past the block
  static constexpr int SLACK = 2 * GC + GE + 8 - NG;                       // = 8 - GE groups
  static constexpr int OB = KSTEPS * BLK + SLACK * 288;
  static constexpr int NPL = K + 2;                                         // staging: K + 2 planes x 128
  static constexpr int SLW = (4 * P + 31 + 15) & ~15, NDW = (4 * K + 31 + 15) & ~15;   // slot / node windows
  static constexpr int STG = NPL * 128 * 16 + SLW + NDW;
  static constexpr int NS = MIS_UMMA_NS;                                   // staging stages
  static constexpr int RT = 52 * P + 20 * K, NITEM = 13 * P + 6 * K;
  static constexpr int NMETA = P + K;
  // dynamic shared memory map (bytes)
  static constexpr int O_OB = 0, O_STG = 2 * OB, O_X = O_STG + NS * STG;
  static constexpr int O_REC = O_X;                                        // the chunk record
  static constexpr int SMEM = O_REC + 4 * RT;

  static_assert(NMETA <= 48, "k <= 8");
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b, uint32_t n = 1) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
// wait for the phase of parity `par` to complete; traps after ~4 s (a lost arrival is a bug: fail
// loudly rather than hang the device)
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(par) : "memory");
    if (done) return;
    if (t0 == 0) t0 = gtimer();
    else if (gtimer() - t0 > 4000000000ull) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {   // K-major, no swizzle, LBO 144, SBO 288
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(144 >> 4) << 16) | ((uint64_t)(288 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {   // F32 accumulate, TF32 A / B, K-major
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
// 16 consecutive columns of this warp's 32 TMEM lanes; the registers are valid after tmem_wait_ld()
__device__ __forceinline__ void tmem_ld16_async(uint32_t addr, float (&v)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                 "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
               : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_regs_ready16(float (&v)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) asm volatile("" : "+f"(v[j]));
}
// after tmem_wait_ld(): makes every use of the loaded registers depend on the wait (an empty asm
// that "rewrites" them, ordered after the volatile wait), so no use is scheduled before it
template <int Q>
__device__ __forceinline__ void tmem_regs_ready(float (&v)[Q][16]) {
#pragma unroll
  for (int q = 0; q < Q; ++q)
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("" : "+f"(v[q][j]));
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

#ifndef MIS_UMMA_NORED
#define MIS_UMMA_NORED 0   // 1: skip the commit atomics (experiments: atomic-throughput bound?)
#endif
#ifndef MIS_UMMA_PROF
#define MIS_UMMA_PROF 0   // 1: CTA 0's role leaders printf their wait / work cycle totals (experiments)
#endif
#if MIS_UMMA_PROF
#define PTIME(acc, stmt) do { const long long _t0 = clock64(); stmt; acc += clock64() - _t0; } while (0)
#else
#define PTIME(acc, stmt) do { stmt; } while (0)
#endif

struct Round {        // one operand buffer's round, builder -> MMA thread
  int rows, stage, first, last;
};
struct StageMeta {    // issuer -> builders: chunk range and where its slots / node ids start in the
  int y, z, slo, ndo;   // stage's copied 16-byte-aligned windows (ints)
};
struct TmemMeta {     // builders -> epilogue, per TMEM stage
  int done, pad[3];
  int slot[48];
};

// One feature group (8 features, hi and lo) of one operand row from the point's state in registers
// (wa[s] = (w_s a_s, w_s), rr = (r', r_pl), nn = (n', 0); zeros for a pad row).  G < GC: c' features
// 8 G .. 8 G + 7, else e' features 8 (G - GC) ...
template <int K, int G>
__device__ __forceinline__ void build_group(const float4 (&wa)[K], const float4& rr, const float4& nn, float* base) {
  using U = UM<K>;
  constexpr int GC = U::GC, GE = U::GE;
  constexpr bool C = G < GC;
  constexpr int f0 = C ? 8 * G : 8 * (G - GC);
  constexpr int ghi = C ? G : 2 * GC + (G - GC), glo = C ? G + GC : 2 * GC + GE + (G - GC);
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int f = f0 + i;
    float x = 0.f;
    if constexpr (C) {
      if (f < 6 * K) {
        const float4 w = wa[f / 6 < K ? f / 6 : K - 1];
        const int c = f % 6;
        x = c == 0 ? w.y * nn.z - w.z * nn.y : c == 1 ? w.z * nn.x - w.x * nn.z : c == 2 ? w.x * nn.y - w.y * nn.x
          : c == 3 ? w.w * nn.x : c == 4 ? w.w * nn.y : w.w * nn.z;
      } else if (f == 6 * K) {
        x = rr.w;
      }
    } else {
      if (f < 4 * K) {
        const float4 w = wa[f / 4 < K ? f / 4 : K - 1];
        const int c = f % 4;
        x = c == 0 ? w.x : c == 1 ? w.y : c == 2 ? w.z : w.w;
      } else if (f < 4 * K + 3) {
        x = f == 4 * K ? rr.x : f == 4 * K + 1 ? rr.y : rr.z;
      }
    }
    v[i] = x;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float hi = __uint_as_float(__float_as_uint(v[i]) & 0xffffe000u);
    base[(ghi * 288 + i * 16) >> 2] = hi;
    base[(glo * 288 + i * 16) >> 2] = v[i] - hi;
  }
}
template <int K, int W>
__device__ __forceinline__ void build_groups(const float4* sg, int pt, float* base) {
  constexpr int NGH = UM<K>::GC + UM<K>::GE;
  static_assert(NGH <= 16, "k <= 8");
  float4 wa[K], rr, nn;   // the whole staged state first: one shared-memory latency
  if (pt >= 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) wa[q] = sg[q * 128 + pt];
    rr = sg[K * 128 + pt];
    nn = sg[(K + 1) * 128 + pt];
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) wa[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    rr = nn = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if constexpr (W < NGH) build_group<K, W>(wa, rr, nn, base);
  if constexpr (W + 4 < NGH) build_group<K, W + 4>(wa, rr, nn, base);
  if constexpr (W + 8 < NGH) build_group<K, W + 8>(wa, rr, nn, base);
  if constexpr (W + 12 < NGH) build_group<K, W + 12>(wa, rr, nn, base);
}

template <int K>
__global__ void __launch_bounds__(320, 2) k_accum_points_umma(AsmPointsArgs a) {
  using U = UM<K>;
  constexpr int P = U::P, FC = U::FC, FE = U::FE, GC = U::GC, GE = U::GE, NS = U::NS;
  constexpr int NIPT = (U::NITEM + 127) / 128;   // record items per epilogue thread
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;   // (the dynamic shared base is 128 B aligned; no integer round trip, so the
                            // compiler keeps shared-space addressing: STS / LDS, not generic ST / LD)
  float* Rec = reinterpret_cast<float*>(sm + U::O_REC);   // the chunk record (k_accum_points' layout)
  float* const a_acc_data = a.acc.data;
  float* const a_acc_mom = a.acc.mom;
  float* const a_acc_rhs = a.acc.rhs_data;
  float* const a_acc_nmom = a.acc.node_mom;
  constexpr int MR = 2;   // chunk metadata ring (builders -> epilogue)
  __shared__ __align__(8) uint64_t bar_sfull[NS], bar_sempty[NS], bar_ofull[2], bar_oempty[2], bar_tfull[U::NT],
      bar_tempty[U::NT], bar_mfull[MR], bar_mempty[MR];
  __shared__ StageMeta smeta[NS];
  __shared__ TmemMeta tmeta[MR];
  __shared__ Round rd[2];
  __shared__ int wcnt[4];
  __shared__ int16_t rowpt[128];   // compacted row -> point of the chunk (builders)
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bar_sfull[i], 1);
      mbar_init(&bar_sempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_ofull[i], 1);
      mbar_init(&bar_oempty[i], 1);
    }
    for (int i = 0; i < U::NT; ++i) {
      mbar_init(&bar_tfull[i], 1);   // the chunk's last MMA commit
      mbar_init(&bar_tempty[i], 1);
    }
    for (int i = 0; i < MR; ++i) {
      mbar_init(&bar_mfull[i], 1);
      mbar_init(&bar_mempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(128 * U::NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the record entries no Gram entry maps to stay zero; the operand buffers' slack is read (as the
  // M = 128 rows past a block's last group) only into D rows the epilogue ignores, but keep it finite
  for (int q = tid; q < 2 * U::OB / 4; q += blockDim.x) reinterpret_cast<float*>(sm + U::O_OB)[q] = 0.f;
  for (int q = tid; q < U::RT; q += blockDim.x) Rec[q] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  pdl_wait();      // K3a's factor state
  pdl_trigger();   // the finalisation may launch (it waits for this grid's completion)

  long long pw0 = 0, pw1 = 0, pw2 = 0, pw3 = 0, pcount = 0;
  const long long pstart = clock64();
  if (warp == 8) {
    // ------------------------------------------------------------ issuer
    const float4* ps = a.pstate;
    const int64_t S = a.pstride;
    int st = 0;
    uint32_t ph = 0;
    // static schedule: CTA b owns chunks b, b + grid, ... (round robin: balanced), visited from a
    // CTA-dependent start so that concurrently committing CTAs work on distant chunks (different
    // node blocks: no same-address atomic contention between SMs)
    const int64_t J = (a.nchunk + gridDim.x - 1) / gridDim.x;
    const int64_t rot = (J * blockIdx.x) / gridDim.x;
    for (int64_t j0 = 0; j0 < J; j0 += 32) {
      int64_t jj = j0 + lane + rot;
      if (jj >= J) jj -= J;
      const int64_t cl = jj * gridDim.x + blockIdx.x;
      const bool valid = j0 + lane < J && cl < a.nchunk;
      int4 h = make_int4(0, 0, 0, 0);
      if (valid) h = a.chunks[cl];
      // chunks without an associated point (K3a by chunk flags them) add nothing: never staged
      const bool live = valid && (a.chunk_live == nullptr || a.chunk_live[cl] != 0);
      const unsigned vmask = __ballot_sync(0xffffffffu, live);
      for (int k = 0; k < 32; ++k) {
        if (!((vmask >> k) & 1u)) continue;
        const int seg = __shfl_sync(0xffffffffu, h.x, k);
        const int y = __shfl_sync(0xffffffffu, h.y, k), z = __shfl_sync(0xffffffffu, h.z, k);
        PTIME(pw0, mbar_wait(&bar_sempty[st], ph ^ 1u));
        ++pcount;
        if (lane == 0) {
          // the chunk's factor-state planes, and 16-byte-aligned windows around its P slots and K
          // node ids, all by TMA bulk copies completing on the stage's barrier
          const int32_t* sp = a.seg_slot + (int64_t)seg * P;
          const int32_t* np = a.seg_nodes + (int64_t)seg * K;
          const uintptr_t s0 = reinterpret_cast<uintptr_t>(sp) & ~uintptr_t(15);
          const uintptr_t s1 = (reinterpret_cast<uintptr_t>(sp + P) + 15) & ~uintptr_t(15);
          const uintptr_t n0 = reinterpret_cast<uintptr_t>(np) & ~uintptr_t(15);
          const uintptr_t n1 = (reinterpret_cast<uintptr_t>(np + K) + 15) & ~uintptr_t(15);
          smeta[st].y = y;
          smeta[st].z = z;
          smeta[st].slo = (int)((reinterpret_cast<uintptr_t>(sp) - s0) >> 2);
          smeta[st].ndo = (int)((reinterpret_cast<uintptr_t>(np) - n0) >> 2);
          const uint32_t bytes = (uint32_t)(z - y) * 16u;
          mbar_arrive_tx(&bar_sfull[st], bytes * U::NPL + (uint32_t)(s1 - s0) + (uint32_t)(n1 - n0));
          uint8_t* dst = sm + U::O_STG + st * U::STG;
          if (bytes > 0)
            for (int s = 0; s < U::NPL; ++s) bulk_g2s(dst + s * 2048, ps + s * S + y, bytes, &bar_sfull[st]);
          bulk_g2s(dst + U::NPL * 2048, reinterpret_cast<const void*>(s0), (uint32_t)(s1 - s0), &bar_sfull[st]);
          bulk_g2s(dst + U::NPL * 2048 + U::SLW, reinterpret_cast<const void*>(n0), (uint32_t)(n1 - n0), &bar_sfull[st]);
        }
        __syncwarp();
        if (++st == NS) { st = 0; ph ^= 1u; }
      }
    }
    mbar_wait(&bar_sempty[st], ph ^ 1u);   // end of work
    if (lane == 0) {
      smeta[st].y = -1;
      mbar_arrive(&bar_sfull[st]);
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ builders
    // compaction with one thread per point; then the rows with lane = row, warp = every 4th feature
    // group (warp-uniform code per group, conflict-free scalar stores)
    const int bt = tid;
    int st = 0, b = 0, s = 0, mi = 0;
    uint32_t ph = 0, pho = 0, pm = 0;
    while (true) {
      PTIME(pw0, mbar_wait(&bar_sfull[st], ph));
      const int y = smeta[st].y, z = smeta[st].z;
      if (y < 0) {   // propagate the end: an empty round to the MMA thread, `done` to the epilogue
        mbar_wait(&bar_oempty[b], pho ^ 1u);
        mbar_wait(&bar_mempty[mi], pm ^ 1u);
        if (bt == 0) {
          rd[b].rows = -1;
          tmeta[mi].done = 1;
          mbar_arrive(&bar_ofull[b]);
          mbar_arrive(&bar_mfull[mi]);
        }
        break;
      }
      const int n = z - y;
      const float4* sg = reinterpret_cast<const float4*>(sm + U::O_STG + st * U::STG);
      bool live = false;
      if (bt < n) {
        if (a.sparse_state) {   // plane K + 1 = (n', associated); the other planes are stale when not
          live = reinterpret_cast<const float*>(sg + (K + 1) * 128 + bt)[3] != 0.f;
        } else {
#pragma unroll
          for (int q = 0; q < K; ++q) live |= reinterpret_cast<const float*>(sg + q * 128 + bt)[3] != 0.f;   // w_q
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      if (lane == 0) wcnt[warp] = __popc(bal);
      named_sync(1, 128);
      int nlive = 0, before = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int cw = wcnt[w];
        before += w < warp ? cw : 0;
        nlive += cw;
      }
      if (live) rowpt[before + __popc(bal & ((1u << lane) - 1u))] = (int16_t)bt;
      if (nlive > 0) {
        PTIME(pw1, mbar_wait(&bar_mempty[mi], pm ^ 1u));
        ++pcount;
        if (bt < U::NMETA) {
          const int32_t* win = reinterpret_cast<const int32_t*>(sm + U::O_STG + st * U::STG + U::NPL * 2048);
          tmeta[mi].slot[bt] = bt < P ? win[smeta[st].slo + bt] : win[U::SLW / 4 + smeta[st].ndo + (bt - P)];
        }
        if (bt == 0) tmeta[mi].done = 0;
      }
      named_sync(1, 128);   // wcnt read; rowpt and the chunk metadata written
      if (bt == 0 && nlive > 0) mbar_arrive(&bar_mfull[mi]);
      if (nlive > 0) {
        const int nr = (nlive + U::ROWS - 1) / U::ROWS;
        for (int r = 0; r < nr; ++r) {
          PTIME(pw2, mbar_wait(&bar_oempty[b], pho ^ 1u));
          uint8_t* ob = sm + U::O_OB + b * U::OB;
          const int rows = min(U::ROWS, nlive - r * U::ROWS), rows8 = (rows + 7) & ~7;
#if MIS_UMMA_PROF
          const long long pbld = clock64();
#endif
          for (int rw = lane; rw < rows8; rw += 32) {   // rows past `rows` up to the K-step: zeros
            const int pt = rw < rows ? rowpt[r * U::ROWS + rw] : -1;
            float* base = reinterpret_cast<float*>(ob + (rw >> 3) * U::BLK + (rw & 3) * 4 + ((rw >> 2) & 1) * 144);
            switch (warp) {
              case 0: build_groups<K, 0>(sg, pt, base); break;
              case 1: build_groups<K, 1>(sg, pt, base); break;
              case 2: build_groups<K, 2>(sg, pt, base); break;
              default: build_groups<K, 3>(sg, pt, base); break;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#if MIS_UMMA_PROF
          pw3 += clock64() - pbld;
#endif
          named_sync(1, 128);
          if (bt == 0) {
            rd[b].rows = rows;
            rd[b].stage = s;
            rd[b].first = r == 0;
            rd[b].last = r == nr - 1;
            mbar_arrive(&bar_ofull[b]);
          }
          if (++b == 2) { b = 0; pho ^= 1u; }
        }
      }
      if (bt == 0) mbar_arrive(&bar_sempty[st]);   // the staging is read (the last named_sync above)
      if (++st == NS) { st = 0; ph ^= 1u; }
      if (nlive > 0) {
        if (++s == U::NT) s = 0;
        if (++mi == MR) { mi = 0; pm ^= 1u; }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    int b = 0;
    uint32_t pho = 0, pht = 0;
    const uint32_t ob0 = su32(sm + U::O_OB);
    while (true) {
      PTIME(pw0, mbar_wait(&bar_ofull[b], pho));
      const Round r = rd[b];
      ++pcount;
      if (r.rows < 0) break;
      if (r.first) {   // the chunk's TMEM stage drained by the epilogue of its previous user
        PTIME(pw1, mbar_wait(&bar_tempty[r.stage], pht ^ 1u));
        if (r.stage == U::NT - 1) pht ^= 1u;
      }
      tc_fence_after();
      if (lane == 0) {
        const uint32_t dc = tm + (uint32_t)(r.stage * 128), de = dc + 64;
        const int nk = (r.rows + 7) >> 3;
        for (int k = 0; k < nk; ++k) {
          const uint32_t blk = ob0 + (uint32_t)(b * U::OB + k * U::BLK);
          const uint32_t acc = (r.first && k == 0) ? 0u : 1u;
          // M = 64: G = HH + HL + LH accumulated in place (D row i = TMEM lane 32 (i / 16) + i % 16)
          const uint32_t ch = blk, cl = blk + GC * 288, eh = blk + 2 * GC * 288, el = eh + GE * 288;
          umma_tf32(dc, sdesc(ch), sdesc(ch), idesc_tf32(64, U::NC), acc);
          umma_tf32(dc, sdesc(ch), sdesc(cl), idesc_tf32(64, U::NC), 1u);
          umma_tf32(dc, sdesc(cl), sdesc(ch), idesc_tf32(64, U::NC), 1u);
          umma_tf32(de, sdesc(eh), sdesc(eh), idesc_tf32(64, U::NE), acc);
          umma_tf32(de, sdesc(eh), sdesc(el), idesc_tf32(64, U::NE), 1u);
          umma_tf32(de, sdesc(el), sdesc(eh), idesc_tf32(64, U::NE), 1u);
        }
        umma_commit(&bar_oempty[b]);
        if (r.last) umma_commit(&bar_tfull[r.stage]);
      }
      __syncwarp();
      if (++b == 2) { b = 0; pho ^= 1u; }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ epilogue (TMEM lane = L)
    // phase A: lane m < 6k holds Gram row m of c' (node j = m / 6, component a = m % 6); its entries
    // (m, n = 6 l + b) of the upper triangle go to record index 52 pair(j, l) + 6 a + b -- a
    // per-lane base plus a compile-time offset 52 l + b, so the scatter is one predicated store per
    // entry -- and column 6k to the node's rhs; e' rows likewise.  Phase B: the record items (lanes =
    // consecutive items: coalesced) as one vector atomic each.  The record entries no Gram entry maps
    // to (pads, the diagonal blocks' lower triangles) stay zero.
    const int L = tid - 128, ew = L >> 5;
    const uint32_t lane_addr = (uint32_t)(32 * ew) << 16;
    // this thread's record items it = L + 128 k: record index | kind (0 data, 1 moments, 2 node rhs,
    // 3 node moments) << 12 | pair / node slot << 14 | destination offset << 22 | valid << 31
    uint32_t idsc[NIPT];
#pragma unroll
    for (int k = 0; k < NIPT; ++k) {
      const int it = L + 128 * k;
      uint32_t dsc = 0;
      if (it < 13 * P) {
        const int pr = it / 13, qq = it - 13 * pr;
        dsc = (uint32_t)(4 * it) | ((qq < 9 ? 0u : 1u) << 12) | ((uint32_t)pr << 14) |
              ((uint32_t)(qq < 9 ? 4 * qq : 4 * (qq - 9)) << 22) | (1u << 31);
      } else if (it < U::NITEM) {
        const int t2 = it - 13 * P, sl = t2 / 6, qq = t2 - 6 * sl;
        dsc = qq < 3 ? ((uint32_t)(52 * P + 20 * sl + 2 * qq) | (2u << 12) | ((uint32_t)sl << 14) | ((uint32_t)(2 * qq) << 22) | (1u << 31))
                     : ((uint32_t)(52 * P + 20 * sl + 8 + 4 * (qq - 3)) | (3u << 12) | ((uint32_t)sl << 14) |
                        ((uint32_t)(4 * (qq - 3)) << 22) | (1u << 31));
      }
      idsc[k] = dsc;
    }
    int s = 0, mi = 0;
    uint32_t pht = 0, pm = 0;
    while (true) {
      mbar_wait(&bar_mfull[mi], pm);
      if (tmeta[mi].done) break;
      PTIME(pw0, mbar_wait(&bar_tfull[s], pht));
      tc_fence_after();
      ++pcount;
#if MIS_UMMA_PROF
      const long long pa = clock64();
#endif
      const uint32_t col = tm + lane_addr + (uint32_t)(s * 128);
      // phase A: Gram row m = 16 ew + lane (lanes < 16 of each warp, the M = 64 data path) -> its
      // upper-triangle entries in the record: c' (m < 6k) then e' (m < 4k)
      {
        const int m = 16 * ew + lane;
        float v[(FC + 15) / 16][16];
#pragma unroll
        for (int q = 0; q < (FC + 15) / 16; ++q) tmem_ld16_async(col + 16 * q, v[q]);
        tmem_wait_ld();
        tmem_regs_ready(v);
        if (lane < 16 && m < 6 * K) {
          const int j = m / 6, a = m - 6 * (m / 6);
          float* rb = Rec + 52 * (j * K - (j * (j - 1)) / 2 - j) + 6 * a;
#pragma unroll
          for (int l = 0; l < K; ++l)
#pragma unroll
            for (int b = 0; b < 6; ++b)
              if (l > j || (l == j && b >= a)) rb[52 * l + b] = v[(6 * l + b) / 16][(6 * l + b) % 16];
          Rec[52 * P + 20 * j + a] = v[(6 * K) / 16][(6 * K) % 16];
        }
      }
      {
        const int m = 16 * ew + lane;
        float u[(FE + 15) / 16][16];
#pragma unroll
        for (int q = 0; q < (FE + 15) / 16; ++q) tmem_ld16_async(col + 64 + 16 * q, u[q]);
        tmem_wait_ld();
        tmem_regs_ready(u);
        if (lane < 16 && m < 4 * K) {
          const int j = m >> 2, a = m & 3;
          float* rb = Rec + 52 * (j * K - (j * (j - 1)) / 2 - j) + 36 + 4 * a;
#pragma unroll
          for (int l = 0; l < K; ++l)
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (l > j || (l == j && b >= a)) rb[52 * l + b] = u[(4 * l + b) / 16][(4 * l + b) % 16];
#pragma unroll
          for (int c = 0; c < 3; ++c) Rec[52 * P + 20 * j + 8 + 3 * a + c] = u[(4 * K + c) / 16][(4 * K + c) % 16];
        }
      }
      tc_fence_before();
      named_sync(2, 128);   // record written, TMEM stage read
      if (L == 0) mbar_arrive(&bar_tempty[s]);
#if MIS_UMMA_PROF
      pw1 += clock64() - pa;
      const long long pb = clock64();
#endif
      // all of this thread's items loaded first (no branch between the loads), then the atomics
      const int* slots = tmeta[mi].slot;
      float4 iv[NIPT];
      float* idst[NIPT];
#pragma unroll
      for (int k = 0; k < NIPT; ++k) {
        const uint32_t dsc = idsc[k];
        const int d = dsc & 4095, kind = (dsc >> 12) & 3, idx = (dsc >> 14) & 255, off = (dsc >> 22) & 63;
        iv[k] = kind == 2 ? make_float4(Rec[d], Rec[d + 1], 0.f, 0.f) : *reinterpret_cast<const float4*>(Rec + d);
        const int sl = slots[kind >= 2 ? P + idx : idx];
        idst[k] = (kind == 0 ? a_acc_data + 36 * (int64_t)sl : kind == 1 ? a_acc_mom + 16 * (int64_t)sl
                  : kind == 2 ? a_acc_rhs + 6 * (int64_t)sl : a_acc_nmom + 12 * (int64_t)sl) + off;
      }
#pragma unroll
      for (int k = 0; k < NIPT; ++k) {
        const uint32_t dsc = idsc[k];
        const float4 v = iv[k];
        const bool nz = (dsc >> 31) && !MIS_UMMA_NORED && (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f);
        if (nz) {
          if (((dsc >> 12) & 3) == 2) atomicAdd(reinterpret_cast<float2*>(idst[k]), make_float2(v.x, v.y));
          else atomicAdd(reinterpret_cast<float4*>(idst[k]), v);
        }
      }
      named_sync(2, 128);   // record and the chunk's slots read
      if (L == 0) mbar_arrive(&bar_mempty[mi]);
#if MIS_UMMA_PROF
      pw2 += clock64() - pb;
#endif
      if (++s == U::NT) { s = 0; pht ^= 1u; }
      if (++mi == MR) { mi = 0; pm ^= 1u; }
    }
  }
#if MIS_UMMA_PROF
  if (blockIdx.x == 0 && (tid == 0 || tid == 128 || tid == 256 || tid == 288))
    printf("umma prof role %s: total %lld  w0 %lld w1 %lld w2 %lld w3 %lld count %lld\n",
           tid == 0 ? "build" : tid == 128 ? "epi" : tid == 256 ? "issue" : "mma", clock64() - pstart, pw0, pw1, pw2,
           pw3, pcount);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128 * U::NT));
  }
}

template <int K>
void launch_umma_k(const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  using U = UM<K>;
  // two CTAs per SM (each allocates 256 of the 512 TMEM columns; registers and >= 80 KB of shared
  // memory keep a third off the SM, whose TMEM allocation would wait for one of them to exit)
  const int smem = U::SMEM > 80 * 1024 ? U::SMEM : 80 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_accum_points_umma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int64_t grid = 2 * (int64_t)num_sms;
  if (a.nchunk < grid) grid = a.nchunk;
  if (grid <= 0) return;
  launch_pdl(k_accum_points_umma<K>, dim3((unsigned)grid), dim3(320), (size_t)smem, s, a);
}

}  // namespace

bool umma_k3b_enabled() {
  static const int on = [] {
    const char* e = getenv("MIS_K3B_UMMA");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

void launch_accum_points_umma(int K, const AsmPointsArgs& a, int num_sms, cudaStream_t s) {
  switch (K) {
    case 5: launch_umma_k<5>(a, num_sms, s); break;
    case 6: launch_umma_k<6>(a, num_sms, s); break;
    case 7: launch_umma_k<7>(a, num_sms, s); break;
    case 8: launch_umma_k<8>(a, num_sms, s); break;
    default: break;
  }
}

}  // namespace mis
