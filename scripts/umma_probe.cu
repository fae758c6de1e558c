// Stand-alone check of the tcgen05 operand layout K3b uses (MN-major, no swizzle, kind::tf32):
// 16 points x 256 features in 2 K-steps of 8 KB, D_c = F[:, 0:128]^T F[:, 0:128] (M = N = 128) and
// D_e = F[:, 128:256]^T F[:, 128:240] (M = 128, N = 112), read back with tcgen05.ld and compared
// on the host with the exact sums (features are TF32-exact small integers / 8).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_probe scripts/umma_probe.cu && /tmp/umma_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int NP = 16, NF = 256;
#ifndef DELAY
#define DELAY 0
#endif
#ifndef KMAJOR
#define KMAJOR 0
#endif
#ifndef PREFILL
#define PREFILL 0
#endif
#ifndef TEST_ST
#define TEST_ST 0
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t sbo, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;   // version (sm_100)
  return d;                  // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void probe(const float* F, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  float* buf = reinterpret_cast<float*>(sm);
  const int tid = threadIdx.x, warp = tid >> 5;
  // layout: point p, feature f -> (p / 8) * 8192 + (f / 4) * 128 + (p % 8) * 16 + (f % 4) * 4 bytes
  for (int q = tid; q < NP * NF; q += blockDim.x) {
    const int p = q / NF, f = q % NF;
    if (KMAJOR)   // (f % 8) * 16 + (f / 8) * 256 + (p % 4) * 4 + ((p % 8) / 4) * 128
      buf[((p / 8) * 8192 + (f % 8) * 16 + (f / 8) * 256 + (p % 4) * 4 + ((p % 8) / 4) * 128) / 4] = F[q];
    else
      buf[((p / 8) * 8192 + (f / 4) * 128 + (p % 8) * 16 + (f % 4) * 4) / 4] = F[q];
  }
  for (int q = tid; q < 2048 / 4; q += blockDim.x) buf[2 * 8192 / 4 + q] = 0.f;   // slack
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (PREFILL && warp < 4) {
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(7.f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(tm + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                    "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t base = smem_u32(buf);
    for (int k = 0; k < NP / 8; ++k) {
      const uint32_t blk = base + k * 8192;
      if (KMAJOR) {
        const uint32_t idk = idesc_tf32(128, 128) & ~((1u << 15) | (1u << 16));
        const uint32_t idk2 = idesc_tf32(128, 112) & ~((1u << 15) | (1u << 16));
        mma_tf32(tm + 0, desc_mn(blk, 256, 128), desc_mn(blk, 256, 128), idk, k > 0 || PREFILL);
        mma_tf32(tm + 128, desc_mn(blk + 16 * 256, 256, 128), desc_mn(blk + 16 * 256, 256, 128), idk2, k > 0 || PREFILL);
      } else {
        mma_tf32(tm + 0, desc_mn(blk, 128, 8192), desc_mn(blk, 128, 8192), idesc_tf32(128, 128), k > 0 || PREFILL);
        mma_tf32(tm + 128, desc_mn(blk + 32 * 128, 128, 8192), desc_mn(blk + 32 * 128, 128, 8192),
                 idesc_tf32(128, 112), k > 0 || PREFILL);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (DELAY) { for (int i = 0; i < 2000; ++i) __nanosleep(1000); }
  if (TEST_ST && warp < 4) {   // tcgen05.st a pattern into D_c column 0 .. 15 and read it back below
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(1000.f + 32 * warp + (tid & 31) + 0.5f * j);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(tm + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                    "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  if (warp < 4) {
    const int lane_row = 32 * warp + (tid & 31);
    for (int c0 = 0; c0 < 240; c0 += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) out[lane_row * 240 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(256));
}

int main() {
  std::vector<float> F(NP * NF), out(128 * 240, -1.f);
  srand(3);
  for (auto& x : F) x = (float)((rand() % 33) - 16) / 8.f;
  float *dF, *dO;
  cudaMalloc(&dF, F.size() * 4);
  cudaMalloc(&dO, out.size() * 4);
  cudaMemcpy(dF, F.data(), F.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 2 * 8192 + 2048 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 256, smem>>>(dF, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
  double maxe_c = 0, maxe_e = 0;
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 240; ++n) {
      double ref = 0;
      const bool isc = n < 128;
      const int nn = isc ? n : n - 128;
      if (!isc && nn >= 112) continue;
      for (int p = 0; p < NP; ++p) ref += (double)F[p * NF + (isc ? m : 128 + m)] * F[p * NF + (isc ? nn : 128 + nn)];
      const double err = fabs(ref - out[m * 240 + n]);
      if (isc) maxe_c = fmax(maxe_c, err); else maxe_e = fmax(maxe_e, err);
      if (err > 1e-3 && bad++ < 10) printf("mismatch m=%d n=%d got %g want %g\n", m, n, out[m * 240 + n], ref);
    }
  printf("max err D_c %g D_e %g bad %d\n", maxe_c, maxe_e, bad);
  printf("out[0][0..3] %g %g %g %g  out[33][0] %g out[0][128] %g\n", out[0], out[1], out[2], out[3], out[33 * 240], out[128]);
  return bad ? 1 : 0;
}
