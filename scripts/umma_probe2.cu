// Check of the K3b tcgen05 operand layout (K-major, no swizzle, kind::tf32, padded strides):
// NP points with c' (49) and e' (35) features split hi / lo (3xTF32), per 8-point K-step block
//   group g (8 features), row r = f % 8, point p8: g * 288 + r * 16 + (p8 % 4) * 4 + (p8 / 4) * 144
// groups: c_hi 0..6, c_lo 7..13, e_hi 14..18, e_lo 19..23; block stride 6944 B.
// D_c = [c_hi|c_lo] x [c_hi|c_lo]^T (M 128, N 112), D_e = [e_hi|e_lo|..] x [e_hi|e_lo]^T (M 128, N 80);
// host: G_c[m][n] = D_c[m][n] + D_c[m][56 + n] + D_c[56 + m][n] vs the fp64 Gram (same for e, 40).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/up2 scripts/umma_probe2.cu && /tmp/up2
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int NP = 40, FC = 49, FE = 35, BLK = 6944;
#ifndef M64
#define M64 0
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k(uint32_t addr, uint32_t sbo, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32_k(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void put(float* buf, int s, int g, int r, float v) {
  const int k = s >> 3, p8 = s & 7;
  buf[(k * BLK + g * 288 + r * 16 + (p8 & 3) * 4 + (p8 >> 2) * 144) >> 2] = v;
}

__global__ void probe(const float* C, const float* E, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  float* buf = reinterpret_cast<float*>(sm);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nk = (NP + 7) / 8;
  for (int q = tid; q < (nk * BLK + 8 * 288) / 4; q += blockDim.x) buf[q] = 0.f;
  __syncthreads();
  if (tid < NP) {
    for (int f = 0; f < 56; ++f) {
      const float x = f < FC ? C[tid * FC + f] : 0.f;
      const float h = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
      put(buf, tid, f >> 3, f & 7, h);
      put(buf, tid, 7 + (f >> 3), f & 7, x - h);
    }
    for (int f = 0; f < 40; ++f) {
      const float x = f < FE ? E[tid * FE + f] : 0.f;
      const float h = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
      put(buf, tid, 14 + (f >> 3), f & 7, h);
      put(buf, tid, 19 + (f >> 3), f & 7, x - h);
    }
  }
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
  if (tid == 0) {
    const uint32_t base = smem_u32(buf);
    for (int k = 0; k < nk; ++k) {
      const uint32_t blk = base + k * BLK;
      if (M64) {
        mma_tf32(tm + 0, desc_k(blk, 288, 144), desc_k(blk, 288, 144), idesc_tf32_k(64, 64), k > 0);
      } else {
      mma_tf32(tm + 0, desc_k(blk, 288, 144), desc_k(blk, 288, 144), idesc_tf32_k(128, 112), k > 0);
      mma_tf32(tm + 128, desc_k(blk + 14 * 288, 288, 144), desc_k(blk + 14 * 288, 288, 144), idesc_tf32_k(128, 80), k > 0);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int row = 32 * warp + (tid & 31);
    for (int c0 = 0; c0 < 208; c0 += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) out[row * 208 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(256));
}

int main() {
  std::vector<float> C(NP * FC), E(NP * FE), out(128 * 208);
  srand(5);
  auto rnd = [] { return (float)(rand() / (double)RAND_MAX * 2 - 1) * powf(10.f, (float)(rand() % 5 - 2)); };
  for (auto& x : C) x = rnd();
  for (auto& x : E) x = rnd();
  float *dC, *dE, *dO;
  cudaMalloc(&dC, C.size() * 4); cudaMalloc(&dE, E.size() * 4); cudaMalloc(&dO, out.size() * 4);
  cudaMemcpy(dC, C.data(), C.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 8 * BLK + 8 * 288 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 256, smem>>>(dC, dE, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
  if (M64) {   // where does D row i (A row = c_hi feature i, i < 56) land? match lane rows against the Gram row i, cols 0..48
    for (int i = 0; i < 56; i += 1) {
      int found = -1;
      for (int ln = 0; ln < 128 && found < 0; ++ln) {
        bool ok = true;
        for (int n = 0; n < FC && ok; ++n) {
          double ref = 0;
          for (int p = 0; p < NP; ++p) ref += (double)(i < FC ? C[p * FC + i] : 0.f) * C[p * FC + n];
          const float hi_i = 0; (void)hi_i;
          if (fabs(ref - out[ln * 208 + n]) > 1e-2 * (1 + fabs(ref))) ok = false;
        }
        if (ok) found = ln;
      }
      if (i < FC) printf("row %d -> lane %d\n", i, found);
    }
    return 0;
  }
  double worst = 0;
  for (int which = 0; which < 2; ++which) {
    const int Fn = which ? FE : FC, off = which ? 40 : 56, col0 = which ? 128 : 0;
    const std::vector<float>& X = which ? E : C;
    for (int m = 0; m < Fn; ++m)
      for (int n = m; n < Fn; ++n) {
        double ref = 0, mag = 0;
        for (int p = 0; p < NP; ++p) {
          ref += (double)X[p * Fn + m] * X[p * Fn + n];
          mag += fabs((double)X[p * Fn + m] * X[p * Fn + n]);
        }
        const double g = (double)out[m * 208 + col0 + n] + out[m * 208 + col0 + off + n] + out[(off + m) * 208 + col0 + n];
        const double rel = fabs(g - ref) / (mag + 1e-30);
        if (rel > worst) worst = rel;
      }
  }
  printf("worst |G - Gram| / sum|products| = %.3g\n", worst);
  return worst < 1e-6 ? 0 : 1;
}
