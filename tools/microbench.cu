// Microbenchmarks for the GEMM design (tuning tool, not part of the library):
//   1. tcgen05.mma kind::tf32 issue rate, M=128, N=128 / N=256, SS operands, 1 CTA/SM
//   2. the same while 8 other warps stream st.shared at full speed (smem contention)
//   3. tcgen05.ld 32x32b.x16 + wait throughput (4 warps), tcgen05.st x16 throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ uint64_t desc_mn32(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(512 >> 4) << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
template <int N, bool STS_NOISE, bool AMN = false, bool BMN = false, int HANDSHAKE = 0>
__global__ void __launch_bounds__(416, 1) mma_rate(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2, bar3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&bar2)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar3)));
    }
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i & 15);
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(smem), sb = sa + 16384;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
                         ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  unsigned long long t0 = clock64(), t1 = t0;
  if (warp == 0) {
    if (lane == 0) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (HANDSHAKE >= 1) {   // chunk boundary of the GEMM: commit, wait a (complete) barrier, fence
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
          asm volatile("{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1;\n\t@!P1 bra W2;\n\t}" ::"r"(smem_u32(&bar3)));
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        for (int k = 0; k < 12; ++k) {
          const uint64_t a = AMN ? desc_mn32(sa + (k & 3) * 8192, 4096) : desc_k128(sa + (k & 3) * 32);
          const uint64_t bd = BMN ? desc_mn32(sb + (k & 3) * (N / 32 * 1024), N / 32 * 512) : desc_k128(sb + (k & 3) * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tmem), "l"(a), "l"(bd), "r"(idesc), "r"(1u));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)));
      t1 = clock64();
      done = 1;
    }
    __syncwarp();
  } else if (STS_NOISE && warp >= 5) {
    // 8 warps: st.shared streams into a region the MMA does not read
    const uint32_t dst = sa + 32768 + ((warp - 5) * 32 + lane) * 4;
    float v = lane;
    unsigned long long n = 0, s0 = clock64();
    while (!done) {
#pragma unroll
      for (int q = 0; q < 8; ++q) asm volatile("st.shared.f32 [%0], %1;" ::"r"(dst + q * 1024), "f"(v));
      v += 1.f;
      ++n;
    }
    if (lane == 0) { out[4096 + blockIdx.x * 16 + (warp - 5)] = n; out[8192 + blockIdx.x * 16 + (warp - 5)] = clock64() - s0; }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
}

__global__ void __launch_bounds__(128, 1) tmem_rate(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tslot + ((uint32_t)(warp * 32) << 16);
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int g = 0; g < 16; ++g) {   // 256 columns per iteration
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(base + g * 16));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += __uint_as_float(r[j]);
    }
  }
  unsigned long long t1 = clock64();
  unsigned long long t2 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int g = 0; g < 16; ++g) {
      uint32_t r = __float_as_uint(acc + g);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                   ::"r"(base + 256 + g * 16), "r"(r));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  unsigned long long t3 = clock64();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t3 - t2; }
  sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(512u));
}

int main() {
  unsigned long long* d_out; float* sink;
  cudaMalloc(&d_out, 16384 * 8); cudaMalloc(&sink, 4096 * 4);
  static unsigned long long h[16384];
  const int iters = 2000;
  auto run_mma = [&](auto kern, const char* name, double flops_per_iter) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    kern<<<148, 416, 64 * 1024>>>(iters, d_out, sink);
    cudaDeviceSynchronize();
    kern<<<148, 416, 64 * 1024>>>(iters, d_out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, 16384 * 8, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
    double stsb = 0, stsc = 0;
    for (int i = 0; i < 148; ++i) for (int w = 0; w < 8; ++w) { stsb += h[4096 + i * 16 + w] * 8.0 * 128; stsc += h[8192 + i * 16 + w]; }
    if (stsc > 0) printf("   STS: %.1f bytes/cycle/SM while MMAs run\n", stsb / (stsc / 8.0) / 148);
    printf("%-40s %s cycles/iter %.1f  (12 MMAs)  => per MMA %.1f cyc, tf32 TF/s @1.9GHz x148 = %.0f\n", name,
           cudaGetErrorString(e), cyc / iters, cyc / iters / 12, flops_per_iter * iters / cyc * 1.9e9 * 148 / 1e12);
  };
  run_mma(mma_rate<128, false>, "mma N=128 alone", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<128, true>, "mma N=128 + 8 warps STS", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<256, false>, "mma N=256 alone", 12.0 * 2 * 128 * 256 * 8);
  run_mma(mma_rate<256, true>, "mma N=256 + 8 warps STS", 12.0 * 2 * 128 * 256 * 8);
  run_mma(mma_rate<128, false, true, false>, "mma N=128 A MN-major", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<128, false, false, true>, "mma N=128 B MN-major", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<128, false, true, true>, "mma N=128 A,B MN-major", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<128, false, false, false, 1>, "mma N=128 + chunk handshake", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<128, true, true, false>, "mma N=128 A MN + 8 warps STS", 12.0 * 2 * 128 * 128 * 8);
  run_mma(mma_rate<256, false, false, false, 1>, "mma N=256 + chunk handshake", 12.0 * 2 * 128 * 256 * 8);
  tmem_rate<<<148, 128>>>(200, d_out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d_out, 2 * 148 * 8, cudaMemcpyDeviceToHost);
  printf("tmem: %s ld 256 cols x 128 lanes: %.1f cycles; st: %.1f cycles (per iteration, 128 KB)\n",
         cudaGetErrorString(e), (double)h[0] / 200, (double)h[1] / 200);
  return 0;
}
