// Probe: does tcgen05.mma kind::tf32 truncate or round the fp32 bits it reads?
// A (128 x 8, K-major SW128) row 0 = x at k = 0, zeros elsewhere; B (N=16 x 8) = 1 at k = 0.
// D[0][0] = tf32(x) as the tensor core sees it.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d;
}
__global__ void probe(const float* xs, int nx, float* out) {
  __shared__ __align__(1024) float A[128 * 32];
  __shared__ __align__(1024) float B[16 * 32];
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  }
  for (int i = tid; i < 128 * 32; i += blockDim.x) A[i] = 0.f;
  for (int i = tid; i < 16 * 32; i += blockDim.x) B[i] = 0.f;
  __syncthreads();
  // row r of A (r < nx), k = 0 -> chunk 0 ^ (r & 7) of row r
  if (tid < nx && tid < 128) A[tid * 32 + ((0 ^ (tid & 7)) << 2)] = xs[tid];
  if (tid < 16) B[tid * 32 + ((0 ^ (tid & 7)) << 2)] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tslot), "l"(desc_k128(smem_u32(A))), "l"(desc_k128(smem_u32(B))), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tslot + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[tid] = __uint_as_float(r);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(32u));
}
int main() {
  const int nx = 8;
  float hx[nx]; uint32_t bits[nx] = {0x3f800000u | 0x1fffu, 0x3f800000u | 0x1000u, 0x3f800000u | 0x0fffu,
                                      0x3f800000u | 0x3000u, 0xbf800000u | 0x1fffu, 0x40490fdbu, 0x3eaaaaabu, 0x3f801001u};
  memcpy(hx, bits, sizeof(bits));
  float *dx, *dout; cudaMalloc(&dx, sizeof(hx)); cudaMalloc(&dout, 128 * 4);
  cudaMemcpy(dx, hx, sizeof(hx), cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dx, nx, dout);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[128]; cudaMemcpy(ho, dout, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  for (int i = 0; i < nx; ++i) {
    uint32_t o; memcpy(&o, &ho[i], 4);
    uint32_t tr = bits[i] & 0xFFFFE000u, rn = (bits[i] + 0x1000u) & 0xFFFFE000u;
    printf("x=%08x  tc=%08x  trunc=%08x  rna=%08x  -> %s\n", bits[i], o, tr, rn,
           o == tr ? (o == rn ? "both" : "TRUNCATES") : (o == rn ? "ROUNDS(rna)" : "other"));
  }
  return 0;
}
