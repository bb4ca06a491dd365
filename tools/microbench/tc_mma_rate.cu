// tcgen05.mma kind::tf32 issue rate on B200: one CTA per SM issues `iters` MMAs
// (M = 128, K = 8, N in {16, 32, 64, 128, 256}) from shared memory into
// `nacc` TMEM accumulators round-robin (nacc = 1: every MMA accumulates into
// the previous one's D), commits once, waits; clock64 around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_mma_rate tc_mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) | (uint64_t((sbo >> 4) & 0x3fff) << 32) |
         (1ull << 46);
}

template <int N, int M>
__global__ void bench(int iters, int nacc, unsigned long long* out, int nis = 1) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 * 8 + N * 8) ; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 7);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(nis));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t d0 = tm;
  if ((tid & 31) == 0 && (tid >> 5) < nis) {
    const uint32_t sa = su32(sm), sb = sa + 128 * 8 * 4;
    const uint64_t ad = desc(sa, 128 * 16, 128), bd = desc(sb, N * 16, 128);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(N) >> 3) << 17) | ((uint32_t(M) >> 4) << 24);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = d0 + ((tid >> 5) * nacc + (i % nacc)) * N;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(i >= nacc ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar)));
    const long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) out[0] = t1 - t0;
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(d0));
}

template <int N, int M>
void run(unsigned long long* d, int ctas_per_sm) {
  const int smem = (128 * 8 + N * 8) * 4 + 1024;
  cudaFuncSetAttribute(bench<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nacc : {1, 4}) {
    if (nacc * N > 256) continue;
    const int iters = 4096;
    bench<N, M><<<148 * ctas_per_sm, 128, smem>>>(iters, nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("M=%3d N=%3d nacc=%d ctas/SM=%d: %.1f cycles/MMA (CTA 0), %.0f tf32 flop/clk/CTA (%s)\n", M, N, nacc,
           ctas_per_sm, double(c) / iters, 2.0 * M * N * 8 * iters / c, cudaGetErrorString(e));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int c : {1, 2}) {
    run<16, 128>(d, c);
    run<64, 128>(d, c);
    run<256, 128>(d, c);
    run<16, 64>(d, c);
    run<64, 64>(d, c);
    run<256, 64>(d, c);
  }
  // several issuing warps in one CTA, each into its own accumulator
  for (int nis : {2, 4}) {
    const int smem = (128 * 8 + 64 * 8) * 4 + 1024;
    cudaFuncSetAttribute(bench<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<64, 64><<<148, 128, smem>>>(4096, 1, d, nis);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("M=64 N=64 issuers/CTA=%d: %.1f cycles per MMA of one issuer (%s)\n", nis, double(c) / 4096,
           cudaGetErrorString(e));
  }
  return 0;
}
