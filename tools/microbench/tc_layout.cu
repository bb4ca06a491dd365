// Where tcgen05.mma kind::tf32 puts D rows in TMEM for M = 64 and M = 128
// (cta_group::1): A[i][0] = i + 1, B[n][0] = n + 1 (other k zero), so
// D[i][n] = (i + 1)(n + 1); each warp w reads lanes 32w..32w+31, columns 0..15
// with tcgen05.ld.32x32b.x16 and prints the row i each lane holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_layout tc_layout.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) | (uint64_t((sbo >> 4) & 0x3fff) << 32) |
         (1ull << 46);
}
__host__ __device__ constexpr int koff(int r, int k, int rows) { return (k / 4) * (rows * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 4) * 4; }

template <int M>
__global__ void probe(float* out) {
  constexpr int N = 16;
  __shared__ __align__(1024) unsigned char sm[128 * 8 * 4 + N * 8 * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* A = reinterpret_cast<float*>(sm);
  float* B = reinterpret_cast<float*>(sm + 128 * 8 * 4);
  for (int i = tid; i < 128 * 8 + N * 8; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  __syncthreads();
  if (tid < M) A[koff(tid, 0, M) / 4] = float(tid + 1);
  if (tid < N) B[koff(tid, 0, N) / 4] = float(tid + 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t d = tm;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(N) >> 3) << 17) | ((uint32_t(M) >> 4) << 24);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(desc(su32(A), M * 16, 128)), "l"(desc(su32(B), N * 16, 128)), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(d + (uint32_t(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 16; ++c) out[(tid * 16) + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(d));
}

template <int M>
void run(float* d) {
  probe<M><<<1, 128>>>(d);
  printf("M=%d: %s\n", M, cudaGetErrorString(cudaDeviceSynchronize()));
  float h[128 * 16];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  for (int w = 0; w < 4; ++w) {
    printf("  warp %d lanes 0..31 -> row (col 0 value / 1 - 1), col 1 check:", w);
    for (int l = 0; l < 32; ++l) {
      const float* v = h + (32 * w + l) * 16;
      printf(" %g%s", v[0] - 1, v[1] == 2 * v[0] ? "" : "!");
    }
    printf("\n");
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  run<128>(d);
  run<64>(d);
  return 0;
}
