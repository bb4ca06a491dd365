// FP64 peak probes for the B200 roofline denominators (DFMA pipe, DMMA pipe,
// HBM store-only bandwidth).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// Prints one JSON line.  Not product code: it only measures the hardware the
// integration kernels are graded against.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m8n8k4 f64 MMA: 8*8*4 = 256 FMA per warp-instruction.
template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = 0; c1[c] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void store_kernel(double2* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  double2 v = make_double2(1.0, 2.0);
  for (; i < n; i += stride) dst[i] = v;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;

  // DFMA: 8 independent chains, 1024 threads/SM worth of blocks.
  const int iters = 1 << 16;
  int blocks = sms * 4, threads = 256;
  dfma_kernel<8><<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double dfma_tf = 2.0 * 8 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;

  // DMMA
  const int mit = 1 << 14;
  dmma_kernel<4><<<blocks, threads>>>(out, 16);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  dmma_kernel<4><<<blocks, threads>>>(out, mit);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)blocks * threads / 32;
  double dmma_tf = 2.0 * 256 * 4 * (double)mit * warps / (ms * 1e-3) / 1e12;

  // HBM store-only bandwidth over 8 GiB.
  size_t bytes = 8ull << 30;
  double2* buf;
  CK(cudaMalloc(&buf, bytes));
  size_t n = bytes / sizeof(double2);
  store_kernel<<<sms * 8, 512>>>(buf, n);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    store_kernel<<<sms * 8, 512>>>(buf, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double store_gbs = bytes / (best * 1e-3) / 1e9;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"store_gbs\": %.1f}\n",
         prop.name, sms, dfma_tf, dmma_tf, store_gbs);
  return 0;
}
