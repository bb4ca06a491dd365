// Diagnostics: on-device FP64 peak probes used as the roofline denominator
// (MEASURED_PEAKS.json carries HBM and bf16 figures only).  The DMMA probe
// issues independent m8n8k4 FP64 MMAs from every warp of a full grid; the
// DFMA probe runs 8 independent FMA chains per thread.
#include <cuda_runtime.h>

#include "kernels_common.cuh"

namespace {

__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) pib::dmma_8x8x4(c[k][0], c[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = fma(acc[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Measures FP64 tensor (DMMA) and FMA-pipe throughput in TFLOP/s on `device`.
int pi_measure_fp64_peak(int device, double* dmma_tflops, double* dfma_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int blocks = prop.multiProcessorCount * 4, threads = 256;
  double* buf = nullptr;
  if (cudaMalloc(&buf, sizeof(double) * blocks * threads) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  const int mit = 1 << 13;
  dmma_peak_kernel<<<blocks, threads>>>(buf, 64);
  cudaEventRecord(e0);
  dmma_peak_kernel<<<blocks, threads>>>(buf, mit);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  *dmma_tflops = 2.0 * 256.0 * 8.0 * mit * (blocks * threads / 32.0) / (ms * 1e-3) / 1e12;
  const int fit = 1 << 15;
  dfma_peak_kernel<<<blocks, threads>>>(buf, 64, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_peak_kernel<<<blocks, threads>>>(buf, fit, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  *dfma_tflops = 2.0 * 8.0 * fit * blocks * threads / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
