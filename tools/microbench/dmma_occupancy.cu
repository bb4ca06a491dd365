// DMMA (FP64 m8n8k4) throughput vs warps per SM, independent accumulator
// chains per warp, and interleaved DFMA work per MMA (the sum-factorised
// kernels compute each B fragment with 3 FMAs).  Prints CSV.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH, int NF>
__global__ void k(double* out, int iters, double s) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double x = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      double g = b;
#pragma unroll
      for (int f = 0; f < NF; ++f) g = fma(g, s, x);
      dmma(c[i][0], c[i][1], a, g);
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int CH, int NF>
void run(int warps_per_sm, double* buf, int sms) {
  const int threads = 32 * warps_per_sm;
  const int iters = 4096 / CH * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<CH, NF><<<sms, threads>>>(buf, 16, 1.0000001);
  cudaEventRecord(e0);
  k<CH, NF><<<sms, threads>>>(buf, iters, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tf = 2.0 * 256 * CH * (double)iters * (threads / 32) * sms / (ms * 1e-3) / 1e12;
  printf("%d,%d,%d,%.2f\n", warps_per_sm, CH, NF, tf);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * sms * 1024);
  printf("warps_per_sm,chains,fma_per_mma,dmma_tflops\n");
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<4, 0>(w, buf, sms);
    run<8, 0>(w, buf, sms);
    run<16, 0>(w, buf, sms);
    run<8, 1>(w, buf, sms);
    run<8, 2>(w, buf, sms);
    run<8, 3>(w, buf, sms);
    run<16, 2>(w, buf, sms);
  }
  return 0;
}
