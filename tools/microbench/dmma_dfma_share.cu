// Does DFMA work steal FP64 tensor (DMMA) throughput, and how much DMMA can
// one SM sub-partition (SMSP) issue?  Each warp runs CH independent DMMA
// accumulator chains; before each MMA it runs NF *live* DFMAs (a carried
// chain per accumulator, so nothing is hoisted).  Prints CSV:
// warps_per_sm, chains, dfma_per_mma, dmma_tflops, dfma_tflops.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH, int NF>
__global__ void k(double* out, int iters, double s) {
  double c[CH][2], g[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0, g[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-9;
  const double a = 1.0 + threadIdx.x * 1e-9, x = threadIdx.x * 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
#pragma unroll
      for (int f = 0; f < NF; ++f) g[i] = fma(g[i], s, x);
      dmma(c[i][0], c[i][1], a, NF ? g[i] : a);
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += c[i][0] + c[i][1] + g[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// Independent DFMA chains (not feeding the MMAs): do the two pipes overlap?
template <int CH, int NF>
__global__ void kind(double* out, int iters, double s) {
  double c[CH][2], g[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    c[i][0] = c[i][1] = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) g[i][f] = 1.0 + i * 1e-3 + f * 1e-4 + threadIdx.x * 1e-9;
  }
  const double a = 1.0 + threadIdx.x * 1e-9, x = threadIdx.x * 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
#pragma unroll
      for (int f = 0; f < NF; ++f) g[i][f & 3] = fma(g[i][f & 3], s, x);
      dmma(c[i][0], c[i][1], a, a);
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += c[i][0] + c[i][1] + g[i][0] + g[i][1] + g[i][2] + g[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int CH, int NF>
void run_ind(int warps_per_sm, double* buf, int sms) {
  const int threads = 32 * warps_per_sm;
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kind<CH, NF><<<sms, threads>>>(buf, 16, 0.9999999);
  cudaEventRecord(e0);
  kind<CH, NF><<<sms, threads>>>(buf, iters, 0.9999999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)CH * iters * (threads / 32) * sms;
  printf("ind,%d,%d,%d,%.2f,%.2f\n", warps_per_sm, CH, NF, 2.0 * 256 * n / (ms * 1e-3) / 1e12,
         2.0 * 32 * NF * n / (ms * 1e-3) / 1e12);
}

template <int CH, int NF>
void run(int warps_per_sm, double* buf, int sms) {
  const int threads = 32 * warps_per_sm;
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<CH, NF><<<sms, threads>>>(buf, 16, 0.9999999);
  cudaEventRecord(e0);
  k<CH, NF><<<sms, threads>>>(buf, iters, 0.9999999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)CH * iters * (threads / 32) * sms;
  printf("%d,%d,%d,%.2f,%.2f\n", warps_per_sm, CH, NF, 2.0 * 256 * n / (ms * 1e-3) / 1e12,
         2.0 * 32 * NF * n / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * sms * 1024);
  printf("warps_per_sm,chains,dfma_per_mma,dmma_tflops,dfma_tflops\n");
  for (int w : {4, 8, 16}) {
    run_ind<8, 1>(w, buf, sms);
    run_ind<8, 2>(w, buf, sms);
    run_ind<8, 4>(w, buf, sms);
    run_ind<8, 8>(w, buf, sms);
  }
  for (int w : {1, 2, 4, 8, 16}) {
    run<8, 0>(w, buf, sms);
    run<8, 1>(w, buf, sms);
    run<8, 2>(w, buf, sms);
    run<8, 4>(w, buf, sms);
    run<16, 0>(w, buf, sms);
    run<16, 2>(w, buf, sms);
  }
  return 0;
}
