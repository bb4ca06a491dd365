// Host interface of the tcgen05 FP32 sum-factorised kernels (kernels_tc32.cuh).
// Internal, not ABI.
#pragma once

#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "kernels_common.cuh"

namespace pib {

struct Tc32Tables;

struct Tc32HostTables {
  std::vector<float> bhi, blo, xg, yline;
  std::vector<double> z;
};

bool tc32_supported(int p, int ne);
bool tc32_build(int p, const double* pts, const double* phi, int n_q, int n_shape, Tc32HostTables& t);
void tc32_attrs(int p);
void tc32_launch(int p, bool general, const LaunchArgs& a, const Tc32Tables& t, cudaStream_t s);

}  // namespace pib
