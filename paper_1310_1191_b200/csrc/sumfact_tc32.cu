// Host side of the tcgen05 FP32 sum-factorised kernels (kernels_tc32.cuh):
// tables from the caller's rule / shape table and the launches, p = 3..7.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels_sumfact.cuh"
#include "kernels_tc32.cuh"
#include "tc32_api.hpp"

namespace pib {
namespace {

template <int P>
bool build_p(const double* pts, const double* phi, int n_q, int n_shape, Tc32HostTables& out) {
  using C = Tc32Shape<P>;
  constexpr int NS = C::NS, NZ = C::NZ, NV = C::NV, NT = C::NT;
  if (n_q != NS * NZ || n_shape != NT * NV) return false;
  auto PHI = [&](int q, int k, int dof) { return phi[(static_cast<size_t>(q) * 4 + k) * n_shape + dof]; };
  // X_x(t, s): x = 0 dm/dxi1, 1 dm/dxi2, 2 m (kernels_sumfact.cuh); read at a = 0, z = 0
  std::vector<double> X(static_cast<size_t>(3) * NT * NS);
  for (int t = 0; t < NT; ++t)
    for (int s = 0; s < NS; ++s) {
      X[(0 * NT + t) * NS + s] = PHI(s, 1, t * NV);
      X[(1 * NT + t) * NS + s] = PHI(s, 2, t * NV);
      X[(2 * NT + t) * NS + s] = PHI(s, 0, t * NV) / PHI(s, 0, 0);
    }
  out.bhi.assign(C::B_BYTES / 4, 0.f);
  out.blo.assign(C::B_BYTES / 4, 0.f);
  for (int x = 0; x < 3; ++x)
    for (int s = 0; s < NS; ++s)
      for (int t = 0; t < NT; ++t) {
        const float v = static_cast<float>(X[(x * NT + t) * NS + s]);
        // round to TF32 (nearest, ties away: cvt.rna) -- the device splits G the same way
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u = (u + 0x1000u) & 0xffffe000u;
        float hi;
        std::memcpy(&hi, &u, 4);
        const int k = x * C::NSP8 + s;
        const int idx = umma_kmajor_offset(t, k, C::NPAD) / 4;
        out.bhi[idx] = hi;
        out.blo[idx] = v - hi;
      }
  out.xg.assign(static_cast<size_t>(3) * NT * C::NSP8, 0.f);
  for (int y = 0; y < 3; ++y)
    for (int t = 0; t < NT; ++t)
      for (int s = 0; s < NS; ++s) out.xg[(y * NT + t) * C::NSP8 + s] = static_cast<float>(X[(y * NT + t) * NS + s]);
  out.yline.assign(2 * NZ * NV, 0.f);
  out.z.assign(NZ, 0.0);
  for (int z = 0; z < NZ; ++z) {
    for (int a = 0; a < NV; ++a) {
      out.yline[2 * (z * NV + a)] = static_cast<float>(PHI(z * NS, 0, a));
      out.yline[2 * (z * NV + a) + 1] = static_cast<float>(PHI(z * NS, 3, a));
    }
    out.z[z] = pts[3 * z * NS + 2];
  }
  return true;
}

template <int P, int FORM>
void go(const LaunchArgs& a, const Tc32Tables& t, cudaStream_t s) {
  using C = Tc32Shape<P>;
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev >= 0 && dev < 64 ? dev : 0];
  int grid = slot.load(std::memory_order_relaxed);
  if (grid == 0) {
    // CTAS resident CTAs per SM by construction (shared memory and TMEM are
    // sized for it; launch bounds cap the registers)
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = std::max(1, sms) * C::CTAS;
    slot.store(grid, std::memory_order_relaxed);
  }
  const unsigned g = static_cast<unsigned>(std::min<int64_t>(a.n_elem, grid));
  sumfact_tc32_kernel<P, FORM><<<g, C::NTHREADS, C::SMEM_BYTES, s>>>(a, t);
}

template <int P>
void attrs_p() {
  cudaFuncSetAttribute(sumfact_tc32_kernel<P, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       Tc32Shape<P>::SMEM_BYTES);
  cudaFuncSetAttribute(sumfact_tc32_kernel<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       Tc32Shape<P>::SMEM_BYTES);
  cudaFuncSetAttribute(sumfact_tc32_kernel<P, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(sumfact_tc32_kernel<P, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

}  // namespace

bool tc32_supported(int p, int ne) { return ne == 1 && p >= 3 && p <= 7; }

bool tc32_build(int p, const double* pts, const double* phi, int n_q, int n_shape, Tc32HostTables& t) {
  switch (p) {
    case 3: return build_p<3>(pts, phi, n_q, n_shape, t);
    case 4: return build_p<4>(pts, phi, n_q, n_shape, t);
    case 5: return build_p<5>(pts, phi, n_q, n_shape, t);
    case 6: return build_p<6>(pts, phi, n_q, n_shape, t);
    case 7: return build_p<7>(pts, phi, n_q, n_shape, t);
  }
  return false;
}

void tc32_attrs(int p) {
  switch (p) {
    case 3: attrs_p<3>(); break;
    case 4: attrs_p<4>(); break;
    case 5: attrs_p<5>(); break;
    case 6: attrs_p<6>(); break;
    case 7: attrs_p<7>(); break;
  }
}

void tc32_launch(int p, bool general, const LaunchArgs& a, const Tc32Tables& t, cudaStream_t s) {
#define PIB_TC_CASE(P) \
  case P: general ? go<P, 1>(a, t, s) : go<P, 0>(a, t, s); break;
  switch (p) {
    PIB_TC_CASE(3)
    PIB_TC_CASE(4)
    PIB_TC_CASE(5)
    PIB_TC_CASE(6)
    PIB_TC_CASE(7)
  }
#undef PIB_TC_CASE
}

}  // namespace pib
