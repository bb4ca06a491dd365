// Template host side of the sum-factorised kernels: table construction,
// launch attributes and the persistent-grid launch for one (P, NE).
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>

#include "kernels_pairs.cuh"
#include "kernels_sumfact.cuh"
#include "sumfact_api.hpp"

namespace pib {

constexpr int kMaxDevices = 64;

// Persistent grid of a kernel on the current device: SMs x resident CTAs per
// SM, computed once per (kernel, device) -- a per-device cache that host
// threads driving different GPUs (pi_integrate_host_multi) share safely.
template <typename K>
int persistent_grid(std::atomic<int>* cache, K kernel, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev >= 0 && dev < kMaxDevices ? dev : 0];
  int c = slot.load(std::memory_order_relaxed);
  if (c == 0) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) {
      cudaGetLastError();
      per_sm = 1;
    }
    c = std::max(1, std::max(1, sms) * std::max(1, per_sm));
    slot.store(c, std::memory_order_relaxed);
  }
  return c;
}

template <int P, int NE>
struct SumFactHost {
  using C = SumFactConfig<P, NE>;         // tables; the general-form kernels
  using CS = SumFactConfig<P, NE, true>;  // the symmetric-form kernels
  static_assert(C::TMAJOR == CS::TMAJOR && C::XPLAIN == CS::XPLAIN && C::XPLAIN_TOTAL == CS::XPLAIN_TOTAL &&
                    C::XFRAG == CS::XFRAG,
                "both launch shapes of a (p, n_eq) read the same tables");
  template <bool SYM>
  using CK = SumFactConfig<P, NE, SYM>;
  template <int FORM, bool SYM>
  static void attr() {
    cudaFuncSetAttribute(sumfact_kernel<P, NE, FORM, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_bytes<SYM>(NE == 1)));
  }
  // dynamic shared memory of a launch (fused load vectors: the dw / u region after the rest)
  template <bool SYM>
  static constexpr size_t smem_bytes(bool load) {
    return load ? CK<SYM>::SMEM_BYTES_LOAD : CK<SYM>::SMEM_BYTES;
  }
  static_assert(NE != 1 || (CK<false>::SMEM_BYTES_LOAD <= 232448 && CK<true>::SMEM_BYTES_LOAD <= 232448),
                "fused load-vector region must fit the SM");
  // Persistent grid: as many CTAs as fit on the device at once (queried per
  // instantiation), each looping over (element group, a'-group, column block) items.
  template <int FORM, bool SYM>
  static int resident_ctas(bool load) {
    static std::atomic<int> cache[2][kMaxDevices] = {};
    return persistent_grid(cache[load], sumfact_kernel<P, NE, FORM, SYM>, CK<SYM>::NTHREADS, smem_bytes<SYM>(load));
  }
  // symmetric forms at high p: the pair-split kernel (kernels_pairs.cuh)
  // (measured: faster for scalar forms at p >= 5; slower for n_eq = 3, whose
  // per-chunk M blocks the pair items would rebuild per item)
#ifndef PI_PAIRS_MINP
#define PI_PAIRS_MINP 5
#endif
  static constexpr bool kPairs = NE == 1 && P >= PI_PAIRS_MINP;
  template <int FORM>
  static void attr_pairs() {
    if constexpr (kPairs) {
      static_assert(PairsConfig<P, NE>::SMEM_BYTES_LOAD <= 232448, "fused load-vector region must fit the SM");
      cudaFuncSetAttribute(sumfact_pairs_kernel<P, NE, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(PairsConfig<P, NE>::SMEM_BYTES_LOAD));
    }
  }
  template <int FORM>
  static bool go_pairs(const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
    if constexpr (kPairs) {
      using PC = PairsConfig<P, NE>;
      static std::atomic<int> cache[2][kMaxDevices] = {};
      const bool load = a.fout != nullptr;
      const size_t smem = load ? PC::SMEM_BYTES_LOAD : PC::SMEM_BYTES;
      const int c = persistent_grid(cache[load], sumfact_pairs_kernel<P, NE, FORM>, PC::NTHREADS, smem);
      const dim3 grid(static_cast<unsigned>(std::min<int64_t>(a.n_elem, c)));  // element-major CTAs
      sumfact_pairs_kernel<P, NE, FORM><<<grid, PC::NTHREADS, smem, s>>>(a, t);
      return true;
    }
    return false;
  }
  template <int FORM, bool SYM>
  static void go(const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
#ifndef PI_NO_PAIRS
    if constexpr (SYM)
      if (go_pairs<FORM>(a, t, s)) return;
#endif
    using K = CK<SYM>;
    const bool load = NE == 1 && a.fout != nullptr;
    const int64_t items = (a.n_elem + K::EPC - 1) / K::EPC * K::NITEM;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>(items, resident_ctas<FORM, SYM>(load))));
    sumfact_kernel<P, NE, FORM, SYM><<<grid, K::NTHREADS, smem_bytes<SYM>(load), s>>>(a, t);
  }

  // Builds the X fragment table, Y table and rule coordinates from the
  // caller's rule and shape table; false if the table is not the tensor
  // product the kernel factorises.
  static bool build(const double* pts, const double* phi, int n_q, int n_shape, SumFactHostTables& out) {
    constexpr int NS = C::NS, NZ = C::NZ, NV = C::NV, NT = C::NT, NSH1 = NT * NV;
    if (n_q != NS * NZ || n_shape != NSH1) return false;
    auto PHI = [&](int q, int k, int dof) { return phi[(static_cast<size_t>(q) * 4 + k) * NSH1 + dof]; };
    for (int z = 0; z < NZ; ++z)
      for (int s = 0; s < NS; ++s) {
        const int q = z * NS + s;
        if (pts[3 * q] != pts[3 * s] || pts[3 * q + 1] != pts[3 * s + 1] || pts[3 * q + 2] != pts[3 * z * NS + 2])
          return false;
      }
    out.tri.assign(2 * NS, 0.0);
    for (int s = 0; s < NS; ++s) {
      out.tri[s] = pts[3 * s];
      out.tri[NS + s] = pts[3 * s + 1];
    }
    // Y: [NZ][NV] pairs (P_a(z), P'_a(z)), P_a(z) = phi_0((t=0,a), (s=0,z)), P'_a(z) = phi_3((0,a),(0,z)) since m_0 = 1.
    auto& yl = out.yline;
    yl.assign(2 * NV * NZ + NZ, 0.0);
    for (int a = 0; a < NV; ++a)
      for (int z = 0; z < NZ; ++z) {
        yl[2 * (z * NV + a)] = PHI(z * NS, 0, a);      // (P, P') interleaved: one 16-byte load
        yl[2 * (z * NV + a) + 1] = PHI(z * NS, 3, a);
      }
    for (int z = 0; z < NZ; ++z) yl[2 * NV * NZ + z] = pts[3 * z * NS + 2];
    yl.resize((yl.size() + 1) / 2 * 2, 0.0);  // 16-byte multiple for the TMA bulk copy
    // X_x(t,s): x=0 dm/dxi1, 1 dm/dxi2, 2 m, read at a=0 (P_0 = 1), z=0.
    std::vector<double> X(static_cast<size_t>(3) * NT * NS);
    for (int t = 0; t < NT; ++t)
      for (int s = 0; s < NS; ++s) {
        X[(0 * NT + t) * NS + s] = PHI(s, 1, t * NV);
        X[(1 * NT + t) * NS + s] = PHI(s, 2, t * NV);
        X[(2 * NT + t) * NS + s] = PHI(s, 0, t * NV) / PHI(s, 0, 0);
      }
    // Structure check: phi_k(i,q) == X(t,s) Y(a,z) to rounding.
    double worst = 0.0, scale = 0.0;
    for (int z = 0; z < NZ; ++z)
      for (int s = 0; s < NS; ++s)
        for (int t = 0; t < NT; ++t)
          for (int a = 0; a < NV; ++a) {
            const int q = z * NS + s, dof = t * NV + a;
            const double Pz = yl[2 * (z * NV + a)], D = yl[2 * (z * NV + a) + 1];
            const double m = X[(2 * NT + t) * NS + s];
            const double ref[4] = {m * Pz, X[(0 * NT + t) * NS + s] * Pz, X[(1 * NT + t) * NS + s] * Pz, m * D};
            for (int k = 0; k < 4; ++k) {
              worst = std::max(worst, std::fabs(PHI(q, k, dof) - ref[k]));
              scale = std::max(scale, std::fabs(ref[k]));
            }
          }
    if (worst > 1e-13 * std::max(1.0, scale)) return false;
    out.xfrag.assign(C::XFRAG, 0.0);
    for (int mt = 0; mt < C::MT; ++mt)
      for (int ks = 0; ks < C::KSTEPS; ++ks)
        for (int lane = 0; lane < 32; ++lane) {
          const int t = mt * 8 + lane / 4, kx = ks * 4 + lane % 4;
          const int s = kx / 3, x = kx % 3;
          double v = 0.0;
          if (t < NT && s < NS) v = X[(x * NT + t) * NS + s];
          out.xfrag[(mt * C::KSTEPS + ks) * 32 + lane] = v;
        }
    out.xplain.assign(C::XPLAIN_TOTAL, 0.0);
    out.ntps = C::NTPS;
    for (int s = 0; s < NS; ++s)
      for (int t = 0; t < NT; ++t)
        for (int x = 0; x < 3; ++x) {
          out.xplain[(static_cast<size_t>(s) * 3 + x) * C::NTPS + t] = X[(x * NT + t) * NS + s];
          if (C::XP4) out.xplain[C::XPLAIN + (static_cast<size_t>(s) * C::NTP + t) * 4 + x] = X[(x * NT + t) * NS + s];
        }
    return true;
  }

  // Fraction of the (t, t') pairs whose MMA tiles the symmetric path computes
  // (t'-major skips t'-blocks below the t-block; natural order skips n-tiles
  // whose largest t' lies below the m-tile).
  static double sym_fraction() {
    if (CS::NAG != 1 || CS::NCB != 1) return 1.0;
    if (CS::PAIRS) {
      // (a', b') pairs with a' <= b' (kernels_sumfact.cuh PAIRS)
      const double mt = CS::MT, nve = CS::NVE;
      return (nve * mt * (mt + 1) / 2 + nve * (nve - 1) / 2 * mt * mt) / (nve * nve * mt * mt);
    }
    long done = 0;
    for (int t = 0; t < CS::NT; ++t)
      for (int tp = 0; tp < CS::NT; ++tp) {
        const int mt = t / 8;
        bool comp;
        if (CS::TMAJOR) {
          comp = tp / 8 >= mt;
        } else {
          const int nt = (tp * CS::NVE) / 8;
          comp = std::min(CS::NT - 1, (nt * 8 + 7) / CS::NVE) >= 8 * mt;
        }
        done += comp;
      }
    return static_cast<double>(done) / (CS::NT * CS::NT);
  }
  // fraction of the B-fragment values the symmetric path forms (PAIRS: a' <= b')
  static double fragment_fraction() {
    if (CS::PAIRS) return (CS::NVE + 1) / (2.0 * CS::NVE);
    return 1.0;
  }
  static void padded(int& cols, int& rows, int& k4) {
    cols = C::NTILE * 8;
    rows = C::MT * 8;
    k4 = C::KSTEPS * 4;
  }
};

}  // namespace pib
