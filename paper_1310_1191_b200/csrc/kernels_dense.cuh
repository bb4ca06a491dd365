// Thread-per-element dense integration (p = 1) and the load-vector kernel.
//
// At p = 1 the element matrix is 6x6 = 36 doubles, so one thread keeps all of
// K in registers and walks the 6 rule points itself (the paper's
// "one element per thread" organisation for the lowest order).  The shape
// table (6 x 4 x 6 doubles) is read from shared memory as warp-wide
// broadcasts; geometry and coefficients arrive as coalesced SoA loads; K
// leaves through a shared-memory transpose so the canonical per-element
// layout is written with contiguous 16-byte stores.
#pragma once

#include "kernels_common.cuh"

namespace pib {

struct DenseTables {
  const double* phi;  // [NQ][4][NSH] (tabulate_shapes order)
  const double* pts;  // [NQ][3]
  const double* w;    // [NQ]
};

// threads (= elements) per CTA: 128 for Laplace; 64 for general tensors,
// whose 2 resident CTAs/SM then interleave their load and compute phases better
template <bool GENERAL>
constexpr int p1_threads() {
  return GENERAL ? 64 : 128;
}
#ifndef PI_P1_MINB  // CTAs per SM of the Laplace thread kernel
#define PI_P1_MINB 4
#endif
#ifndef PI_P1_MINB_GENERAL
#define PI_P1_MINB_GENERAL 2
#endif

// Structural zeros of the reference basis (reference_element.cpp:255-266):
// dof = t*(P+1) + a with triangle monomial t = xi1^e1 xi2^e2 (enumerated by
// total degree d, then e1 = 0..d, reference_element.cpp:195-205) and
// Legendre degree a.  d/dxi1 vanishes iff e1 = 0, d/dxi2 iff e2 = 0 and the
// xi3 derivative iff a = 0; the table holds exact 0.0 there (dm1, dm2 and
// dleg are assigned 0.0, :218-225, :258-259), which the context checks.
template <int P>
struct BasisPattern {
  static constexpr int NV = P + 1;
  // branch-free so the optimiser folds it once the callers' loops unroll
  static constexpr int tri_d(int t) {
    return (t >= 1) + (t >= 3) + (t >= 6) + (t >= 10) + (t >= 15) + (t >= 21) + (t >= 28);
  }
  static constexpr int tri_e1(int t) { return t - tri_d(t) * (tri_d(t) + 1) / 2; }
  static constexpr int tri_e2(int t) { return tri_d(t) - tri_e1(t); }
  static constexpr bool nz(int k, int dof) {
    return k == 0 ? true : k == 1 ? tri_e1(dof / NV) > 0 : k == 2 ? tri_e2(dof / NV) > 0 : (dof % NV) > 0;
  }
};

// Thread per element.  K_ij = sum_q sum_kl phi_k(i) M_kl phi_l(j) with the
// per-point block M (kernels_common.cuh); the basis' structural zeros are
// skipped at compile time (13 of the 24 phi entries per point are non-zero),
// so the contraction costs about half the dense loop nest's FMAs.
// LOAD: also the load vector F_i = sum_q det w_q f phi_0(i, q) (6 more accumulators).
// T = float: the FP32 arithmetic variant (pi_integrate_f32): Jacobian, point
// block, phi, the accumulation, the staging and the stores in FP32 (half the
// registers, staging and output bytes).
template <bool GENERAL, bool LOAD = false, typename T = double>
__global__ void __launch_bounds__(p1_threads<GENERAL>(), GENERAL ? 2 * PI_P1_MINB_GENERAL : PI_P1_MINB)
    p1_thread_kernel(LaunchArgs args, DenseTables tab) {
  constexpr int kP1Threads = p1_threads<GENERAL>();
  constexpr int NQ = 6, NSH = 6, KK = NSH * NSH;
  constexpr bool F32 = sizeof(T) == 4;
  static_assert(!(F32 && LOAD), "fused load vectors are FP64");
  using BP = BasisPattern<1>;
  __shared__ T sPhi[NQ * 4 * NSH];
  __shared__ double sPts[NQ * 3];
  __shared__ double sW[NQ];
  __shared__ __align__(16) double sOut[kP1Threads * KK + kP1Threads];  // 36 KB staging

  const int tid = threadIdx.x;
  for (int i = tid; i < NQ * 4 * NSH; i += kP1Threads) sPhi[i] = static_cast<T>(tab.phi[i]);
  if (tid < NQ * 3) sPts[tid] = tab.pts[tid];
  if (tid < NQ) sW[tid] = tab.w[tid];
  __syncthreads();

  const int64_t e = static_cast<int64_t>(blockIdx.x) * kP1Threads + tid;
  const bool live = e < args.n_elem;
  const int64_t ec = live ? e : args.n_elem - 1;
  // Per-thread edge vectors (and coefficient tensor) in shared memory, odd
  // pitch so a warp's accesses are conflict-free; they alias the output
  // staging buffer, which is only used after the loop.  This keeps the 36
  // accumulators and their operands in registers without spilling.
  constexpr int PITCH = GENERAL ? 37 : 21;
  static_assert(PITCH * kP1Threads <= kP1Threads * KK + kP1Threads, "staging alias");
  double* d = sOut + tid * PITCH;
  double* cf = d + 21;
  {
    double x[18], dd[21];
#pragma unroll
    for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + ec];
    prism_edges(x, dd);
#pragma unroll
    for (int c = 0; c < 21; ++c) d[c] = dd[c];
  }
  if (GENERAL) {
#pragma unroll
    for (int c = 0; c < 16; ++c) cf[c] = args.coeff ? args.coeff[c * args.coeff_ld + ec] : args.cu[c];
  }

  T K[KK];
#pragma unroll
  for (int i = 0; i < KK; ++i) K[i] = T(0);
  double F[LOAD ? NSH : 1];
  const double fe = LOAD ? load_f(args, ec) : 0.0;
#pragma unroll
  for (int i = 0; i < (LOAD ? NSH : 1); ++i) F[i] = 0.0;
  bool inverted = false;

#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    // FP32 variant: the Jacobian and point block in FP32 too (det relative error ~1e-7)
    T M[16];
    const T det = point_block<GENERAL, 1, 1, T>(d, static_cast<T>(sPts[3 * q]), static_cast<T>(sPts[3 * q + 1]),
                                                static_cast<T>(sPts[3 * q + 2]), static_cast<T>(sW[q]), cf, M);
    inverted |= !(det > T(0));
    const T* ph = sPhi + q * 4 * NSH;
    if constexpr (LOAD) {
      const double dwf = det * sW[q] * fe;
#pragma unroll
      for (int i = 0; i < NSH; ++i) F[i] = fma(dwf, ph[i], F[i]);
    }
    constexpr int K0 = GENERAL ? 0 : 1;  // Laplace has no value row
    // G_l(i) = sum_k phi_k(i) M_kl ; K_ij += sum_l G_l(i) phi_l(j)
#pragma unroll
    for (int i = 0; i < NSH; ++i) {
      T g[4];
#pragma unroll
      for (int l = K0; l < 4; ++l) {
        T s = T(0);
#pragma unroll
        for (int k = K0; k < 4; ++k)
          if (BP::nz(k, i)) s = fma(ph[k * NSH + i], M[k * 4 + l], s);
        g[l] = s;
      }
#pragma unroll
      for (int j = GENERAL ? 0 : i; j < NSH; ++j) {
        T s = K[i * NSH + j];
#pragma unroll
        for (int l = K0; l < 4; ++l)
          if (BP::nz(l, j)) s = fma(g[l], ph[l * NSH + j], s);
        K[i * NSH + j] = s;
      }
    }
  }
  if (!GENERAL) {  // Laplace: mirror the strict upper triangle
#pragma unroll
    for (int i = 0; i < NSH; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) K[i * NSH + j] = K[j * NSH + i];
  }
  if (inverted && live) flag_inverted(args.bad, args.element_id_base + e);
  if (LOAD && live) {
#pragma unroll
    for (int i = 0; i < NSH; ++i) args.fout[e * NSH + i] = F[i];
  }

  if (args.out_layout == PI_OUT_SOA) {
    if (live) {
#pragma unroll
      for (int i = 0; i < KK; ++i) store_out(args, i * args.ld_out + e, K[i]);
    }
    return;
  }
  if constexpr (F32) {
    // FP32 staging [thread][36] (odd float2 pitch 19: conflict-free), then the
    // CTA's contiguous block (144 B per element): one TMA bulk store when the
    // output base is 16-byte aligned, else coalesced 8- / 4-byte stores.
    constexpr int P2F = KK / 2 + 1;
    static_assert(kP1Threads * (P2F + KK / 2) <= kP1Threads * KK + kP1Threads, "FP32 staging fits sOut");
    float2* so = reinterpret_cast<float2*>(sOut);
    __syncthreads();  // every thread is done with its edge vectors / coefficients
#pragma unroll
    for (int i = 0; i < KK / 2; ++i) so[tid * P2F + i] = make_float2(K[2 * i], K[2 * i + 1]);
    __syncthreads();
    const int64_t first = static_cast<int64_t>(blockIdx.x) * kP1Threads;
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kP1Threads), args.n_elem - first));
    float2* pk = reinterpret_cast<float2*>(sOut) + kP1Threads * P2F;  // packed image after the padded staging
    for (int i = tid; i < n_here * (KK / 2); i += kP1Threads) pk[i] = so[(i / (KK / 2)) * P2F + i % (KK / 2)];
    __syncthreads();
    const uintptr_t ob = reinterpret_cast<uintptr_t>(args.out32 + first * KK);
    if ((ob & 15) == 0) {
      if (tid == 0) {
        fence_proxy_async_smem();
        bulk_store(reinterpret_cast<double*>(args.out32 + first * KK), reinterpret_cast<const double*>(pk),
                   static_cast<unsigned>(n_here) * KK * 4u);
        bulk_commit();
        bulk_wait_read();
      }
    } else if ((ob & 7) == 0) {
      float2* dst = reinterpret_cast<float2*>(args.out32 + first * KK);
      for (int i = tid; i < n_here * (KK / 2); i += kP1Threads) dst[i] = pk[i];
    } else {
      const float* src = reinterpret_cast<const float*>(pk);
      for (int i = tid; i < n_here * KK; i += kP1Threads) args.out32[first * KK + i] = src[i];
    }
    return;
  } else {
  // Canonical: stage [thread][36] in smem (odd stride in 16B units avoids
  // bank conflicts: 36 doubles = 18 x 16 B), then write the CTA's contiguous
  // block of 128 * 288 B with coalesced 16-byte stores.
  double2* so2 = reinterpret_cast<double2*>(sOut);
  __syncthreads();  // every thread is done with its edge vectors / coefficients
#pragma unroll
  for (int i = 0; i < KK / 2; ++i) so2[tid * (KK / 2) + i] = make_double2(K[2 * i], K[2 * i + 1]);
  __syncthreads();
  const int64_t first = static_cast<int64_t>(blockIdx.x) * kP1Threads;
  const int64_t n_here = min(static_cast<int64_t>(kP1Threads), args.n_elem - first);
  const int total2 = static_cast<int>(n_here) * (KK / 2);
  if (args.out32) {
    if ((reinterpret_cast<uintptr_t>(args.out32) & 7) == 0) {
      float2* dst = reinterpret_cast<float2*>(args.out32 + first * KK);
      for (int i = tid; i < total2; i += kP1Threads)
        dst[i] = make_float2(static_cast<float>(so2[i].x), static_cast<float>(so2[i].y));
    } else {  // 4-byte aligned output base
      const double* so = sOut;
      for (int i = tid; i < 2 * total2; i += kP1Threads) args.out32[first * KK + i] = static_cast<float>(so[i]);
    }
  } else {
#ifndef PI_P1_NO_BULK
    // the staging is the tile's exact global image: one TMA bulk store (16-byte
    // aligned when the output base is; 288 B per element)
    if ((reinterpret_cast<uintptr_t>(args.out) & 15) == 0) {
      if (tid == 0) {
        fence_proxy_async_smem();
        bulk_store(args.out + first * KK, sOut, static_cast<unsigned>(n_here) * KK * 8u);
        bulk_commit();
        bulk_wait_read();  // the CTA's shared memory must outlive the copy
      }
      return;
    }
#endif
    if ((reinterpret_cast<uintptr_t>(args.out) & 15) == 0) {
      double2* dst = reinterpret_cast<double2*>(args.out + first * KK);
      for (int i = tid; i < total2; i += kP1Threads) dst[i] = so2[i];
    } else {  // 8-byte aligned output base
      for (int i = tid; i < 2 * total2; i += kP1Threads) args.out[first * KK + i] = sOut[i];
    }
  }
  }
}

// Load vectors: F_i = sum_q det_q w_q f phi_i(q) (value row).  One warp per
// element: lanes split the shape functions; det*w per point is computed once
// per element into shared memory.
constexpr int kLoadWarps = 4;
__global__ void __launch_bounds__(32 * kLoadWarps)
    load_vector_kernel(LaunchArgs args, DenseTables tab, int nq, int nsh, const double* f, double f_const) {
  extern __shared__ double sdw[];  // [kLoadWarps][nq]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kLoadWarps + warp;
  if (e >= args.n_elem) return;
  double x[18];
#pragma unroll
  for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];
  const double fe = f ? f[e] : f_const;
  double* dw = sdw + warp * nq;
  bool inverted = false;
  for (int q = lane; q < nq; q += 32) {
    double inv[3][3];
    const double det = prism_jacobian(x, tab.pts[3 * q], tab.pts[3 * q + 1], tab.pts[3 * q + 2], inv);
    inverted |= !(det > 0.0);
    dw[q] = det * tab.w[q] * fe;
  }
  if (__any_sync(0xffffffffu, inverted) && lane == 0) flag_inverted(args.bad, args.element_id_base + e);
  __syncwarp();
  for (int i = lane; i < nsh; i += 32) {
    double s = 0.0;
    for (int q = 0; q < nq; ++q) s += dw[q] * tab.phi[static_cast<int64_t>(q) * 4 * nsh + i];
    args.out[e * nsh + i] = s;
  }
}

// Load vectors at p = 1 (no tensor tables): thread per element, det at the 6
// rule points, F staged per CTA and stored as one contiguous block.
constexpr int kLoadP1Threads = 128;
__global__ void __launch_bounds__(kLoadP1Threads)
    load_vector_p1_kernel(LaunchArgs args, DenseTables tab, const double* f, double f_const) {
  constexpr int NQ = 6, NSH = 6;
  __shared__ double sPhi0[NQ * NSH], sPts[NQ * 3], sW[NQ];
  __shared__ double sF[kLoadP1Threads * NSH];
  const int tid = threadIdx.x;
  if (tid < NQ * NSH) sPhi0[tid] = tab.phi[(tid / NSH) * 4 * NSH + tid % NSH];  // value row phi_0(i, q)
  if (tid < NQ * 3) sPts[tid] = tab.pts[tid];
  if (tid < NQ) sW[tid] = tab.w[tid];
  __syncthreads();
  const int64_t first = static_cast<int64_t>(blockIdx.x) * kLoadP1Threads, e = first + tid;
  if (e < args.n_elem) {
    double x[18], d[21];
#pragma unroll
    for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];
    prism_edges(x, d);
    const double fe = f ? f[e] : f_const;
    double F[NSH] = {0, 0, 0, 0, 0, 0};
    bool inverted = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double det = jacobian_det(d, sPts[3 * q], sPts[3 * q + 1], sPts[3 * q + 2]);
      inverted |= !(det > 0.0);
      const double dw = det * sW[q] * fe;
#pragma unroll
      for (int i = 0; i < NSH; ++i) F[i] = fma(dw, sPhi0[q * NSH + i], F[i]);
    }
    if (inverted) flag_inverted(args.bad, args.element_id_base + e);
#pragma unroll
    for (int i = 0; i < NSH; ++i) sF[tid * NSH + i] = F[i];
  }
  __syncthreads();
  const int n_here = static_cast<int>(min(static_cast<int64_t>(kLoadP1Threads), args.n_elem - first));
  for (int i = tid; i < n_here * NSH; i += kLoadP1Threads) args.out[first * NSH + i] = sF[i];
}

// Load vectors through the tensor-product structure (p >= 2 with the
// sum-factorisation tables): phi_0(t*NV + a, (s, z)) = m_t(s) P_a(z), so
//     F(t,a) = sum_s X_2(t,s) u(s,a),   u(s,a) = sum_z P_a(z) dw(s,z),
// dw = det w f at every rule point (q = z*NS + s, reference order).  A CTA
// takes kLoadSfElems elements: (1) coalesced SoA geometry into shared memory,
// (2) one thread per (element, triangle point s) walks the NZ Gauss points:
// det, dw and u(s, .) in registers, (3) one thread per (element, dof) forms F
// and stores it (consecutive dofs of consecutive elements: coalesced).  Per
// element: 144 B of geometry (+8 B of f) read, 8 N_sh bytes written, N_q
// determinants -- HBM-bound at low p, FP64-bound at high p; the per-p tables
// are a few KB and stay in L1.
struct LoadSfTables {
  const double* tri;     // xi1 [NS], xi2 [NS]
  const double* yline;   // (P, P') [NZ][NV] pairs, xi3 [NZ]
  const double* xplain;  // X as [NSP][3][ntps]; y = 2 is m_t(s)
  const double* w;       // [NQ] reference order
  int ns, nz, nv, nt, ntps;
};
constexpr int kLoadSfThreads = 256;
// elements per CTA: 64 at p <= 4, fewer where u (NS x NV per element) grows
constexpr int load_sf_elems(int ns, int nv) { return ns * nv <= 80 ? 64 : ns * nv <= 150 ? 32 : 16; }
constexpr size_t load_sf_smem(int ns, int nv) {
  return sizeof(double) * (18 * (load_sf_elems(ns, nv) + 1) + load_sf_elems(ns, nv) * ns * nv);
}
// P: the degree (compile-time loop bounds: the kernel is instruction-issue
// bound, ~160 warp instructions per element with runtime bounds at p = 2)
template <int P>
__global__ void __launch_bounds__(kLoadSfThreads)
    load_vector_sf_kernel(LaunchArgs args, LoadSfTables tb, const double* f, double f_const) {
  constexpr int nv = P + 1, nz = P + 1, nt = (P + 1) * (P + 2) / 2, nsh = nt * nv;
  constexpr int ns = P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : P == 5 ? 25 : P == 6 ? 33 : 42;
  constexpr int kLoadSfElems = load_sf_elems(ns, nv), kLoadSfPitch = kLoadSfElems + 1;
  extern __shared__ __align__(16) double sl[];
  double* sX = sl;                          // vertices [18][kLoadSfPitch]
  double* sU = sX + 18 * kLoadSfPitch;      // u [E][ns][nv]
  const int tid = threadIdx.x;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * kLoadSfElems;
  const int64_t left = args.n_elem - e0;
  const int ne = left < kLoadSfElems ? static_cast<int>(left) : kLoadSfElems;
  for (int i = tid; i < 18 * kLoadSfElems; i += kLoadSfThreads) {
    const int c = i / kLoadSfElems, el = i % kLoadSfElems;
    if (el < ne) sX[c * kLoadSfPitch + el] = args.geom[c * args.geom_ld + e0 + el];
  }
  __syncthreads();
  for (int i = tid; i < ne * ns; i += kLoadSfThreads) {
    const int el = i / ns, s = i - el * ns;
    double x[18], d[21];
#pragma unroll
    for (int c = 0; c < 18; ++c) x[c] = sX[c * kLoadSfPitch + el];
    prism_edges(x, d);
    const double fe = f ? f[e0 + el] : f_const;
    const double xi1 = __ldg(tb.tri + s), xi2 = __ldg(tb.tri + ns + s);
    double u[nv];
#pragma unroll
    for (int a = 0; a < nv; ++a) u[a] = 0.0;
    bool inverted = false;
#pragma unroll
    for (int z = 0; z < nz; ++z) {
      const double det = jacobian_det(d, xi1, xi2, __ldg(tb.yline + 2 * nv * nz + z));
      inverted |= !(det > 0.0);
      const double dw = det * __ldg(tb.w + z * ns + s) * fe;
#pragma unroll
      for (int a = 0; a < nv; ++a) u[a] = fma(__ldg(tb.yline + 2 * (z * nv + a)), dw, u[a]);
    }
    if (inverted) flag_inverted(args.bad, args.element_id_base + e0 + el);
#pragma unroll
    for (int a = 0; a < nv; ++a) sU[(el * ns + s) * nv + a] = u[a];
  }
  __syncthreads();
  // thread = (element, t): the nv values F(t, .) share each X_2(t, s) load
  for (int i = tid; i < ne * nt; i += kLoadSfThreads) {
    const int el = i / nt, t = i - el * nt;
    const double* u = sU + el * ns * nv;
    double acc[nv];
#pragma unroll
    for (int a = 0; a < nv; ++a) acc[a] = 0.0;
#pragma unroll 4
    for (int s = 0; s < ns; ++s) {
      const double x2 = __ldg(tb.xplain + (s * 3 + 2) * tb.ntps + t);
#pragma unroll
      for (int a = 0; a < nv; ++a) acc[a] = fma(x2, u[s * nv + a], acc[a]);
    }
    double* dst = args.out + (e0 + el) * nsh + t * nv;
#pragma unroll
    for (int a = 0; a < nv; ++a) dst[a] = acc[a];
  }
}

}  // namespace pib
