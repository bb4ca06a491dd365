// p = 2: dense per-point accumulation with the basis' structural zeros
// skipped at compile time, lane = element.
//
// At p = 2 the sum-factorised MMA path feeds each tensor-core fragment from
// three shared-memory loads (the triangle factor has only 6 rows, so every
// G value is used by one MMA) and is shared-memory bound.  The dense loop
// nest of integrate_generic (integrate_ref.cpp:72-89) in reference
// coordinates, K_ij += sum_kl phi_k(i) M_kl phi_l(j), is cheaper here once
// the zeros of the reference basis are skipped (BasisPattern: 2/3 of the
// d/dxi entries vanish on average), so it runs on the FP64 FMA pipe:
//
//  * a CTA integrates groups of 32 elements; lane l of every warp owns
//    element l of the group;
//  * symmetric tensors: warp w (of 9) owns the upper-triangle parts of K
//    rows w and 17-w (19 accumulators, mirrored at the store); general
//    tensors: warp w (of 18) owns row w (18 accumulators);
//  * the per-point blocks M (kernels_common.cuh) of the 18 rule points are
//    computed once per element into shared memory;
//  * phi is read with warp-uniform addresses from the constant bank;
//  * element matrices leave through shared-memory staging (reusing the M
//    buffer) as contiguous, coalesced blocks.
#pragma once

#include "kernels_common.cuh"
#include "kernels_dense.cuh"

namespace pib {

constexpr int kP2NQ = 18, kP2NSH = 18, kP2KK = kP2NSH * kP2NSH;
// The context's rule and shape table travel with every launch as a kernel
// parameter (constant bank 0, warp-uniform reads like __constant__), so
// contexts with different tables never race on a shared symbol.
struct P2Tables {
  double phi[kP2NQ * 4 * kP2NSH];  // tabulate_shapes order [q][k][dof]
  double pts[kP2NQ * 4];           // xi1, xi2, xi3, w
  float phif[kP2NQ * 4 * kP2NSH];  // the same table in FP32 (FP32 arithmetic variant)
};

// Compute type T: double (the 1e-12 path) or float (FP32 variant, bound 5e-5).
template <typename T>
__device__ __forceinline__ const T* p2_phi(const P2Tables& tb);
template <>
__device__ __forceinline__ const double* p2_phi<double>(const P2Tables& tb) {
  return tb.phi;
}
template <>
__device__ __forceinline__ const float* p2_phi<float>(const P2Tables& tb) {
  return tb.phif;
}

// staged element pitch: 16-byte multiple (TMA bulk stores of whole elements),
// 2-way bank conflicts at most for the staging writes
constexpr int kP2Pitch = kP2KK + 2;
constexpr int kP2Half = 16;  // elements per bulk-store half (symmetric kernel)
#ifdef PI_P2_ONEHALF  // A/B: one round of 32 element stores (2.5 % slower, Laplace)
constexpr bool kP2OneHalf = true;
#else
constexpr bool kP2OneHalf = false;
#endif

// GENERAL: full 4x4 tensor (uniform in args.cu, or per element in
// args.coeff); SYM: the tensor is symmetric, so K is (upper triangle only).
//  SYM:  9 warps, warp w owns rows (w, 17-w)  -> 19 accumulators per lane;
//  !SYM: 18 warps, warp w owns row w          -> 18 accumulators per lane.
template <bool GENERAL, bool SYM>
struct P2Cfg {
  static constexpr int NW = SYM ? 9 : 18;
  static constexpr int NACC = SYM ? kP2NSH + 1 : kP2NSH;
  static constexpr int NTHREADS = 32 * NW;
  static constexpr int NM = GENERAL ? 16 : 6;            // stored M entries per point
#ifndef PI_P2_ROUND_SYM
#define PI_P2_ROUND_SYM 32
#endif
#ifndef PI_P2_ROUND_GEN
#define PI_P2_ROUND_GEN 32
#endif
  // elements staged per output round (32: the whole group, one round)
  static constexpr int ROUND = SYM ? PI_P2_ROUND_SYM : PI_P2_ROUND_GEN;
  static constexpr int MBUF = kP2NQ * NM * 32;           // doubles
  static constexpr int SBUF = ROUND * kP2Pitch;
  static constexpr int BUF = MBUF > SBUF ? MBUF : SBUF;
  static constexpr int OFF_D = BUF;                      // edge vectors [21][32]
  static constexpr int OFF_G = OFF_D + 21 * 32;          // raw geometry, double buffered [2][18][32]
  static constexpr int OFF_C = OFF_G + 2 * 18 * 32;      // coefficients, double buffered [2][16][32]
  static constexpr int SMEM_DOUBLES = OFF_C + (GENERAL ? 2 * 16 * 32 : 0);
  static constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);
  // fused load vectors: det w f per (point, lane) after the rest
  static constexpr int OFF_DW = SMEM_DOUBLES;
  static constexpr size_t SMEM_BYTES_LOAD = (SMEM_DOUBLES + kP2NQ * 32) * sizeof(double);
  // per-SMSP register file (16K regs; warps dealt round-robin to the 4 SMSPs):
  // 9-warp CTAs x3 need <= 72 registers, one 18-warp CTA <= 96
  // per-SMSP register file (16K regs; warps dealt round-robin to the 4 SMSPs):
  // 9-warp CTAs x3 need <= 72 registers, one 18-warp CTA <= 96
  static constexpr int MAXREG = SYM ? 72 : 96;
};

// M entry (k, l) of the lane's element at point q; Laplace stores the
// symmetric 3x3 derivative block [11, 12, 13, 22, 23, 33].
template <bool GENERAL>
__device__ __forceinline__ int p2_mslot(int k, int l) {
  if (GENERAL) return k * 4 + l;
  const int a = (k < l ? k : l) - 1, b = (k < l ? l : k) - 1;
  return a == 0 ? b : (a == 1 ? 2 + b : 5);
}

// Symmetric tensors: warp w owns the upper-triangle parts of rows w and 17 - w
// (19 accumulators).  Dealing rows by their per-point cost instead (the
// busiest warp 48 FMAs per point instead of 53) needs up to 31 accumulators
// and measured 2.3x slower: the register budget drops the kernel to one CTA
// per SM.
__host__ __device__ constexpr int p2_sym_row(int w, int r) { return r == 0 ? w : r == 1 ? 17 - w : -1; }
template <bool SYM, int W>
__device__ __forceinline__ constexpr int p2_nr() {
  return !SYM ? 1 : (p2_sym_row(W, 2) >= 0 ? 3 : p2_sym_row(W, 1) >= 0 ? 2 : 1);
}
template <bool SYM, int W>
__device__ __forceinline__ constexpr int p2_row(int r) {
  return SYM ? p2_sym_row(W, r) : W;
}

// The warp's rows over all rule points.
template <typename T, bool GENERAL, bool SYM, int W>
__device__ __forceinline__ void p2_rows(const P2Tables& tb, const T* __restrict__ sM, int lane, T* acc) {
  using BP = BasisPattern<2>;
  using C = P2Cfg<GENERAL, SYM>;
  constexpr int K0 = GENERAL ? 0 : 1, NR = p2_nr<SYM, W>(), NM = C::NM;
#pragma unroll 1
  for (int q = 0; q < kP2NQ; ++q) {
    const T* ph = p2_phi<T>(tb) + q * 4 * kP2NSH;
    const T* mq = sM + q * NM * 32 + lane;
    // G_l(i) = sum_k phi_k(i) M_kl, M read one row k at a time (only the
    // rows k the warp's basis functions do not annihilate)
    T g[NR][4];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int l = 0; l < 4; ++l) g[r][l] = T(0);
#pragma unroll
    for (int k = K0; k < 4; ++k) {
      bool need = false;
#pragma unroll
      for (int r = 0; r < NR; ++r) need = need || BP::nz(k, p2_row<SYM, W>(r));
      if (!need) continue;
      T mk[4];
#pragma unroll
      for (int l = K0; l < 4; ++l) mk[l] = mq[p2_mslot<GENERAL>(k, l) * 32];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = p2_row<SYM, W>(r);
        if (BP::nz(k, i)) {
          const T f = ph[k * kP2NSH + i];
#pragma unroll
          for (int l = K0; l < 4; ++l) g[r][l] = fma(f, mk[l], g[r][l]);
        }
      }
    }
    int off = 0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int i = p2_row<SYM, W>(r);
#pragma unroll
      for (int j = SYM ? i : 0; j < kP2NSH; ++j) {
        T s = acc[off + j - (SYM ? i : 0)];
#pragma unroll
        for (int l = K0; l < 4; ++l)
          if (BP::nz(l, j)) s = fma(g[r][l], ph[l * kP2NSH + j], s);
        acc[off + j - (SYM ? i : 0)] = s;
      }
      off += SYM ? kP2NSH - i : kP2NSH;
    }
  }
}

// General (non-symmetric) tensors: every warp owns one full row i (runtime,
// warp-uniform), so all 18 warps run the same instruction stream: G is
// formed densely from the warp-uniform phi_k(i), the column loop skips the
// structural zeros of phi_l(j) at compile time.
template <typename T>
__device__ __forceinline__ void p2_row_general(const P2Tables& tb, const T* __restrict__ sM, int lane, int i, T* acc) {
  using BP = BasisPattern<2>;
#pragma unroll 1
  for (int q = 0; q < kP2NQ; ++q) {
    const T* ph = p2_phi<T>(tb) + q * 4 * kP2NSH;
    const T* mq = sM + q * 16 * 32 + lane;
    T g[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T f = ph[k * kP2NSH + i];
      if (f != T(0)) {  // warp-uniform: skips the M rows the basis function annihilates
#pragma unroll
        for (int l = 0; l < 4; ++l) g[l] = fma(f, mq[(k * 4 + l) * 32], g[l]);
      }
    }
#pragma unroll
    for (int j = 0; j < kP2NSH; ++j) {
      T s = acc[j];
#pragma unroll
      for (int l = 0; l < 4; ++l)
        if (BP::nz(l, j)) s = fma(g[l], ph[l * kP2NSH + j], s);
      acc[j] = s;
    }
  }
}

// Writes the lane's accumulators as rows of its staged element matrix.
template <bool SYM, int W, typename T>
__device__ __forceinline__ void p2_stage(T* st, const T* acc) {
  constexpr int NR = p2_nr<SYM, W>();
  int off = 0;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int i = p2_row<SYM, W>(r);
#pragma unroll
    for (int j = SYM ? i : 0; j < kP2NSH; ++j) {
      const T v = acc[off + j - (SYM ? i : 0)];
      st[i * kP2NSH + j] = v;
      if (SYM && j > i) st[j * kP2NSH + i] = v;
    }
    off += SYM ? kP2NSH - i : kP2NSH;
  }
}

template <bool SYM, int W, typename T>
__device__ __forceinline__ void p2_store_soa(const LaunchArgs& args, int64_t e, const T* acc) {
  constexpr int NR = p2_nr<SYM, W>();
  int off = 0;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int i = p2_row<SYM, W>(r);
#pragma unroll
    for (int j = SYM ? i : 0; j < kP2NSH; ++j) {
      const double v = acc[off + j - (SYM ? i : 0)];
      store_out(args, (i * kP2NSH + j) * args.ld_out + e, v);
      if (SYM && j > i) store_out(args, (j * kP2NSH + i) * args.ld_out + e, v);
    }
    off += SYM ? kP2NSH - i : kP2NSH;
  }
}

// warp -> compile-time row set (only the NW cases of the instantiation are
// emitted, keeping the kernel within the instruction cache)
// warp -> compile-time row pair (symmetric tensors)
#define P2_WARP_SWITCH(CALL) \
  switch (warp) {            \
    case 0: CALL(0); break;  \
    case 1: CALL(1); break;  \
    case 2: CALL(2); break;  \
    case 3: CALL(3); break;  \
    case 4: CALL(4); break;  \
    case 5: CALL(5); break;  \
    case 6: CALL(6); break;  \
    case 7: CALL(7); break;  \
    default: CALL(8); break; \
  }

// LOAD (FP64 only): also the load vector F_i = sum_q det w_q f phi_0(i, q);
// det w f per point is kept from the M pass, each warp sums its own rows.
template <bool GENERAL, bool SYM, typename T = double, bool LOAD = false>
__global__ void __maxnreg__((P2Cfg<GENERAL, SYM>::MAXREG)) p2_lane_kernel(const __grid_constant__ LaunchArgs args,
                                                                         const __grid_constant__ P2Tables tb) {
  using C = P2Cfg<GENERAL, SYM>;
  extern __shared__ __align__(16) double p2_smem[];
  T* sM = reinterpret_cast<T*>(p2_smem);  // M [q][NM][32], then the output staging (same byte size as FP64)
  double* sD = p2_smem + C::OFF_D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t groups = (args.n_elem + 31) / 32;
  // FP64 canonical output: whole staged elements leave by TMA bulk stores
  // (measured: faster for the 9-warp symmetric kernel, slower for the 18-warp one)
  const bool bulk = SYM && C::ROUND == 32 && !args.out32 && args.out_layout == PI_OUT_CANONICAL &&
                    (reinterpret_cast<uintptr_t>(args.out) & 15) == 0;
  // The next group's geometry (warp 0) and coefficients (warp 1) stream into
  // shared memory with cp.async while the current group is integrated; each
  // lane copies and later reads its own element's values.
  auto prefetch = [&](int64_t g, int buf) {
    const int64_t ec = min(g * 32 + lane, args.n_elem - 1);
    if (warp == 0) {
      double* dst = p2_smem + C::OFF_G + buf * 18 * 32 + lane;
#pragma unroll
      for (int c = 0; c < 18; ++c) cp_async8(dst + c * 32, args.geom + c * args.geom_ld + ec);
    } else if (GENERAL && warp == 1 && args.coeff) {
      double* dst = p2_smem + C::OFF_C + buf * 16 * 32 + lane;
#pragma unroll
      for (int c = 0; c < 16; ++c) cp_async8(dst + c * 32, args.coeff + c * args.coeff_ld + ec);
    }
    cp_async_commit();
  };
  if (blockIdx.x < groups) prefetch(blockIdx.x, 0);
  int buf = 0;
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x, buf ^= 1) {
    const int64_t e = g * 32 + lane;
    const bool live = e < args.n_elem;
    if (g + gridDim.x < groups) prefetch(g + gridDim.x, buf ^ 1);
    else cp_async_commit();  // keep the group count uniform
    cp_async_wait<1>();      // this group's copies have landed
    // previous group's first-half element stores no longer read sM (M lives in
    // that half); the second half may still be draining to HBM
    if (bulk && kP2OneHalf && threadIdx.x < 32) bulk_wait_read();
    if (bulk && !kP2OneHalf && threadIdx.x < kP2Half) {
      if constexpr (C::MBUF <= kP2Half * kP2Pitch)
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else  // general tensors: M (16 entries per point) spans both halves
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    double* sC = p2_smem + C::OFF_C + buf * 16 * 32;
    if (warp == 0) {
      const double* sx = p2_smem + C::OFF_G + buf * 18 * 32 + lane;
      double x[18], d[21];
#pragma unroll
      for (int c = 0; c < 18; ++c) x[c] = sx[c * 32];
      prism_edges(x, d);
#pragma unroll
      for (int c = 0; c < 21; ++c) sD[c * 32 + lane] = d[c];
    } else if (GENERAL && warp == 1 && !args.coeff) {
#pragma unroll
      for (int c = 0; c < 16; ++c) sC[c * 32 + lane] = args.cu[c];
    }
    __syncthreads();
    // M for the 18 points (18 / NW per warp)
    {
      bool inverted = false;
#pragma unroll
      for (int q = warp; q < kP2NQ; q += C::NW) {
        double M[16];
        const double det = point_block<GENERAL, 32, 32>(sD + lane, tb.pts[4 * q], tb.pts[4 * q + 1],
                                                        tb.pts[4 * q + 2], tb.pts[4 * q + 3], sC + lane, M);
        inverted |= !(det > 0.0);
        if constexpr (LOAD) p2_smem[C::OFF_DW + q * 32 + lane] = det * tb.pts[4 * q + 3] * load_f(args, min(e, args.n_elem - 1));
        if (GENERAL) {
#pragma unroll
          for (int k = 0; k < 16; ++k) sM[(q * 16 + k) * 32 + lane] = static_cast<T>(M[k]);
        } else {
          const int src[6] = {5, 6, 7, 10, 11, 15};
#pragma unroll
          for (int k = 0; k < 6; ++k) sM[(q * 6 + k) * 32 + lane] = static_cast<T>(M[src[k]]);
        }
      }
      if (inverted && live) flag_inverted(args.bad, args.element_id_base + e);
    }
    __syncthreads();
    T acc[C::NACC];
#pragma unroll
    for (int i = 0; i < C::NACC; ++i) acc[i] = T(0);
    if constexpr (SYM) {
#define P2_ACC(W) p2_rows<T, GENERAL, SYM, W>(tb, sM, lane, acc)
      P2_WARP_SWITCH(P2_ACC)
#undef P2_ACC
    } else {
      p2_row_general(tb, sM, lane, warp, acc);
    }
    __syncthreads();  // M no longer read: the buffer becomes the output staging
    if constexpr (LOAD) {
      static_assert(sizeof(T) == 8, "fused load vectors are FP64");
      if (live) {
#pragma unroll
        for (int i = warp; i < kP2NSH; i += C::NW) {  // F rows dealt round-robin over the warps
          double fi = 0.0;
#pragma unroll
          for (int q = 0; q < kP2NQ; ++q) fi = fma(p2_smem[C::OFF_DW + q * 32 + lane], tb.phi[q * 4 * kP2NSH + i], fi);
          args.fout[e * kP2NSH + i] = fi;
        }
      }
    }
    if (args.out_layout == PI_OUT_SOA) {
      if (live) {
        if constexpr (SYM) {
#define P2_SOA(W) p2_store_soa<SYM, W>(args, e, acc)
          P2_WARP_SWITCH(P2_SOA)
#undef P2_SOA
        } else {
#pragma unroll
          for (int j = 0; j < kP2NSH; ++j) store_out(args, (warp * kP2NSH + j) * args.ld_out + e, acc[j]);
        }
      }
      continue;
    }
    if (bulk && !kP2OneHalf) {
      // Two halves of 16 elements, each one TMA bulk store per element (2592 B,
      // 16-byte aligned on both sides) issued by threads 0..15 as soon as that
      // half is staged: the half holding M drains first, so the next group's M
      // pass waits only for it (about half the former drain wait).
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        if (h == 1) {  // the second half's previous stores (one group ago) are read
          if (threadIdx.x < kP2Half) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncthreads();
        }
        if (lane / kP2Half == h) {
          T* st = sM + lane * kP2Pitch;
#define P2_STAGE(W) p2_stage<SYM, W>(st, acc)
          P2_WARP_SWITCH(P2_STAGE)
#undef P2_STAGE
        }
        const int64_t first = g * 32 + kP2Half * h;
        const int64_t left = args.n_elem - first;
        const int n_here = left <= 0 ? 0 : (left < kP2Half ? static_cast<int>(left) : kP2Half);
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x < kP2Half) {
          if (threadIdx.x < n_here)
            bulk_store(args.out + (first + threadIdx.x) * kP2KK,
                       reinterpret_cast<const double*>(sM) + (kP2Half * h + threadIdx.x) * kP2Pitch, kP2KK * 8u);
          bulk_commit();  // one group per half and issuing thread (empty when n_here is short)
        }
      }
      continue;
    }
#pragma unroll 1
    for (int h = 0; h < 32 / C::ROUND; ++h) {
      if (lane / C::ROUND == h) {
        T* st = sM + (lane % C::ROUND) * kP2Pitch;
        if constexpr (SYM) {
#define P2_STAGE(W) p2_stage<SYM, W>(st, acc)
          P2_WARP_SWITCH(P2_STAGE)
#undef P2_STAGE
        } else {
#pragma unroll
          for (int j = 0; j < kP2NSH; ++j) st[warp * kP2NSH + j] = acc[j];
        }
      }
      const int64_t first = g * 32 + C::ROUND * h;
      const int64_t left = args.n_elem - first;
      const int n_here = left <= 0 ? 0 : (left < C::ROUND ? static_cast<int>(left) : C::ROUND);
      if (bulk) {  // kP2OneHalf
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x < n_here) {
          bulk_store(args.out + (first + threadIdx.x) * kP2KK,
                     reinterpret_cast<const double*>(sM) + threadIdx.x * kP2Pitch, kP2KK * 8u);
          bulk_commit();
        }
        continue;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < n_here * kP2KK; r += C::NTHREADS) {
        const int el = r / kP2KK, c = r - el * kP2KK;
        store_out(args, first * kP2KK + r, sM[el * kP2Pitch + c]);
      }
      __syncthreads();
    }
  }
  if (threadIdx.x < 32) bulk_wait_all();  // outstanding element stores of the last group
}
#undef P2_WARP_SWITCH

}  // namespace pib
