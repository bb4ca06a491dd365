// p = 1 isotropic elasticity (n_eq = 3, K 18x18): lane = element, in
// physical coordinates like the reference's integrate_optimized
// (integrate_ref.cpp:93-130, the 21-term / 63-flop block of flop_costs.hpp):
//   K[(i,ie),(j,je)] += dw [lam g_ie(i) g_je(j) + mu g_je(i) g_ie(j)
//                           + mu d_(ie,je) g(i).g(j)]
// with g_d(i) = psi_(d+1)(i) = sum_k phi_(k+1)(i) inv[k][d] (geometry.cpp:85-102).
//
// At p = 1 the sum-factorised kernel's per-item overhead dominates (one
// 4-point chunk, a 6-row triangle factor), so this kernel keeps K in
// registers instead:
//  * a CTA integrates groups of 32 elements; lane l of every warp owns
//    element l;
//  * warp w (of 3) owns the upper-triangle 3x3 blocks of block rows w and
//    5-w (7 blocks, 57 accumulators);
//  * the 6 rule points' physical gradients (18 values) and dw*lam, dw*mu are
//    computed once per element (2 points per warp) into shared memory, the
//    structural zeros of the basis skipped at compile time (BasisPattern);
//  * K leaves through shared-memory staging as contiguous coalesced blocks.
#pragma once

#include "kernels_common.cuh"
#include "kernels_dense.cuh"

namespace pib {

constexpr int kE1NQ = 6, kE1NSH = 6, kE1DIM = 18, kE1KK = kE1DIM * kE1DIM;
// The context's rule and shape table, passed with every launch (kernel
// parameter space: no shared __constant__ symbol between contexts).
struct E1Tables {
  double phi[kE1NQ * 4 * kE1NSH];  // tabulate_shapes order [q][k][dof]
  double pts[kE1NQ * 4];           // xi1, xi2, xi3, w
};

constexpr int kE1Warps = 3;
constexpr int kE1Pitch = kE1KK + 2;  // 16-byte multiple: staged elements leave by TMA bulk stores
#ifndef PI_E1_ROUND
#define PI_E1_ROUND 16
#endif
#ifndef PI_E1_MINB
#define PI_E1_MINB 4
#endif
constexpr int kE1Round = PI_E1_ROUND;  // elements staged per output round
constexpr int kE1NG = 20;            // per point: g_d(i) (18), dw*lam, dw*mu
struct E1Smem {
  static constexpr int GBUF = kE1NQ * kE1NG * 32;
  static constexpr int SBUF = kE1Round * kE1Pitch;
  static constexpr int BUF = GBUF > SBUF ? GBUF : SBUF;
  static constexpr int OFF_D = BUF;             // edge vectors [21][32]
  static constexpr int OFF_MAT = OFF_D + 21 * 32;  // lam, mu [2][32]
  static constexpr int DOUBLES = OFF_MAT + 2 * 32;
  static constexpr size_t BYTES = DOUBLES * sizeof(double);
};

// block rows of warp W: W and 5-W; blocks (bi, bj >= bi); diagonal blocks keep
// the 6 entries ie <= je.
template <int W>
__device__ __forceinline__ constexpr int e1_brow(int r) {
  return r == 0 ? W : kE1NSH - 1 - W;
}

template <int W>
__device__ __forceinline__ void e1_accumulate(const double* __restrict__ sG, int lane, double* acc) {
#pragma unroll 1
  for (int q = 0; q < kE1NQ; ++q) {
    const double* gq = sG + q * kE1NG * 32 + lane;
    double g[kE1NSH][3];
#pragma unroll
    for (int i = 0; i < kE1NSH; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) g[i][d] = gq[(i * 3 + d) * 32];
    const double lam = gq[18 * 32], mu = gq[19 * 32];
    int off = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int bi = e1_brow<W>(r);
      double lg[3], mg[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        lg[d] = lam * g[bi][d];
        mg[d] = mu * g[bi][d];
      }
#pragma unroll
      for (int bj = bi; bj < kE1NSH; ++bj) {
        const double dot = mu * fma(g[bi][0], g[bj][0], fma(g[bi][1], g[bj][1], g[bi][2] * g[bj][2]));
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = (bj == bi ? ie : 0); je < 3; ++je) {
            double v = fma(lg[ie], g[bj][je], fma(mg[je], g[bj][ie], acc[off]));
            if (ie == je) v += dot;
            acc[off++] = v;
          }
      }
    }
  }
}

template <int W, typename T>
__device__ __forceinline__ void e1_store(T* st, int64_t ld, const double* acc) {
  int off = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int bi = e1_brow<W>(r);
#pragma unroll
    for (int bj = bi; bj < kE1NSH; ++bj)
#pragma unroll
      for (int ie = 0; ie < 3; ++ie)
#pragma unroll
        for (int je = (bj == bi ? ie : 0); je < 3; ++je) {
          const int row = bi * 3 + ie, col = bj * 3 + je;
          const double v = acc[off++];
          st[(row * kE1DIM + col) * ld] = static_cast<T>(v);
          if (row != col) st[(col * kE1DIM + row) * ld] = static_cast<T>(v);
        }
  }
}

#define E1_WARP_SWITCH(CALL) \
  switch (warp) {            \
    case 0: CALL(0); break;  \
    case 1: CALL(1); break;  \
    default: CALL(2); break; \
  }

__global__ void __launch_bounds__(32 * kE1Warps, PI_E1_MINB) p1_elastic_lane_kernel(const __grid_constant__ LaunchArgs args,
                                                                           const __grid_constant__ E1Tables tb) {
  using BP = BasisPattern<1>;
  constexpr int NACC = 57;
  extern __shared__ __align__(16) double e1_smem[];
  double* sG = e1_smem;  // per-point data, then the output staging
  double* sD = e1_smem + E1Smem::OFF_D;
  double* sMat = e1_smem + E1Smem::OFF_MAT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t groups = (args.n_elem + 31) / 32;
  const bool bulk = !args.out32 && args.out_layout == PI_OUT_CANONICAL && (reinterpret_cast<uintptr_t>(args.out) & 15) == 0;
  for (int64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
    const int64_t e = grp * 32 + lane;
    const bool live = e < args.n_elem;
    const int64_t ec = live ? e : args.n_elem - 1;
    if (bulk && threadIdx.x < kE1Round) bulk_wait_read();  // last group's stores no longer read sG
    if (warp == 0) {
      double x[18], d[21];
#pragma unroll
      for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + ec];
      prism_edges(x, d);
#pragma unroll
      for (int c = 0; c < 21; ++c) sD[c * 32 + lane] = d[c];
    } else if (warp == 1) {
      const double young = args.coeff ? args.coeff[ec] : args.cu[0];
      const double nu = args.coeff ? args.coeff[args.coeff_ld + ec] : args.cu[1];
      if (live) check_material(args, e, young, nu);
      lame(young, nu, sMat[lane], sMat[32 + lane]);
    }
    __syncthreads();
    // physical gradients at the warp's points
    {
      bool inverted = false;
#pragma unroll
      for (int q = warp; q < kE1NQ; q += kE1Warps) {
        double cf[3][3];
        const double det = jacobian_cofactors<32>(sD + lane, tb.pts[4 * q], tb.pts[4 * q + 1],
                                                  tb.pts[4 * q + 2], cf);
        inverted |= !(det > 0.0);
        const double id = __drcp_rn(det), dw = det * tb.pts[4 * q + 3];
        const double* ph = tb.phi + q * 4 * kE1NSH;
        double* gq = sG + q * kE1NG * 32 + lane;
#pragma unroll
        for (int i = 0; i < kE1NSH; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            // inv[k][d] = cf[d][k] / det
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (BP::nz(k + 1, i)) s = fma(ph[(k + 1) * kE1NSH + i], cf[d][k], s);
            gq[(i * 3 + d) * 32] = s * id;
          }
        gq[18 * 32] = dw * sMat[lane];
        gq[19 * 32] = dw * sMat[32 + lane];
      }
      if (inverted && live) flag_inverted(args.bad, args.element_id_base + e);
    }
    __syncthreads();
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
#define E1_ACC(W) e1_accumulate<W>(sG, lane, acc)
    E1_WARP_SWITCH(E1_ACC)
#undef E1_ACC
    __syncthreads();  // per-point data no longer read: the buffer becomes the output staging
    if (args.out_layout == PI_OUT_SOA) {
      if (live) {
        if (args.out32) {
#define E1_SOA(W) e1_store<W>(args.out32 + e, args.ld_out, acc)
          E1_WARP_SWITCH(E1_SOA)
#undef E1_SOA
        } else {
#define E1_SOA(W) e1_store<W>(args.out + e, args.ld_out, acc)
          E1_WARP_SWITCH(E1_SOA)
#undef E1_SOA
        }
      }
      continue;
    }
#pragma unroll 1
    for (int h = 0; h < 32 / kE1Round; ++h) {
      if (bulk && h > 0) {  // the previous round's bulk stores have read the staging
        if (threadIdx.x < kE1Round) bulk_wait_read();
        __syncthreads();
      }
      if (lane / kE1Round == h) {
        double* st = sG + (lane % kE1Round) * kE1Pitch;
#define E1_STAGE(W) e1_store<W>(st, 1, acc)
        E1_WARP_SWITCH(E1_STAGE)
#undef E1_STAGE
      }
      const int64_t first = grp * 32 + kE1Round * h;
      const int64_t left = args.n_elem - first;
      const int n_here = left <= 0 ? 0 : (left < kE1Round ? static_cast<int>(left) : kE1Round);
      if (bulk) {  // one TMA bulk store per staged element (2592 B)
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x < n_here) {
          bulk_store(args.out + (first + threadIdx.x) * kE1KK, sG + threadIdx.x * kE1Pitch, kE1KK * 8u);
          bulk_commit();
        }
        continue;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < n_here * kE1KK; r += 32 * kE1Warps) {
        const int el = r / kE1KK, c = r - el * kE1KK;
        store_out(args, first * kE1KK + r, sG[el * kE1Pitch + c]);
      }
      __syncthreads();
    }
  }
  if (threadIdx.x < kE1Round) bulk_wait_all();
}
#undef E1_WARP_SWITCH

}  // namespace pib

namespace pib {

// ---------------------------------------------------------------------------
// p = 2 isotropic elasticity (K 54x54): one warp per element, lanes own 3x3
// blocks.  The 171 upper-triangle shape blocks (i, j >= i) are dealt to the
// 32 lanes round-robin (5 or 6 blocks, 54 accumulators); per rule point a
// lane reads the physical gradients g(i), g(j) of its blocks (computed once
// per element into the warp's shared memory, structural zeros skipped) and
// updates the 63-flop block of integrate_optimized.  The element matrix is
// staged in the warp's shared memory (mirrors included) and leaves with
// coalesced 16-byte stores.
constexpr int kE2NQ = 18, kE2NSH = 18, kE2DIM = 54, kE2KK = kE2DIM * kE2DIM, kE2NBLK = 171;
struct E2Tables {
  double phi[kE2NQ * 4 * kE2NSH];  // tabulate_shapes order [q][k][dof]
  double pts[kE2NQ * 4];           // xi1, xi2, xi3, w
};

constexpr int kE2Warps = 4;
constexpr int kE2BPL = 6;                          // blocks per lane (ceil(171 / 32))
constexpr int kE2G = kE2NQ * (kE2NSH * 3 + 2);     // per point: g_d(i) (54), dw*lam, dw*mu
constexpr int kE2WarpDoubles = kE2KK > kE2G ? kE2KK : kE2G;  // staging aliases the gradients
constexpr int kE2Phi = kE2NQ * 4 * kE2NSH;          // the shape table, staged per CTA
constexpr size_t kE2SmemBytes = sizeof(double) * ((kE2WarpDoubles + 2) * kE2Warps + kE2Phi);

__global__ void __launch_bounds__(32 * kE2Warps, 2) p2_elastic_warp_kernel(const __grid_constant__ LaunchArgs args,
                                                                  const __grid_constant__ E2Tables tb) {
  using BP = BasisPattern<2>;
  extern __shared__ __align__(16) double e2_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sw = e2_smem + warp * (kE2WarpDoubles + 2);  // this warp's region (16-byte aligned)
  // lanes read the table at different points: shared memory, not the constant bank
  double* sPhi = e2_smem + (kE2WarpDoubles + 2) * kE2Warps;
  for (int i = threadIdx.x; i < kE2Phi; i += 32 * kE2Warps) sPhi[i] = tb.phi[i];
  __syncthreads();
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kE2Warps;
  // the lane's blocks (i, j)
  int bi[kE2BPL], bj[kE2BPL];
#pragma unroll
  for (int k = 0; k < kE2BPL; ++k) {
    // upper-triangle block b = (i, j >= i) in row-major order (padding: b >= 171)
    int b = lane + 32 * k, i = 0;
    if (b >= kE2NBLK) b = kE2NBLK - 1;
    while (b >= kE2NSH - i) b -= kE2NSH - i++;
    bi[k] = i;
    bj[k] = i + b;
  }
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * kE2Warps + warp; e < args.n_elem; e += nwarps) {
    // ---- geometry, material, then per-point gradients (lane = point) ----
    double lam, mu;
    {
      const double young = args.coeff ? args.coeff[e] : args.cu[0];
      const double nu = args.coeff ? args.coeff[args.coeff_ld + e] : args.cu[1];
      if (threadIdx.x % 32 == 0) check_material(args, e, young, nu);
      lame(young, nu, lam, mu);
    }
    double x[18], d[21];
#pragma unroll
    for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];  // warp-uniform (broadcast) loads
    prism_edges(x, d);
    bool inverted = false;
    if (lane < kE2NQ) {
      const int q = lane;
      double cf[3][3];
      const double det = jacobian_cofactors(d, tb.pts[4 * q], tb.pts[4 * q + 1], tb.pts[4 * q + 2], cf);
      inverted = !(det > 0.0);
      const double id = __drcp_rn(det), dw = det * tb.pts[4 * q + 3];
      double* gq = sw + q * (kE2NSH * 3 + 2);
#pragma unroll
      for (int i = 0; i < kE2NSH; ++i)
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (BP::nz(k + 1, i)) s = fma(sPhi[(q * 4 + k + 1) * kE2NSH + i], cf[dd][k], s);
          gq[i * 3 + dd] = s * id;
        }
      gq[kE2NSH * 3] = dw * lam;
      gq[kE2NSH * 3 + 1] = dw * mu;
    }
    if (__any_sync(0xffffffffu, inverted) && lane == 0) flag_inverted(args.bad, args.element_id_base + e);
    __syncwarp();
    // ---- accumulate the lane's blocks over the rule points ----
    double acc[kE2BPL][9];
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k)
#pragma unroll
      for (int m = 0; m < 9; ++m) acc[k][m] = 0.0;
#pragma unroll 1
    for (int q = 0; q < kE2NQ; ++q) {
      const double* gq = sw + q * (kE2NSH * 3 + 2);
      const double l = gq[kE2NSH * 3], m_ = gq[kE2NSH * 3 + 1];
#pragma unroll
      for (int k = 0; k < kE2BPL; ++k) {
        if (k == kE2BPL - 1 && lane + 32 * k >= kE2NBLK) break;  // lanes 11..31 own 5 blocks
        const double* gi = gq + bi[k] * 3;
        const double* gj = gq + bj[k] * 3;
        const double a0 = gi[0], a1 = gi[1], a2 = gi[2], b0 = gj[0], b1 = gj[1], b2 = gj[2];
        const double dot = m_ * fma(a0, b0, fma(a1, b1, a2 * b2));
        const double la[3] = {l * a0, l * a1, l * a2}, ma[3] = {m_ * a0, m_ * a1, m_ * a2};
        const double bb[3] = {b0, b1, b2};
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = 0; je < 3; ++je) {
            double v = fma(la[ie], bb[je], fma(ma[je], bb[ie], acc[k][ie * 3 + je]));
            if (ie == je) v += dot;
            acc[k][ie * 3 + je] = v;
          }
      }
    }
    __syncwarp();  // gradients no longer read: the region becomes the staging of K
    // ---- stage the element matrix (mirrors included), then coalesced stores ----
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k) {
      if (k == kE2BPL - 1 && lane + 32 * k >= kE2NBLK) break;
#pragma unroll
      for (int ie = 0; ie < 3; ++ie)
#pragma unroll
        for (int je = 0; je < 3; ++je) {
          const int r = bi[k] * 3 + ie, c = bj[k] * 3 + je;
          const double v = acc[k][ie * 3 + je];
          if (bi[k] != bj[k] || ie <= je) {
            sw[r * kE2DIM + c] = v;
            sw[c * kE2DIM + r] = v;
          }
        }
    }
    __syncwarp();
    if (args.out_layout == PI_OUT_SOA) {
      for (int r = lane; r < kE2KK; r += 32) store_out(args, static_cast<int64_t>(r) * args.ld_out + e, sw[r]);
    } else if (args.out32) {
      for (int r = lane; r < kE2KK; r += 32) args.out32[e * kE2KK + r] = static_cast<float>(sw[r]);
    } else if ((reinterpret_cast<uintptr_t>(args.out) & 15) == 0) {
      // 2916 doubles per element, 16-byte aligned: one TMA bulk store
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_store(args.out + e * kE2KK, sw, kE2KK * 8u);
        bulk_commit();
        bulk_wait_read();  // the next element's gradients overwrite the staging
      }
    } else {  // 8-byte aligned output base (kE2KK is even: every element keeps the base's alignment)
      for (int r = lane; r < kE2KK; r += 32) args.out[e * kE2KK + r] = sw[r];
    }
    __syncwarp();  // staging read out before the next element's gradients overwrite it
  }
}

}  // namespace pib

namespace pib {

// ---------------------------------------------------------------------------
// p = 3 isotropic elasticity (K 120x120): one CTA (4 warps) per element.  The
// 820 upper-triangle 3x3 shape blocks are dealt to the 128 threads
// round-robin (6-7 blocks, 63 accumulators).  Inverse Jacobians of the 48
// rule points, then the 40 x 3 physical gradients per point are computed
// into shared memory by the whole CTA; the block form is the 63-flop one of
// integrate_optimized.  K is 115 KB per element, so blocks are stored
// straight from registers (3-double row segments, the mirrored block
// transposed); the CTA's writes to one element merge in L2.
constexpr int kE3NQ = 48, kE3NSH = 40, kE3DIM = 120, kE3KK = kE3DIM * kE3DIM, kE3NBLK = 820;
constexpr int kE3Threads = 128, kE3BPT = (kE3NBLK + kE3Threads - 1) / kE3Threads;  // 7
constexpr int kE3GP = kE3NSH * 3 + 2;  // per point: g_d(i), dw*lam, dw*mu
struct E3Smem {  // the 61 KB shape table is read through L1 (read-only loads), not staged
  static constexpr int OFF_PTS = 0;                                // [NQ][4]
  static constexpr int OFF_INV = OFF_PTS + kE3NQ * 4;              // [NQ][10]: inverse, dw
  static constexpr int OFF_G = OFF_INV + kE3NQ * 10;               // [NQ][GP]
  static constexpr int DOUBLES = OFF_G + kE3NQ * kE3GP;
  static constexpr size_t BYTES = DOUBLES * sizeof(double);
};

__global__ void __launch_bounds__(kE3Threads, 2) p3_elastic_cta_kernel(LaunchArgs args, DenseTables tab) {
  extern __shared__ __align__(16) double e3_smem[];
  double* sPts = e3_smem + E3Smem::OFF_PTS;
  double* sInv = e3_smem + E3Smem::OFF_INV;
  double* sG = e3_smem + E3Smem::OFF_G;
  const int tid = threadIdx.x;
  for (int q = tid; q < kE3NQ; q += kE3Threads) {
    sPts[4 * q] = tab.pts[3 * q];
    sPts[4 * q + 1] = tab.pts[3 * q + 1];
    sPts[4 * q + 2] = tab.pts[3 * q + 2];
    sPts[4 * q + 3] = tab.w[q];
  }
  // this thread's blocks (i, j >= i), upper-triangle enumeration b -> (i, j)
  int bi[kE3BPT], bj[kE3BPT];
#pragma unroll
  for (int k = 0; k < kE3BPT; ++k) {
    int b = tid + kE3Threads * k, i = 0;
    if (b >= kE3NBLK) b = kE3NBLK - 1;
    while (b >= kE3NSH - i) b -= kE3NSH - i++;
    bi[k] = i;
    bj[k] = i + b;
  }
  __syncthreads();
  for (int64_t e = blockIdx.x; e < args.n_elem; e += gridDim.x) {
    double lam, mu;
    {
      const double young = args.coeff ? args.coeff[e] : args.cu[0];
      const double nu = args.coeff ? args.coeff[args.coeff_ld + e] : args.cu[1];
      if (threadIdx.x % 32 == 0) check_material(args, e, young, nu);
      lame(young, nu, lam, mu);
    }
    // (1) inverse Jacobian and dw per point (threads 0..47)
    bool inverted = false;
    if (tid < kE3NQ) {
      double x[18], d[21];
#pragma unroll
      for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];
      prism_edges(x, d);
      const int q = tid;
      double cf[3][3];
      const double det = jacobian_cofactors(d, sPts[4 * q], sPts[4 * q + 1], sPts[4 * q + 2], cf);
      inverted = !(det > 0.0);
      const double id = __drcp_rn(det);
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) sInv[q * 10 + k * 3 + dd] = cf[dd][k] * id;  // inv[k][dd]
      sInv[q * 10 + 9] = det * sPts[4 * q + 3];
    }
    if (__syncthreads_or(inverted) && tid == 0) flag_inverted(args.bad, args.element_id_base + e);
    // (2) gradients g_d(i) at every point, (q, i) pairs over the CTA
    for (int t = tid; t < kE3NQ * kE3NSH; t += kE3Threads) {
      const int q = t / kE3NSH, i = t - q * kE3NSH;
      const double* ph = tab.phi + q * 4 * kE3NSH + i;
      const double f1 = __ldg(ph + kE3NSH), f2 = __ldg(ph + 2 * kE3NSH), f3 = __ldg(ph + 3 * kE3NSH);
      const double* inv = sInv + q * 10;
      double* g = sG + q * kE3GP + i * 3;
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) g[dd] = fma(f1, inv[dd], fma(f2, inv[3 + dd], f3 * inv[6 + dd]));
    }
    for (int q = tid; q < kE3NQ; q += kE3Threads) {
      sG[q * kE3GP + kE3NSH * 3] = sInv[q * 10 + 9] * lam;
      sG[q * kE3GP + kE3NSH * 3 + 1] = sInv[q * 10 + 9] * mu;
    }
    __syncthreads();
    // (3) accumulate the thread's blocks
    double acc[kE3BPT][9];
#pragma unroll
    for (int k = 0; k < kE3BPT; ++k)
#pragma unroll
      for (int m = 0; m < 9; ++m) acc[k][m] = 0.0;
#pragma unroll 1
    for (int q = 0; q < kE3NQ; ++q) {
      const double* gq = sG + q * kE3GP;
      const double l = gq[kE3NSH * 3], m_ = gq[kE3NSH * 3 + 1];
#pragma unroll
      for (int k = 0; k < kE3BPT; ++k) {
        const double* gi = gq + bi[k] * 3;
        const double* gj = gq + bj[k] * 3;
        const double a0 = gi[0], a1 = gi[1], a2 = gi[2], b0 = gj[0], b1 = gj[1], b2 = gj[2];
        const double dot = m_ * fma(a0, b0, fma(a1, b1, a2 * b2));
        const double la[3] = {l * a0, l * a1, l * a2}, ma[3] = {m_ * a0, m_ * a1, m_ * a2};
        const double bb[3] = {b0, b1, b2};
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = 0; je < 3; ++je) {
            double v = fma(la[ie], bb[je], fma(ma[je], bb[ie], acc[k][ie * 3 + je]));
            if (ie == je) v += dot;
            acc[k][ie * 3 + je] = v;
          }
      }
    }
    // (4) store the blocks (and their mirrors) straight from registers
#pragma unroll
    for (int k = 0; k < kE3BPT; ++k) {
      if (tid + kE3Threads * k >= kE3NBLK) break;
#pragma unroll
      for (int ie = 0; ie < 3; ++ie)
#pragma unroll
        for (int je = 0; je < 3; ++je) {
          const int r = bi[k] * 3 + ie, c = bj[k] * 3 + je;
          if (bi[k] == bj[k] && ie > je) continue;
          const double v = acc[k][ie * 3 + je];
          if (args.out_layout == PI_OUT_SOA) {
            store_out(args, static_cast<int64_t>(r * kE3DIM + c) * args.ld_out + e, v);
            if (r != c) store_out(args, static_cast<int64_t>(c * kE3DIM + r) * args.ld_out + e, v);
          } else {
            store_out(args, e * kE3KK + r * kE3DIM + c, v);
            if (r != c) store_out(args, e * kE3KK + c * kE3DIM + r, v);
          }
        }
    }
    __syncthreads();  // gradients read before the next element overwrites them
  }
}

}  // namespace pib
