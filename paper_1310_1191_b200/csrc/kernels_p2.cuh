// p = 2 symmetric weak forms (Laplace, symmetric uniform tensors): dense
// per-point accumulation in registers, lane = element.
//
// At p = 2 the sum-factorised MMA path feeds each tensor-core fragment from
// three shared-memory loads (the triangle factor has only 6 rows, so every
// G value is used by one MMA) and is shared-memory bound.  Here each group of
// 32 elements is handled by 3 warps; lane l of every warp owns element l, and
// warp r owns the upper-triangle part of the row blocks (r, 5-r) of 3 rows
// each (63 accumulators, balanced).  Per rule point a thread forms
// G_l(i) = sum_k phi_k(i) M_kl for its 6 rows and K_ij += sum_l G_l(i) phi_l(j);
// phi is read with warp-uniform addresses from the constant bank, M (per
// element and point) is built once by the group and shared through shared
// memory.  The 32 elements' matrices are staged in shared memory (mirroring
// the lower triangle) and leave as one contiguous coalesced block.
#pragma once

#include "kernels_common.cuh"

namespace pib {

constexpr int kP2NQ = 18, kP2NSH = 18, kP2KK = kP2NSH * kP2NSH;
__constant__ double c_phi_p2[kP2NQ * 4 * kP2NSH];  // tabulate_shapes order [q][k][dof]
__constant__ double c_pts_p2[kP2NQ * 4];           // xi1, xi2, xi3, w

constexpr int kP2Warps = 3;
constexpr int kP2Pitch = kP2KK + 1;  // odd pitch: lanes (elements) hit distinct banks

struct P2Smem {
  double M[kP2NQ][6][32];           // Laplace-type symmetric block (k,l = 1..3), per point and lane
  double D[21][32];                 // edge vectors per lane
  double K[16 * kP2Pitch];          // staged element matrices (half of the lanes at a time)
};

template <int R>
__device__ __forceinline__ void p2_accumulate(const P2Smem& sm, int lane, double acc[63]) {
  // row blocks (R, 5-R): rows 3R..3R+2 with columns >= 3R, rows 15-3R.. with columns >= 15-3R
  constexpr int RA = 3 * R, RB = 15 - 3 * R;
  constexpr int NA = 3 * (kP2NSH - RA), NB = 3 * (kP2NSH - RB);
  static_assert(NA + NB == 63, "balanced blocks");
#pragma unroll 1
  for (int q = 0; q < kP2NQ; ++q) {
    double m[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) m[k] = sm.M[q][k][lane];
    const double* ph = c_phi_p2 + q * 4 * kP2NSH;
    // M (symmetric 3x3): m = [11, 12, 13, 22, 23, 33]
    auto Ml = [&](int k, int l) {
      const int a = k < l ? k : l, b = k < l ? l : k;
      return a == 0 ? m[b] : (a == 1 ? m[2 + b] : m[5]);
    };
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const int r0 = blk == 0 ? RA : RB;
      const int off = blk == 0 ? 0 : NA;
#pragma unroll
      for (int ii = 0; ii < 3; ++ii) {
        const int i = r0 + ii;
        double g[3];
#pragma unroll
        for (int l = 0; l < 3; ++l)
          g[l] = fma(ph[1 * kP2NSH + i], Ml(0, l), fma(ph[2 * kP2NSH + i], Ml(1, l), ph[3 * kP2NSH + i] * Ml(2, l)));
#pragma unroll
        for (int j = r0; j < kP2NSH; ++j) {
          double& a = acc[off + ii * (kP2NSH - r0) + (j - r0)];
          a = fma(g[0], ph[1 * kP2NSH + j], fma(g[1], ph[2 * kP2NSH + j], fma(g[2], ph[3 * kP2NSH + j], a)));
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void p2_stage(P2Smem& sm, int slot, const double acc[63]) {
  constexpr int RA = 3 * R, RB = 15 - 3 * R, NA = 3 * (kP2NSH - RA);
  double* k = sm.K + slot * kP2Pitch;
#pragma unroll
  for (int blk = 0; blk < 2; ++blk) {
    const int r0 = blk == 0 ? RA : RB;
    const int off = blk == 0 ? 0 : NA;
#pragma unroll
    for (int ii = 0; ii < 3; ++ii)
#pragma unroll
      for (int j = r0; j < kP2NSH; ++j) {
        const int i = r0 + ii;
        const double v = acc[off + ii * (kP2NSH - r0) + (j - r0)];
        k[i * kP2NSH + j] = v;
        if (j >= r0 + 3) k[j * kP2NSH + i] = v;  // mirror outside the diagonal block
      }
  }
}

// SYMMETRIC coefficient tensors only (Laplace, or a symmetric UNIFORM
// tensor with no value-row terms, checked by the launcher).
template <bool GENERAL>
__global__ void __launch_bounds__(32 * kP2Warps) p2_lane_kernel(LaunchArgs args) {
  extern __shared__ __align__(16) unsigned char p2_smem_raw[];
  P2Smem& sm = *reinterpret_cast<P2Smem*>(p2_smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t groups = (args.n_elem + 31) / 32;
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const int64_t e = g * 32 + lane;
    const bool live = e < args.n_elem;
    const int64_t ec = live ? e : args.n_elem - 1;
    if (warp == 0) {
      double x[18], d[21];
#pragma unroll
      for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + ec];
      prism_edges(x, d);
#pragma unroll
      for (int c = 0; c < 21; ++c) sm.D[c][lane] = d[c];
    }
    __syncthreads();
    // M for the 18 points, 6 per warp
    {
      double d[21];
#pragma unroll
      for (int c = 0; c < 21; ++c) d[c] = sm.D[c][lane];
      bool inverted = false;
#pragma unroll 1
      for (int q = warp; q < kP2NQ; q += kP2Warps) {
        double M[16];
        const double det = point_block<GENERAL>(d, c_pts_p2[4 * q], c_pts_p2[4 * q + 1], c_pts_p2[4 * q + 2],
                                                c_pts_p2[4 * q + 3], args.cu, M);
        inverted |= !(det > 0.0);
        sm.M[q][0][lane] = M[5];
        sm.M[q][1][lane] = M[6];
        sm.M[q][2][lane] = M[7];
        sm.M[q][3][lane] = M[10];
        sm.M[q][4][lane] = M[11];
        sm.M[q][5][lane] = M[15];
      }
      if (inverted && live) flag_inverted(args.bad, args.element_id_base + e);
    }
    __syncthreads();
    double acc[63];
#pragma unroll
    for (int i = 0; i < 63; ++i) acc[i] = 0.0;
    if (warp == 0)
      p2_accumulate<0>(sm, lane, acc);
    else if (warp == 1)
      p2_accumulate<1>(sm, lane, acc);
    else
      p2_accumulate<2>(sm, lane, acc);
    // two rounds of 16 elements through the staging buffer
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if ((lane >> 4) == h) {
        if (warp == 0)
          p2_stage<0>(sm, lane & 15, acc);
        else if (warp == 1)
          p2_stage<1>(sm, lane & 15, acc);
        else
          p2_stage<2>(sm, lane & 15, acc);
      }
      __syncthreads();
      const int64_t first = g * 32 + 16 * h;
      const int64_t left = args.n_elem - first;
      const int n_here = left <= 0 ? 0 : (left < 16 ? static_cast<int>(left) : 16);
      for (int el = 0; el < n_here; ++el) {
        const double* src = sm.K + el * kP2Pitch;
        if (args.out_layout == PI_OUT_CANONICAL) {
          double* dst = args.out + (first + el) * kP2KK;
          for (int r = threadIdx.x; r < kP2KK; r += 32 * kP2Warps) dst[r] = src[r];
        } else {
          for (int r = threadIdx.x; r < kP2KK; r += 32 * kP2Warps) args.out[r * args.ld_out + first + el] = src[r];
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace pib
