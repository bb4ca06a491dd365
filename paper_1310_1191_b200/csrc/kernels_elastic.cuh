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
//  * the 6 rule points' physical gradients (18 values) and dw are computed
//    once per element (2 points per warp) into shared memory, the
//    structural zeros of the basis skipped at compile time (BasisPattern);
//  * lam, mu are constant per element, so the lanes accumulate
//    S_(ie,je) = sum_q dw g_ie(i) g_je(j) (9 FMAs per block and point) and form
//    K = lam S + mu S^T + mu tr(S) I per block at the end;
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
#define PI_E1_MINB 3
#endif
constexpr int kE1Round = PI_E1_ROUND;  // elements staged per output round
constexpr int kE1NG = 19;            // per point: g_d(i) (18), dw
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

// S_(ie,je)(bi, bj) = sum_q dw g_ie(bi) g_je(bj) of the warp's blocks (diagonal
// blocks: the 6 entries ie <= je of the symmetric S); e1_finish then forms
// K = lam S + mu S^T + mu tr(S) I per block (lam, mu constant per element):
// 9 FMAs per block and point instead of the 27-FLOP update.
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
    const double dw = gq[18 * 32];
    int off = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int bi = e1_brow<W>(r);
      double wg[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) wg[d] = dw * g[bi][d];
#pragma unroll
      for (int bj = bi; bj < kE1NSH; ++bj)
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = (bj == bi ? ie : 0); je < 3; ++je) {
            acc[off] = fma(wg[ie], g[bj][je], acc[off]);
            ++off;
          }
    }
  }
}

template <int W>
__device__ __forceinline__ void e1_finish(double* acc, double lam, double mu) {
  int off = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int bi = e1_brow<W>(r);
#pragma unroll
    for (int bj = bi; bj < kE1NSH; ++bj) {
      if (bj == bi) {  // entries (0,0) (0,1) (0,2) (1,1) (1,2) (2,2)
        const double tr = mu * (acc[off] + acc[off + 3] + acc[off + 5]), lm = lam + mu;
#pragma unroll
        for (int m = 0; m < 6; ++m) acc[off + m] = fma(lm, acc[off + m], (m == 0 || m == 3 || m == 5) ? tr : 0.0);
        off += 6;
      } else {
        const double tr = mu * (acc[off] + acc[off + 4] + acc[off + 8]), lm = lam + mu;
#pragma unroll
        for (int ie = 0; ie < 3; ++ie) {
          acc[off + ie * 4] = fma(lm, acc[off + ie * 4], tr);
#pragma unroll
          for (int je = ie + 1; je < 3; ++je) {
            const double a = acc[off + ie * 3 + je], b = acc[off + je * 3 + ie];
            acc[off + ie * 3 + je] = fma(lam, a, mu * b);
            acc[off + je * 3 + ie] = fma(lam, b, mu * a);
          }
        }
        off += 9;
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
        gq[18 * 32] = dw;
      }
      if (inverted && live) flag_inverted(args.bad, args.element_id_base + e);
    }
    __syncthreads();
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
#define E1_ACC(W) e1_accumulate<W>(sG, lane, acc), e1_finish<W>(acc, sMat[lane], sMat[32 + lane])
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
// lane reads the physical gradients dw g(i), g(j) of its blocks (computed
// once per element into the warp's shared memory, structural zeros skipped)
// and accumulates S_(ie,je) = sum_q dw g_ie(i) g_je(j) (9 FMAs); with lam, mu
// constant per element the block of integrate_optimized is then
// lam S + mu S^T + mu tr(S) I (see p3_elastic_mma_kernel).  The element matrix is
// staged in the warp's shared memory (mirrors included) and leaves with
// coalesced 16-byte stores.
constexpr int kE2NQ = 18, kE2NSH = 18, kE2DIM = 54, kE2KK = kE2DIM * kE2DIM, kE2NBLK = 171;
struct E2Tables {
  double phi[kE2NQ * 4 * kE2NSH];  // tabulate_shapes order [q][k][dof]
  double pts[kE2NQ * 4];           // xi1, xi2, xi3, w
};

#ifndef PI_E2_WARPS
#define PI_E2_WARPS 4
#endif
#ifndef PI_E2_MINB
#define PI_E2_MINB 2
#endif
constexpr int kE2Warps = PI_E2_WARPS;
constexpr int kE2BPL = 6;                          // blocks per lane (ceil(171 / 32))
constexpr int kE2GP = kE2NSH * 6 + 1;             // per point: g_d(i) (54), dw g_d(i) (54); odd pitch:
                                                   // the 18 point lanes write distinct banks
constexpr int kE2G = kE2NQ * kE2GP;
constexpr int kE2WarpDoubles = kE2KK > kE2G ? kE2KK : kE2G;  // staging aliases the gradients
// per CTA: the factors of the tensor basis phi_(t,a) = m_t(xi1, xi2) P_a(xi3)
// at the rule points q = (z, s) -- m_t(s), dm1_t(s), dm2_t(s) [3][6][6] and
// P_a(z), P'_a(z) [2][3][3] -- and the rule [18][4]
constexpr int kE2NT = 6, kE2NS = 6, kE2NZ = 3, kE2NV = 3;
constexpr int kE2OffPz = 3 * kE2NT * kE2NS, kE2OffPts = kE2OffPz + 2 * kE2NV * kE2NZ;
constexpr int kE2Phi = kE2OffPts + 4 * kE2NQ;
constexpr size_t kE2SmemBytes = sizeof(double) * ((kE2WarpDoubles + 2) * kE2Warps + kE2Phi);

__global__ void __launch_bounds__(32 * kE2Warps, PI_E2_MINB) p2_elastic_warp_kernel(const __grid_constant__ LaunchArgs args,
                                                                  const __grid_constant__ E2Tables tb) {
  using BP = BasisPattern<2>;
  extern __shared__ __align__(16) double e2_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sw = e2_smem + warp * (kE2WarpDoubles + 2);  // this warp's region (16-byte aligned)
  // lanes read the tables at different points: shared memory, not the constant bank
  double* sMt = e2_smem + (kE2WarpDoubles + 2) * kE2Warps;
  double* sPz = sMt + kE2OffPz;
  double* sPts = sMt + kE2OffPts;
  // read off the shape table (tabulate_shapes order [q][k][dof], q = z*6 + s,
  // dof = t*3 + a): at z = 0, a = 0 (P_0 = 1) phi_k = m_t(s), dm1_t(s), dm2_t(s);
  // at t = 0 (m_0 = 1) phi_0 / phi_3 = P_a(z) / P'_a(z)
  for (int i = threadIdx.x; i < kE2Phi; i += 32 * kE2Warps) {
    double v;
    if (i < kE2OffPz) {
      const int c = i / (kE2NT * kE2NS), t = (i / kE2NS) % kE2NT, sp = i % kE2NS;
      v = tb.phi[(sp * 4 + c) * kE2NSH + t * kE2NV];
    } else if (i < kE2OffPts) {
      const int j = i - kE2OffPz, c = j / (kE2NV * kE2NZ), a = (j / kE2NZ) % kE2NV, z = j % kE2NZ;
      v = tb.phi[(z * kE2NS * 4 + (c ? 3 : 0)) * kE2NSH + a];
    } else {
      v = tb.pts[i - kE2OffPts];
    }
    sMt[i] = v;
  }
  __syncthreads();
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kE2Warps;
  // The lane's blocks (i, j): column segments.  Rows fall in three bands of
  // six (6s .. 6s+5); a lane owns up to six blocks of one column j in one
  // band, so per point it reads g(j) once (b operand in registers) and
  // slot k reads dw g(6s + k), which lanes of the same band share
  // (broadcast): about half the shared-memory wavefronts of a round-robin
  // deal.  Lanes 0..20 own the 21 full segments (j >= 6s + 5); lanes 21..29
  // pair the partial diagonal segments of each band (sizes 1 + 5, 2 + 4, 3);
  // lanes 30, 31 idle.  171 blocks, at most 6 per lane.
  int bi[kE2BPL], bj[kE2BPL], c0 = 0, c1 = 0;
  unsigned live = 0u, sel = 0u;  // per slot: stored / reads column c1
  if (lane < 21) {
    const int s = lane < 13 ? 0 : lane < 20 ? 1 : 2;
    const int j = s == 0 ? 5 + lane : s == 1 ? 11 + (lane - 13) : 17;
    c0 = c1 = j;
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k) {
      bi[k] = 6 * s + k;
      bj[k] = j;
    }
    live = 0x3fu;
  } else {
    const int m = lane < 30 ? lane - 21 : 8, s = m / 3, r = m % 3;
    const int ca = 6 * s + r, na = r + 1;                     // column 6s+r: rows 6s .. 6s+r
    const int cb = 6 * s + 4 - r, nb = r < 2 ? 5 - r : 0;     // column 6s+4-r: rows 6s .. 6s+4-r
    c0 = nb > 0 ? cb : ca;
    c1 = ca;
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k) {
      const bool first = k < nb;
      bi[k] = 6 * s + (first ? k : k - nb);
      bj[k] = first ? cb : ca;
      if (!first) sel |= 1u << k;
      if (lane < 30 && k < nb + na) live |= 1u << k;
      if (bi[k] > 17) bi[k] = 17;  // dead slots: any valid address
    }
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
      const int q = lane, z = q / kE2NS, sp = q % kE2NS;
      double cf[3][3];
      const double det = jacobian_cofactors(d, sPts[4 * q], sPts[4 * q + 1], sPts[4 * q + 2], cf);
      inverted = !(det > 0.0);
      const double id = __drcp_rn(det), dw = det * sPts[4 * q + 3];
      double* gq = sw + q * kE2GP;
      double pz[kE2NV], dpz[kE2NV];
#pragma unroll
      for (int a = 0; a < kE2NV; ++a) {
        pz[a] = a == 0 ? 1.0 : sPz[a * kE2NZ + z];
        dpz[a] = a == 0 ? 0.0 : sPz[(kE2NV + a) * kE2NZ + z];
      }
      // g_d((t,a), q) = [(cf[d][0] dm1_t + cf[d][1] dm2_t) P_a + cf[d][2] m_t P'_a] / det
#pragma unroll
      for (int t = 0; t < kE2NT; ++t) {
        const int i0 = t * kE2NV;
        const double m = sMt[t * kE2NS + sp];
        const double m1 = BP::nz(1, i0) ? sMt[(kE2NT + t) * kE2NS + sp] : 0.0;
        const double m2 = BP::nz(2, i0) ? sMt[(2 * kE2NT + t) * kE2NS + sp] : 0.0;
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
          const double u = fma(cf[dd][0], m1, cf[dd][1] * m2), w = cf[dd][2] * m;
#pragma unroll
          for (int a = 0; a < kE2NV; ++a) {
            const double g = (a == 0 ? u : fma(u, pz[a], w * dpz[a])) * id;
            gq[(i0 + a) * 3 + dd] = g;
            gq[kE2NSH * 3 + (i0 + a) * 3 + dd] = dw * g;
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, inverted) && lane == 0) flag_inverted(args.bad, args.element_id_base + e);
    __syncwarp();
    // ---- S_(ie,je)(i, j) = sum_q dw g_ie(i) g_je(j) of the lane's blocks ----
    // (lam, mu are per element: K = lam S + mu S^T + mu tr(S) I per block
    // afterwards -- 9 FMAs per block and point instead of the 27-FLOP update)
    double acc[kE2BPL][9];
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k)
#pragma unroll
      for (int m = 0; m < 9; ++m) acc[k][m] = 0.0;
#pragma unroll 1
    for (int q = 0; q < kE2NQ; ++q) {
      const double* gq = sw + q * kE2GP;
      const double b0[3] = {gq[c0 * 3], gq[c0 * 3 + 1], gq[c0 * 3 + 2]};
      const double b1[3] = {gq[c1 * 3], gq[c1 * 3 + 1], gq[c1 * 3 + 2]};
#pragma unroll
      for (int k = 0; k < kE2BPL; ++k) {
        const double* gi = gq + kE2NSH * 3 + bi[k] * 3;  // dw g(i)
        // slots 0..3 always read column c0, slot 5 column c1 (equal to c0 on
        // single-column lanes); only slot 4 differs between lanes
        const bool s1 = k == 5 || (k == 4 && ((sel >> 4) & 1u));
        const double a[3] = {gi[0], gi[1], gi[2]};
        const double b[3] = {s1 ? b1[0] : b0[0], s1 ? b1[1] : b0[1], s1 ? b1[2] : b0[2]};
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = 0; je < 3; ++je) acc[k][ie * 3 + je] = fma(a[ie], b[je], acc[k][ie * 3 + je]);
      }
    }
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k) {
      const double tr = mu * (acc[k][0] + acc[k][4] + acc[k][8]);
      double kb[9];
#pragma unroll
      for (int ie = 0; ie < 3; ++ie)
#pragma unroll
        for (int je = 0; je < 3; ++je)
          kb[ie * 3 + je] = fma(lam, acc[k][ie * 3 + je], fma(mu, acc[k][je * 3 + ie], ie == je ? tr : 0.0));
#pragma unroll
      for (int m = 0; m < 9; ++m) acc[k][m] = kb[m];
    }
    __syncwarp();  // gradients no longer read: the region becomes the staging of K
    // ---- stage the element matrix (mirrors included), then coalesced stores ----
#pragma unroll
    for (int k = 0; k < kE2BPL; ++k) {
      if (!((live >> k) & 1u)) continue;
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

namespace pib {

// ---------------------------------------------------------------------------
// Isotropic elasticity as one FP64 tensor-core product per element
// (p3_elastic_mma_kernel, the p = 3 default).  Lam and mu are constant per
// element, so the block form of integrate_optimized (integrate_ref.cpp:93-130)
//   K[(i,ie),(j,je)] = sum_q dw [lam g_ie(i) g_je(j) + mu g_je(i) g_ie(j) + mu d_(ie,je) g(i).g(j)]
// is an epilogue over the nine products
//   S_(ie,je)(i, j) = sum_q (dw_q g_ie(i, q)) g_je(j, q),
//   K[(i,ie),(j,je)] = lam S_(ie,je)(i,j) + mu S_(je,ie)(i,j) + mu d_(ie,je) (S_00 + S_11 + S_22)(i,j):
// a [3 N_sh x N_q] x [N_q x 3 N_sh] product on DMMA m8n8k4 (9 FMAs per block
// and point instead of the 27-FLOP update, and on the tensor pipe).
//  * one CTA per element (persistent, two per SM); the last N_q threads
//    form the inverse Jacobian and dw of their rule point -- for element
//    e+1 between the products and the epilogue of element e, its vertices
//    prefetched by cp.async during the products;
//  * the CTA writes B_d(q, i) = g_d(i, q) and A_d(q, i) = dw_q g_d(i, q) to
//    shared memory ([d][q][i], row pitch = 8 mod 16 doubles: a warp's
//    fragment load is two conflict-free wavefronts), the gradients formed
//    from the factors of the tensor basis phi_(t,a) = m_t P_a;
//  * warp w owns PPW (t_i, t_j >= t_i) pairs of 8 x 8 (i, j) tiles and
//    accumulates the nine S_(ie,je) tiles of each (18 doubles per pair);
//  * the epilogue forms K in registers (a lane holds every (ie, je) of its
//    (i, j) positions), stages each tile pair as a 24 x 24 block of K over
//    the dead operands and writes it as 192-byte row segments, the mirror of
//    an off-diagonal pair as the transposed block (other layouts / FP32:
//    scalar stores from registers).
#ifndef PI_EMMA_NW3
#define PI_EMMA_NW3 5
#endif
#ifndef PI_EMMA_GUNROLL
#define PI_EMMA_GUNROLL 4
#endif
constexpr int kEmmaGUnroll = PI_EMMA_GUNROLL;  // gradient-loop unroll (phi loads in flight)
#ifndef PI_EMMA_KUNROLL
#define PI_EMMA_KUNROLL 1
#endif
constexpr int kEmmaKUnroll = PI_EMMA_KUNROLL;  // product k-loop unroll
template <int P>
struct EMma {
  static constexpr int NV = P + 1, NTR = (P + 1) * (P + 2) / 2;
  static constexpr int NSH = NTR * NV;
  static constexpr int NS = P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : 25, NZ = P + 1;
  static constexpr int NQ = NS * NZ;  // q = z * NS + s (host_refelem.cpp prism_quadrature)
  static constexpr int NT = (NSH + 7) / 8;                 // 8-wide (i) tiles
  static constexpr int NSHP = NT * 8 % 16 == 8 ? NT * 8 : NT * 8 + 8;
  static constexpr int NQP = (NQ + 3) / 4 * 4, KS = NQP / 4;
  static constexpr int DIM = 3 * NSH;
  static constexpr int NPAIR = NT * (NT + 1) / 2;
  static constexpr int NW = P == 3 ? PI_EMMA_NW3 : (NPAIR + 2) / 3;   // warps
  static constexpr int PPW = (NPAIR + NW - 1) / NW;          // tile pairs per warp
  static constexpr int NTHREADS = 32 * NW;
  static constexpr int OFF_A = 0, OFF_B = 3 * NQP * NSHP, OFF_INV = 6 * NQP * NSHP;  // sInv [NQ][10]: inv, dw
  static constexpr int OFF_X = OFF_INV + NQ * 10;
  static constexpr int OFF_MT = OFF_X + 18;
  static constexpr int OFF_PZ = OFF_MT + 3 * NTR * NS;
  static constexpr int DOUBLES = OFF_PZ + 2 * NV * NZ;
  // staged epilogue: whole tiles only; a warp's 24 x 24 block (row pitch PT)
  // fits in the dead operands
  static constexpr int PT = 26;
#ifdef PI_EMMA_NOSTAGE
  static constexpr bool STAGED = false;
#else
  static constexpr bool STAGED = NSH % 8 == 0;
#endif
  static_assert(!STAGED || NW * 24 * PT <= OFF_INV, "staging fits in the operands");
  static constexpr size_t BYTES = DOUBLES * sizeof(double);
  static_assert(NQ <= NTHREADS, "one thread per rule point");
};

// (t_i, t_j >= t_i) of pair index k in row-major order
template <int NT>
__device__ __forceinline__ void emma_pair(int k, int& ti, int& tj) {
  ti = 0;
  while (k >= NT - ti) k -= NT - ti++;
  tj = ti + k;
}

template <int P>
__global__ void __launch_bounds__(EMma<P>::NTHREADS, 2) p3_elastic_mma_kernel(LaunchArgs args, DenseTables tab) {
  using C = EMma<P>;
  constexpr int NSH = C::NSH, NQ = C::NQ, NQP = C::NQP, NSHP = C::NSHP, NT = C::NT, PPW = C::PPW, DIM = C::DIM;
  constexpr int64_t KK = static_cast<int64_t>(DIM) * DIM;
  constexpr int PT = C::PT;
  extern __shared__ __align__(16) double em_smem[];
  double* sA = em_smem + C::OFF_A;
  double* sB = em_smem + C::OFF_B;
  double* sInv = em_smem + C::OFF_INV;
  double* sX = em_smem + C::OFF_X;  // the element's 18 vertex coordinates (prefetched)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* sMt = em_smem + C::OFF_MT;  // m_t(s), dm1_t(s), dm2_t(s): [3][NTR][NS]
  double* sPz = em_smem + C::OFF_PZ;  // P_a(z), P'_a(z): [2][NV][NZ]
  // padding rows (q >= NQ) and columns (i >= NSH) stay zero
  for (int k = tid; k < C::OFF_INV; k += C::NTHREADS) em_smem[k] = 0.0;
  // the factors of the tensor basis, read off the shape table: at level z = 0
  // and a = 0 (P_0 = 1) phi_k((t,0), (0,s)) = m_t(s), dm1_t(s), dm2_t(s); at
  // t = 0 (m_0 = 1) phi_0 / phi_3((0,a), (z,0)) = P_a(z) / P'_a(z)
  for (int k = tid; k < 3 * C::NTR * C::NS; k += C::NTHREADS) {
    const int c = k / (C::NTR * C::NS), t = (k / C::NS) % C::NTR, sp = k % C::NS;
    sMt[k] = tab.phi[(sp * 4 + c) * NSH + t * C::NV];
  }
  for (int k = tid; k < 2 * C::NV * C::NZ; k += C::NTHREADS) {
    const int c = k / (C::NV * C::NZ), a = (k / C::NZ) % C::NV, z = k % C::NZ;
    sPz[k] = tab.phi[((z * C::NS) * 4 + (c ? 3 : 0)) * NSH + a];
  }
  int ti[PPW], tj[PPW];
#pragma unroll
  for (int k = 0; k < PPW; ++k) {
    const int pk = warp * PPW + k;
    emma_pair<NT>(pk < C::NPAIR ? pk : C::NPAIR - 1, ti[k], tj[k]);
  }
  // whole 8 x 8 tiles, canonical FP64 16-byte aligned output: each tile pair
  // is staged as a 24 x 24 block of K (over the dead A / B operands) and
  // leaves as 192-byte row segments, its mirror as the transposed block
  const bool staged = C::STAGED && args.out_layout == PI_OUT_CANONICAL && !args.out32 &&
                      (reinterpret_cast<uintptr_t>(args.out) & 15) == 0;
  // (1) inverse Jacobian and dw per rule point of element ee, from sX, by the
  // last NQ threads: for element e+1 this runs between the products and the
  // epilogue of element e (warp 4 owns the two diagonal tile pairs, the
  // lightest epilogue), off the critical path of the other warps
  const int qj = tid - (C::NTHREADS - NQ);
  auto jacobians = [&](int64_t ee) -> bool {
    if (qj < 0 || ee >= args.n_elem) return false;
    double x[18], d[21];
#pragma unroll
    for (int c = 0; c < 18; ++c) x[c] = sX[c];
    prism_edges(x, d);
    double cf[3][3];
    const double det = jacobian_cofactors(d, __ldg(tab.pts + 3 * qj), __ldg(tab.pts + 3 * qj + 1), __ldg(tab.pts + 3 * qj + 2), cf);
    const double id = __drcp_rn(det);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) sInv[qj * 10 + k * 3 + dd] = cf[dd][k] * id;  // inv[k][dd]
    sInv[qj * 10 + 9] = det * __ldg(tab.w + qj);
    return !(det > 0.0);
  };
  if (tid < 18 && blockIdx.x < args.n_elem) sX[tid] = args.geom[tid * args.geom_ld + blockIdx.x];
  __syncthreads();
  if (__syncthreads_or(jacobians(blockIdx.x)) && tid == 0) flag_inverted(args.bad, args.element_id_base + blockIdx.x);
  for (int64_t e = blockIdx.x; e < args.n_elem; e += gridDim.x) {
    double lam, mu;
    {
      const double young = args.coeff ? args.coeff[e] : args.cu[0];
      const double nu = args.coeff ? args.coeff[args.coeff_ld + e] : args.cu[1];
      if (tid == 0) check_material(args, e, young, nu);
      lame(young, nu, lam, mu);
    }
    // (2) B_d(q, i) = g_d(i, q), A_d(q, i) = dw_q g_d(i, q); with the tensor
    // basis phi_(t,a) = m_t(xi1, xi2) P_a(xi3) and q = (z, s):
    //   g_d((t,a), (z,s)) = (inv[0][d] dm1_t(s) + inv[1][d] dm2_t(s)) P_a(z) + inv[2][d] m_t(s) P'_a(z)
    // one item = (q, t), all a (tables in shared memory, 16-byte stores)
#pragma unroll kEmmaGUnroll
    for (int it = tid; it < NQ * C::NTR; it += C::NTHREADS) {
      const int q = it / C::NTR, t = it - q * C::NTR, z = q / C::NS, sp = q - z * C::NS;
      const double m = sMt[(0 * C::NTR + t) * C::NS + sp], m1 = sMt[(1 * C::NTR + t) * C::NS + sp],
                   m2 = sMt[(2 * C::NTR + t) * C::NS + sp];
      const double* inv = sInv + q * 10;
      const double dw = inv[9];
      double u[3], w[3];
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) {
        u[dd] = fma(inv[dd], m1, inv[3 + dd] * m2);
        w[dd] = inv[6 + dd] * m;
      }
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) {
        double g[C::NV];
#pragma unroll
        for (int a = 0; a < C::NV; ++a) g[a] = fma(u[dd], sPz[a * C::NZ + z], w[dd] * sPz[(C::NV + a) * C::NZ + z]);
        double* rb = sB + (dd * NQP + q) * NSHP + t * C::NV;
        double* ra = sA + (dd * NQP + q) * NSHP + t * C::NV;
        if constexpr (C::NV % 2 == 0 && NSHP % 2 == 0) {
#pragma unroll
          for (int a = 0; a < C::NV; a += 2) {
            *reinterpret_cast<double2*>(rb + a) = make_double2(g[a], g[a + 1]);
            *reinterpret_cast<double2*>(ra + a) = make_double2(dw * g[a], dw * g[a + 1]);
          }
        } else {
#pragma unroll
          for (int a = 0; a < C::NV; ++a) {
            rb[a] = g[a];
            ra[a] = dw * g[a];
          }
        }
      }
    }
    __syncthreads();
    // the next element's vertices, in flight during the products
    // (cp.async: no registers held across the products)
    const int64_t en = e + gridDim.x;
    if (tid < 18 && en < args.n_elem) cp_async8(sX + tid, args.geom + tid * args.geom_ld + en);
    cp_async_commit();
    // (3) S_(ie,je) tiles of the warp's pairs
    double acc[PPW][9][2];
#pragma unroll
    for (int k = 0; k < PPW; ++k)
#pragma unroll
      for (int m = 0; m < 9; ++m) acc[k][m][0] = acc[k][m][1] = 0.0;
    const int fo = (lane & 3) * NSHP + (lane >> 2);  // fragment offset: row q = lane % 4, column lane / 4
#pragma unroll kEmmaKUnroll
    for (int ks = 0; ks < C::KS; ++ks) {
      const int ko = 4 * ks * NSHP + fo;
#pragma unroll
      for (int k = 0; k < PPW; ++k) {
        double a[3], b[3];
#pragma unroll
        for (int dd = 0; dd < 3; ++dd) {
          a[dd] = sA[dd * NQP * NSHP + ko + 8 * ti[k]];
          b[dd] = sB[dd * NQP * NSHP + ko + 8 * tj[k]];
        }
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int je = 0; je < 3; ++je) dmma_8x8x4(acc[k][ie * 3 + je][0], acc[k][ie * 3 + je][1], a[ie], b[je]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // every warp's products done: A / B become the staging, sInv is free, sX holds e+1
    const bool inverted_next = jacobians(en);
    // (4) epilogue: K from S in registers
    double* sT = em_smem + warp * (24 * PT);  // the warp's 24 x 24 block
#pragma unroll
    for (int k = 0; k < PPW; ++k) {
      if (warp * PPW + k >= C::NPAIR) break;
      const int il = lane >> 2, jl0 = 2 * (lane & 3);
      const int i = 8 * ti[k] + il, j0 = 8 * tj[k] + jl0;
      const bool diag = ti[k] == tj[k];
      const double tr[2] = {mu * (acc[k][0][0] + acc[k][4][0] + acc[k][8][0]),
                            mu * (acc[k][0][1] + acc[k][4][1] + acc[k][8][1])};
      // K row (i, ie), column (j0 + h, je)
      auto kv = [&](int ie, int je, int h) {
        return fma(lam, acc[k][ie * 3 + je][h], fma(mu, acc[k][je * 3 + ie][h], ie == je ? tr[h] : 0.0));
      };
      const int64_t base = e * KK;
      if (staged) {
        // block rows 3 il + ie, columns 3 jl + je; diagonal tiles keep the
        // upper triangle and mirror it in the block
#pragma unroll
        for (int ie = 0; ie < 3; ++ie)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int je = 0; je < 3; ++je) {
              const int rr = 3 * il + ie, cc = 3 * (jl0 + h) + je;
              if (diag) {
                if (rr <= cc) {
                  const double val = kv(ie, je, h);
                  sT[rr * PT + cc] = val;
                  sT[cc * PT + rr] = val;
                }
              } else {
                sT[rr * PT + cc] = kv(ie, je, h);
              }
            }
        __syncwarp();
        double* rowblk = args.out + base + static_cast<int64_t>(24 * ti[k]) * DIM + 24 * tj[k];
        // half-warp per row: 24 rows x 12 double2 (lanes 12..15 of each half idle)
        const int hr = lane >> 4, c2 = lane & 15;
        if (c2 < 12) {
#pragma unroll 4
          for (int rr = hr; rr < 24; rr += 2) {
            const double2 w = *reinterpret_cast<const double2*>(sT + rr * PT + 2 * c2);
            *reinterpret_cast<double2*>(rowblk + static_cast<int64_t>(rr) * DIM + 2 * c2) = w;
          }
          if (!diag) {  // transposed: row cc of the mirror = column cc of the block
            double* colblk = args.out + base + static_cast<int64_t>(24 * tj[k]) * DIM + 24 * ti[k];
#pragma unroll 4
            for (int cc = hr; cc < 24; cc += 2) {
              const double2 w = make_double2(sT[(2 * c2) * PT + cc], sT[(2 * c2 + 1) * PT + cc]);
              *reinterpret_cast<double2*>(colblk + static_cast<int64_t>(cc) * DIM + 2 * c2) = w;
            }
          }
        }
        __syncwarp();  // block read out before the warp's next pair overwrites it
      } else if (i < NSH) {
#pragma unroll
      for (int ie = 0; ie < 3; ++ie) {
        const int r = 3 * i + ie;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = j0 + h;
          if (j >= NSH) continue;
#pragma unroll
          for (int je = 0; je < 3; ++je) {
            const int c = 3 * j + je;
            if (diag && r > c) continue;  // the lane owning (j, i) writes it
            const double val = kv(ie, je, h);
            if (args.out_layout == PI_OUT_SOA) {
              store_out(args, static_cast<int64_t>(r * DIM + c) * args.ld_out + e, val);
              if (r != c) store_out(args, static_cast<int64_t>(c * DIM + r) * args.ld_out + e, val);
            } else {
              store_out(args, base + static_cast<int64_t>(r) * DIM + c, val);
              if (r != c) store_out(args, base + static_cast<int64_t>(c) * DIM + r, val);
            }
          }
        }
      }
      }
    }
    // element e+1's Jacobians visible; the staging read out before its gradients
    if (__syncthreads_or(inverted_next) && tid == 0) flag_inverted(args.bad, args.element_id_base + en);
  }
}

}  // namespace pib
