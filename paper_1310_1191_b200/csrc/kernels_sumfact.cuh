// Sum-factorised element stiffness on the FP64 tensor pipe (p = 2..7).
//
// The prism basis is a tensor product, phi_(t,a)(xi) = m_t(xi1,xi2) P_a(xi3)
// (reference_element.cpp:230-270, dof = t*(p+1)+a), and the rule is a tensor
// product of a triangle rule (points s) and Gauss-Legendre (points z)
// (reference_element.cpp:175-193, q = z*N_s + s).  Grouping the reference
// derivative index k by its triangle factor
//     x = 0: d/dxi1 m (k=1, P)    x = 1: d/dxi2 m (k=2, P)
//     x = 2: m        (k=0, P  and k=3, P')
// the integral of integrate_generic (integrate_ref.cpp:79-88) re-associates as
//     H_xy(s,a,b) = sum_z sum_{k in x, l in y} Y_k(a,z) M_kl(s,z) Y_l(b,z)
//     G_x(s,a,j)  = sum_y H_xy(s,a,b_j) X_y(t'_j, s)          j = t'*(p+1)+b
//     K[(t,a), j] = sum_(s,x) X_x(t,s) G_x(s,a,j)             <- DMMA GEMM
// with M = T (det w C) T^T the per-point 4x4 block (kernels_common.cuh).
// Only the last line is O(N_sh^2 N_s); it runs as m8n8k4 FP64 MMAs with the
// element-independent X table as the A operand (staged once per CTA in
// fragment order) and G (element-specific) staged per chunk of 4 triangle
// points in fragment order by the warp that consumes it.
#pragma once

#include "kernels_common.cuh"

namespace pib {

template <int P>
struct SumFactShape {
  static constexpr int NV = P + 1;                    // Legendre modes / GL points
  static constexpr int NZ = P + 1;
  static constexpr int NT = (P + 1) * (P + 2) / 2;    // triangle monomials
  static constexpr int NS = (P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : P == 5 ? 25 : P == 6 ? 33 : 42);
  static constexpr int NSP = (NS + 3) / 4 * 4;        // padded to whole chunks
  static constexpr int NSH = NT * NV;
  static constexpr int NQ = NS * NZ;
  static constexpr int MT = (NT + 7) / 8;             // m-tiles of the X operand
  static constexpr int NTILE = (NSH + 7) / 8;         // n-tiles of one K row block
  static constexpr int KSTEPS = 3 * NSP / 4;          // k4-steps over (s, x)
  static constexpr int NCHUNK = NSP / 4;              // 4 triangle points per chunk
  static constexpr int XFRAG = MT * KSTEPS * 32;      // doubles in the A-fragment table
};

// Launch shape: EPC elements x AG Legendre rows `a` per CTA; each warp owns
// WA rows a x NB n-tiles x all MT m-tiles of accumulators (WA*NB*MT frags).
template <int P>
struct SumFactLaunch;
template <> struct SumFactLaunch<2> { static constexpr int EPC = 8, AG = 3, WA = 3, NB = 3; };
template <> struct SumFactLaunch<3> { static constexpr int EPC = 4, AG = 4, WA = 2, NB = 5; };
template <> struct SumFactLaunch<4> { static constexpr int EPC = 2, AG = 5, WA = 1, NB = 10; };
template <> struct SumFactLaunch<5> { static constexpr int EPC = 1, AG = 6, WA = 1, NB = 8; };
template <> struct SumFactLaunch<6> { static constexpr int EPC = 1, AG = 1, WA = 1, NB = 5; };
template <> struct SumFactLaunch<7> { static constexpr int EPC = 1, AG = 1, WA = 1, NB = 4; };

template <int P>
struct SumFactConfig : SumFactShape<P>, SumFactLaunch<P> {
  using S = SumFactShape<P>;
  using L = SumFactLaunch<P>;
  static constexpr int NBLK = (S::NTILE + L::NB - 1) / L::NB;
  static constexpr int WPE = (L::AG / L::WA) * NBLK;   // warps per element
  static constexpr int NWARPS = L::EPC * WPE;
  static constexpr int NTHREADS = 32 * NWARPS;
  static constexpr int NAG = S::NV / L::AG;            // CTAs per element group
  static_assert(S::NV % L::AG == 0 && L::AG % L::WA == 0, "bad a-grouping");
  static_assert(S::NTILE % L::NB == 0, "n-tiles must split evenly");
  // shared memory layout (doubles)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_M = OFF_X + S::XFRAG;
  static constexpr int OFF_H = OFF_M + L::EPC * S::NQ * 16;
  static constexpr int H_PER_BUF = L::EPC * L::AG * 4 * S::NV * 9;
  static constexpr int OFF_G = OFF_H + 2 * H_PER_BUF;
  static constexpr int G_PER_WARP = L::WA * L::NB * 3 * 32;
  static constexpr int OFF_GEOM = OFF_G + NWARPS * G_PER_WARP;
  static constexpr int OFF_C = OFF_GEOM + L::EPC * 18;
  static constexpr int OFF_LINE = OFF_C + L::EPC * 16;  // Y tables [2][NV][NZ], xi3 [NZ]
  static constexpr int OFF_TRI = OFF_LINE + 2 * S::NV * S::NZ + S::NZ;  // xi1, xi2 [NS]
  static constexpr int OFF_W = OFF_TRI + 2 * S::NS;                     // weights [NQ]
  static constexpr int SMEM_DOUBLES = OFF_W + S::NQ;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
};

// Per-p constant tables in device memory (built by the host from the shape
// table, pi_context.cu): X in A-fragment order, Y = (P, P') at GL points,
// the triangle and line coordinates, and the rule weights in rule order.
struct SumFactTables {
  const double* xfrag;  // [MT][KSTEPS][32]
  const double* yline;  // [2][NV][NZ] then xi3 [NZ]
  const double* tri;    // [2][NS]: xi1 then xi2
  const double* w;      // [NQ]
};

template <int P, bool GENERAL>
__global__ void __launch_bounds__(SumFactConfig<P>::NTHREADS)
    sumfact_kernel(LaunchArgs args, SumFactTables tab) {
  using C = SumFactConfig<P>;
  constexpr int NV = C::NV, NZ = C::NZ, NT = C::NT, NS = C::NS, NSH = C::NSH, NQ = C::NQ;
  constexpr int MT = C::MT, KSTEPS = C::KSTEPS, EPC = C::EPC, AG = C::AG, WA = C::WA, NB = C::NB;
  extern __shared__ __align__(16) double smem[];
  double* sX = smem + C::OFF_X;
  double* sM = smem + C::OFF_M;
  double* sH = smem + C::OFF_H;
  double* sGeom = smem + C::OFF_GEOM;
  double* sC = smem + C::OFF_C;
  double* sY = smem + C::OFF_LINE;
  double* sTri = smem + C::OFF_TRI;
  double* sW = smem + C::OFF_W;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t egroup = blockIdx.x / C::NAG;
  const int agroup = blockIdx.x % C::NAG;
  const int64_t e0 = egroup * EPC;

  // ---- stage per-p tables and per-element inputs ----
  for (int i = tid; i < C::XFRAG; i += C::NTHREADS) sX[i] = tab.xfrag[i];
  for (int i = tid; i < 2 * NV * NZ + NZ; i += C::NTHREADS) sY[i] = tab.yline[i];
  for (int i = tid; i < 2 * NS; i += C::NTHREADS) sTri[i] = tab.tri[i];
  for (int i = tid; i < NQ; i += C::NTHREADS) sW[i] = tab.w[i];
  for (int i = tid; i < EPC * 18; i += C::NTHREADS) {
    const int el = i / 18, c = i % 18;
    const int64_t e = e0 + el;
    const int64_t ec = e < args.n_elem ? e : args.n_elem - 1;  // pad with a valid element
    sGeom[i] = args.geom[c * args.geom_ld + ec];
  }
  if (GENERAL) {
    for (int i = tid; i < EPC * 16; i += C::NTHREADS) {
      const int el = i / 16, c = i % 16;
      const int64_t e = e0 + el;
      const int64_t ec = e < args.n_elem ? e : args.n_elem - 1;
      sC[i] = args.coeff ? args.coeff[c * args.coeff_ld + ec] : args.cu[c];
    }
  }
  __syncthreads();

  // ---- M(s,z) for every rule point of every element of the CTA ----
  for (int i = tid; i < EPC * NQ; i += C::NTHREADS) {
    const int el = i / NQ, q = i % NQ;
    const int s = q % NS, z = q / NS;
    double inv[3][3];
    const double det = prism_jacobian(sGeom + 18 * el, sTri[s], sTri[NS + s], sY[2 * NV * NZ + z], inv);
    const int64_t e = e0 + el;
    if (!(det > 0.0) && e < args.n_elem && agroup == 0) flag_inverted(args.bad, args.element_id_base + e);
    double M[16];
    coefficient_block<GENERAL>(inv, det * sW[q], sC + 16 * el, M);
    double* dst = sM + (el * NQ + q) * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) dst[k] = M[k];
  }

  // ---- warp task ----
  const int el_w = warp / C::WPE;
  const int r_w = warp % C::WPE;
  const int a_w0 = agroup * AG + (r_w / C::NBLK) * WA;  // first Legendre row a of this warp
  const int nt0 = (r_w % C::NBLK) * NB;
  double* sG = smem + C::OFF_G + warp * C::G_PER_WARP;

  double acc[WA][MT][NB][2];
#pragma unroll
  for (int wa = 0; wa < WA; ++wa)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) acc[wa][mt][nb][0] = acc[wa][mt][nb][1] = 0.0;

  const double* Pv = sY;            // P_a(z)  [NV][NZ]
  const double* Pd = sY + NV * NZ;  // P'_a(z) [NV][NZ]

  for (int chunk = 0; chunk < C::NCHUNK; ++chunk) {
    double* Hb = sH + (chunk & 1) * C::H_PER_BUF;
    __syncthreads();  // M ready (first pass) / previous H buffer reuse is safe
    // ---- H_xy(s,a,b) for the chunk's 4 triangle points ----
    for (int i = tid; i < C::H_PER_BUF; i += C::NTHREADS) {
      // i = (((el*AG + al)*4 + sl)*NV + b)*9 + xy
      const int xy = i % 9, b = (i / 9) % NV, sl = (i / (9 * NV)) % 4;
      const int al = (i / (36 * NV)) % AG, el = i / (36 * NV * AG);
      const int s = chunk * 4 + sl, a = agroup * AG + al;
      const int x = xy / 3, y = xy % 3;
      double h = 0.0;
      if (s < NS) {
#pragma unroll
        for (int z = 0; z < NZ; ++z) {
          const double* M = sM + (el * NQ + z * NS + s) * 16;
          const double pa = Pv[a * NZ + z], pb = Pv[b * NZ + z];
          const double da = Pd[a * NZ + z], db = Pd[b * NZ + z];
          // left factor: sum_{k in x} Y_k(a) M_k. ; right: sum_{l in y} ... Y_l(b)
          double u[4];
          if (x < 2) {
#pragma unroll
            for (int l = 0; l < 4; ++l) u[l] = pa * M[(x + 1) * 4 + l];
          } else {
#pragma unroll
            for (int l = 0; l < 4; ++l) u[l] = GENERAL ? pa * M[l] + da * M[12 + l] : da * M[12 + l];
          }
          if (y < 2) {
            h += u[y + 1] * pb;
          } else {
            h += GENERAL ? u[0] * pb + u[3] * db : u[3] * db;
          }
        }
      }
      Hb[i] = h;
    }
    __syncthreads();

    // ---- G for this warp's (a, n-tile) block, written in B-fragment order ----
    __syncwarp();
#pragma unroll 1
    for (int f = 0; f < WA * NB * 3; ++f) {
      const int ks = f % 3, nb = (f / 3) % NB, wa = f / (3 * NB);
      const int kk = ks * 4 + (lane & 3);  // 0..11 within the chunk
      const int sl = kk / 3, x = kk % 3;
      const int s = chunk * 4 + sl;
      const int j = (nt0 + nb) * 8 + (lane >> 2);
      double g = 0.0;
      if (s < NS && j < NSH) {
        const int tp = j / NV, b = j % NV;
        const int al = a_w0 + wa - agroup * AG;
        const double* H = Hb + (((el_w * AG + al) * 4 + sl) * NV + b) * 9 + x * 3;
#pragma unroll
        for (int yy = 0; yy < 3; ++yy) {
          const int kx = s * 3 + yy;
          const double X = sX[((tp >> 3) * KSTEPS + (kx >> 2)) * 32 + (tp & 7) * 4 + (kx & 3)];
          g += H[yy] * X;
        }
      }
      sG[f * 32 + lane] = g;
    }
    __syncwarp();

    // ---- K[t][(a, j)] += X[t][(s,x)] G[(s,x)][(a,j)] on the tensor pipe ----
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      const int kstep = chunk * 3 + ks;
      double afr[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) afr[mt] = sX[(mt * KSTEPS + kstep) * 32 + lane];
#pragma unroll
      for (int wa = 0; wa < WA; ++wa)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const double bfr = sG[((wa * NB + nb) * 3 + ks) * 32 + lane];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma_8x8x4(acc[wa][mt][nb][0], acc[wa][mt][nb][1], afr[mt], bfr);
        }
    }
  }

  // ---- epilogue: fragments -> K rows (t*NV + a), columns j ----
  const int64_t e = e0 + el_w;
  if (e >= args.n_elem) return;
  const int64_t kk_elem = static_cast<int64_t>(NSH) * NSH;
#pragma unroll
  for (int wa = 0; wa < WA; ++wa)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int t = mt * 8 + (lane >> 2);
      if (t >= NT) continue;
      const int row = t * NV + a_w0 + wa;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int j = (nt0 + nb) * 8 + 2 * (lane & 3);
        if (args.out_layout == PI_OUT_CANONICAL) {
          double* dst = args.out + e * kk_elem + static_cast<int64_t>(row) * NSH + j;
          if ((NSH % 2 == 0) && j + 1 < NSH) {
            *reinterpret_cast<double2*>(dst) = make_double2(acc[wa][mt][nb][0], acc[wa][mt][nb][1]);
          } else {
            if (j < NSH) dst[0] = acc[wa][mt][nb][0];
            if (j + 1 < NSH) dst[1] = acc[wa][mt][nb][1];
          }
        } else {
          const int64_t base = static_cast<int64_t>(row) * NSH + j;
          if (j < NSH) args.out[base * args.ld_out + e] = acc[wa][mt][nb][0];
          if (j + 1 < NSH) args.out[(base + 1) * args.ld_out + e] = acc[wa][mt][nb][1];
        }
      }
    }
}

}  // namespace pib
