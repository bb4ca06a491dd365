// Symmetric sum factorisation over (a', b') PAIRS across CTAs (scalar forms,
// p >= 5; at p <= 4 a CTA holds whole elements and kernels_sumfact.cuh pairs
// within the CTA; for n_eq = 3 the row split measured faster).
//
// For a symmetric coefficient tensor K is symmetric:
//     K[(t,a'),(t',b')] = K[(t',b'),(t,a')],
// so only the vertical-index pairs a' <= b' need the GEMM of
// kernels_sumfact.cuh.  At p >= 5 one element's K is split over several CTAs
// by rows a' there, which forbids skipping the mirrored half.  This kernel
// splits an element by PAIRS instead: a work item is (element, group of
// pairs); each consumer warp owns PPW pairs and, t'-major, all MT x MT tiles
// of each (MT (MT+1) / 2 for a diagonal pair).  For the pair (a', b') and the
// k-row (s, x) a lane's B fragment is
//     G = sum_y H_xy(s, a', b') X_y(t', s),     t' = 8 g + lane/4,
// so only H for the item's own pairs is formed by the producers (no H for
// a' > b').  Blocks are stored straight from registers together with their
// mirrors; a CTA walks all pair items of its element, whose 32-byte sectors
// are completed across items and merge in L2.
// About 56 % of the MMAs and fragment FMAs of the row split.
#pragma once

#include "kernels_sumfact.cuh"

namespace pib {

#ifndef PI_PAIRS_NBUF  // H ring depth (p = 5: +3 %, p = 6: +1.4 % over 3)
#define PI_PAIRS_NBUF 4
#endif
#ifndef PI_PAIRS_NBUF7  // p = 7: 4 buffers measured -1.5 %
#define PI_PAIRS_NBUF7 3
#endif

template <int P, int NE>
struct PairsConfig {
  using SF = SumFactConfig<P, NE>;  // shares the per-p tables (X fragments, X plain, Y, rule)
  static constexpr int NV = P + 1, NZ = P + 1, NVE = NE * NV, NT = SF::NT, NS = SF::NS, NSP = SF::NSP;
  static constexpr int NSH = NT * NVE, NQ = SF::NQ, MT = SF::MT, KSTEPS = SF::KSTEPS, NCHUNK = SF::NCHUNK;
  static constexpr int NTPS = SF::NTPS;
  static_assert(NTPS >= MT * 8, "t'-major columns need MT*8 rows of the X table");
  static constexpr int NPAIR = NVE * (NVE + 1) / 2;
  // pairs per consumer warp (accumulators PPW*MT*MT*2), consumer / producer warps
#ifndef PI_PAIRS_CFG7
#define PI_PAIRS_CFG7 1, 9, 3
#endif
  struct Cfg {
    int ppw, ncw, npw;
  };
#ifndef PI_PAIRS_CFG5
#define PI_PAIRS_CFG5 1, 7, 3
#endif
#ifndef PI_PAIRS_CFG6
#define PI_PAIRS_CFG6 1, 7, 3
#endif
  static constexpr Cfg cfg() {
    if (NE == 1 && P == 7) {
      constexpr int v[3] = {PI_PAIRS_CFG7};
      return {v[0], v[1], v[2]};
    }
    if (NE == 1 && P == 6) {
      constexpr int v[3] = {PI_PAIRS_CFG6};
      return {v[0], v[1], v[2]};
    }
    if (NE == 1 && P == 5) {
      constexpr int v[3] = {PI_PAIRS_CFG5};
      return {v[0], v[1], v[2]};
    }
    if (NE == 1) return {1, 7, 3};
    return {MT <= 2 ? 4 : MT == 3 ? 2 : 1, 8, 4};
  }
  static constexpr int PPW = cfg().ppw, NCW = cfg().ncw, NPW = cfg().npw;
  static constexpr int NWARPS = NCW + NPW, NTHREADS = 32 * NWARPS, NPT = 32 * NPW;
  static constexpr int PPI = NCW * PPW;         // pairs per work item
  static constexpr int NITEM = (NPAIR + PPI - 1) / PPI;  // items per element
  static constexpr int NCOEF = 16 * NE * NE;
  // H ring: [PPI][4 s][3 x][HY] (HY = 4: y + pad; odd-ish s stride against bank conflicts)
  static constexpr int HX = 4, HSL = 3 * HX + 2, HPAIR = 4 * HSL + 2;
  static constexpr int H_PER_BUF = PPI * HPAIR;
  static constexpr int NBUF = P == 7 ? PI_PAIRS_NBUF7 : PI_PAIRS_NBUF;
  // M: all points of the element (scalar forms), double buffered across items
  static constexpr bool MALL = NE == 1;
#ifdef PI_SF_MS_EVEN
  static constexpr int MS = NZ;
#else
  static constexpr int MS = NZ | 1;  // odd point stride per s (kernels_sumfact.cuh MS)
#endif
  static constexpr int MITEMS = (MALL ? NSP : 4) * MS;
  static constexpr int MPITCH = MITEMS | 1;
  static constexpr int M_PER_BUF = NE * NE * 16 * MPITCH;
  static constexpr int OFF_XA = 0;
  static constexpr int OFF_XP = OFF_XA + SF::XFRAG;
  static constexpr int OFF_H = OFF_XP + SF::XPLAIN;
  static constexpr int OFF_M = OFF_H + NBUF * H_PER_BUF;
  static constexpr int OFF_GEOM = OFF_M + (MALL ? 2 : 1) * M_PER_BUF;
  static constexpr int OFF_C = OFF_GEOM + 22;
  static constexpr int OFF_LINE = OFF_C + NCOEF;
  static constexpr int OFF_TRI = OFF_LINE + (2 * NV * NZ + NZ + 1) / 2 * 2;
  static constexpr int OFF_W = OFF_TRI + 2 * NS;
  static constexpr int SMEM_DOUBLES = OFF_W + (NQ + 1) / 2 * 2;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
  // fused load vectors (sumfact_load_vectors): dw [NSP][NZ], u [NSP][NV]
  static constexpr int OFF_LDW = SMEM_DOUBLES, OFF_LU = OFF_LDW + NSP * NZ;
  static constexpr size_t SMEM_BYTES_LOAD = sizeof(double) * (OFF_LU + NSP * NV);
  // named barriers: FULL 1..3, EMPTY 4..6, producers 7
  static constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + NBUF, BAR_PROD = 1 + 2 * NBUF;
};

// pair index -> (a', b') with a' <= b'.  Pairs are ordered by 4 x 4 blocks of
// the (a', b') triangle (blocks row-major, pairs row-major inside a block), so
// consecutive items complete whole 32-byte sectors of K -- 4 consecutive b'
// of a row, and in the mirrored rows 4 consecutive a' -- while they are in L2.
__device__ __forceinline__ void pair_decode(int k, int nve, int& a, int& b) {
  const int nb = (nve + 3) / 4;
  for (int bi = 0; bi < nb; ++bi)
    for (int bj = bi; bj < nb; ++bj) {
      const int a0 = 4 * bi, a1 = min(nve, a0 + 4), b0 = 4 * bj, b1 = min(nve, b0 + 4);
      const int cnt = bi == bj ? (a1 - a0) * (a1 - a0 + 1) / 2 : (a1 - a0) * (b1 - b0);
      if (k < cnt) {
        if (bi == bj) {  // upper triangle of a diagonal block
          int i = 0;
          while (k >= (a1 - a0) - i) k -= (a1 - a0) - i++;
          a = a0 + i;
          b = a0 + i + k;
        } else {
          a = a0 + k / (b1 - b0);
          b = b0 + k % (b1 - b0);
        }
        return;
      }
      k -= cnt;
    }
  a = b = 0;
}

template <int P, int NE, int FORM>
__global__ void __launch_bounds__(PairsConfig<P, NE>::NTHREADS, 1)
    sumfact_pairs_kernel(LaunchArgs args, SumFactTables tab) {
  using C = PairsConfig<P, NE>;
  constexpr bool GENERAL = FORM == kFormGeneral;
  constexpr int NV = C::NV, NVE = C::NVE, NZ = C::NZ, NT = C::NT, NS = C::NS, NSH = C::NSH, NQ = C::NQ;
  constexpr int NTPS = C::NTPS, MT = C::MT, KSTEPS = C::KSTEPS, NCHUNK = C::NCHUNK, PPW = C::PPW;
  constexpr int NCOEF = C::NCOEF;
  extern __shared__ __align__(16) double smem[];
  double* sXA = smem + C::OFF_XA;
  double* sXP = smem + C::OFF_XP;
  double* sH = smem + C::OFF_H;
  double* sM = smem + C::OFF_M;
  double* sGeom = smem + C::OFF_GEOM;
  double* sC = smem + C::OFF_C;
  double* sY = smem + C::OFF_LINE;
  double* sTri = smem + C::OFF_TRI;
  double* sW = smem + C::OFF_W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- per-p tables by TMA bulk copies ----
  __shared__ __align__(8) uint64_t s_tables;
  if (tid == 0) mbar_init(&s_tables, 1);
  __syncthreads();
  if (tid == 0) {
    constexpr unsigned BX = 8u * C::SF::XFRAG, BP = 8u * C::SF::XPLAIN, BY = 8u * ((2 * NV * NZ + NZ + 1) / 2 * 2),
                       BT = 8u * 2 * NS, BW = 8u * ((NQ + 1) / 2 * 2);
    mbar_arrive_expect_tx(&s_tables, BX + BP + BY + BT + BW);
    bulk_load(sXA, tab.xfrag, BX, &s_tables);
    bulk_load(sXP, tab.xplain, BP, &s_tables);
    bulk_load(sY, tab.yline, BY, &s_tables);
    bulk_load(sTri, tab.tri, BT, &s_tables);
    bulk_load(sW, tab.w, BW, &s_tables);
  }
  mbar_wait(&s_tables, 0);
  const double2* PD = reinterpret_cast<const double2*>(sY);  // (P_a(z), P'_a(z)) [NZ][NV]

  // Element-major: a CTA takes elements blockIdx.x + k * gridDim.x and walks
  // all NITEM pair groups of each, so M is built once per element.
  const int64_t my_elems = blockIdx.x < args.n_elem ? (args.n_elem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_items = my_elems * C::NITEM;
  const int64_t total_chunks = my_items * NCHUNK;

  if (warp >= C::NCW) {
    // ======================= producer warps =======================
    const int ptid = tid - 32 * C::NCW;
    int64_t gc = 0;
    int64_t loaded = -1;  // element whose geometry / M is in shared memory
    int mb = 0;
    auto prepare = [&](int64_t e, int buf, int s_first, int s_count) {
      if (ptid == 0) {
        double x[18], d[21];
#pragma unroll
        for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];
        prism_edges(x, d);
#pragma unroll
        for (int c = 0; c < 21; ++c) sGeom[c] = d[c];
      }
      if (FORM == kFormGeneral) {
        for (int i = ptid; i < NCOEF; i += C::NPT) sC[i] = args.coeff ? args.coeff[i * args.coeff_ld + e] : args.cu[i];
      } else if (FORM == kFormElasticity) {
        if (ptid == 0) {
          const double young = args.coeff ? args.coeff[e] : args.cu[0];
          const double nu = args.coeff ? args.coeff[args.coeff_ld + e] : args.cu[1];
          check_material(args, e, young, nu);
          lame(young, nu, sC[0], sC[1]);
        }
      }
      named_sync(C::BAR_PROD, C::NPT);
      double* sMb = sM + buf * C::M_PER_BUF;
      for (int i = ptid; i < s_count * NZ; i += C::NPT) {
        const int z = i % NZ, s = s_first + i / NZ;
        double* Mi = sMb + (i / NZ) * C::MS + z;
        if (s < NS) {
          double cf[3][3];
          const double det = jacobian_cofactors(sGeom, sTri[s], sTri[NS + s], sY[2 * NV * NZ + z], cf);
          const double w8 = sW[z * NS + s], wd = w8 * __drcp_rn(det);
          if (!(det > 0.0)) flag_inverted(args.bad, args.element_id_base + e);
          if (NE == 1 && args.fout) smem[C::OFF_LDW + s * NZ + z] = det * w8 * load_f(args, e);
#pragma unroll
          for (int blk = 0; blk < NE * NE; ++blk) {
            double M[16];
            if (FORM == kFormElasticity)
              elasticity_block(cf, wd, sC[0], sC[1], blk / NE, blk % NE, M);
            else
              block_from_cofactors<GENERAL>(cf, det, w8, wd, sC + 16 * blk, M);
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (GENERAL || (k >= 4 && (k & 3) != 0)) Mi[(blk * 16 + k) * C::MPITCH] = M[k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16 * NE * NE; ++k) Mi[k * C::MPITCH] = 0.0;
          if (NE == 1 && args.fout) smem[C::OFF_LDW + s * NZ + z] = 0.0;
        }
      }
      named_sync(C::BAR_PROD, C::NPT);
      if (NE == 1 && C::MALL && args.fout) {
        sumfact_load_vectors<NS, C::NSP, NZ, NV, NT, NTPS>(args, e, 1, smem + C::OFF_LDW, smem + C::OFF_LU, sXP, PD,
                                                         ptid, C::NPT, C::BAR_PROD);
        named_sync(C::BAR_PROD, C::NPT);
      }
    };
    for (int64_t it = 0; it < my_items; ++it) {
      const int64_t e = blockIdx.x + (it / C::NITEM) * gridDim.x;
      const int p0 = static_cast<int>(it % C::NITEM) * C::PPI;  // first pair of the item
      if (C::MALL) {
        if (e != loaded) {  // a new element: M for all its points into the other buffer
          mb = loaded < 0 ? 0 : mb ^ 1;
          prepare(e, mb, 0, C::NSP);
          loaded = e;
        }
      }
      for (int chunk = 0; chunk < NCHUNK; ++chunk, ++gc) {
        if (!C::MALL) prepare(e, 0, chunk * 4, 4);
        const int buf = static_cast<int>(gc % C::NBUF);
        if (gc >= C::NBUF) named_sync(C::BAR_EMPTY + buf, C::NTHREADS);
        double* Hb = sH + buf * C::H_PER_BUF;
        // H_x,y(s, a', b'), y = 0..2 for the item's pairs: items (pair, s, x)
        for (int i = ptid; i < C::PPI * 12; i += C::NPT) {
          const int x = i % 3, sl = (i / 3) % 4, pl = i / 12;
          const int pk = p0 + pl;
          double h0 = 0.0, h1 = 0.0, h2 = 0.0;
          if (pk < C::NPAIR) {
            int ap, bp;
            pair_decode(pk, NVE, ap, bp);
            const int a = ap / NE, ie = ap % NE, b = bp / NE, je = bp % NE;
            const int kx = x < 2 ? x + 1 : 3;
            const int s_row = C::MALL ? chunk * 4 + sl : sl;
            const double* Mp = sM + mb * C::M_PER_BUF + s_row * C::MS + ((ie * NE + je) * 16) * C::MPITCH;
#pragma unroll
            for (int z = 0; z < NZ; ++z) {
              auto M = [Mp, z](int k) { return Mp[k * C::MPITCH + z]; };
              const double2 yab = PD[z * NV + a];
              const double pa = yab.x, da = yab.y;
              const double wr = x < 2 ? pa : da;
              const double w0 = (GENERAL && x == 2) ? pa : 0.0;
              const double L0 = GENERAL ? wr * M(kx * 4 + 0) + w0 * M(0) : 0.0;
              const double L1 = wr * M(kx * 4 + 1) + (GENERAL ? w0 * M(1) : 0.0);
              const double L2 = wr * M(kx * 4 + 2) + (GENERAL ? w0 * M(2) : 0.0);
              const double L3 = wr * M(kx * 4 + 3) + (GENERAL ? w0 * M(3) : 0.0);
              const double2 ybb = PD[z * NV + b];
              const double pb = ybb.x, db = ybb.y;
              h0 = fma(L1, pb, h0);
              h1 = fma(L2, pb, h1);
              h2 = GENERAL ? fma(L0, pb, fma(L3, db, h2)) : fma(L3, db, h2);
            }
          }
          double* dst = Hb + pl * C::HPAIR + sl * C::HSL + x * C::HX;
          *reinterpret_cast<double2*>(dst) = make_double2(h0, h1);
          dst[2] = h2;
        }
        smem_release();
        named_arrive(C::BAR_FULL + buf, C::NTHREADS);
        if (!C::MALL) named_sync(C::BAR_PROD, C::NPT);
      }
    }
    return;
  }

  // ======================= consumer warps =======================
  const int cpos = lane >> 2;
  const int64_t kk_elem = static_cast<int64_t>(NSH) * NSH;
  int sl_k[3], x_k[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) {
    const int kk = ks * 4 + (lane & 3);
    sl_k[ks] = kk / 3;
    x_k[ks] = kk % 3;
  }
  int64_t gc = 0;
  for (int64_t it = 0; it < my_items; ++it) {
    const int64_t e = blockIdx.x + (it / C::NITEM) * gridDim.x;
    const int p0 = static_cast<int>(it % C::NITEM) * C::PPI + warp * PPW;
    int pa[PPW], pb[PPW];
    bool live[PPW];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
      live[pp] = p0 + pp < C::NPAIR;
      pair_decode(live[pp] ? p0 + pp : 0, NVE, pa[pp], pb[pp]);
    }
    double acc[PPW][MT][MT][2];
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int g = 0; g < MT; ++g) acc[pp][mt][g][0] = acc[pp][mt][g][1] = 0.0;

#pragma unroll 1
    for (int chunk = 0; chunk < NCHUNK; ++chunk, ++gc) {
      double afr3[3][MT];
#pragma unroll
      for (int ks = 0; ks < 3; ++ks)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) afr3[ks][mt] = sXA[(mt * KSTEPS + chunk * 3 + ks) * 32 + lane];
      const int buf = static_cast<int>(gc % C::NBUF);
      named_sync(C::BAR_FULL + buf, C::NTHREADS);
      const double* Hb = sH + buf * C::H_PER_BUF;
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) {
        const double* afr = afr3[ks];
        const int s = chunk * 4 + sl_k[ks];
        double xv[MT][3];
#pragma unroll
        for (int g = 0; g < MT; ++g) {
          const double* xp = sXP + s * 3 * NTPS + g * 8 + cpos;
          xv[g][0] = xp[0];
          xv[g][1] = xp[NTPS];
          xv[g][2] = xp[2 * NTPS];
        }
#pragma unroll
        for (int pp = 0; pp < PPW; ++pp) {
          const bool diag = pa[pp] == pb[pp];
          const double* Hs = Hb + (warp * PPW + pp) * C::HPAIR + sl_k[ks] * C::HSL + x_k[ks] * C::HX;
          const double2 h01 = *reinterpret_cast<const double2*>(Hs);
          const double h2 = Hs[2];
#pragma unroll
          for (int g = 0; g < MT; ++g) {
            const double gv = fma(h01.x, xv[g][0], fma(h01.y, xv[g][1], h2 * xv[g][2]));
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
              if (mt <= g || !diag) dmma_8x8x4(acc[pp][mt][g][0], acc[pp][mt][g][1], afr[mt], gv);
          }
        }
      }
      if (gc + C::NBUF < total_chunks) named_arrive(C::BAR_EMPTY + buf, C::NTHREADS);
    }
    // ---- epilogue: the pair's blocks and their mirrors, straight to global ----
#pragma unroll
    for (int pp = 0; pp < PPW; ++pp) {
      if (!live[pp]) continue;
      const bool diag = pa[pp] == pb[pp];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int t = mt * 8 + (lane >> 2);
#pragma unroll
        for (int g = 0; g < MT; ++g) {
          if (diag && g < mt) continue;  // mirrored from (mt, g) = (g, mt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int tp = g * 8 + 2 * (lane & 3) + h;
            if (t >= NT || tp >= NT) continue;
            const double v = acc[pp][mt][g][h];
            const int64_t row = t * NVE + pa[pp], col = tp * NVE + pb[pp];
            const bool mirror = !diag || g > mt;
            if (args.out_layout == PI_OUT_CANONICAL) {
              store_out(args, e * kk_elem + row * NSH + col, v);
              if (mirror) store_out(args, e * kk_elem + col * NSH + row, v);
            } else {
              store_out(args, (row * NSH + col) * args.ld_out + e, v);
              if (mirror) store_out(args, (col * NSH + row) * args.ld_out + e, v);
            }
          }
        }
      }
    }
  }
}

}  // namespace pib
