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
//
// Warp specialisation inside each CTA:
//  * producer warps, per chunk of 4 triangle points: Jacobians and M for the
//    chunk's points, then H -> shared memory (double buffered, named
//    barriers FULL/EMPTY);
//  * consumer warps own accumulator fragments K[t][(a, j)] (all m-tiles of
//    the element-independent X operand, NB n-tiles, WA rows a).  Each lane
//    computes exactly the B-fragment value G[k][j] its own m8n8k4 FP64 MMA
//    consumes (3 FMAs from H and X in shared memory), so G never touches
//    memory; the A fragments (X) are staged once per CTA in fragment order.
//
// Systems (n_eq = NE > 1, e.g. linear elasticity): the canonical row
// i_dof*NE + i_e = (t*(p+1) + a)*NE + i_e = t*NVE + a' with the combined
// vertical index a' = a*NE + i_e (NVE = NE*(p+1)), and likewise for columns.
// The GEMM above is unchanged with (a, b) -> (a', b'); only H changes:
//     H_xy(s,a',b') = sum_z sum_{k in x, l in y} Y_k(a,z) M^{ie,je}_kl(s,z) Y_l(b,z)
// with one 4x4 block M^{ie,je} per equation pair and point.
#pragma once

#include "kernels_common.cuh"

namespace pib {

// Weak forms the kernel instantiates.
enum SumFactForm {
  kFormLaplace = 0,     // c[0][0][d][d] = 1 (derivative-only, built in)
  kFormGeneral = 1,     // any element-constant tensor c[ie][je][4][4]
  kFormElasticity = 2   // isotropic elasticity from (E, nu) per element (coefficients.cpp:23-59)
};

// Column order of a K row block inside the GEMM ("n-tiles" of 8 columns):
//  natural: n-tile nt = columns j = 8 nt .. 8 nt + 7, j = t'*(p+1) + b;
//  t'-major (TMAJOR): n-tile (g, b) = columns t' = 8g .. 8g+7 at fixed b, so
//  a lane's X values are shared by every b-tile and H is warp-uniform per
//  tile (the better order when p+1 does not divide 8).
template <int P, int NE, bool TMAJOR>
struct SumFactShape {
  static constexpr int NV = P + 1;                    // Legendre modes / GL points
  static constexpr int NZ = P + 1;
  static constexpr int NVE = NE * NV;                 // combined vertical index a' = a*NE + ie
  static constexpr int NT = (P + 1) * (P + 2) / 2;    // triangle monomials
  static constexpr int NS = (P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : P == 5 ? 25 : P == 6 ? 33 : 42);
  static constexpr int NSP = (NS + 3) / 4 * 4;        // padded to whole chunks
  static constexpr int NSH = NT * NVE;                // K dimension (n_eq * shape_count)
  static constexpr int NQ = NS * NZ;
  static constexpr int MT = (NT + 7) / 8;             // m-tiles of the X operand (rows t)
  static constexpr int KSTEPS = 3 * NSP / 4;          // k4-steps over (s, x)
  static constexpr int NCHUNK = NSP / 4;              // 4 triangle points per chunk
  static constexpr int XFRAG = MT * KSTEPS * 32;      // doubles in the A-fragment table
};

// Launch shape: EPC elements x AG vertical rows a' per CTA; each consumer
// warp owns WA rows a' x NB n-tiles x all MT m-tiles (WA*NB*MT fragments);
// NPW producer warps; NCB column blocks (CTAs) per (element, a'-group).
// TMAJOR warps own NG t'-groups x NBB b values (NB = NG*NBB).
template <bool TMAJOR_, int EPC_, int AG_, int WA_, int NG_, int NBB_, int NB_, int NPW_, int BSPLIT_, int MINB_,
          int NCB_>
struct SumFactLaunchP {
  static constexpr bool TMAJOR = TMAJOR_;
  static constexpr int EPC = EPC_, AG = AG_, WA = WA_, NG = NG_, NBB = NBB_, NB = NB_, NPW = NPW_, BSPLIT = BSPLIT_,
                       MINB = MINB_, NCB = NCB_;
};
template <int P, int NE>
struct SumFactLaunch;
// Per (p, n_eq): TMAJOR, EPC, AG, WA, NG, NBB, NB, NPW, BSPLIT, MINB, NCB.
// Each can be overridden at build time (A/B runs, tools/ab_build.sh): a header
// named by -DPI_SF_OVERRIDE (included by kernels_common.cuh) defining PI_SF_<p>_<n_eq>.
// H ring depth per (p, n_eq): PI_SF_NBUF_<p>_<n_eq> (4 for p >= 4: +2 % at
// p = 4), else PI_SF_NBUF (3: p = 3 keeps two CTAs per SM); 2..6 (named
// barriers: FULL/EMPTY per buffer + 2 <= 16).
#ifndef PI_SF_NBUF
#define PI_SF_NBUF 3
#endif
#ifndef PI_SF_2_1
#define PI_SF_2_1 true, 8, 3, 3, 1, 3, 3, 4, 1, 1, 1
#endif
template <> struct SumFactLaunch<2, 1> : SumFactLaunchP<PI_SF_2_1> {};
#ifndef PI_SF_3_1
#define PI_SF_3_1 false, 2, 4, 2, 0, 0, 5, 2, 1, 2, 1
#endif
template <> struct SumFactLaunch<3, 1> : SumFactLaunchP<PI_SF_3_1> {};
#ifndef PI_SF_4_1
#define PI_SF_4_1 true, 2, 5, 1, 2, 5, 10, 2, 1, 1, 1
#endif
template <> struct SumFactLaunch<4, 1> : SumFactLaunchP<PI_SF_4_1> {};
#ifndef PI_SF_5_1
#define PI_SF_5_1 false, 1, 3, 1, 0, 0, 8, 2, 2, 1, 1
#endif
template <> struct SumFactLaunch<5, 1> : SumFactLaunchP<PI_SF_5_1> {};
#ifndef PI_SF_6_1  // NB = 3 (9 consumer warps), 3 producer warps: CDR +11 % over NB = 5, NPW = 2
#define PI_SF_6_1 false, 1, 1, 1, 0, 0, 3, 3, 4, 1, 1
#endif
template <> struct SumFactLaunch<6, 1> : SumFactLaunchP<PI_SF_6_1> {};
#ifndef PI_SF_7_1
#define PI_SF_7_1 false, 1, 1, 1, 0, 0, 3, 4, 4, 1, 1
#endif
template <> struct SumFactLaunch<7, 1> : SumFactLaunchP<PI_SF_7_1> {};
// n_eq = 3 (elasticity): K is 9x larger; p >= 6 also splits columns over CTAs
// (column blocks of whole t' rows: 42 tiles = 16 t' at p = 6, 36 = 12 at p = 7).
#ifndef PI_SF_1_3
#define PI_SF_1_3 false, 2, 6, 3, 0, 0, 3, 2, 2, 1, 1
#endif
template <> struct SumFactLaunch<1, 3> : SumFactLaunchP<PI_SF_1_3> {};
#ifndef PI_SF_2_3
#define PI_SF_2_3 false, 1, 9, 3, 0, 0, 7, 2, 3, 1, 1
#endif
template <> struct SumFactLaunch<2, 3> : SumFactLaunchP<PI_SF_2_3> {};
#ifndef PI_SF_3_3
#define PI_SF_3_3 false, 1, 4, 2, 0, 0, 5, 2, 3, 1, 1
#endif
template <> struct SumFactLaunch<3, 3> : SumFactLaunchP<PI_SF_3_3> {};
#ifndef PI_SF_4_3
#define PI_SF_4_3 false, 1, 3, 1, 0, 0, 10, 3, 5, 1, 1
#endif
template <> struct SumFactLaunch<4, 3> : SumFactLaunchP<PI_SF_4_3> {};
#ifndef PI_SF_5_3
#define PI_SF_5_3 false, 1, 1, 1, 0, 0, 8, 2, 6, 1, 1
#endif
template <> struct SumFactLaunch<5, 3> : SumFactLaunchP<PI_SF_5_3> {};
#ifndef PI_SF_6_3
#define PI_SF_6_3 false, 1, 1, 1, 0, 0, 6, 2, 7, 1, 2
#endif
template <> struct SumFactLaunch<6, 3> : SumFactLaunchP<PI_SF_6_3> {};
#ifndef PI_SF_7_3
#define PI_SF_7_3 false, 1, 1, 1, 0, 0, 4, 2, 8, 1, 3
#endif
template <> struct SumFactLaunch<7, 3> : SumFactLaunchP<PI_SF_7_3> {};
template <int P, int NE>
struct SumFactNbuf {
  static constexpr int value = PI_SF_NBUF;
};
#define PI_SF_NBUF_SPEC(p, ne, v) \
  template <>                     \
  struct SumFactNbuf<p, ne> {     \
    static constexpr int value = v; \
  };
#ifndef PI_SF_NBUF_4_3
#define PI_SF_NBUF_4_3 4
#endif
PI_SF_NBUF_SPEC(4, 3, PI_SF_NBUF_4_3)
#ifndef PI_SF_NBUF_5_3
#define PI_SF_NBUF_5_3 4
#endif
PI_SF_NBUF_SPEC(5, 3, PI_SF_NBUF_5_3)
#ifndef PI_SF_NBUF_6_3
#define PI_SF_NBUF_6_3 4
#endif
PI_SF_NBUF_SPEC(6, 3, PI_SF_NBUF_6_3)
#ifndef PI_SF_NBUF_7_3
#define PI_SF_NBUF_7_3 4
#endif
PI_SF_NBUF_SPEC(7, 3, PI_SF_NBUF_7_3)
#ifndef PI_SF_NBUF_4_1
#define PI_SF_NBUF_4_1 4
#endif
PI_SF_NBUF_SPEC(4, 1, PI_SF_NBUF_4_1)
#ifndef PI_SF_NBUF_5_1
#define PI_SF_NBUF_5_1 4
#endif
PI_SF_NBUF_SPEC(5, 1, PI_SF_NBUF_5_1)
#ifndef PI_SF_NBUF_6_1
#define PI_SF_NBUF_6_1 4
#endif
PI_SF_NBUF_SPEC(6, 1, PI_SF_NBUF_6_1)
#ifndef PI_SF_NBUF_7_1
#define PI_SF_NBUF_7_1 4
#endif
PI_SF_NBUF_SPEC(7, 1, PI_SF_NBUF_7_1)

// Symmetric forms may take their own launch shape and ring depth
// (PI_SF_<p>_<ne>_SYM): p = 4 Laplace runs one element per CTA at two CTAs
// per SM (+1.2 %), a shape that costs the general (CDR) form 5 %; p = 3
// splits the producers' H items over two b' halves.  Both
// shapes of a (p, n_eq) must share the per-p tables (same TMAJOR).
template <int P, int NE>
struct SumFactLaunchSym : SumFactLaunch<P, NE> {
  static constexpr int NBUF = SumFactNbuf<P, NE>::value;
};
#ifndef PI_SF_4_1_SYM
#define PI_SF_4_1_SYM true, 1, 5, 1, 2, 5, 10, 1, 1, 2, 1
#endif
#ifndef PI_SF_NBUF_4_1_SYM
#define PI_SF_NBUF_4_1_SYM 3
#endif
template <>
struct SumFactLaunchSym<4, 1> : SumFactLaunchP<PI_SF_4_1_SYM> {
  static constexpr int NBUF = PI_SF_NBUF_4_1_SYM;
};
#ifndef PI_SF_3_1_SYM  // H items split over two b' halves: Laplace +1.6 %, CDR -1.7 %
#define PI_SF_3_1_SYM false, 2, 4, 2, 0, 0, 5, 2, 2, 2, 1
#endif
template <>
struct SumFactLaunchSym<3, 1> : SumFactLaunchP<PI_SF_3_1_SYM> {
  static constexpr int NBUF = SumFactNbuf<3, 1>::value;
};
template <int P, int NE, bool SYMV>
struct SumFactLaunchSel : SumFactLaunch<P, NE> {
  static constexpr int NBUF = SumFactNbuf<P, NE>::value;
};
template <int P, int NE>
struct SumFactLaunchSel<P, NE, true> : SumFactLaunchSym<P, NE> {};

template <int P, int NE = 1, bool SYMV = false>
struct SumFactConfig : SumFactShape<P, NE, SumFactLaunchSel<P, NE, SYMV>::TMAJOR>, SumFactLaunchSel<P, NE, SYMV> {
  using S = SumFactShape<P, NE, SumFactLaunchSel<P, NE, SYMV>::TMAJOR>;
  using L = SumFactLaunchSel<P, NE, SYMV>;
  // n-tiles of 8 columns: t'-major (g, b') tiles, or natural tiles padded to
  // a whole number of NB x NCB blocks (padding columns are computed from
  // zero X rows and never stored)
  static constexpr int NTILE = L::TMAJOR ? S::MT * S::NVE : ((S::NSH + 7) / 8 + L::NB * L::NCB - 1) / (L::NB * L::NCB) * (L::NB * L::NCB);
  static constexpr int NTP = L::TMAJOR ? S::MT * 8 : (NTILE * 8 + S::NVE - 1) / S::NVE;  // t' rows of the X table
  // X as [s][y][t'] with a row pitch NTPS = NTP rounded up to 8 (mod 16):
  // rows s and s+1 then start 64 bytes apart modulo 128, so the two s a
  // warp reads per k-step land in disjoint bank halves.
  static constexpr int NTPS = (NTP + 7) / 16 * 16 + 8;
  static constexpr int XPLAIN = S::NSP * 3 * NTPS;
  // natural order: X also as [s][t'][4] (y = 0, 1 in one 16-byte load, y = 2
  // in an 8-byte one) after the [s][y][t'] table (A/B: PI_SF_NO_XP4)
#ifdef PI_SF_NO_XP4
  static constexpr bool XP4 = false;
#else
  static constexpr bool XP4 = !L::TMAJOR && S::NV <= 4;  // p <= 3: the table grows as N_s N_t
#endif
  static constexpr int XP4_DOUBLES = XP4 ? S::NSP * NTP * 4 : 0;
  static constexpr int XPLAIN_TOTAL = XPLAIN + XP4_DOUBLES;       // the device table holds both
  static constexpr int XP_SMEM = XP4 ? XP4_DOUBLES : XPLAIN;     // the consumers stage only the one they read
  static constexpr int NBLK = NTILE / (L::NB * L::NCB);  // n-tile blocks (warps) per CTA and row group
  static constexpr int WPE = (L::AG / L::WA) * NBLK;      // consumer warps per element
  // t'-major warps own whole K rows (all t'-groups, all b), so they stage
  // and store their rows without CTA-level synchronisation.
  static_assert(!L::TMAJOR || (L::NB == L::NG * L::NBB && L::NG == S::MT && L::NBB == S::NVE && L::NCB == 1),
                "t'-major warp tiling");
  static constexpr int NCW = L::EPC * WPE;
  static constexpr int NWARPS = NCW + L::NPW;
  static constexpr int NTHREADS = 32 * NWARPS;
  static constexpr int NPT = 32 * L::NPW;              // producer threads
  static constexpr int NAG = S::NVE / L::AG;           // a'-groups per element
  static constexpr int NITEM = NAG * L::NCB;           // CTA work items per element group
  static constexpr int BPER = (S::NVE + L::BSPLIT - 1) / L::BSPLIT;  // b' values per H item
  // Along a consumer lane's n-tiles, b' = (8*nb + lane/4) mod NVE repeats with
  // period R = NVE / gcd(8, NVE); its H values are cached in registers.
  static constexpr int R = S::NVE / (S::NVE % 8 == 0 ? 8 : S::NVE % 4 == 0 ? 4 : S::NVE % 2 == 0 ? 2 : 1);
  static constexpr int RC = R < L::NB ? R : L::NB;     // distinct b' values a lane touches
  static_assert(S::NVE % L::AG == 0 && L::AG % L::WA == 0, "bad a-grouping");
  static_assert(NTILE % (L::NB * L::NCB) == 0, "n-tiles must split evenly");
  // H for one chunk, two planes per ring buffer, indexed by one offset
  //   o = ((el*AG + a')*4 + s)*HS2 + b'*HB2 + x:
  //     y = 0, 1 at H[2o], H[2o + 1]   (16-byte loads / stores)
  //     y = 2    at H[H2OFF + o]        (8-byte loads / stores)
  // The strides are padded at compile time by counting the shared-memory
  // wavefronts of one warp's consumer loads and producer stores in both
  // planes (hwave): the 16-byte plane is bank-conflict free when the o of a
  // quarter warp differ mod 8, the 8-byte plane when those of a half warp
  // differ mod 16.
  static constexpr int hwave_cons(int hb2, int hs2) {
    int total = 0;
    constexpr int NBM = L::TMAJOR ? (S::NVE < 8 ? S::NVE : 8) : (NTILE < 8 ? NTILE : 8);
    for (int ks = 0; ks < 3; ++ks)
      for (int nb = 0; nb < NBM; ++nb)
        for (int plane = 0; plane < 2; ++plane) {
          const int width = plane == 0 ? 8 : 16, mod = plane == 0 ? 8 : 16;
          for (int q = 0; q < 32; q += width) {
            int cnt[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, worst = 0;
            // natural order: b' = (8 nt + lane/4) mod NVE, every lane distinct;
            // t'-major: one b' per warp, lanes 4..7 of a group repeat lanes 0..3
            for (int l = 0; l < (L::TMAJOR ? 4 : width); ++l) {
              const int lane = q + l, kk = 4 * ks + (lane & 3);
              const int b = L::TMAJOR ? nb : (nb * 8 + (lane >> 2)) % S::NVE;
              const int k = ((kk / 3) * hs2 + b * hb2 + (kk % 3)) % mod;
              ++cnt[k];
              worst = worst > cnt[k] ? worst : cnt[k];
            }
            total += worst;
          }
        }
    return total;
  }
  // producers: consecutive items (b'-group, x, s, (el, a')) per lane, b' looped
  static constexpr int hwave_prod(int hb2, int hs2) {
    constexpr int items = L::EPC * L::AG * 4 * 3 * L::BSPLIT;
    int total = 0;
    for (int w0 = 0; w0 < items; w0 += 32)
      for (int bb = 0; bb < BPER; ++bb)
        for (int plane = 0; plane < 2; ++plane) {
          const int width = plane == 0 ? 8 : 16, mod = plane == 0 ? 8 : 16;
          for (int q0 = w0; q0 < w0 + 32 && q0 < items; q0 += width) {
            int cnt[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, worst = 0;
            for (int i = q0; i < q0 + width && i < items; ++i) {
              const int bg = i % L::BSPLIT, x = (i / L::BSPLIT) % 3, sl = (i / (3 * L::BSPLIT)) % 4;
              const int alg = i / (12 * L::BSPLIT);  // (el, a')
              const int bp = bg * BPER + bb;
              if (bp >= S::NVE) continue;
              const int k = (alg * 4 * hs2 + sl * hs2 + bp * hb2 + x) % mod;
              ++cnt[k];
              worst = worst > cnt[k] ? worst : cnt[k];
            }
            total += worst;
          }
        }
    return total;
  }
  static constexpr int hpick() {  // returns hb2 * 1024 + hs2
    long long best = 1LL << 62;
    int pick = 3 * 1024 + S::NVE * 3;
    for (int hb2 = 3; hb2 <= 8; ++hb2)
      for (int pad = 0; pad < 16; ++pad) {
        const int hs2 = S::NVE * hb2 + pad;
        // consumer loads weigh 4x: every consumer warp reads H, two producer warps write it
        const long long score = (4LL * hwave_cons(hb2, hs2) + hwave_prod(hb2, hs2)) * 100000LL + hs2;
        if (score < best) best = score, pick = hb2 * 1024 + hs2;
      }
    return pick;
  }
  static constexpr int HPICK = hpick();
  static constexpr int HB2 = HPICK / 1024;
  static constexpr int HS2 = HPICK % 1024;
  static constexpr int H2OFF = 2 * L::EPC * L::AG * 4 * HS2;  // the y = 2 plane
  static constexpr int H_PER_BUF = (H2OFF + L::EPC * L::AG * 4 * HS2 + 1) / 2 * 2;
  static constexpr int NBUF = L::NBUF;  // H ring depth (producers run up to NBUF chunks ahead)
  static_assert(NBUF >= 2 && NBUF <= 6, "named barriers: FULL/EMPTY per buffer + 2 <= 16");
  // Scalar forms build M for every point of the item up front (one wide,
  // latency-bound pass instead of one per chunk); systems (9 blocks per
  // point) build it per chunk of 4 triangle points.
  static constexpr bool MALL = NE == 1;
  // M stored k-major: [NE*NE][16][MPITCH], point (el, s, z) at el*MEL + s*MS + z
  // (an odd k-row pitch; padding MEL / MPITCH against the producers' read
  // conflicts measured no gain).
  // point stride per triangle point s: NZ made odd, so the producers' reads of
  // one M row at different (x, s) fall into distinct banks (k-row offsets are
  // multiples of 4 doubles, s offsets then are not)
#ifdef PI_SF_MS_EVEN  // A/B: the former stride NZ
  static constexpr int MS = S::NZ;
#else
  static constexpr int MS = S::NZ | 1;
#endif
  static constexpr int MEL = (MALL ? S::NSP : 4) * MS;  // point slots per element per M pass
  static constexpr int MPITCH = (L::EPC * MEL) | 1;
  static constexpr int M_PER_CHUNK = NE * NE * 16 * MPITCH;
  static constexpr int NCOEF = 16 * NE * NE;            // coefficient tensor per element
  // shared memory layout (doubles; every block 16-byte aligned)
  static constexpr int OFF_XA = 0;
  static constexpr int OFF_XP = OFF_XA + S::XFRAG;
  static constexpr int OFF_H = OFF_XP + XP_SMEM;
  static constexpr int OFF_M = OFF_H + NBUF * H_PER_BUF;
  static constexpr int OFF_GEOM = OFF_M + (MALL ? 2 : 1) * M_PER_CHUNK;
  static constexpr int OFF_C = OFF_GEOM + (L::EPC * 21 + 1) / 2 * 2;
  static constexpr int OFF_LINE = OFF_C + L::EPC * NCOEF;  // (P, P') [NZ][NV] pairs, xi3 [NZ]
  static constexpr int OFF_TRI = OFF_LINE + (2 * S::NV * S::NZ + S::NZ + 1) / 2 * 2;
  static constexpr int OFF_W = OFF_TRI + 2 * S::NS;
  // t'-major epilogue: each consumer warp stages its WA*NT K rows
  // t'-major with whole elements in the CTA: element matrices staged in
  // canonical order (one spare double to match the global address mod 16)
  // and stored by the TMA bulk engine.
  static constexpr bool BULK = NAG == 1 && L::NCB == 1;  // whole elements per CTA: staged, TMA bulk stores
  // symmetric forms: warps own (a', b') pairs a' <= b' (kernel PAIRS), when
  // the diagonal and off-diagonal pairs split evenly over an element's warps
  static constexpr bool PAIRS = L::TMAJOR && BULK && S::NVE % WPE == 0 && (S::NVE * (S::NVE - 1) / 2) % WPE == 0;
  static constexpr int ESTRIDE = (S::NSH * S::NSH + 3) / 2 * 2;
  static constexpr int STAGE_PER_WARP = L::TMAJOR ? (L::WA * S::NT * S::NSH + 1) / 2 * 2 : 0;
  static constexpr int OFF_STAGE = (OFF_W + S::NQ + 1) / 2 * 2;
  static constexpr int STAGE_DOUBLES = BULK ? L::EPC * ESTRIDE : NCW * STAGE_PER_WARP;
  static constexpr int SMEM_DOUBLES = OFF_STAGE + STAGE_DOUBLES;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
  // fused load vectors (n_eq = 1): det w f per point [EPC][NSP][NZ] and
  // u(s, a) [EPC][NSP][NV] after the rest; launched with SMEM_BYTES_LOAD
  static constexpr int OFF_LDW = SMEM_DOUBLES;
  static constexpr int OFF_LU = OFF_LDW + L::EPC * S::NSP * S::NZ;
  static constexpr size_t SMEM_BYTES_LOAD = sizeof(double) * (OFF_LU + L::EPC * S::NSP * S::NV);
};

// Fused load vector of the producers' current elements (pi_integrate_load):
// phi_0(t*NV + a, (s, z)) = m_t(s) P_a(z) = X_2(t, s) P_a(z), so
//     F(t, a) = sum_s X_2(t, s) u(s, a),   u(s, a) = sum_z P_a(z) dw(s, z)
// from dw = det w f per point (sDW [ne][NSP][NZ], zero at padded s); one
// contiguous coalesced store of N_sh doubles per element.
// X_2(t, s) in shared memory: [s][y][t'] with pitch NTPS, or (XP4 > 0) [s][t'][4] with XP4 = NTP rows
template <int NS, int NSP, int NZ, int NV, int NT, int NTPS, int XP4 = 0>
__device__ __forceinline__ void sumfact_load_vectors(const LaunchArgs& args, int64_t e0, int ne, const double* sDW,
                                                     double* sU, const double* sXP, const double2* PD, int ptid,
                                                     int npt, int bar) {
  for (int i = ptid; i < ne * NSP * NV; i += npt) {
    const int el = i / (NSP * NV), r = i % (NSP * NV), s = r / NV, a = r % NV;
    const double* dw = sDW + (el * NSP + s) * NZ;
    double u = 0.0;
#pragma unroll
    for (int z = 0; z < NZ; ++z) u = fma(PD[z * NV + a].x, dw[z], u);
    sU[i] = u;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(npt) : "memory");
  constexpr int NSH = NT * NV;
  for (int i = ptid; i < ne * NSH; i += npt) {
    const int el = i / NSH, dof = i % NSH, t = dof / NV, a = dof % NV;
    if (e0 + el >= args.n_elem) continue;
    const double* u = sU + el * NSP * NV + a;
    double acc = 0.0;
#pragma unroll 4
    for (int s = 0; s < NS; ++s)
      acc = fma(XP4 ? sXP[(s * XP4 + t) * 4 + 2] : sXP[(s * 3 + 2) * NTPS + t], u[s * NV], acc);
    args.fout[(e0 + el) * NSH + dof] = acc;
  }
}

// Per-p constant tables in device memory (built by the host from the shape
// table, pi_context.cu).
struct SumFactTables {
  const double* xfrag;   // X in A-fragment order [MT][KSTEPS][32]
  const double* xplain;  // X as [NSP][3][NTPS] (zero padded)
  const double* yline;   // (P, P') [NZ][NV] pairs, xi3 [NZ]
  const double* tri;     // xi1 [NS], xi2 [NS]
  const double* w;       // [NQ] rule weights (reference order)
};

// Named barriers (id 0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// named barrier ids: FULL and EMPTY per ring buffer, producers, consumers
constexpr int kBarFull0 = 1, kBarEmpty0 = 7, kBarProd = 13, kBarCons = 14;

// Release fence for the shared-memory hand-off before bar.arrive (MEMBAR.ALL.CTA).
__device__ __forceinline__ void smem_release() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }

// FORM: SumFactForm.  SYM: the coefficient tensor is symmetric, so K is.
// Where a CTA holds all rows of an element (t'-major, NAG == 1) only the
// blocks with t'-block >= t-block are multiplied; the rest are mirrored
// from the CTA's staged K.
template <int P, int NE, int FORM, bool SYM>
__global__ void __launch_bounds__(SumFactConfig<P, NE, SYM>::NTHREADS, SumFactConfig<P, NE, SYM>::MINB)
    sumfact_kernel(LaunchArgs args, SumFactTables tab) {
  using C = SumFactConfig<P, NE, SYM>;
  constexpr bool GENERAL = FORM == kFormGeneral;  // value row/column present in M
  constexpr bool SYMK = SYM && C::TMAJOR && C::NAG == 1;
  // Symmetric t'-major with one warp per vertical row (WPE == NVE, odd): the
  // warps take (a', b') PAIRS with a' <= b' instead -- the diagonal pair plus
  // (NVE-1)/2 off-diagonal ones each -- so the blocks below the (a', b')
  // diagonal are neither multiplied nor their B fragments formed (27 % fewer
  // MMAs, 40 % fewer fragment FMAs at p = 4); mirrors come from the staging.
  constexpr int NPAIR = C::NVE * (C::NVE + 1) / 2;
  constexpr bool PAIRS = C::PAIRS && SYM;
  constexpr int PPW = PAIRS ? NPAIR / C::WPE : 1;     // pairs per warp
  constexpr int NDW = PAIRS ? C::NVE / C::WPE : 1;    // diagonal pairs per warp (first NDW)
  constexpr int NV = C::NV, NVE = C::NVE, NZ = C::NZ, NT = C::NT, NS = C::NS, NSH = C::NSH, NQ = C::NQ;
  constexpr int NTPS = C::NTPS, MT = C::MT, KSTEPS = C::KSTEPS, EPC = C::EPC, AG = C::AG, WA = C::WA, NB = C::NB;
  constexpr int NCHUNK = C::NCHUNK, NCOEF = C::NCOEF;
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

  // ---- per-p tables: staged once per (persistent) CTA by TMA bulk copies ----
  // (contiguous device arrays, sizes padded to 16 bytes by the host)
  __shared__ __align__(8) uint64_t s_tables;
  if (tid == 0) mbar_init(&s_tables, 1);
  __syncthreads();
  if (tid == 0) {
    constexpr unsigned BX = 8u * C::XFRAG, BP = 8u * C::XP_SMEM, BY = 8u * ((2 * NV * NZ + NZ + 1) / 2 * 2),
                       BT = 8u * 2 * NS, BW = 8u * ((NQ + 1) / 2 * 2);
    mbar_arrive_expect_tx(&s_tables, BX + BP + BY + BT + BW);
    bulk_load(sXA, tab.xfrag, BX, &s_tables);
    bulk_load(sXP, tab.xplain + (C::XP4 ? C::XPLAIN : 0), BP, &s_tables);
    bulk_load(sY, tab.yline, BY, &s_tables);
    bulk_load(sTri, tab.tri, BT, &s_tables);
    bulk_load(sW, tab.w, BW, &s_tables);
  }
  mbar_wait(&s_tables, 0);

  const double2* PD = reinterpret_cast<const double2*>(sY);  // (P_a(z), P'_a(z)) [NZ][NV]

  // Work items: (element group, a'-group, column block); this CTA takes
  // items blockIdx.x + k*gridDim.x.
  const int64_t n_items = (args.n_elem + EPC - 1) / EPC * C::NITEM;
  const int64_t my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total_chunks = my_items * NCHUNK;

  if (warp >= C::NCW) {
    // ======================= producer warps =======================
    const int ptid = tid - 32 * C::NCW;
    int64_t gc = 0;  // chunk counter across items: selects the H buffer
    // Geometry / coefficients of item `it` into shared memory.
    auto load_item = [&](int64_t it) {
      const int64_t w = blockIdx.x + it * gridDim.x;
      const int64_t e0 = (w / C::NITEM) * EPC;
      if (ptid < EPC) {  // edge vectors of the item's elements
        const int64_t e = e0 + ptid;
        const int64_t ec = e < args.n_elem ? e : args.n_elem - 1;  // pad with a valid element
        double x[18], d[21];
#pragma unroll
        for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + ec];
        prism_edges(x, d);
#pragma unroll
        for (int c = 0; c < 21; ++c) sGeom[ptid * 21 + c] = d[c];
      }
      if (FORM == kFormGeneral) {
        for (int i = ptid; i < EPC * NCOEF; i += C::NPT) {
          const int el = i / NCOEF, c = i % NCOEF;
          const int64_t e = e0 + el;
          const int64_t ec = e < args.n_elem ? e : args.n_elem - 1;
          sC[i] = args.coeff ? args.coeff[c * args.coeff_ld + ec] : args.cu[c];
        }
      } else if (FORM == kFormElasticity) {
        if (ptid < EPC) {  // Lame parameters from (E, nu)
          const int64_t e = e0 + ptid;
          const int64_t ec = e < args.n_elem ? e : args.n_elem - 1;
          const double young = args.coeff ? args.coeff[ec] : args.cu[0];
          const double nu = args.coeff ? args.coeff[args.coeff_ld + ec] : args.cu[1];
          if (e < args.n_elem && (w % C::NITEM) == 0) check_material(args, e, young, nu);
          lame(young, nu, sC[2 * ptid], sC[2 * ptid + 1]);
        }
      }
      named_sync(kBarProd, C::NPT);
    };
    // (1) M blocks of item `it`: points (el, s, z), s in [s_first, s_first + s_count),
    // into M buffer mb (MALL: two buffers, so item it+1 is prepared while the
    // consumers still drain item it's chunks from the H ring).
    auto build_m = [&](int64_t it, int mb, int s_first, int s_count) {
      const int64_t w = blockIdx.x + it * gridDim.x;
      const int64_t e0 = (w / C::NITEM) * EPC;
      const bool flagger = (w % C::NITEM) == 0;  // one item per element group reports inversions
      double* sMb = sM + mb * C::M_PER_CHUNK;
      for (int i = ptid; i < EPC * s_count * NZ; i += C::NPT) {
        const int z = i % NZ, sl = (i / NZ) % s_count, el = i / (s_count * NZ);
        const int s = s_first + sl;
        double* Mi = sMb + el * C::MEL + sl * C::MS + z;
        if (s < NS) {
          double cf[3][3];
          const double det = jacobian_cofactors(sGeom + 21 * el, sTri[s], sTri[NS + s], sY[2 * NV * NZ + z], cf);
          const double w8 = sW[z * NS + s], wd = w8 * __drcp_rn(det);
          const int64_t e = e0 + el;
          if (!(det > 0.0) && e < args.n_elem && flagger) flag_inverted(args.bad, args.element_id_base + e);
          if (NE == 1 && args.fout && flagger)
            smem[C::OFF_LDW + (el * C::NSP + s) * NZ + z] = det * w8 * load_f(args, e < args.n_elem ? e : args.n_elem - 1);
#pragma unroll
          for (int blk = 0; blk < NE * NE; ++blk) {
            double M[16];
            if (FORM == kFormElasticity)
              elasticity_block(cf, wd, sC[2 * el], sC[2 * el + 1], blk / NE, blk % NE, M);
            else
              block_from_cofactors<GENERAL>(cf, det, w8, wd, sC + NCOEF * el + 16 * blk, M);
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (GENERAL || (k >= 4 && (k & 3) != 0)) Mi[(blk * 16 + k) * C::MPITCH] = M[k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16 * NE * NE; ++k) Mi[k * C::MPITCH] = 0.0;
          if (NE == 1 && args.fout && flagger) smem[C::OFF_LDW + (el * C::NSP + s) * NZ + z] = 0.0;
        }
      }
      named_sync(kBarProd, C::NPT);
      if (NE == 1 && C::MALL && args.fout && flagger) {
        sumfact_load_vectors<NS, C::NSP, NZ, NV, NT, C::NTPS, C::XP4 ? C::NTP : 0>(args, e0, EPC, smem + C::OFF_LDW,
                                                                                 smem + C::OFF_LU, sXP,
                                                            PD, ptid, C::NPT, kBarProd);
        named_sync(kBarProd, C::NPT);
      }
    };
    if (C::MALL && my_items > 0) {
      load_item(0);
      build_m(0, 0, 0, C::NSP);
    }
    for (int64_t it = 0; it < my_items; ++it) {
      const int64_t w = blockIdx.x + it * gridDim.x;
      const int agroup = static_cast<int>((w % C::NITEM) / C::NCB);
      const int mb = C::MALL ? static_cast<int>(it & 1) : 0;
      if (!C::MALL) load_item(it);
      for (int chunk = 0; chunk < NCHUNK; ++chunk, ++gc) {
        if (!C::MALL) build_m(it, 0, chunk * 4, 4);
        const int buf = static_cast<int>(gc % C::NBUF);
        if (gc >= C::NBUF) named_sync(kBarEmpty0 + buf, C::NTHREADS);  // consumers released this buffer
        double* Hb = sH + buf * C::H_PER_BUF;
        // (2) H_x,y(s,a',b'), y = 0..2: items (el, al, sl, x, b'-group), b' looped
        for (int i = ptid; i < EPC * AG * 4 * 3 * C::BSPLIT; i += C::NPT) {
          const int bg = i % C::BSPLIT, x = (i / C::BSPLIT) % 3, sl = (i / (3 * C::BSPLIT)) % 4;
          const int al = (i / (12 * C::BSPLIT)) % AG, el = i / (12 * C::BSPLIT * AG);
          const int ap = agroup * AG + al;          // a' = a*NE + ie
          const int a = ap / NE, ie = ap % NE;
          const int kx = x < 2 ? x + 1 : 3;
          double h[C::BPER][3];
#pragma unroll
          for (int bb = 0; bb < C::BPER; ++bb) h[bb][0] = h[bb][1] = h[bb][2] = 0.0;
          // M_k of point z at Mp[k*MPITCH + z]
          const double* Mp = sM + mb * C::M_PER_CHUNK + el * C::MEL + (C::MALL ? chunk * 4 + sl : sl) * C::MS;
#pragma unroll
          for (int z = 0; z < NZ; ++z) {
            const double* Mz = Mp + z;
            const double2 yab = PD[z * NV + a];
            const double pa = yab.x, da = yab.y;
            // left factor L_l = sum_{k in x} Y_k(a) M_kl (row kx weighted by P or P',
            // plus row 0 weighted by P for x = 2 in the general case); with one
            // equation it does not depend on b', so it is formed once per z
            const double wr = x < 2 ? pa : da;
            const double w0 = (GENERAL && x == 2) ? pa : 0.0;
            auto left = [&](int je, double (&L)[4]) {
              auto M = [Mz, ie, je](int k) { return Mz[((ie * NE + je) * 16 + k) * C::MPITCH]; };
              L[0] = GENERAL ? wr * M(kx * 4 + 0) + w0 * M(0) : 0.0;
              L[1] = wr * M(kx * 4 + 1) + (GENERAL ? w0 * M(1) : 0.0);
              L[2] = wr * M(kx * 4 + 2) + (GENERAL ? w0 * M(2) : 0.0);
              L[3] = wr * M(kx * 4 + 3) + (GENERAL ? w0 * M(3) : 0.0);
            };
            double L1e[4];
            if (NE == 1) left(0, L1e);
#pragma unroll
            for (int bb = 0; bb < C::BPER; ++bb) {
              const int bp = bg * C::BPER + bb;      // b' = b*NE + je
              if (bp < NVE) {
                const int b = bp / NE, je = bp % NE;
                double Lb[4];
                if (NE != 1) left(je, Lb);
                const double L0 = NE == 1 ? L1e[0] : Lb[0], L1 = NE == 1 ? L1e[1] : Lb[1];
                const double L2 = NE == 1 ? L1e[2] : Lb[2], L3 = NE == 1 ? L1e[3] : Lb[3];
                const double2 ybb = PD[z * NV + b];
                const double pb = ybb.x, db = ybb.y;
                h[bb][0] = fma(L1, pb, h[bb][0]);
                h[bb][1] = fma(L2, pb, h[bb][1]);
                h[bb][2] = GENERAL ? fma(L0, pb, fma(L3, db, h[bb][2])) : fma(L3, db, h[bb][2]);
              }
            }
          }
#pragma unroll
          for (int bb = 0; bb < C::BPER; ++bb) {
            const int bp = bg * C::BPER + bb;
            if (bp < NVE) {
              const int o = ((el * AG + al) * 4 + sl) * C::HS2 + bp * C::HB2 + x;
              *reinterpret_cast<double2*>(Hb + 2 * o) = make_double2(h[bb][0], h[bb][1]);
              Hb[C::H2OFF + o] = h[bb][2];
            }
          }
        }
        smem_release();
        named_arrive(kBarFull0 + buf, C::NTHREADS);
        // per-chunk M: all producers done with sM before the next chunk rewrites it
        if (!C::MALL) named_sync(kBarProd, C::NPT);
      }
      // MALL: the next item's geometry and M go into the other buffer while the
      // consumers work through this item's buffered chunks
      if (C::MALL && it + 1 < my_items) {
        load_item(it + 1);
        build_m(it + 1, mb ^ 1, 0, C::NSP);
      }
    }
    return;
  }

  // ======================= consumer warps =======================
  const int el_w = warp / C::WPE;
  const int r_w = warp % C::WPE;
  const int al0 = (r_w / C::NBLK) * WA;  // first local a' of this warp
  const int nblk = r_w % C::NBLK;
  const int cpos = lane >> 2;            // B-fragment column within an n-tile
  const int64_t kk_elem = static_cast<int64_t>(NSH) * NSH;
  // PAIRS: pairs 0..NDW-1 = diagonal (d, d), d = NDW r_w + pp; the rest are
  // off-diagonal pairs (a < b) number (PPW - NDW) r_w + pp - NDW
  int pa[PPW], pb[PPW];
#pragma unroll
  for (int pp = 0; pp < PPW; ++pp) {
    pa[pp] = pb[pp] = NDW * r_w + pp;
    if (pp >= NDW) {
      int o = (PPW - NDW) * r_w + pp - NDW, a = 0;
      while (o >= C::NVE - 1 - a) o -= C::NVE - 1 - a++;
      pa[pp] = a;
      pb[pp] = a + 1 + o;
    }
  }

  // B-fragment row kk = ks*4 + lane%4 -> (sl, x) for the three k-steps of a chunk
  int sl_k[3], x_k[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) {
    const int kk = ks * 4 + (lane & 3);
    sl_k[ks] = kk / 3;
    x_k[ks] = kk % 3;
  }
  // Natural order: the warp's n-tiles (of its column block, set per item).
  // With a symmetric tensor the tiles entirely below the t-block diagonal
  // are skipped, so tiles are dealt to warps zig-zag (or strided, when the
  // H register cache needs a fixed b' period) to balance the remaining work.
  constexpr bool SYMN = SYM && !C::TMAJOR && C::NAG == 1 && C::NCB == 1;  // mirrors stay inside the CTA's element
  constexpr int NTB = C::NTILE / C::NCB;  // n-tiles per column block
  int ntl0[NB], hoff[NB], xoff0[NB];
  unsigned need[NB];
  if constexpr (!C::TMAJOR) {
    constexpr bool ZIGZAG = (C::R == 1) || (C::RC == NB);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      ntl0[nb] = SYMN ? (ZIGZAG ? nb * C::NBLK + ((nb & 1) ? C::NBLK - 1 - nblk : nblk) : nb * C::NBLK + nblk)
                      : nblk * NB + nb;
      // column j = (cb*NTB + ntl0)*8 + cpos; NTB*8 is a multiple of NVE only
      // when NCB == 1, so b' and t' are resolved per item below for NCB > 1.
      const int j = ntl0[nb] * 8 + cpos;
      const int tp = j / NVE, b = j - tp * NVE;
      hoff[nb] = b * C::HB2;  // + (el, a', s) and x at use
      xoff0[nb] = tp;     // + s*3*NTPS at use
      const int tmax = min(NT - 1, (ntl0[nb] * 8 + 7) / NVE);
      unsigned m = 0;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        if (!SYMN || tmax >= 8 * mt) m |= 1u << mt;
      need[nb] = m;
    }
  }
  static_assert(C::NCB == 1 || (NTB * 8) % NVE == 0, "column blocks must start at a t' boundary");

  int64_t gc = 0;
  for (int64_t it = 0; it <= my_items; ++it) {
    if (it == my_items) {  // drain the TMA bulk stores before the CTA exits
      if (C::BULK && tid < EPC) bulk_wait_all();
      break;
    }
    const int64_t w = blockIdx.x + it * gridDim.x;
    const int64_t e = (w / C::NITEM) * EPC + el_w;
    const int agroup = static_cast<int>((w % C::NITEM) / C::NCB);
    const int cb = static_cast<int>(w % C::NCB);
    const int tp_cb = cb * (NTB * 8 / NVE);  // first t' of the column block
    int xoff[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) xoff[nb] = xoff0[nb] + tp_cb;

    double acc[PAIRS ? 1 : WA][MT][PAIRS ? 1 : NB][2];
    double accp[PPW][MT][PAIRS ? MT : 1][2];  // PAIRS: [pair][m-tile][t'-group]
    if constexpr (PAIRS) {
#pragma unroll
      for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int g = 0; g < MT; ++g) accp[pp][mt][g][0] = accp[pp][mt][g][1] = 0.0;
    } else {
#pragma unroll
      for (int wa = 0; wa < WA; ++wa)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) acc[wa][mt][nb][0] = acc[wa][mt][nb][1] = 0.0;
    }

#pragma unroll 1
    for (int chunk = 0; chunk < NCHUNK; ++chunk, ++gc) {
      // A fragments of the chunk (static table) before waiting for H
      double afr3[3][MT];
#pragma unroll
      for (int ks = 0; ks < 3; ++ks)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) afr3[ks][mt] = sXA[(mt * KSTEPS + chunk * 3 + ks) * 32 + lane];
      const int buf = static_cast<int>(gc % C::NBUF);
#ifndef PI_SF_NO_XPRE
      // t'-major: the first k-step's X values (static table) before waiting for H
      double xv0[C::TMAJOR ? MT : 1][3];
      if constexpr (C::TMAJOR) {
#pragma unroll
        for (int g = 0; g < MT; ++g) {
          const double* xp = sXP + (chunk * 4 + sl_k[0]) * 3 * NTPS + g * 8 + cpos;
          xv0[g][0] = xp[0];
          xv0[g][1] = xp[NTPS];
          xv0[g][2] = xp[2 * NTPS];
        }
      }
#endif
      named_sync(kBarFull0 + buf, C::NTHREADS);
      const double* Hb = sH + buf * C::H_PER_BUF;
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) {
        const double* afr = afr3[ks];
        const int s = chunk * 4 + sl_k[ks];
        if constexpr (C::TMAJOR) {
          // n-tile (g, b'): columns t' = 8g + cpos at fixed b'; lane's X shared by all b'
          double xv[MT][3];
#pragma unroll
          for (int g = 0; g < MT; ++g) {
#ifndef PI_SF_NO_XPRE
            if (ks == 0) {
              xv[g][0] = xv0[g][0];
              xv[g][1] = xv0[g][1];
              xv[g][2] = xv0[g][2];
              continue;
            }
#endif
            const double* xp = sXP + s * 3 * NTPS + g * 8 + cpos;
            xv[g][0] = xp[0];
            xv[g][1] = xp[NTPS];
            xv[g][2] = xp[2 * NTPS];
          }
          if constexpr (PAIRS) {
#pragma unroll
            for (int pp = 0; pp < PPW; ++pp) {
              const int o = ((el_w * AG + pa[pp]) * 4 + sl_k[ks]) * C::HS2 + x_k[ks] + pb[pp] * C::HB2;
              const double2 h01 = *reinterpret_cast<const double2*>(Hb + 2 * o);
              const double h2 = Hb[C::H2OFF + o];
#pragma unroll
              for (int g = 0; g < MT; ++g) {
                const double gv = fma(h01.x, xv[g][0], fma(h01.y, xv[g][1], h2 * xv[g][2]));
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                  if (pp >= NDW || g >= mt) dmma_8x8x4(accp[pp][mt][g][0], accp[pp][mt][g][1], afr[mt], gv);
              }
            }
          } else {
#pragma unroll
          for (int wa = 0; wa < WA; ++wa) {
            const int o = ((el_w * AG + al0 + wa) * 4 + sl_k[ks]) * C::HS2 + x_k[ks];
#pragma unroll
            for (int b = 0; b < NVE; ++b) {
              const double2 h01 = *reinterpret_cast<const double2*>(Hb + 2 * (o + b * C::HB2));
              const double h2 = Hb[C::H2OFF + o + b * C::HB2];
#pragma unroll
              for (int g = 0; g < MT; ++g) {
                const double gv = fma(h01.x, xv[g][0], fma(h01.y, xv[g][1], h2 * xv[g][2]));
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                  if (!SYMK || g >= mt) dmma_8x8x4(acc[wa][mt][g * NVE + b][0], acc[wa][mt][g * NVE + b][1], afr[mt], gv);
              }
            }
          }
          }
        } else {
          const double* Xs = sXP + s * 3 * NTPS;
          // X values of the lane's n-tiles, shared by the WA rows a'
          double xr[WA > 1 ? NB : 1][3];
          if constexpr (WA > 1) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              if constexpr (C::XP4) {
                const double* xq = sXP + (s * C::NTP + xoff[nb]) * 4;
                const double2 x01 = *reinterpret_cast<const double2*>(xq);
                xr[nb][0] = x01.x;
                xr[nb][1] = x01.y;
                xr[nb][2] = xq[2];
              } else {
                const double* xp = Xs + xoff[nb];
                xr[nb][0] = xp[0];
                xr[nb][1] = xp[NTPS];
                xr[nb][2] = xp[2 * NTPS];
              }
            }
          }
#pragma unroll
          for (int wa = 0; wa < WA; ++wa) {
            const int o = ((el_w * AG + al0 + wa) * 4 + sl_k[ks]) * C::HS2 + x_k[ks];
            // b' for n-tile nb is b'_(nb mod R): load each distinct one once
            double hr[C::RC][3];
#pragma unroll
            for (int m = 0; m < C::RC; ++m) {
              const double2 h01 = *reinterpret_cast<const double2*>(Hb + 2 * (o + hoff[m]));
              hr[m][0] = h01.x;
              hr[m][1] = h01.y;
              hr[m][2] = Hb[C::H2OFF + o + hoff[m]];
            }
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              const double* h = hr[nb % C::R];
              double gv;
              if constexpr (WA > 1) {
                gv = fma(h[0], xr[nb][0], fma(h[1], xr[nb][1], h[2] * xr[nb][2]));
              } else if constexpr (C::XP4) {
                const double* xq = sXP + (s * C::NTP + xoff[nb]) * 4;
                const double2 x01 = *reinterpret_cast<const double2*>(xq);
                gv = fma(h[0], x01.x, fma(h[1], x01.y, h[2] * xq[2]));
              } else {
                const double* xp = Xs + xoff[nb];
                gv = fma(h[0], xp[0], fma(h[1], xp[NTPS], h[2] * xp[2 * NTPS]));
              }
#pragma unroll
              for (int mt = 0; mt < MT; ++mt)
                if (!SYMN || ((need[nb] >> mt) & 1u)) dmma_8x8x4(acc[wa][mt][nb][0], acc[wa][mt][nb][1], afr[mt], gv);
            }
          }
        }
      }
      if (gc + C::NBUF < total_chunks) named_arrive(kBarEmpty0 + buf, C::NTHREADS);
    }

    // ---- epilogue (overlaps the producers' next item) ----
    if constexpr (C::BULK) {
      // Whole element matrices in canonical order, mirrors included, then one
      // TMA bulk store per element (FP64, or rounded to FP32 in the staging
      // buffer for the FP32 output variant).
      const bool f32 = args.out32 != nullptr;
      const uintptr_t obase = f32 ? reinterpret_cast<uintptr_t>(args.out32) : reinterpret_cast<uintptr_t>(args.out);
      const bool bulk = args.out_layout == PI_OUT_CANONICAL && (obase & 15) == 0;
      const int amask = f32 ? 3 : 1;  // staging offset so smem and global agree modulo 16 bytes
      if (tid < EPC) bulk_wait_read();  // the issuing threads: previous stores no longer read the staging buffer
      named_sync(kBarCons, 32 * C::NCW);
      const int64_t ecl = e < args.n_elem ? e : 0;
      const int soff = bulk ? static_cast<int>((ecl * kk_elem) & amask) : 0;
      double* st = smem + C::OFF_STAGE + el_w * C::ESTRIDE + soff;
      float* stf = reinterpret_cast<float*>(smem + C::OFF_STAGE + el_w * C::ESTRIDE) + soff;
      auto stage = [&](auto put) {
      if constexpr (PAIRS) {
#pragma unroll
        for (int pp = 0; pp < PPW; ++pp)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int t = mt * 8 + (lane >> 2);
#pragma unroll
            for (int g = (pp < NDW ? mt : 0); g < MT; ++g)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int tp = g * 8 + 2 * (lane & 3) + h;
                if (t < NT && tp < NT) {
                  const double v = accp[pp][mt][g][h];
                  const int row = t * NVE + pa[pp], col = tp * NVE + pb[pp];
                  put(row * NSH + col, v);
                  if (pp >= NDW || g > mt) put(col * NSH + row, v);  // the skipped mirror block
                }
              }
          }
      } else if constexpr (C::TMAJOR) {
#pragma unroll
      for (int wa = 0; wa < WA; ++wa)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t = mt * 8 + (lane >> 2);
          const int row = t * NVE + al0 + wa;
#pragma unroll
          for (int g = SYMK ? mt : 0; g < MT; ++g)
#pragma unroll
            for (int b = 0; b < NVE; ++b)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int tp = g * 8 + 2 * (lane & 3) + h;
                if (t < NT && tp < NT) {
                  const double v = acc[wa][mt][g * NVE + b][h];
                  put(row * NSH + tp * NVE + b, v);
                  if (SYMK && g > mt) put((tp * NVE + b) * NSH + row, v);  // mirror of the skipped block
                }
              }
        }
      } else {
        // natural order, whole elements in the CTA (NAG == 1, NCB == 1)
#pragma unroll
        for (int wa = 0; wa < WA; ++wa)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int t = mt * 8 + (lane >> 2);
            const int row = t * NVE + al0 + wa;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              if (SYMN && !((need[nb] >> mt) & 1u)) continue;  // filled by the transposed tile's mirror
              if (t >= NT) continue;
              const int j = ntl0[nb] * 8 + 2 * (lane & 3);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int jj = j + h;
                if (jj >= NSH) continue;
                const double v = acc[wa][mt][nb][h];
                put(row * NSH + jj, v);
                if (SYMN) {
                  const int mt2 = (jj / NVE) >> 3;
                  const int tmax2 = min(NT - 1, ((row >> 3) * 8 + 7) / NVE);
                  if (tmax2 < 8 * mt2) put(jj * NSH + row, v);
                }
              }
            }
          }
      }
      };
      stage([&](int idx, double v) {
        if (f32)
          stf[idx] = static_cast<float>(v);
        else
          st[idx] = v;
      });
      fence_proxy_async_smem();
      named_sync(kBarCons, 32 * C::NCW);
      if (bulk) {
        if (tid < EPC) {
          const int64_t ee = (w / C::NITEM) * EPC + tid;
          if (ee < args.n_elem) {
            const int o = static_cast<int>((ee * kk_elem) & amask);
            if (f32)
              bulk_store_floats(args.out32 + ee * kk_elem,
                                reinterpret_cast<const float*>(smem + C::OFF_STAGE + tid * C::ESTRIDE) + o,
                                static_cast<int>(kk_elem));
            else
              bulk_store_doubles(args.out + ee * kk_elem, smem + C::OFF_STAGE + tid * C::ESTRIDE + o,
                                 static_cast<int>(kk_elem));
            bulk_commit();
          }
        }
      } else {
        for (int el = 0; el < EPC; ++el) {
          const int64_t ee = (w / C::NITEM) * EPC + el;
          if (ee >= args.n_elem) break;
          const double* src = smem + C::OFF_STAGE + el * C::ESTRIDE;
          const float* srcf = reinterpret_cast<const float*>(src);
          for (int i = tid; i < kk_elem; i += 32 * C::NCW) {
            const double v = f32 ? static_cast<double>(srcf[i]) : src[i];
            if (args.out_layout == PI_OUT_CANONICAL)
              store_out(args, ee * kk_elem + i, v);
            else
              store_out(args, i * args.ld_out + ee, v);
          }
        }
      }
      continue;
    }
    if (e >= args.n_elem) continue;
    if constexpr (C::TMAJOR) {
      // warp-private staging of its WA*NT full K rows, then row-wise coalesced stores
      double* st = smem + C::OFF_STAGE + warp * C::STAGE_PER_WARP;
#pragma unroll
      for (int wa = 0; wa < WA; ++wa)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t = mt * 8 + (lane >> 2);
#pragma unroll
          for (int g = 0; g < MT; ++g)
#pragma unroll
            for (int b = 0; b < NVE; ++b)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int tp = g * 8 + 2 * (lane & 3) + h;
                if (t < NT && tp < NT) st[(wa * NT + t) * NSH + tp * NVE + b] = acc[wa][mt][g * NVE + b][h];
              }
        }
      __syncwarp();
      const int64_t row0 = agroup * AG + al0;  // row of (t = 0, wa = 0); row(t, wa) = row0 + t*NVE + wa
      if (args.out_layout == PI_OUT_CANONICAL) {
        const int64_t dst = e * kk_elem + row0 * NSH;
#pragma unroll
        for (int wa = 0; wa < WA; ++wa)
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int j0 = 0; j0 < NSH; j0 += 32)
              if (j0 + lane < NSH)
                store_out(args, dst + (t * NVE + wa) * NSH + j0 + lane, st[(wa * NT + t) * NSH + j0 + lane]);
      } else {
        for (int r = 0; r < WA * NT; ++r) {
          const int wa = r / NT, t = r % NT;
          const int64_t row = row0 + t * NVE + wa;
          for (int j = lane; j < NSH; j += 32) store_out(args, (row * NSH + j) * args.ld_out + e, st[r * NSH + j]);
        }
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int wa = 0; wa < WA; ++wa)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t = mt * 8 + (lane >> 2);
          const int row = t * NVE + agroup * AG + al0 + wa;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            if (SYMN && !((need[nb] >> mt) & 1u)) continue;  // filled by the transposed tile's mirror
            if (t >= NT) continue;
            const int j = (cb * NTB + ntl0[nb]) * 8 + 2 * (lane & 3);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int jj = j + h;
              if (jj >= NSH) continue;
              const double v = acc[wa][mt][nb][h];
              bool mirror = false;
              if (SYMN) {
                // the transposed entry (jj, row) sits in tile (m-tile of t' = jj/NVE, n-tile of row);
                // write it here when that tile is skipped
                const int mt2 = (jj / NVE) >> 3;
                const int tmax2 = min(NT - 1, ((row >> 3) * 8 + 7) / NVE);
                mirror = tmax2 < 8 * mt2;
              }
              if (args.out_layout == PI_OUT_CANONICAL) {
                store_out(args, e * kk_elem + static_cast<int64_t>(row) * NSH + jj, v);
                if (mirror) store_out(args, e * kk_elem + static_cast<int64_t>(jj) * NSH + row, v);
              } else {
                store_out(args, (static_cast<int64_t>(row) * NSH + jj) * args.ld_out + e, v);
                if (mirror) store_out(args, (static_cast<int64_t>(jj) * NSH + row) * args.ld_out + e, v);
              }
            }
          }
        }
    }
  }
}

}  // namespace pib
