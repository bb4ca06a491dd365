// FP32 variant of the sum-factorised element stiffness on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM), p = 3..7,
// scalar weak forms.  Stated bound 5e-5 (test_kernels.cpp:41-61); measured <= 4.2e-7.
//
// With the factorisation of kernels_sumfact.cuh,
//     K[(t,a), j] = sum_(x,s) X_x(t,s) G_x(s,a,j),
//     G_x(s,a,j)  = sum_y H_xy(s,a,b_j) X_y(t'_j,s),   j = t'*(p+1) + b,
// every Legendre row a is one GEMM with the element-dependent operand in the
// M role:
//     D_a[j][t] = sum_k A_a[j][k] B[k][t],  A_a[j][(x,s)] = G_x(s,a,j),
//     B[(x,s)][t] = X_x(t,s)  (element independent),  K[(t,a), j] = D_a[j][t],
// M = 128 rows j per tile (ceil(N_sh/128) tiles), N = N_t padded to 16,
// K = 3 x (N_s padded to 8).  TF32 keeps 10 mantissa bits, so each operand is
// split hi + lo (hi = cvt.rna.tf32(v), lo = v - hi exactly) and three MMAs
// accumulate A_hi B_hi + A_hi B_lo + A_lo B_hi in FP32 (3xTF32): the dropped
// A_lo B_lo term and the truncation of lo are ~2^-21 relative.
//
// CUDA cores do what the tensor cores cannot: per element the Jacobians and
// point blocks M (FP64, rounded once), per row a the small H_a (FP32), and the
// G values (3 FMAs + the split each) written straight into the UMMA canonical
// K-major SWIZZLE_NONE layout (8-row x 16-byte core matrices; 16-byte stores).
// Lane 0 of one of the first four warps (round-robin over the rows a) issues
// a row's MMAs (tcgen05.mma; one thread's stream completes one MMA per ~150
// cycles whatever its shape, streams of different threads and CTAs overlap)
// and commits them to mbarriers that free the A buffer (double buffered per
// (a, m-tile, x)) and publish D; all warps then drain D from TMEM
// (tcgen05.ld 32x32b: warp w reads lanes 32(w%4)..+31 = rows j) and store K
// rows (t, a) as coalesced 128-byte segments (lanes = consecutive columns j).
// Opt-in (PI_VARIANT_TC32): slower than rounding the FP64 DMMA result, the
// CUDA-core work around the MMAs bounds it.
#pragma once

#include "kernels_common.cuh"

namespace pib {

template <int P>
struct Tc32Shape {
  static constexpr int NV = P + 1, NZ = P + 1;
  static constexpr int NT = (P + 1) * (P + 2) / 2;
  static constexpr int NS = (P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : P == 5 ? 25 : P == 6 ? 33 : 42);
  static constexpr int NQ = NS * NZ;
  static constexpr int NSH = NT * NV;
  static constexpr int NSP8 = (NS + 7) / 8 * 8;   // s padded to whole MMA k-steps
  static constexpr int KST = NSP8 / 8;            // k-steps (K = 8 tf32) per x
  static constexpr int KTOT = 3 * NSP8;
  static constexpr int MTJ = (NSH + 127) / 128;   // m-tiles of 128 rows j
  static constexpr int NPAD = (NT + 15) / 16 * 16;  // MMA N (multiple of 16 for M = 128)
  // A tcgen05.mma issue stream runs one MMA per ~152 cycles whatever its shape
  // (tools/microbench/tc_mma_rate.cu: M = 64 / 128, N = 16..256, K = 8), and
  // the streams of co-resident CTAs overlap: small CTAs, several per SM.
  static constexpr int CTAS = P <= 4 ? 4 : 1;
  static constexpr int NTHREADS = P <= 4 ? 128 : 256;
  static constexpr int NISSUE = 4;  // MMA-issuing threads per CTA (lane 0 of warps 0..3)
  // A ring: (a, m-tile, x) units, hi + lo tiles each
  static constexpr int NAB = 2;
  // TMEM: a ring of D slots, one per Legendre row a (MTJ x NPAD columns each);
  // CTAS_TMEM CTAs per SM share the 512 columns
  static constexpr int SLOTC = MTJ * NPAD;
  static constexpr int CTAS_TMEM = CTAS;
  static constexpr int NDS_MAX = 512 / CTAS_TMEM / SLOTC;
  static constexpr int NDS = NDS_MAX > 8 ? 8 : NDS_MAX;
  static constexpr int TNEED = NDS * SLOTC;
  static constexpr int TCOLS = TNEED <= 32 ? 32 : TNEED <= 64 ? 64 : TNEED <= 128 ? 128 : TNEED <= 256 ? 256 : 512;
  static_assert(NDS >= 2, "TMEM: at least two D slots");
  // shared memory (bytes); every operand block 1024-aligned
  static constexpr int A_BYTES = 128 * NSP8 * 4;          // one (hi or lo) A tile
  static constexpr int B_BYTES = NPAD * KTOT * 4;         // one (hi or lo) B
  static constexpr int H_FLOATS = 9 * NV * NSP8;
  static constexpr int OFF_A = 0;                         // [NAB buffers][hi, lo]
  static constexpr int OFF_B = OFF_A + 2 * NAB * A_BYTES;  // [hi, lo]
  static constexpr int OFF_XG = OFF_B + 2 * B_BYTES;      // X_y(t', s) float [3][NT][NSP8]
  static constexpr int OFF_H = OFF_XG + 3 * NT * NSP8 * 4;  // H_xy(s, a, b) float [2][3][3][NV][NSP8]
  static constexpr int OFF_M = OFF_H + 2 * H_FLOATS * 4;    // M_kl(s, z) float [16][NQ]
  static constexpr int OFF_Y = (OFF_M + 16 * NQ * 4 + 15) / 16 * 16;  // (P, P') float2 [NZ][NV]
  static constexpr int OFF_D = (OFF_Y + NZ * NV * 8 + 15) / 16 * 16;  // doubles: edges 21, coeff 16, xi1/xi2 [NS], xi3 [NZ], w [NQ]
  static constexpr int D_DOUBLES = 21 + 16 + 2 * NS + NZ + NQ;
  static constexpr int SMEM_BYTES = OFF_D + D_DOUBLES * 8;
  static_assert(SMEM_BYTES <= 232448 - 1024, "shared memory");
  static_assert(CTAS * (SMEM_BYTES + 2048) <= 233472 && CTAS * TCOLS <= 512, "CTAS resident CTAs per SM");
  // one MMA: M = 128, N = NPAD, K = 8, kind::tf32, FP32 accumulate, both operands K-major
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t(NPAD) >> 3) << 17) |
                                    ((128u >> 4) << 24);
};

struct Tc32Tables {
  const float* bhi;    // X in the UMMA B layout (hi), B_BYTES
  const float* blo;    // ... (lo)
  const float* xg;     // X_y(t', s) [3][NT][NSP8]
  const float* yline;  // (P, P') [NZ][NV]
  const double* tri;   // xi1 [NS], xi2 [NS]
  const double* z;     // xi3 [NZ]
  const double* w;     // [NQ] reference order (q = z*NS + s)
};

// Canonical K-major SWIZZLE_NONE byte offset of (row r, k) in an operand tile
// with `rows` rows: core matrices of 8 rows x 16 bytes, 8-row groups 128 bytes
// apart (SBO), 4-column k groups rows*16 bytes apart (LBO).
__host__ __device__ constexpr int umma_kmajor_offset(int r, int k, int rows) {
  return (k / 4) * (rows * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (static_cast<uint64_t>((lbo >> 4) & 0x3fff) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            bool accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ float tf32_hi(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
// 16 consecutive TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// FORM: kFormLaplace (0) or kFormGeneral (1) (kernels_sumfact.cuh SumFactForm).
//
// Pipeline (all 256 threads run the same program; thread 0 also issues the MMAs):
//   per element: M for every rule point (FP64 -> FP32)                     [sync]
//   per row a:   H_a into one of two H buffers                              [sync]
//                units (a, m-tile, x): G -> A ring buffer (waits `empty`),
//                arrive `full`; thread 0 waits `full`, issues 3 x KST MMAs
//                into D slot(a), commits `empty` (and `dfull` after x = 2)
//                epilogue of row a-1 (its MMAs were issued one phase earlier):
//                wait `dfull`, tcgen05.ld, coalesced FP32 stores
// The D slot of row a is overwritten no earlier than NDS rows later, after at
// least one CTA barrier that follows its epilogue.
template <int P, int FORM>
__global__ void __launch_bounds__(Tc32Shape<P>::NTHREADS, Tc32Shape<P>::CTAS) sumfact_tc32_kernel(LaunchArgs args, Tc32Tables tab) {
  using C = Tc32Shape<P>;
  constexpr bool GENERAL = FORM == 1;
  constexpr int NV = C::NV, NZ = C::NZ, NT = C::NT, NS = C::NS, NQ = C::NQ, NSH = C::NSH, NSP8 = C::NSP8;
  constexpr int KST = C::KST, MTJ = C::MTJ, NPAD = C::NPAD, NTH = C::NTHREADS, NAB = C::NAB, NDS = C::NDS;
  extern __shared__ __align__(1024) unsigned char tsm[];
  float* sXg = reinterpret_cast<float*>(tsm + C::OFF_XG);
  float* sM = reinterpret_cast<float*>(tsm + C::OFF_M);
  const float2* sY = reinterpret_cast<const float2*>(tsm + C::OFF_Y);
  double* sD = reinterpret_cast<double*>(tsm + C::OFF_D);
  double* sEdge = sD;
  double* sCoef = sD + 21;
  double* sTri = sD + 37;
  double* sZ = sTri + 2 * NS;
  double* sW = sZ + NZ;
  __shared__ __align__(8) uint64_t bar_full[NAB];   // A buffer written by all threads
  __shared__ __align__(8) uint64_t bar_empty[NAB];  // its MMAs completed
  __shared__ __align__(8) uint64_t bar_dfull[NDS];  // D slot complete
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NAB; ++i) {
      mbar_init(&bar_full[i], NTH);
      mbar_init(&bar_empty[i], 1);
    }
    for (int i = 0; i < NDS; ++i) mbar_init(&bar_dfull[i], 1);
  }
  // static tables: B (hi, lo) in UMMA layout, X for G, (P, P'), rule
  for (int i = tid; i < C::B_BYTES / 16; i += NTH) {
    reinterpret_cast<float4*>(tsm + C::OFF_B)[i] = reinterpret_cast<const float4*>(tab.bhi)[i];
    reinterpret_cast<float4*>(tsm + C::OFF_B + C::B_BYTES)[i] = reinterpret_cast<const float4*>(tab.blo)[i];
  }
  for (int i = tid; i < 3 * NT * NSP8; i += NTH) sXg[i] = tab.xg[i];
  for (int i = tid; i < NZ * NV; i += NTH)
    reinterpret_cast<float2*>(tsm + C::OFF_Y)[i] = make_float2(tab.yline[2 * i], tab.yline[2 * i + 1]);
  for (int i = tid; i < 2 * NS; i += NTH) sTri[i] = tab.tri[i];
  for (int i = tid; i < NZ; i += NTH) sZ[i] = tab.z[i];
  for (int i = tid; i < NQ; i += NTH) sW[i] = tab.w[i];
  // A tiles: rows j >= N_sh are never written; zero them once (their D rows are not stored)
  for (int i = tid; i < 2 * NAB * C::A_BYTES / 16; i += NTH)
    reinterpret_cast<float4*>(tsm + C::OFF_A)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = tid; i < 2 * C::H_FLOATS; i += NTH) reinterpret_cast<float*>(tsm + C::OFF_H)[i] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t sbase = smem_u32(tsm);

  uint32_t full_ph = 0, empty_ph = 0, dfull_ph = 0;  // parity bit per buffer / slot
  unsigned empty_used = 0;                            // buffers that have been committed at least once
  int ab = 0;          // next A buffer
  int64_t arow = 0;    // rows a processed by this CTA (D slot = arow % NDS)
  const int64_t kk = static_cast<int64_t>(NSH) * NSH;

  // epilogue of the row issued as `row` (element e, Legendre row a)
  auto epilogue = [&](int64_t row, int64_t e, int a) {
    const int slot = static_cast<int>(row % NDS);
    mbar_wait(&bar_dfull[slot], (dfull_ph >> slot) & 1u);
    dfull_ph ^= 1u << slot;
    tc_fence_after();
    constexpr int NCG = NTH / 128;  // warps per TMEM lane quarter: they split the 16-column chunks
    const int quarter = warp & 3, colgroup = warp >> 2;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + slot * C::SLOTC;
#pragma unroll
    for (int mt = 0; mt < MTJ; ++mt) {
      const int j = mt * 128 + 32 * quarter + lane;
#pragma unroll
      for (int c0 = 0; c0 < NPAD; c0 += 16) {
        if ((c0 / 16) % NCG != colgroup) continue;
        float v[16];
        tc_ld16(tbase + mt * NPAD + c0, v);
        if (j < NSH) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int t = c0 + c;
            if (t < NT) {
              const int64_t r = t * NV + a;
              if (args.out_layout == PI_OUT_CANONICAL)
                args.out32[e * kk + r * NSH + j] = v[c];
              else
                args.out32[(r * NSH + j) * args.ld_out + e] = v[c];
            }
          }
        }
      }
    }
    tc_fence_before();  // these TMEM reads precede the next barrier (and any MMA that reuses the slot)
  };

  int64_t pend_row = -1, pend_e = 0;
  int pend_a = 0;
  for (int64_t e = blockIdx.x; e < args.n_elem; e += gridDim.x) {
    // ---- geometry, coefficients, point blocks M (FP64, rounded to FP32) ----
    if (tid == 0) {
      double x[18], d[21];
#pragma unroll
      for (int c = 0; c < 18; ++c) x[c] = args.geom[c * args.geom_ld + e];
      prism_edges(x, d);
#pragma unroll
      for (int c = 0; c < 21; ++c) sEdge[c] = d[c];
    }
    if (GENERAL && tid < 16) sCoef[tid] = args.coeff ? args.coeff[tid * args.coeff_ld + e] : args.cu[tid];
    __syncthreads();
    for (int q = tid; q < NQ; q += NTH) {  // point q = s*NZ + z (H walks z for fixed s)
      const int s = q / NZ, z = q % NZ;
      double cf[3][3];
      const double det = jacobian_cofactors(sEdge, sTri[s], sTri[NS + s], sZ[z], cf);
      if (!(det > 0.0)) flag_inverted(args.bad, args.element_id_base + e);
      const double w8 = sW[z * NS + s];
      double M[16];
      block_from_cofactors<GENERAL>(cf, det, w8, w8 * __drcp_rn(det), sCoef, M);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (GENERAL || (k >= 4 && (k & 3) != 0)) sM[k * NQ + q] = static_cast<float>(M[k]);
    }
    __syncthreads();

    for (int a = 0; a < NV; ++a, ++arow) {
      // ---- H_xy(s, a, b) for this row a: items (x, y, b, s) ----
      float* sH = reinterpret_cast<float*>(tsm + C::OFF_H) + (arow & 1) * C::H_FLOATS;
      for (int i = tid; i < 9 * NV * NS; i += NTH) {
        const int s = i % NS, b = (i / NS) % NV, xy = i / (NS * NV), x = xy / 3, y = xy % 3;
        const int kx = x < 2 ? x + 1 : 3, ly = y < 2 ? y + 1 : 3;
        float h = 0.f;
#pragma unroll
        for (int z = 0; z < NZ; ++z) {
          const float2 ya = sY[z * NV + a], yb = sY[z * NV + b];
          const float wa = x < 2 ? ya.x : ya.y, wb = y < 2 ? yb.x : yb.y;
          const float* Mz = sM + s * NZ + z;
          const float m = Mz[(kx * 4 + ly) * NQ];
          if (GENERAL) {
            // x = 2 also holds k = 0 (weight P), y = 2 also l = 0 (weight P)
            float v = wa * m * wb;
            if (x == 2) v = fmaf(ya.x * Mz[(0 * 4 + ly) * NQ], wb, v);
            if (y == 2) v = fmaf(wa * Mz[(kx * 4 + 0) * NQ], yb.x, v);
            if (x == 2 && y == 2) v = fmaf(ya.x * Mz[0], yb.x, v);
            h += v;
          } else {
            h = fmaf(wa * m, wb, h);
          }
        }
        sH[((x * 3 + y) * NV + b) * NSP8 + s] = h;
      }
      __syncthreads();  // H_a complete; every earlier epilogue's TMEM reads are ordered before later MMAs
      if (tid == 0) tc_fence_after();
      const int slot = static_cast<int>(arow % NDS);

      for (int mt = 0; mt < MTJ; ++mt) {
        for (int x = 0; x < 3; ++x) {
          const int buf = ab;
          ab = ab + 1 == NAB ? 0 : ab + 1;
          // the MMAs that last read this A buffer are complete
          if (empty_used & (1u << buf)) {
            mbar_wait(&bar_empty[buf], (empty_ph >> buf) & 1u);
            empty_ph ^= 1u << buf;
          }
          // ---- G_x(s, a, j) -> A (hi, lo): thread = (row r, part of the s range) ----
          unsigned char* Ahi = tsm + C::OFF_A + buf * 2 * C::A_BYTES;
          unsigned char* Alo = Ahi + C::A_BYTES;
          {
            constexpr int NPART = NTH / 128;
            const int r = tid & 127, half = tid >> 7;
            const int j = mt * 128 + r;
            if (j < NSH) {
              const int tp = j / NV, b = j % NV;
              const float* h0 = sH + ((x * 3 + 0) * NV + b) * NSP8;
              const float* h1 = h0 + NV * NSP8;
              const float* h2 = h1 + NV * NSP8;
              const float* x0 = sXg + (0 * NT + tp) * NSP8;
              const float* x1 = x0 + NT * NSP8;
              const float* x2 = x1 + NT * NSP8;
              constexpr int S4 = NSP8 / 4;
#pragma unroll 2
              for (int s4 = half; s4 < S4; s4 += NPART) {
                const float4 a0 = reinterpret_cast<const float4*>(h0)[s4];
                const float4 a1 = reinterpret_cast<const float4*>(h1)[s4];
                const float4 a2 = reinterpret_cast<const float4*>(h2)[s4];
                const float4 b0 = reinterpret_cast<const float4*>(x0)[s4];
                const float4 b1 = reinterpret_cast<const float4*>(x1)[s4];
                const float4 b2 = reinterpret_cast<const float4*>(x2)[s4];
                float g[4];
                g[0] = fmaf(a0.x, b0.x, fmaf(a1.x, b1.x, a2.x * b2.x));
                g[1] = fmaf(a0.y, b0.y, fmaf(a1.y, b1.y, a2.y * b2.y));
                g[2] = fmaf(a0.z, b0.z, fmaf(a1.z, b1.z, a2.z * b2.z));
                g[3] = fmaf(a0.w, b0.w, fmaf(a1.w, b1.w, a2.w * b2.w));
                float4 hi, lo;
                hi.x = tf32_hi(g[0]);
                hi.y = tf32_hi(g[1]);
                hi.z = tf32_hi(g[2]);
                hi.w = tf32_hi(g[3]);
                lo = make_float4(g[0] - hi.x, g[1] - hi.y, g[2] - hi.z, g[3] - hi.w);
                const int off = umma_kmajor_offset(r, 4 * s4, 128);
                *reinterpret_cast<float4*>(Ahi + off) = hi;
                *reinterpret_cast<float4*>(Alo + off) = lo;
              }
            }
          }
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_full[buf])) : "memory");
          // one issuing thread per row a, dealt round-robin over the first warps:
          // each thread's tcgen05.mma stream completes one MMA per ~150 cycles, and
          // streams of different threads overlap (tools/microbench/tc_mma_rate.cu);
          // the MMAs of one D slot stay in one stream, in order
          if (lane == 0 && warp == static_cast<int>(arow % C::NISSUE)) {
            mbar_wait(&bar_full[buf], (full_ph >> buf) & 1u);
            tc_fence_after();
            const uint32_t d = tmem + slot * C::SLOTC + mt * NPAD;
            const uint32_t ahi = sbase + C::OFF_A + buf * 2 * C::A_BYTES, alo = ahi + C::A_BYTES;
            const uint32_t bhi = sbase + C::OFF_B, blo = bhi + C::B_BYTES;
            constexpr uint32_t LBO_A = 128 * 16, LBO_B = NPAD * 16, SBO = 128;
#pragma unroll
            for (int ks = 0; ks < KST; ++ks) {
              const uint32_t ao = ks * 2 * LBO_A;                     // k = 8 ks within this x
              const uint32_t bo = ((x * NSP8 + 8 * ks) / 4) * LBO_B;  // k = x*NSP8 + 8 ks in B
              const bool acc0 = !(x == 0 && ks == 0);
              tc_mma_tf32(d, umma_desc(ahi + ao, LBO_A, SBO), umma_desc(blo + bo, LBO_B, SBO), C::IDESC, acc0);
              tc_mma_tf32(d, umma_desc(alo + ao, LBO_A, SBO), umma_desc(bhi + bo, LBO_B, SBO), C::IDESC, true);
              tc_mma_tf32(d, umma_desc(ahi + ao, LBO_A, SBO), umma_desc(bhi + bo, LBO_B, SBO), C::IDESC, true);
            }
            tc_commit(&bar_empty[buf]);
            if (x == 2 && mt == MTJ - 1) tc_commit(&bar_dfull[slot]);
          }
          full_ph ^= 1u << buf;
          empty_used |= 1u << buf;
        }
      }
      // epilogue of the previous row (its MMAs were issued one phase earlier)
      if (pend_row >= 0) epilogue(pend_row, pend_e, pend_a);
      pend_row = arow;
      pend_e = e;
      pend_a = a;
    }
  }
  if (pend_row >= 0) epilogue(pend_row, pend_e, pend_a);
  // every issued MMA has completed (the last D slot was waited for); free TMEM
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TCOLS));
}

}  // namespace pib
