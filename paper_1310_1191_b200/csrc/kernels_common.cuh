// Device helpers shared by the integration kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/prism_b200.h"

// A/B builds (tools/ab_build.sh): build-time overrides of launch shapes and switches.
#ifdef PI_SF_OVERRIDE
#include PI_SF_OVERRIDE
#endif

namespace pib {

// Per-launch arguments common to every strategy.
struct LaunchArgs {
  int64_t n_elem;
  int64_t element_id_base;
  const double* geom;   // SoA [18][geom_ld]
  int64_t geom_ld;
  const double* coeff;  // PER_ELEMENT: SoA [16][coeff_ld]; else nullptr
  int64_t coeff_ld;
  double cu[144];       // UNIFORM coefficient tensor [n_eq][n_eq][4][4] (or E, nu)
  double* out;
  float* out32;         // FP32 output variant (out unused): K rounded to float at the store
  int out_layout;
  int64_t ld_out;
  unsigned long long* bad;      // min offending global element id (atomicMin): inverted element
  unsigned long long* bad_mat;  // ... invalid material (E, nu) of an elasticity element
  // Fused load vectors (pi_integrate_load, n_eq = 1): when fout != nullptr the
  // stiffness kernels also write F_i = sum_q det w_q f phi_i(q) as [n_elem][n_shape],
  // f = fsrc[e] (per element) or fconst.
  double* fout;
  const double* fsrc;
  double fconst;
};

// f of element e for the fused load vector.
__device__ __forceinline__ double load_f(const LaunchArgs& a, int64_t e) { return a.fsrc ? a.fsrc[e] : a.fconst; }

// Jacobian of the multilinear prism map at xi (geometry.cpp:32-58) for the
// SoA/smem vertex array x[v*3+i], its determinant and the cofactor inverse
// inv[k][i] = dxi_k/dx_i (geometry.cpp:60-83).  Returns det.
__device__ __forceinline__ double prism_jacobian(const double* __restrict__ x, double xi1, double xi2,
                                                 double xi3, double inv[3][3]) {
  const double zm = 0.5 * (1.0 - xi3), zp = 0.5 * (1.0 + xi3);
  const double l0 = 0.5 * (1.0 - xi1 - xi2), l1 = 0.5 * xi1, l2 = 0.5 * xi2;
  double j[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    j[i][0] = zm * (x[3 + i] - x[0 + i]) + zp * (x[12 + i] - x[9 + i]);
    j[i][1] = zm * (x[6 + i] - x[0 + i]) + zp * (x[15 + i] - x[9 + i]);
    j[i][2] = l0 * (x[9 + i] - x[0 + i]) + l1 * (x[12 + i] - x[3 + i]) + l2 * (x[15 + i] - x[6 + i]);
  }
  const double c00 = j[1][1] * j[2][2] - j[1][2] * j[2][1];
  const double c01 = j[1][2] * j[2][0] - j[1][0] * j[2][2];
  const double c02 = j[1][0] * j[2][1] - j[1][1] * j[2][0];
  const double det = j[0][0] * c00 + j[0][1] * c01 + j[0][2] * c02;
  const double id = 1.0 / det;
  inv[0][0] = c00 * id;
  inv[0][1] = (j[0][2] * j[2][1] - j[0][1] * j[2][2]) * id;
  inv[0][2] = (j[0][1] * j[1][2] - j[0][2] * j[1][1]) * id;
  inv[1][0] = c01 * id;
  inv[1][1] = (j[0][0] * j[2][2] - j[0][2] * j[2][0]) * id;
  inv[1][2] = (j[0][2] * j[1][0] - j[0][0] * j[1][2]) * id;
  inv[2][0] = c02 * id;
  inv[2][1] = (j[0][1] * j[2][0] - j[0][0] * j[2][1]) * id;
  inv[2][2] = (j[0][0] * j[1][1] - j[0][1] * j[1][0]) * id;
  return det;
}

// Reference-coordinate coefficient block M = T (dw C) T^T with
// T = diag(1, inv): then K_ij = sum_q sum_kl phi_k(i,q) M_kl(q) phi_l(j,q),
// an exact re-association of integrate_generic's
// sum_q sum_ab (dw c_ab) psi_a(i) psi_b(j) (integrate_ref.cpp:79-88), with
// psi from physical_derivatives (geometry.cpp:85-102).  M is 4x4 row-major.
template <bool GENERAL>
__device__ __forceinline__ void coefficient_block(const double inv[3][3], double dw, const double* c,
                                                  double M[16]) {
  if (!GENERAL) {
    // Laplace: c[d][d] = 1 (d = 1..3): M_kl = dw * sum_d inv[k][d] inv[l][d].
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int l = k; l < 3; ++l) {
        const double v = dw * (inv[k][0] * inv[l][0] + inv[k][1] * inv[l][1] + inv[k][2] * inv[l][2]);
        M[(k + 1) * 4 + (l + 1)] = v;
        M[(l + 1) * 4 + (k + 1)] = v;
      }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      M[k] = 0.0;
      M[k * 4] = 0.0;
    }
  } else {
    double cd[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) cd[i] = dw * c[i];
    // W = C' T^T: W[a][l] = sum_b C'[a][b] T[l][b]
    double W[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      W[a][0] = cd[a * 4 + 0];
#pragma unroll
      for (int l = 1; l < 4; ++l)
        W[a][l] = cd[a * 4 + 1] * inv[l - 1][0] + cd[a * 4 + 2] * inv[l - 1][1] + cd[a * 4 + 3] * inv[l - 1][2];
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      M[0 * 4 + l] = W[0][l];
#pragma unroll
      for (int k = 1; k < 4; ++k)
        M[k * 4 + l] = inv[k - 1][0] * W[1][l] + inv[k - 1][1] * W[2][l] + inv[k - 1][2] * W[3][l];
    }
  }
}


// Per-element geometry as the seven edge vectors the multilinear map needs
// (geometry.cpp:32-58): d = [x1-x0, x4-x3, x2-x0, x5-x3, x3-x0, x4-x1, x5-x2],
// each [3].  Then J[:,0] = zm d0 + zp d1, J[:,1] = zm d2 + zp d3,
// J[:,2] = (l0 d4 + l1 d5 + l2 d6)/2.
__device__ __forceinline__ void prism_edges(const double* __restrict__ x, double d[21]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    d[0 + i] = x[3 + i] - x[0 + i];
    d[3 + i] = x[12 + i] - x[9 + i];
    d[6 + i] = x[6 + i] - x[0 + i];
    d[9 + i] = x[15 + i] - x[9 + i];
    d[12 + i] = x[9 + i] - x[0 + i];
    d[15 + i] = x[12 + i] - x[3 + i];
    d[18 + i] = x[15 + i] - x[6 + i];
  }
}

// det J only (load vectors): three cofactors instead of nine.
template <int DS = 1>
__device__ __forceinline__ double jacobian_det(const double* __restrict__ dp, double xi1, double xi2, double xi3) {
  auto d = [dp](int i) { return dp[i * DS]; };
  const double zm = 0.5 * (1.0 - xi3), zp = 0.5 * (1.0 + xi3);
  const double l0 = 0.5 * (1.0 - xi1 - xi2), l1 = 0.5 * xi1, l2 = 0.5 * xi2;
  double j[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    j[i][0] = fma(zm, d(0 + i), zp * d(3 + i));
    j[i][1] = fma(zm, d(6 + i), zp * d(9 + i));
    j[i][2] = fma(l0, d(12 + i), fma(l1, d(15 + i), l2 * d(18 + i)));
  }
  const double c0 = j[1][1] * j[2][2] - j[1][2] * j[2][1];
  const double c1 = j[1][2] * j[2][0] - j[1][0] * j[2][2];
  const double c2 = j[1][0] * j[2][1] - j[1][1] * j[2][0];
  return j[0][0] * c0 + j[0][1] * c1 + j[0][2] * c2;
}

// The per-point block M = T (det w C) T^T of coefficient_block, built from
// the cofactors c_ik of J without forming J^-1 (inv[k][i] = c_ik / det,
// geometry.cpp:60-83):
//   Laplace  M_kl = (w/det) sum_i c_i,k-1 c_i,l-1            (k, l >= 1)
//   general  M_00 = w det C_00,  M_0l = w sum_b C_0b c_b-1,l-1,
//            M_k0 = w sum_a c_a-1,k-1 C_a0,
//            M_kl = (w/det) sum_ab c_a-1,k-1 C_ab c_b-1,l-1.
// Returns det (<= 0 flags an inverted element, geometry.cpp:67-69).
// Jacobian of the multilinear map at xi from the edge vectors (stride DS)
// and its cofactors cf[i][k] (of J[i][k] = dx_i/dxi_k); returns det.
// inv[k][i] = cf[i][k] / det (geometry.cpp:60-83).
// T: the arithmetic type (double; float for the FP32 variant), edges stored as double.
template <int DS = 1, typename T = double>
__device__ __forceinline__ T jacobian_cofactors(const double* __restrict__ dp, T xi1, T xi2, T xi3, T cf[3][3]) {
  auto d = [dp](int i) { return static_cast<T>(dp[i * DS]); };
  const T zm = T(0.5) * (T(1) - xi3), zp = T(0.5) * (T(1) + xi3);
  const T l0 = T(0.5) * (T(1) - xi1 - xi2), l1 = T(0.5) * xi1, l2 = T(0.5) * xi2;
  T j[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    j[i][0] = fma(zm, d(0 + i), zp * d(3 + i));
    j[i][1] = fma(zm, d(6 + i), zp * d(9 + i));
    j[i][2] = fma(l0, d(12 + i), fma(l1, d(15 + i), l2 * d(18 + i)));
  }
  cf[0][0] = j[1][1] * j[2][2] - j[1][2] * j[2][1];
  cf[0][1] = j[1][2] * j[2][0] - j[1][0] * j[2][2];
  cf[0][2] = j[1][0] * j[2][1] - j[1][1] * j[2][0];
  cf[1][0] = j[0][2] * j[2][1] - j[0][1] * j[2][2];
  cf[1][1] = j[0][0] * j[2][2] - j[0][2] * j[2][0];
  cf[1][2] = j[0][1] * j[2][0] - j[0][0] * j[2][1];
  cf[2][0] = j[0][1] * j[1][2] - j[0][2] * j[1][1];
  cf[2][1] = j[0][2] * j[1][0] - j[0][0] * j[1][2];
  cf[2][2] = j[0][0] * j[1][1] - j[0][1] * j[1][0];
  return j[0][0] * cf[0][0] + j[0][1] * cf[0][1] + j[0][2] * cf[0][2];
}

// The per-point block M = T (det w C) T^T of coefficient_block, built from
// the cofactors c_ik of J without forming J^-1:
//   Laplace  M_kl = (w/det) sum_i c_i,k-1 c_i,l-1            (k, l >= 1)
//   general  M_00 = w det C_00,  M_0l = w sum_b C_0b c_b-1,l-1,
//            M_k0 = w sum_a c_a-1,k-1 C_a0,
//            M_kl = (w/det) sum_ab c_a-1,k-1 C_ab c_b-1,l-1.
// wd = w / det.  CS: element stride of the coefficient array.
template <bool GENERAL, int CS = 1, typename T = double>
__device__ __forceinline__ void block_from_cofactors(const T cf[3][3], T det, T w, T wd, const double* cp, T M[16]) {
  auto c = [cp](int i) { return static_cast<T>(cp[i * CS]); };
  if (!GENERAL) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int l = k; l < 3; ++l) {
        const T v = wd * fma(cf[0][k], cf[0][l], fma(cf[1][k], cf[1][l], cf[2][k] * cf[2][l]));
        M[(k + 1) * 4 + (l + 1)] = v;
        M[(l + 1) * 4 + (k + 1)] = v;
      }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      M[k] = T(0);
      M[k * 4] = T(0);
    }
  } else {
    T W[4][3];  // W[a][l-1] = sum_b C_ab c_b-1,l-1
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int l = 0; l < 3; ++l)
        W[a][l] = fma(c(a * 4 + 1), cf[0][l], fma(c(a * 4 + 2), cf[1][l], c(a * 4 + 3) * cf[2][l]));
    M[0] = w * det * c(0);
#pragma unroll
    for (int l = 0; l < 3; ++l) M[l + 1] = w * W[0][l];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      M[(k + 1) * 4] = w * fma(cf[0][k], c(4), fma(cf[1][k], c(8), cf[2][k] * c(12)));
#pragma unroll
      for (int l = 0; l < 3; ++l)
        M[(k + 1) * 4 + (l + 1)] = wd * fma(cf[0][k], W[1][l], fma(cf[1][k], W[2][l], cf[2][k] * W[3][l]));
    }
  }
}

// Isotropic elasticity block (ie, je) (elasticity_tensor, coefficients.cpp:40-59:
// c[ie][je][a+1][b+1] = lam d_(ie,a) d_(je,b) + mu d_(ie,je) d_ab + mu d_(ie,b) d_(je,a)):
//   M_(k+1)(l+1) = (w/det) [lam c_ie,k c_je,l + mu c_je,k c_ie,l + mu d_(ie,je) sum_a c_a,k c_a,l]
// (derivative rows/columns only; row/column 0 are not written).
__device__ __forceinline__ void elasticity_block(const double cf[3][3], double wd, double lam, double mu, int ie,
                                                 int je, double M[16]) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      double v = fma(lam * cf[ie][k], cf[je][l], mu * cf[je][k] * cf[ie][l]);
      if (ie == je) v = fma(mu, fma(cf[0][k], cf[0][l], fma(cf[1][k], cf[1][l], cf[2][k] * cf[2][l])), v);
      M[(k + 1) * 4 + (l + 1)] = wd * v;
    }
}

// lame_parameters' domain checks (coefficients.cpp:23-32): E > 0 and
// -1 < nu < 0.5; a violation flags the element (DomainError on the host).
__device__ __forceinline__ void check_material(const LaunchArgs& a, int64_t e, double young, double nu) {
  if (!(young > 0.0) || !(nu > -1.0) || !(nu < 0.5))
    atomicMin(a.bad_mat, static_cast<unsigned long long>(a.element_id_base + e));
}

// Lame parameters (lame_parameters, coefficients.cpp:33-36).
__device__ __forceinline__ void lame(double young, double nu, double& lam, double& mu) {
  mu = young / (2.0 * (1.0 + nu));
  lam = young * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
}

// DS / CS: element strides of the edge-vector and coefficient arrays (1 for
// per-thread arrays; 32 for lane-interleaved shared-memory arrays).
// Returns det (<= 0 flags an inverted element, geometry.cpp:67-69).
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
template <bool GENERAL, int DS = 1, int CS = 1, typename T = double>
__device__ __forceinline__ T point_block(const double* __restrict__ dp, T xi1, T xi2, T xi3, T w, const double* cp,
                                         T M[16]) {
  T cf[3][3];
  const T det = jacobian_cofactors<DS, T>(dp, xi1, xi2, xi3, cf);
  block_from_cofactors<GENERAL, CS, T>(cf, det, w, w * rcp_rn(det), cp, M);
  return det;
}

// ---- TMA bulk copies global -> shared completing on an mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- asynchronous global -> shared copies (cp.async, SASS LDGSTS) ----
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- TMA bulk store (cp.async.bulk, SASS UBLKCP) from shared to global ----
__device__ __forceinline__ void bulk_store(double* gdst, const double* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Stores n doubles from shared memory to global with the TMA bulk engine:
// scalar head/tail where the global address is only 8-byte aligned.  The
// caller guarantees src and dst have the same address modulo 16.
__device__ __forceinline__ void bulk_store_doubles(double* gdst, const double* ssrc, int n) {
  int head = (reinterpret_cast<uintptr_t>(gdst) & 15) ? 1 : 0;
  if (head) gdst[0] = ssrc[0];
  const int body = (n - head) & ~1;
  if (body > 0) bulk_store(gdst + head, ssrc + head, static_cast<unsigned>(body) * 8u);
  if (head + body < n) gdst[n - 1] = ssrc[n - 1];
}

// Stores one entry of K: FP64, or rounded to FP32 for the FP32 output variant.
__device__ __forceinline__ void store_out(const LaunchArgs& a, int64_t idx, double v) {
  if (a.out32)
    a.out32[idx] = static_cast<float>(v);
  else
    a.out[idx] = v;
}

// FP32 variant of bulk_store_doubles: scalar head / tail where the global
// address is not 16-byte aligned; src and dst agree modulo 16 bytes.
__device__ __forceinline__ void bulk_store_floats(float* gdst, const float* ssrc, int n) {
  int head = static_cast<int>(((16 - (reinterpret_cast<uintptr_t>(gdst) & 15)) & 15) / 4);
  head = head < n ? head : n;
  for (int i = 0; i < head; ++i) gdst[i] = ssrc[i];
  const int body = (n - head) & ~3;
  if (body > 0) bulk_store(reinterpret_cast<double*>(gdst + head), reinterpret_cast<const double*>(ssrc + head),
                           static_cast<unsigned>(body) * 4u);
  for (int i = head + body; i < n; ++i) gdst[i] = ssrc[i];
}

__device__ __forceinline__ void flag_inverted(unsigned long long* bad, int64_t gid) {
  atomicMin(bad, static_cast<unsigned long long>(gid));
}

// D = A(8x4) * B(4x8) + D, FP64 tensor core (SASS DMMA.8x8x4).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// d0,d1 = D[lane/4][2*(lane%4) + {0,1}].
// Not volatile: the MMA is a pure function of its operands, so the compiler
// may schedule independent MMAs and their operand arithmetic freely.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace pib
