// C-ABI implementation: contexts, per-p table upload, strategy dispatch,
// error reporting and the host-buffer streaming path.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "kernels_dense.cuh"
#include "kernels_elastic.cuh"
#include "kernels_p2.cuh"
#include "kernels_sumfact.cuh"
#include "sumfact_api.hpp"
#include "tc32_api.hpp"
#include "kernels_tc32.cuh"
#include "pi_internal.hpp"

using namespace pib;

struct CallRecord {
  const double* geom;
  int64_t ld, base, n;
};

// Completion of the context's work on one caller stream (pi_check waits on
// these events instead of the whole device).
struct StreamMark {
  cudaStream_t stream;
  cudaEvent_t done;
};

struct pi_context {
  int device = 0, p = 0, n_eq = 1, n_q = 0, n_shape = 0;
  int variant = PI_VARIANT_AUTO;
  int load_fusion = PI_LOAD_AUTO;  // pi_integrate_load strategy
  cudaStream_t stream = nullptr;
  std::vector<double> h_pts, h_w, h_phi;
  double *d_phi = nullptr, *d_pts = nullptr, *d_w = nullptr;
  double *d_xfrag = nullptr, *d_xplain = nullptr, *d_yline = nullptr, *d_tri = nullptr;
  bool tensor_ok = false;
  // FP32 variant on tcgen05 (kernels_tc32.cuh), p = 3..7 scalar forms
  bool tc_ok = false;
  float *d_tc_bhi = nullptr, *d_tc_blo = nullptr, *d_tc_xg = nullptr, *d_tc_y = nullptr;
  double* d_tc_z = nullptr;
  int sf_ntps = 0;          // row pitch of d_xplain
  bool p2_ok = false;       // p = 2 register-dense kernel available
  int p2_ctas[3] = {0, 0, 0};  // persistent grid per p2_lane_kernel instantiation
  int p2_ctas_f[3] = {0, 0, 0};  // ... and per FP32-arithmetic instantiation
  int p2_ctas_l[3] = {0, 0, 0};  // ... and per fused-load-vector instantiation
  // per-context rule / shape tables of the p <= 2 register kernels, passed by
  // value with every launch (kernel parameter space)
  std::unique_ptr<P2Tables> p2tab;
  std::unique_ptr<E1Tables> e1tab;
  std::unique_ptr<E2Tables> e2tab;
  int e1_ctas = 0;             // persistent grid of p1_elastic_lane_kernel
  int e2_ctas = 0;             // persistent grid of p2_elastic_warp_kernel
  int e3_ctas = 0;             // persistent grid of p3_elastic_cta_kernel
  double* d_pts4 = nullptr; // rule as [n_q][xi1, xi2, xi3, w]
  unsigned long long* d_bad = nullptr;  // [0] lowest inverted element id, [1] lowest invalid material id
  std::vector<CallRecord> calls;
  std::vector<StreamMark> marks;
  // host streaming path
  cudaStream_t hs[2] = {nullptr, nullptr};
  double* hbuf = nullptr;
  size_t hbuf_bytes = 0;
};

namespace {

pi_status cuda_fail(pi_error_info* err, cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    // out of device memory is a capacity problem of the request, not a CUDA
    // failure (CapacityError, errors.hpp:16); the error is not sticky
    cudaGetLastError();
    if (err) err->cuda_error = static_cast<int>(e);
    return set_error(err, PI_E_CAPACITY, "%s: device memory exhausted", what);
  }
  if (err) err->cuda_error = static_cast<int>(e);
  return set_error(err, PI_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// lame_parameters' checks (coefficients.cpp:23-32).
pi_status check_material_host(double young, double nu, int64_t element, pi_error_info* err) {
  const char* why = nullptr;
  if (!(young > 0.0))
    why = "material: Young modulus must be positive";
  else if (!(nu > -1.0) || nu > 0.5)
    why = "material: Poisson ratio must lie in (-1, 0.5]";
  else if (nu == 0.5)
    why = "material: nu = 0.5 (incompressible) has no finite Lame lambda";
  if (!why) return PI_OK;
  pi_status st = set_error(err, PI_E_DOMAIN, "%s (element %lld)", why, (long long)element);
  if (err) err->element = element;
  return st;
}

#define PI_CUDA(call, what)                                   \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(err, e_, what);   \
  } while (0)

// Structure-of-arrays transpose for the host path: AoS [n][w] -> SoA [w][ld].
__global__ void aos_to_soa_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t n, int w,
                                  int64_t ld) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  const int64_t e = i / w;
  const int c = static_cast<int>(i % w);
  out[c * ld + e] = in[i];
}

template <typename T>
pi_status upload(T** dst, const std::vector<T>& src, pi_error_info* err) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(sizeof(T), src.size() * sizeof(T)));
  if (e == cudaSuccess && !src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e == cudaSuccess ? PI_OK : cuda_fail(err, e, "upload per-p tables");
}

// Records the completion of the context's latest work on stream s.
pi_status mark_stream(pi_context* ctx, cudaStream_t s, pi_error_info* err) {
  if (s == ctx->stream) return PI_OK;  // pi_check synchronises the context's own stream directly
  for (auto& m : ctx->marks)
    if (m.stream == s) {
      PI_CUDA(cudaEventRecord(m.done, s), "record completion");
      return PI_OK;
    }
  if (ctx->marks.size() >= 64) {  // bound the table: wait for the oldest stream and forget it
    PI_CUDA(cudaEventSynchronize(ctx->marks.front().done), "completion wait");
    cudaEventDestroy(ctx->marks.front().done);
    ctx->marks.erase(ctx->marks.begin());
  }
  StreamMark m{s, nullptr};
  PI_CUDA(cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming), "completion event");
  PI_CUDA(cudaEventRecord(m.done, s), "record completion");
  ctx->marks.push_back(m);
  return PI_OK;
}

int resolve_variant(const pi_context* ctx) {
  if (ctx->variant == PI_VARIANT_TC32) return PI_VARIANT_SUMFACT;  // FP64 calls: the DMMA kernels
  if (ctx->variant != PI_VARIANT_AUTO) return ctx->variant;
  if ((ctx->n_eq == 1 && ctx->p <= 2) || (ctx->n_eq == 3 && ctx->p <= 3)) return PI_VARIANT_DENSE;
  return ctx->tensor_ok ? PI_VARIANT_SUMFACT : PI_VARIANT_DENSE;
}

}  // namespace

extern "C" {

const char* pi_version(void) { return "prism_b200 0.1 (sm_100a)"; }

const char* pi_status_name(pi_status s) {
  static const char* names[] = {"ok",      "config",          "domain",   "unsupported_degree", "inverted_element",
                                "capacity", "shared_memory_exhausted", "contract_violation", "io", "cuda"};
  return (s >= 0 && s <= PI_E_CUDA) ? names[s] : "unknown";
}

pi_status pi_context_create(int device, int p, int n_eq, int n_q, int n_shape, const double* points,
                            const double* weights, const double* shape_table, pi_context** out,
                            pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!out) return set_error(err, PI_E_CONTRACT, "pi_context_create: out is NULL");
  *out = nullptr;
  if (p < 1 || p > kMaxP)
    return set_error(err, PI_E_DOMAIN, "approximation order p=%d outside supported range [1, 7]", p);
  if (n_eq != 1 && n_eq != 3)
    return set_error(err, PI_E_CONFIG, "n_eq=%d: supported systems are n_eq = 1 (scalar) and 3 (elasticity)", n_eq);
  const int nsh = shape_count(p), nq = quad_count(p);
  if ((points || weights || shape_table) && !(points && weights && shape_table))
    return set_error(err, PI_E_CONTRACT, "pi_context_create: pass all of points/weights/shape_table or none");
  if (points && (n_q != nq || n_shape != nsh))
    return set_error(err, PI_E_CONFIG, "integrator: tables have n_q=%d n_shape=%d, p=%d needs %d and %d", n_q,
                     n_shape, p, nq, nsh);

  auto* ctx = new pi_context();
  ctx->device = device;
  ctx->p = p;
  ctx->n_eq = n_eq;
  ctx->n_q = nq;
  ctx->n_shape = nsh;
  ctx->h_pts.resize(3 * nq);
  ctx->h_w.resize(nq);
  ctx->h_phi.resize(static_cast<size_t>(nq) * 4 * nsh);
  if (points) {
    std::memcpy(ctx->h_pts.data(), points, sizeof(double) * 3 * nq);
    std::memcpy(ctx->h_w.data(), weights, sizeof(double) * nq);
    std::memcpy(ctx->h_phi.data(), shape_table, sizeof(double) * ctx->h_phi.size());
  } else {
    prism_quadrature(p, ctx->h_pts.data(), ctx->h_w.data());
    for (int q = 0; q < nq; ++q) shape_values(p, &ctx->h_pts[3 * q], &ctx->h_phi[static_cast<size_t>(q) * 4 * nsh]);
  }

  pi_status st = PI_OK;
  auto fail = [&](pi_status s) {
    pi_context_destroy(ctx);
    return s;
  };
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return fail(cuda_fail(err, ce, "cudaSetDevice"));
  ce = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return fail(cuda_fail(err, ce, "cudaStreamCreate"));
  if ((st = upload(&ctx->d_phi, ctx->h_phi, err)) != PI_OK) return fail(st);
  if ((st = upload(&ctx->d_pts, ctx->h_pts, err)) != PI_OK) return fail(st);
  {
    std::vector<double> wpad(ctx->h_w);  // padded to 16 bytes for TMA bulk copies
    wpad.resize((wpad.size() + 1) / 2 * 2, 0.0);
    if ((st = upload(&ctx->d_w, wpad, err)) != PI_OK) return fail(st);
  }
  ce = cudaMalloc(&ctx->d_bad, 2 * sizeof(unsigned long long));
  if (ce != cudaSuccess) return fail(cuda_fail(err, ce, "cudaMalloc"));
  ce = cudaMemset(ctx->d_bad, 0xff, 2 * sizeof(unsigned long long));
  if (ce != cudaSuccess) return fail(cuda_fail(err, ce, "cudaMemset"));
  for (auto k : {load_vector_sf_kernel<1>, load_vector_sf_kernel<2>, load_vector_sf_kernel<3>, load_vector_sf_kernel<4>,
                 load_vector_sf_kernel<5>, load_vector_sf_kernel<6>, load_vector_sf_kernel<7>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);  // >= load_sf_smem at every p

  // The kernels skip the basis' structural zeros (BasisPattern): the table
  // must hold exact zeros there, as tabulate_shapes does.
  for (int q = 0; q < nq; ++q)
    for (int k = 1; k < 4; ++k)
      for (int dof = 0; dof < nsh; ++dof) {
        const int t = dof / (p + 1), a = dof % (p + 1);
        int d = 0, r = t;
        while (r > d) r -= ++d;
        const bool nz = k == 1 ? r > 0 : k == 2 ? (d - r) > 0 : a > 0;
        if (!nz && ctx->h_phi[(static_cast<size_t>(q) * 4 + k) * nsh + dof] != 0.0)
          return fail(set_error(err, PI_E_CONFIG,
                                "shape table entry (q=%d, d=%d, dof=%d) is not the reference basis' structural zero",
                                q, k, dof));
      }
  if (sumfact_supported(p, n_eq)) {
    SumFactHostTables tb;
    const bool ok = sumfact_build(p, n_eq, ctx->h_pts.data(), ctx->h_phi.data(), nq, nsh, tb);
    ctx->tensor_ok = ok;
    ctx->sf_ntps = tb.ntps;
    if (ok) {
      if ((st = upload(&ctx->d_xfrag, tb.xfrag, err)) != PI_OK) return fail(st);
      if ((st = upload(&ctx->d_xplain, tb.xplain, err)) != PI_OK) return fail(st);
      if ((st = upload(&ctx->d_yline, tb.yline, err)) != PI_OK) return fail(st);
      if ((st = upload(&ctx->d_tri, tb.tri, err)) != PI_OK) return fail(st);
      sumfact_set_attrs(p, n_eq);
      if (tc32_supported(p, n_eq)) {
        Tc32HostTables tt;
        if (tc32_build(p, ctx->h_pts.data(), ctx->h_phi.data(), nq, nsh, tt)) {
          if ((st = upload(&ctx->d_tc_bhi, tt.bhi, err)) != PI_OK) return fail(st);
          if ((st = upload(&ctx->d_tc_blo, tt.blo, err)) != PI_OK) return fail(st);
          if ((st = upload(&ctx->d_tc_xg, tt.xg, err)) != PI_OK) return fail(st);
          if ((st = upload(&ctx->d_tc_y, tt.yline, err)) != PI_OK) return fail(st);
          if ((st = upload(&ctx->d_tc_z, tt.z, err)) != PI_OK) return fail(st);
          tc32_attrs(p);
          ctx->tc_ok = true;
        }
      }
    } else {
      return fail(set_error(err, PI_E_CONFIG,
                            "shape table / rule are not the tensor-product prism basis the kernels factorise"));
    }
  }
  if (p == 2 && n_eq == 1) {
    ctx->p2tab = std::make_unique<P2Tables>();
    std::memcpy(ctx->p2tab->phi, ctx->h_phi.data(), sizeof(ctx->p2tab->phi));
    for (int i = 0; i < kP2NQ * 4 * kP2NSH; ++i) ctx->p2tab->phif[i] = static_cast<float>(ctx->h_phi[i]);
  }
  if (p == 2 && n_eq == 3) {
    ctx->e2tab = std::make_unique<E2Tables>();
    std::memcpy(ctx->e2tab->phi, ctx->h_phi.data(), sizeof(ctx->e2tab->phi));
  }
  if (p == 1 && n_eq == 3) {
    ctx->e1tab = std::make_unique<E1Tables>();
    std::memcpy(ctx->e1tab->phi, ctx->h_phi.data(), sizeof(ctx->e1tab->phi));
  }
  for (int q = 0; q < nq && p <= 2; ++q)
    for (int c = 0; c < 4; ++c) {
      const double v = c < 3 ? ctx->h_pts[3 * q + c] : ctx->h_w[q];
      if (ctx->p2tab) ctx->p2tab->pts[4 * q + c] = v;
      if (ctx->e2tab) ctx->e2tab->pts[4 * q + c] = v;
      if (ctx->e1tab) ctx->e1tab->pts[4 * q + c] = v;
    }
  if (p == 3 && n_eq == 3) {
    int per_sm = 0, sms = 0;
#ifdef PI_E3_CTA  // A/B: the scalar block-update kernel
    cudaFuncSetAttribute(p3_elastic_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(E3Smem::BYTES));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p3_elastic_cta_kernel, kE3Threads, E3Smem::BYTES);
#else
    cudaFuncSetAttribute(p3_elastic_mma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(EMma<3>::BYTES));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p3_elastic_mma_kernel<3>, EMma<3>::NTHREADS, EMma<3>::BYTES);
#endif
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->e3_ctas = std::max(1, per_sm) * sms;
  }
  if (p == 2 && n_eq == 3) {
    int per_sm = 0, sms = 0;
#ifndef PI_E2_MMA
    cudaFuncSetAttribute(p2_elastic_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kE2SmemBytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p2_elastic_warp_kernel, 32 * kE2Warps, kE2SmemBytes);
#else
    cudaFuncSetAttribute(p3_elastic_mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(EMma<2>::BYTES));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p3_elastic_mma_kernel<2>, EMma<2>::NTHREADS, EMma<2>::BYTES);
#endif
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->e2_ctas = std::max(1, per_sm) * sms;
  }
  if (p == 1 && n_eq == 3) {
    cudaFuncSetAttribute(p1_elastic_lane_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(E1Smem::BYTES));
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p1_elastic_lane_kernel, 32 * kE1Warps, E1Smem::BYTES);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->e1_ctas = std::max(1, per_sm) * sms;
  }
  if (p <= 2) {
    std::vector<double> p4(4 * nq);
    for (int q = 0; q < nq; ++q) {
      p4[4 * q] = ctx->h_pts[3 * q];
      p4[4 * q + 1] = ctx->h_pts[3 * q + 1];
      p4[4 * q + 2] = ctx->h_pts[3 * q + 2];
      p4[4 * q + 3] = ctx->h_w[q];
    }
    if ((st = upload(&ctx->d_pts4, p4, err)) != PI_OK) return fail(st);
  }
  if (p == 2 && n_eq == 1) {
    cudaFuncSetAttribute(p2_lane_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<false, true>::SMEM_BYTES));
    cudaFuncSetAttribute(p2_lane_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, true>::SMEM_BYTES));
    cudaFuncSetAttribute(p2_lane_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, false>::SMEM_BYTES));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    auto ctas = [&](auto kern, int threads, size_t smem) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      return std::max(1, per_sm) * sms;
    };
    ctx->p2_ctas[0] = ctas(p2_lane_kernel<false, true>, P2Cfg<false, true>::NTHREADS, P2Cfg<false, true>::SMEM_BYTES);
    ctx->p2_ctas[1] = ctas(p2_lane_kernel<true, true>, P2Cfg<true, true>::NTHREADS, P2Cfg<true, true>::SMEM_BYTES);
    ctx->p2_ctas[2] = ctas(p2_lane_kernel<true, false>, P2Cfg<true, false>::NTHREADS, P2Cfg<true, false>::SMEM_BYTES);
    cudaFuncSetAttribute(p2_lane_kernel<false, true, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<false, true>::SMEM_BYTES));
    cudaFuncSetAttribute(p2_lane_kernel<true, true, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, true>::SMEM_BYTES));
    cudaFuncSetAttribute(p2_lane_kernel<true, false, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, false>::SMEM_BYTES));
    ctx->p2_ctas_f[0] = ctas(p2_lane_kernel<false, true, float>, P2Cfg<false, true>::NTHREADS, P2Cfg<false, true>::SMEM_BYTES);
    ctx->p2_ctas_f[1] = ctas(p2_lane_kernel<true, true, float>, P2Cfg<true, true>::NTHREADS, P2Cfg<true, true>::SMEM_BYTES);
    ctx->p2_ctas_f[2] = ctas(p2_lane_kernel<true, false, float>, P2Cfg<true, false>::NTHREADS, P2Cfg<true, false>::SMEM_BYTES);
    cudaFuncSetAttribute(p2_lane_kernel<false, true, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<false, true>::SMEM_BYTES_LOAD));
    cudaFuncSetAttribute(p2_lane_kernel<true, true, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, true>::SMEM_BYTES_LOAD));
    cudaFuncSetAttribute(p2_lane_kernel<true, false, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(P2Cfg<true, false>::SMEM_BYTES_LOAD));
    ctx->p2_ctas_l[0] = ctas(p2_lane_kernel<false, true, double, true>, P2Cfg<false, true>::NTHREADS,
                             P2Cfg<false, true>::SMEM_BYTES_LOAD);
    ctx->p2_ctas_l[1] = ctas(p2_lane_kernel<true, true, double, true>, P2Cfg<true, true>::NTHREADS,
                             P2Cfg<true, true>::SMEM_BYTES_LOAD);
    ctx->p2_ctas_l[2] = ctas(p2_lane_kernel<true, false, double, true>, P2Cfg<true, false>::NTHREADS,
                             P2Cfg<true, false>::SMEM_BYTES_LOAD);
    ctx->p2_ok = true;
  }
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return fail(cuda_fail(err, ce, "context setup"));
  *out = ctx;
  return PI_OK;
}

pi_status pi_context_destroy(pi_context* ctx) {
  if (!ctx) return PI_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& s : ctx->hs)
    if (s) cudaStreamDestroy(s);
  cudaFree(ctx->d_phi);
  cudaFree(ctx->d_pts);
  cudaFree(ctx->d_w);
  cudaFree(ctx->d_xfrag);
  cudaFree(ctx->d_xplain);
  cudaFree(ctx->d_yline);
  cudaFree(ctx->d_tri);
  cudaFree(ctx->d_tc_bhi);
  cudaFree(ctx->d_tc_blo);
  cudaFree(ctx->d_tc_xg);
  cudaFree(ctx->d_tc_y);
  cudaFree(ctx->d_tc_z);
  cudaFree(ctx->d_bad);
  cudaFree(ctx->d_pts4);
  for (auto& m : ctx->marks) cudaEventDestroy(m.done);
  if (ctx->hbuf) cudaFree(ctx->hbuf);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PI_OK;
}

pi_status pi_context_set_variant(pi_context* ctx, int variant, pi_error_info* err) {
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if (variant < PI_VARIANT_AUTO || variant > PI_VARIANT_TC32)
    return set_error(err, PI_E_CONFIG, "unknown variant %d", variant);
  if (variant == PI_VARIANT_TC32 && !ctx->tc_ok)
    return set_error(err, PI_E_CONFIG, "the tcgen05 FP32 kernels need a scalar weak form at p = 3..7");
  if (variant == PI_VARIANT_SUMFACT && !ctx->tensor_ok)
    return set_error(err, PI_E_CONFIG, "sum factorisation needs p >= 2 and the tensor-product tables");
  if (variant == PI_VARIANT_DENSE && ctx->p > (ctx->n_eq == 3 ? 3 : 2))
    return set_error(err, PI_E_CONFIG, "dense variant is built for scalar forms at p <= 2 and elasticity at p <= 3");
  ctx->variant = variant;
  return PI_OK;
}

int pi_context_variant(const pi_context* ctx, int coeff_mode) {
  (void)coeff_mode;
  return ctx ? resolve_variant(ctx) : -1;
}

void* pi_context_stream(pi_context* ctx) { return ctx ? ctx->stream : nullptr; }

}  // extern "C"

namespace {
// pi_integrate / pi_integrate_f32: exactly one of out, out32 is non-NULL.
pi_status integrate_impl(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                         int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld, double* out,
                         float* out32, int out_layout, int64_t ld_out, void* stream, pi_error_info* err,
                         const double* f = nullptr, double f_const = 0.0, double* fout = nullptr) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if (n_elem < 0) return set_error(err, PI_E_CONTRACT, "n_elem < 0");
  if (n_elem == 0) return PI_OK;
  if (!geom || (!out && !out32)) return set_error(err, PI_E_CONTRACT, "geometry/output buffers must be non-NULL");
  if (geom_ld < n_elem) return set_error(err, PI_E_CONTRACT, "geom_ld (%lld) < n_elem (%lld)", (long long)geom_ld,
                                         (long long)n_elem);
  if (out_layout != PI_OUT_CANONICAL && out_layout != PI_OUT_SOA)
    return set_error(err, PI_E_CONFIG, "unknown output layout %d", out_layout);
  if (out_layout == PI_OUT_SOA && ld_out < n_elem) return set_error(err, PI_E_CONTRACT, "ld_out < n_elem");
  LaunchArgs a{};
  a.n_elem = n_elem;
  a.element_id_base = element_id_base;
  a.geom = geom;
  a.geom_ld = geom_ld;
  a.out = out;
  a.out32 = out32;
  a.out_layout = out_layout;
  a.ld_out = ld_out;
  a.bad = ctx->d_bad;
  a.bad_mat = ctx->d_bad + 1;
  a.fout = fout;
  a.fsrc = f;
  a.fconst = f_const;
  const int ne = ctx->n_eq, ncoef = 16 * ne * ne;
  if (fout && (ne != 1 || out32))
    return set_error(err, PI_E_CONFIG, "fused load vectors need a scalar weak form (n_eq = 1) and FP64 output");
  bool general = false, symmetric = true;
  int form = kFormLaplace;
  switch (coeff_mode) {
    case PI_COEFF_LAPLACE:
      if (ne != 1) return set_error(err, PI_E_CONFIG, "Laplace coefficients need n_eq = 1 (context has %d)", ne);
      break;
    case PI_COEFF_UNIFORM:
      if (!coeff) return set_error(err, PI_E_CONTRACT, "uniform coefficient tensor is NULL");
      std::memcpy(a.cu, coeff, sizeof(double) * ncoef);
      general = true;
      form = kFormGeneral;
      // major symmetry c[ie][je][k][l] == c[je][ie][l][k] makes K symmetric
      for (int ie = 0; ie < ne; ++ie)
        for (int je = 0; je < ne; ++je)
          for (int k = 0; k < 4; ++k)
            for (int l = 0; l < 4; ++l)
              symmetric = symmetric && a.cu[((ie * ne + je) * 4 + k) * 4 + l] == a.cu[((je * ne + ie) * 4 + l) * 4 + k];
      break;
    case PI_COEFF_PER_ELEMENT:
      if (!coeff || coeff_ld < n_elem) return set_error(err, PI_E_CONTRACT, "per-element coefficients: bad buffer/ld");
      a.coeff = coeff;
      a.coeff_ld = coeff_ld;
      general = true;
      symmetric = false;
      form = kFormGeneral;
      break;
    case PI_COEFF_ELASTICITY:
    case PI_COEFF_ELASTICITY_UNIFORM:
      if (ne != 3) return set_error(err, PI_E_CONFIG, "elasticity needs n_eq = 3 (context has %d)", ne);
      if (!coeff) return set_error(err, PI_E_CONTRACT, "elasticity material buffer is NULL");
      if (coeff_mode == PI_COEFF_ELASTICITY) {
        if (coeff_ld < n_elem) return set_error(err, PI_E_CONTRACT, "per-element material: coeff_ld < n_elem");
        a.coeff = coeff;
        a.coeff_ld = coeff_ld;
      } else {
        const pi_status ms = check_material_host(coeff[0], coeff[1], -1, err);
        if (ms != PI_OK) return ms;
        a.cu[0] = coeff[0];
        a.cu[1] = coeff[1];
      }
      form = kFormElasticity;
      break;
    default:
      return set_error(err, PI_E_CONFIG, "unknown coefficient mode %d", coeff_mode);
  }
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  PI_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int v = resolve_variant(ctx);
  const bool e1_lane = ne == 3 && ctx->p == 1 && v == PI_VARIANT_DENSE && form == kFormElasticity;
  const bool e2_warp = ne == 3 && ctx->p == 2 && v == PI_VARIANT_DENSE && form == kFormElasticity;
  const bool e3_cta = ne == 3 && ctx->p == 3 && v == PI_VARIANT_DENSE && form == kFormElasticity;
  if (e3_cta) {
    DenseTables t{ctx->d_phi, ctx->d_pts, ctx->d_w};
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n_elem, ctx->e3_ctas));
#ifdef PI_E3_CTA
    p3_elastic_cta_kernel<<<grid, kE3Threads, E3Smem::BYTES, s>>>(a, t);
#else
    p3_elastic_mma_kernel<3><<<grid, EMma<3>::NTHREADS, EMma<3>::BYTES, s>>>(a, t);
#endif
  } else if (e2_warp) {
#ifndef PI_E2_MMA
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n_elem + kE2Warps - 1) / kE2Warps, ctx->e2_ctas));
    p2_elastic_warp_kernel<<<grid, 32 * kE2Warps, kE2SmemBytes, s>>>(a, *ctx->e2tab);
#else
    DenseTables t{ctx->d_phi, ctx->d_pts, ctx->d_w};
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n_elem, ctx->e2_ctas));
    p3_elastic_mma_kernel<2><<<grid, EMma<2>::NTHREADS, EMma<2>::BYTES, s>>>(a, t);
#endif
  } else if (e1_lane) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n_elem + 31) / 32, ctx->e1_ctas));
    p1_elastic_lane_kernel<<<grid, 32 * kE1Warps, E1Smem::BYTES, s>>>(a, *ctx->e1tab);
  } else if (ctx->p == 2 && ne == 1 && v == PI_VARIANT_DENSE) {
    const int64_t groups = (n_elem + 31) / 32;
    const int which = !general ? 0 : (symmetric ? 1 : 2);
    const P2Tables& tb = *ctx->p2tab;
    if (out32) {
      // FP32 output variant: FP32 arithmetic too (the table in FP32, M rounded
      // after the FP64 point block); bound 5e-5
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>(groups, ctx->p2_ctas_f[which]));
      if (!general)
        p2_lane_kernel<false, true, float><<<grid, P2Cfg<false, true>::NTHREADS, P2Cfg<false, true>::SMEM_BYTES, s>>>(a, tb);
      else if (symmetric)
        p2_lane_kernel<true, true, float><<<grid, P2Cfg<true, true>::NTHREADS, P2Cfg<true, true>::SMEM_BYTES, s>>>(a, tb);
      else
        p2_lane_kernel<true, false, float><<<grid, P2Cfg<true, false>::NTHREADS, P2Cfg<true, false>::SMEM_BYTES, s>>>(a, tb);
    } else if (fout) {
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>(groups, ctx->p2_ctas_l[which]));
      if (!general)
        p2_lane_kernel<false, true, double, true>
            <<<grid, P2Cfg<false, true>::NTHREADS, P2Cfg<false, true>::SMEM_BYTES_LOAD, s>>>(a, tb);
      else if (symmetric)
        p2_lane_kernel<true, true, double, true>
            <<<grid, P2Cfg<true, true>::NTHREADS, P2Cfg<true, true>::SMEM_BYTES_LOAD, s>>>(a, tb);
      else
        p2_lane_kernel<true, false, double, true>
            <<<grid, P2Cfg<true, false>::NTHREADS, P2Cfg<true, false>::SMEM_BYTES_LOAD, s>>>(a, tb);
    } else {
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>(groups, ctx->p2_ctas[which]));
      if (!general)
        p2_lane_kernel<false, true><<<grid, P2Cfg<false, true>::NTHREADS, P2Cfg<false, true>::SMEM_BYTES, s>>>(a, tb);
      else if (symmetric)
        p2_lane_kernel<true, true><<<grid, P2Cfg<true, true>::NTHREADS, P2Cfg<true, true>::SMEM_BYTES, s>>>(a, tb);
      else
        p2_lane_kernel<true, false><<<grid, P2Cfg<true, false>::NTHREADS, P2Cfg<true, false>::SMEM_BYTES, s>>>(a, tb);
    }
  } else if (v == PI_VARIANT_DENSE && ne == 1) {
    DenseTables t{ctx->d_phi, ctx->d_pts, ctx->d_w};
    constexpr int TG = p1_threads<true>(), TL = p1_threads<false>();
    const unsigned gg = static_cast<unsigned>((n_elem + TG - 1) / TG), gl = static_cast<unsigned>((n_elem + TL - 1) / TL);
    if (general && out32)
      p1_thread_kernel<true, false, float><<<gg, TG, 0, s>>>(a, t);
    else if (out32)
      p1_thread_kernel<false, false, float><<<gl, TL, 0, s>>>(a, t);
    else if (general && fout)
      p1_thread_kernel<true, true><<<gg, TG, 0, s>>>(a, t);
    else if (general)
      p1_thread_kernel<true><<<gg, TG, 0, s>>>(a, t);
    else if (fout)
      p1_thread_kernel<false, true><<<gl, TL, 0, s>>>(a, t);
    else
      p1_thread_kernel<false><<<gl, TL, 0, s>>>(a, t);
  } else if (out32 && ctx->variant == PI_VARIANT_TC32 && form != kFormElasticity) {
    // FP32 output on the tcgen05 tensor cores (3xTF32, kernels_tc32.cuh); opt-in:
    // measured slower than the FP64 DMMA kernels rounding at the store
    Tc32Tables t{ctx->d_tc_bhi, ctx->d_tc_blo, ctx->d_tc_xg, ctx->d_tc_y, ctx->d_tri, ctx->d_tc_z, ctx->d_w};
    tc32_launch(ctx->p, general, a, t, s);
  } else {
    SumFactTables t{ctx->d_xfrag, ctx->d_xplain, ctx->d_yline, ctx->d_tri, ctx->d_w};
    sumfact_launch(ctx->p, ne, form, symmetric, a, t, s);
  }
  PI_CUDA(cudaGetLastError(), "kernel launch");
  ctx->calls.push_back({geom, geom_ld, element_id_base, n_elem});
  if (ctx->calls.size() > 4096) ctx->calls.erase(ctx->calls.begin(), ctx->calls.begin() + 2048);
  return mark_stream(ctx, s, err);
}
}  // namespace

extern "C" {

pi_status pi_integrate(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                       int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld, double* out,
                       int out_layout, int64_t ld_out, void* stream, pi_error_info* err) {
  if (!out && n_elem > 0) {
    if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
    return set_error(err, PI_E_CONTRACT, "geometry/output buffers must be non-NULL");
  }
  return integrate_impl(ctx, n_elem, element_id_base, geom, geom_ld, coeff_mode, coeff, coeff_ld, out, nullptr,
                        out_layout, ld_out, stream, err);
}

pi_status pi_integrate_f32(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                           int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld, float* out,
                           int out_layout, int64_t ld_out, void* stream, pi_error_info* err) {
  if (!out && n_elem > 0) {
    if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
    return set_error(err, PI_E_CONTRACT, "geometry/output buffers must be non-NULL");
  }
  return integrate_impl(ctx, n_elem, element_id_base, geom, geom_ld, coeff_mode, coeff, coeff_ld, nullptr, out,
                        out_layout, ld_out, stream, err);
}

pi_status pi_integrate_load(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                            int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld, double* out,
                            int out_layout, int64_t ld_out, const double* f, double f_const, double* load_out,
                            void* stream, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if ((!out || !load_out) && n_elem > 0)
    return set_error(err, PI_E_CONTRACT, "stiffness and load-vector output buffers must be non-NULL");
  if (ctx->n_eq != 1)
    return set_error(err, PI_E_CONFIG, "load vectors need a scalar weak form (n_eq = 1; context has %d)", ctx->n_eq);
  // Fused (the stiffness kernel also forms F from its own Jacobians) or a
  // second, sum-factorised launch on the same stream.  Measured (bench.py
  // load_vectors): fusing pays where K is cheap (p = 1: the geometry is read
  // once); at p >= 2 the extra producer work on the stiffness kernel's
  // critical path costs more (7-21 %) than re-reading 144 B of geometry.
  const bool fuse = ctx->load_fusion == PI_LOAD_FUSED || (ctx->load_fusion == PI_LOAD_AUTO && ctx->p == 1);
  if (fuse)
    return integrate_impl(ctx, n_elem, element_id_base, geom, geom_ld, coeff_mode, coeff, coeff_ld, out, nullptr,
                          out_layout, ld_out, stream, err, f, f_const, load_out);
  const pi_status st = integrate_impl(ctx, n_elem, element_id_base, geom, geom_ld, coeff_mode, coeff, coeff_ld, out,
                                      nullptr, out_layout, ld_out, stream, err);
  if (st != PI_OK || n_elem == 0) return st;
  return pi_load_vectors(ctx, n_elem, element_id_base, geom, geom_ld, f, f_const, load_out, stream, err);
}

pi_status pi_context_set_load_fusion(pi_context* ctx, int mode, pi_error_info* err) {
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if (mode < PI_LOAD_AUTO || mode > PI_LOAD_SEPARATE) return set_error(err, PI_E_CONFIG, "unknown load mode %d", mode);
  ctx->load_fusion = mode;
  return PI_OK;
}

pi_status pi_load_vectors(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                          int64_t geom_ld, const double* f, double f_const, double* out, void* stream,
                          pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if (n_elem <= 0) return n_elem == 0 ? PI_OK : set_error(err, PI_E_CONTRACT, "n_elem < 0");
  if (!geom || !out || geom_ld < n_elem) return set_error(err, PI_E_CONTRACT, "bad geometry/output buffers");
  LaunchArgs a{};
  a.n_elem = n_elem;
  a.element_id_base = element_id_base;
  a.geom = geom;
  a.geom_ld = geom_ld;
  a.out = out;
  a.bad = ctx->d_bad;
  a.bad_mat = ctx->d_bad + 1;
  DenseTables t{ctx->d_phi, ctx->d_pts, ctx->d_w};
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  PI_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (ctx->tensor_ok) {  // sum-factorised: X_2 and P tables instead of the dense phi table
    const int ns = ctx->n_q / (ctx->p + 1);
    LoadSfTables lt{ctx->d_tri, ctx->d_yline, ctx->d_xplain, ctx->d_w, ns, ctx->p + 1, ctx->p + 1,
                    ctx->n_shape / (ctx->p + 1), ctx->sf_ntps};
    const size_t smem = load_sf_smem(ns, ctx->p + 1);
    const int epc = load_sf_elems(ns, ctx->p + 1);
    const unsigned grid = static_cast<unsigned>((n_elem + epc - 1) / epc);
    switch (ctx->p) {
#define PIB_LOAD_CASE(P) \
  case P: load_vector_sf_kernel<P><<<grid, kLoadSfThreads, smem, s>>>(a, lt, f, f_const); break;
      PIB_LOAD_CASE(1) PIB_LOAD_CASE(2) PIB_LOAD_CASE(3) PIB_LOAD_CASE(4) PIB_LOAD_CASE(5) PIB_LOAD_CASE(6)
      PIB_LOAD_CASE(7)
#undef PIB_LOAD_CASE
    }
  } else if (ctx->p == 1 && ctx->n_shape == 6 && ctx->n_q == 6) {
    const unsigned grid = static_cast<unsigned>((n_elem + kLoadP1Threads - 1) / kLoadP1Threads);
    load_vector_p1_kernel<<<grid, kLoadP1Threads, 0, s>>>(a, t, f, f_const);
  } else {
    const unsigned grid = static_cast<unsigned>((n_elem + kLoadWarps - 1) / kLoadWarps);
    load_vector_kernel<<<grid, 32 * kLoadWarps, sizeof(double) * kLoadWarps * ctx->n_q, s>>>(a, t, ctx->n_q,
                                                                                              ctx->n_shape, f, f_const);
  }
  PI_CUDA(cudaGetLastError(), "load-vector launch");
  ctx->calls.push_back({geom, geom_ld, element_id_base, n_elem});
  return mark_stream(ctx, s, err);
}

namespace {
// Describes an inverted element like InvertedElementError (errors.cpp:33-41):
// the first failing rule point in rule order and its determinant.  g: AoS
// [6][3] geometry of the element, or NULL when it is no longer available.
pi_status report_inverted(pi_context* ctx, int64_t gid, const double* g, pi_error_info* err) {
  double xi[3] = {0, 0, 0}, det = 0.0;
  if (g)
    for (int q = 0; q < ctx->n_q; ++q) {
      double inv[9], d;
      if (!jacobian_terms(g, &ctx->h_pts[3 * q], d, inv)) {
        std::memcpy(xi, &ctx->h_pts[3 * q], sizeof xi);
        det = d;
        break;
      }
    }
  pi_status st = set_error(err, PI_E_INVERTED_ELEMENT, "inverted element %lld: det=%f at xi=(%f, %f, %f)",
                           (long long)gid, det, xi[0], xi[1], xi[2]);
  if (err) {
    err->element = gid;
    err->det = det;
    std::memcpy(err->xi, xi, sizeof xi);
  }
  return st;
}

// Waits for every stream the context launched on since the last check (its
// own stream and the recorded caller streams -- never the whole device),
// then reads and resets the error flags.  Returns the flags through bad[2].
pi_status drain(pi_context* ctx, unsigned long long bad[2], pi_error_info* err) {
  bad[0] = bad[1] = ~0ull;
  PI_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  PI_CUDA(cudaStreamSynchronize(ctx->stream), "stream synchronize");
  for (auto& m : ctx->marks) PI_CUDA(cudaEventSynchronize(m.done), "stream synchronize");
  for (auto& h : ctx->hs)
    if (h) PI_CUDA(cudaStreamSynchronize(h), "stream synchronize");
  PI_CUDA(cudaMemcpy(bad, ctx->d_bad, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "read error flags");
  if (bad[0] != ~0ull || bad[1] != ~0ull)
    PI_CUDA(cudaMemset(ctx->d_bad, 0xff, 2 * sizeof(unsigned long long)), "reset error flags");
  return PI_OK;
}

pi_status material_error(int64_t gid, pi_error_info* err) {
  pi_status st = set_error(err, PI_E_DOMAIN,
                           "material of element %lld: lame_parameters needs E > 0 and -1 < nu < 0.5", (long long)gid);
  if (err) err->element = gid;
  return st;
}
}  // namespace

pi_status pi_check(pi_context* ctx, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  unsigned long long bad[2];
  const pi_status ds = drain(ctx, bad, err);
  if (ds != PI_OK) return ds;
  if (bad[1] != ~0ull) {
    ctx->calls.clear();
    return material_error(static_cast<int64_t>(bad[1]), err);
  }
  if (bad[0] == ~0ull) {
    ctx->calls.clear();
    return PI_OK;
  }
  const int64_t gid = static_cast<int64_t>(bad[0]);
  double g[18];
  bool got = false;
  for (auto it = ctx->calls.rbegin(); it != ctx->calls.rend(); ++it) {
    if (gid < it->base || gid >= it->base + it->n) continue;
    const int64_t le = gid - it->base;
    got = true;
    for (int c = 0; c < 18; ++c)  // SoA [18][ld] -> AoS [6][3]
      if (cudaMemcpy(&g[c], it->geom + c * it->ld + le, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        got = false;
    break;
  }
  ctx->calls.clear();
  return report_inverted(ctx, gid, got ? g : nullptr, err);
}

namespace {
// pi_integrate_host / pi_integrate_host_load: f, load_out (host) != NULL also
// stream the load vectors (f per element, or f_const when f == NULL).
pi_status integrate_host_impl(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom_aos,
                              int coeff_mode, const double* coeff, double* out, int64_t chunk_elems,
                              pi_error_info* err, const double* f, double f_const, double* load_out) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctx) return set_error(err, PI_E_CONTRACT, "NULL context");
  if (n_elem <= 0) return n_elem == 0 ? PI_OK : set_error(err, PI_E_CONTRACT, "n_elem < 0");
  if (!geom_aos || !out) return set_error(err, PI_E_CONTRACT, "NULL host buffers");
  if ((coeff_mode == PI_COEFF_PER_ELEMENT || coeff_mode == PI_COEFF_ELASTICITY) && !coeff)
    return set_error(err, PI_E_CONTRACT, "per-element coefficient buffer is NULL");
  // Errors of earlier asynchronous calls on this context surface here first
  // (the header's contract), so this call's flags are its own.
  {
    const pi_status prev = pi_check(ctx, err);
    if (prev != PI_OK) return prev;
  }
  // run_batch validates every material before integrating (lame_parameters)
  if (coeff_mode == PI_COEFF_ELASTICITY)
    for (int64_t e = 0; e < n_elem; ++e) {
      const pi_status ms = check_material_host(coeff[2 * e], coeff[2 * e + 1], element_id_base + e, err);
      if (ms != PI_OK) return ms;
    }
  const int64_t dim = static_cast<int64_t>(ctx->n_shape) * ctx->n_eq;
  const int64_t kk = dim * dim;
  // per-element coefficient width: the tensor, or (E, nu) for elasticity
  const int cw = coeff_mode == PI_COEFF_PER_ELEMENT ? 16 * ctx->n_eq * ctx->n_eq
                                                    : coeff_mode == PI_COEFF_ELASTICITY ? 2 : 0;
  const int64_t nsh = ctx->n_shape;
  const int lw = load_out ? static_cast<int>(nsh) + 1 : 0;  // F and f per element
  const size_t per_elem = sizeof(double) * (kk + 2 * 18 + 2 * cw + lw);
  if (chunk_elems <= 0) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t budget = std::min<size_t>(free_b / 4, size_t(4) << 30);  // per slot
    chunk_elems = std::max<int64_t>(1, static_cast<int64_t>(budget / per_elem));
  }
  chunk_elems = std::min(chunk_elems, n_elem);
  const size_t slot_bytes = per_elem * chunk_elems;
  if (ctx->hbuf_bytes < 2 * slot_bytes) {
    if (ctx->hbuf) cudaFree(ctx->hbuf);
    ctx->hbuf = nullptr;
    ctx->hbuf_bytes = 0;
    PI_CUDA(cudaMalloc(&ctx->hbuf, 2 * slot_bytes), "allocate streaming buffers");
    ctx->hbuf_bytes = 2 * slot_bytes;
  }
  for (auto& s : ctx->hs)
    if (!s) PI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
  // Every exit waits for both slots' copies: no DMA into or out of the
  // caller's host buffers may still be pending when this call returns.
  auto settle = [&](pi_status st) {
    cudaStreamSynchronize(ctx->hs[0]);
    cudaStreamSynchronize(ctx->hs[1]);
    return st;
  };
#define PI_CUDA_SETTLE(call, what)                                       \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) return settle(cuda_fail(err, e_, what));      \
  } while (0)
  int64_t done = 0;
  int slot = 0;
  while (done < n_elem) {
    const int64_t cnt = std::min(chunk_elems, n_elem - done);
    cudaStream_t s = ctx->hs[slot];
    double* base = ctx->hbuf + slot * (slot_bytes / sizeof(double));
    double* d_out = base;
    double* d_aos = d_out + kk * chunk_elems;
    double* d_geom = d_aos + 18 * chunk_elems;
    double* d_caos = d_geom + 18 * chunk_elems;
    double* d_coef = d_caos + cw * chunk_elems;
    double* d_load = d_coef + cw * chunk_elems;   // [cnt][nsh]
    double* d_f = d_load + nsh * chunk_elems;      // [cnt]
    PI_CUDA_SETTLE(cudaMemcpyAsync(d_aos, geom_aos + 18 * done, sizeof(double) * 18 * cnt, cudaMemcpyHostToDevice, s),
                   "H2D geometry");
    aos_to_soa_kernel<<<static_cast<unsigned>((18 * cnt + 255) / 256), 256, 0, s>>>(d_aos, d_geom, cnt, 18, cnt);
    const double* cptr = coeff;
    int64_t cld = 0;
    if (cw) {
      PI_CUDA_SETTLE(cudaMemcpyAsync(d_caos, coeff + cw * done, sizeof(double) * cw * cnt, cudaMemcpyHostToDevice, s),
                     "H2D coefficients");
      aos_to_soa_kernel<<<static_cast<unsigned>((cw * cnt + 255) / 256), 256, 0, s>>>(d_caos, d_coef, cnt, cw, cnt);
      cptr = d_coef;
      cld = cnt;
    }
    pi_status st;
    if (load_out) {
      if (f)
        PI_CUDA_SETTLE(cudaMemcpyAsync(d_f, f + done, sizeof(double) * cnt, cudaMemcpyHostToDevice, s), "H2D f");
      st = pi_integrate_load(ctx, cnt, element_id_base + done, d_geom, cnt, coeff_mode, cptr, cld, d_out,
                             PI_OUT_CANONICAL, 0, f ? d_f : nullptr, f_const, d_load, s, err);
    } else {
      st = pi_integrate(ctx, cnt, element_id_base + done, d_geom, cnt, coeff_mode, cptr, cld, d_out,
                        PI_OUT_CANONICAL, 0, s, err);
    }
    if (st != PI_OK) return settle(st);
    if (load_out)
      PI_CUDA_SETTLE(cudaMemcpyAsync(load_out + nsh * done, d_load, sizeof(double) * nsh * cnt,
                                     cudaMemcpyDeviceToHost, s),
                     "D2H F");
    PI_CUDA_SETTLE(cudaMemcpyAsync(out + kk * done, d_out, sizeof(double) * kk * cnt, cudaMemcpyDeviceToHost, s),
                   "D2H K");
    done += cnt;
    slot ^= 1;
  }
#undef PI_CUDA_SETTLE
  settle(PI_OK);
  unsigned long long bad[2];
  const pi_status ds = drain(ctx, bad, err);
  ctx->calls.clear();
  if (ds != PI_OK) return ds;
  if (bad[1] != ~0ull) return material_error(static_cast<int64_t>(bad[1]), err);
  if (bad[0] == ~0ull) return PI_OK;
  // Device geometry of the streamed chunks is gone: describe the element from
  // the caller's host buffer (the flag can only hold this call's ids, the
  // earlier calls were drained above).
  const int64_t gid = static_cast<int64_t>(bad[0]);
  const bool mine = gid >= element_id_base && gid < element_id_base + n_elem;
  return report_inverted(ctx, gid, mine ? geom_aos + 18 * (gid - element_id_base) : nullptr, err);
}

}  // namespace

pi_status pi_integrate_host(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom_aos,
                            int coeff_mode, const double* coeff, double* out, int64_t chunk_elems,
                            pi_error_info* err) {
  return integrate_host_impl(ctx, n_elem, element_id_base, geom_aos, coeff_mode, coeff, out, chunk_elems, err,
                             nullptr, 0.0, nullptr);
}

pi_status pi_integrate_host_load(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom_aos,
                                 int coeff_mode, const double* coeff, const double* f, double f_const, double* out,
                                 double* load_out, int64_t chunk_elems, pi_error_info* err) {
  if (!load_out && n_elem > 0) {
    if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
    return set_error(err, PI_E_CONTRACT, "NULL load-vector buffer");
  }
  return integrate_host_impl(ctx, n_elem, element_id_base, geom_aos, coeff_mode, coeff, out, chunk_elems, err, f,
                             f_const, load_out);
}

pi_status pi_integrate_host_multi(pi_context* const* ctxs, int n_ctx, int64_t n_elem, int64_t element_id_base,
                                  const double* geom_aos, int coeff_mode, const double* coeff, double* out,
                                  int64_t chunk_elems, pi_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err)), err->element = -1;
  if (!ctxs || n_ctx < 1) return set_error(err, PI_E_CONTRACT, "pi_integrate_host_multi: no contexts");
  for (int g = 0; g < n_ctx; ++g) {
    if (!ctxs[g]) return set_error(err, PI_E_CONTRACT, "pi_integrate_host_multi: NULL context %d", g);
    if (ctxs[g]->p != ctxs[0]->p || ctxs[g]->n_eq != ctxs[0]->n_eq)
      return set_error(err, PI_E_CONFIG, "pi_integrate_host_multi: contexts disagree on (p, n_eq)");
    for (int h = 0; h < g; ++h)
      if (ctxs[h] == ctxs[g]) return set_error(err, PI_E_CONTRACT, "pi_integrate_host_multi: context %d repeated", g);
  }
  if (n_elem <= 0) return n_elem == 0 ? PI_OK : set_error(err, PI_E_CONTRACT, "n_elem < 0");
  const int ne = ctxs[0]->n_eq;
  const int64_t dim = static_cast<int64_t>(ctxs[0]->n_shape) * ne, kk = dim * dim;
  // per-element coefficient stride (uniform modes share one buffer)
  const int64_t cw = coeff_mode == PI_COEFF_PER_ELEMENT ? 16 * ne * ne : coeff_mode == PI_COEFF_ELASTICITY ? 2 : 0;
  std::vector<pi_status> st(n_ctx, PI_OK);
  std::vector<pi_error_info> errs(n_ctx);
  auto work = [&](int g) {
    // contiguous element range of context g (partition.py)
    const int64_t lo = n_elem * g / n_ctx, hi = n_elem * (g + 1) / n_ctx;
    if (hi <= lo) return;
    st[g] = pi_integrate_host(ctxs[g], hi - lo, element_id_base + lo, geom_aos + 18 * lo, coeff_mode,
                              coeff ? coeff + cw * lo : nullptr, out + kk * lo, chunk_elems, &errs[g]);
  };
  std::vector<std::thread> pool;
  for (int g = 1; g < n_ctx; ++g) pool.emplace_back(work, g);
  work(0);
  for (auto& t : pool) t.join();
  // report like a single call would: the lowest inverted element, else the first failure
  int pick = -1;
  for (int g = 0; g < n_ctx; ++g) {
    if (st[g] == PI_OK) continue;
    if (pick < 0) pick = g;
    if (st[g] == PI_E_INVERTED_ELEMENT &&
        (st[pick] != PI_E_INVERTED_ELEMENT || errs[g].element < errs[pick].element))
      pick = g;
  }
  if (pick < 0) return PI_OK;
  if (err) *err = errs[pick];
  return st[pick];
}

double pi_flops_dense_per_element(int p, int n_eq, int coeff_mode) {
  const double nsh = shape_count(p), nq = quad_count(p);
  if (coeff_mode == PI_COEFF_ELASTICITY || coeff_mode == PI_COEFF_ELASTICITY_UNIFORM)
    // the reference's own elasticity model: 63-flop 3x3 block per shape pair,
    // psi 15/shape, Jacobian 150 + dw 1 + 3 scaled moduli (flop_costs.hpp:15-41)
    return nq * (63.0 * nsh * nsh + 15.0 * nsh + 154.0);
  const double r = coeff_mode == PI_COEFF_LAPLACE ? 3.0 : 4.0, ne2 = static_cast<double>(n_eq) * n_eq;
  return nq * (ne2 * (2.0 * r * nsh * nsh + 2.0 * r * r * nsh) + 15.0 * nsh + 151.0);
}

double pi_bytes_per_element(int p, int n_eq, int coeff_mode) {
  const double dim = static_cast<double>(n_eq) * shape_count(p);
  const double coeff_bytes = coeff_mode == PI_COEFF_PER_ELEMENT ? 128.0 * n_eq * n_eq
                             : coeff_mode == PI_COEFF_ELASTICITY ? 16.0
                                                                  : 0.0;
  return 8.0 * dim * dim + 144.0 + coeff_bytes;
}

double pi_flops_executed_per_element(const pi_context* ctx, int coeff_mode) {
  if (!ctx) return 0.0;
  const int p = ctx->p;
  const bool general = coeff_mode != PI_COEFF_LAPLACE;
  const double nq = quad_count(p), nsh = shape_count(p);
  // Per rule point: Jacobian from edge vectors 21 FMA, cofactors/det 32,
  // reciprocal ~6, M block 24 (Laplace) / ~100 (general), in FLOPs.
  const double per_point = 2.0 * (21 + 16) + 6 + (general ? 200.0 : 48.0);
  const int v = resolve_variant(ctx);
  if (v == PI_VARIANT_DENSE && ctx->n_eq == 3 && p == 3) {
#ifdef PI_E3_CTA
    // p3_elastic_cta_kernel: inverse per point, 40 gradient triples (9 FMA each),
    // 820 blocks x (3-FMA dot + 9 x 2 FMA + 6 scalings)
    return nq * (2.0 * (21 + 16) + 6 + 2.0 * 40 * 9 + 2.0 * 820 * (3 + 18 + 6));
#else
    // p3_elastic_mma_kernel: inverse per point, 40 gradient triples (9 FMA +
    // 3 dw scalings each); 15 tile pairs x 9 DMMA m8n8k4 (512 FLOPs) per 4
    // points; the epilogue (about 5 FLOPs per stored upper-triangle entry)
    return nq * (2.0 * (21 + 16) + 6 + 40 * (2.0 * 9 + 3)) + EMma<3>::NPAIR * 9.0 * 512 * EMma<3>::KS +
           5.0 * 120 * 121 / 2;
#endif
  }
  if (v == PI_VARIANT_DENSE && ctx->n_eq == 3 && p == 2) {
    // p2_elastic_warp_kernel: per point 18 gradient triples (about 2 FMA + 2
    // scalings each), then 171 blocks x 9 FMA; the epilogue 171 x 9 x 2 FMA + 3
    return nq * (2.0 * (21 + 16) + 6 + 18 * 3 * (2.0 * 2 + 2) + 2.0 * 171 * 9) + 171 * (2.0 * 18 + 3);
  }
  if (v == PI_VARIANT_DENSE && ctx->n_eq == 3) {
    // p1_elastic_lane_kernel: Jacobian/cofactors, 18 physical gradients
    // (7 structural non-zeros x 3), then 3 warps x (57 FMA + 6 dw scalings)
    // per point; the epilogue about 4 FLOPs per accumulator
    return nq * (2.0 * (21 + 16) + 6 + 2.0 * 7 * 3 + 3.0 * (57 * 2 + 6)) + 3.0 * 57 * 4;
  }
  if (v == PI_VARIANT_DENSE) {
    // G_l(i) = sum_k phi_k(i) M_kl and K_ij += sum_l G_l(i) phi_l(j) over the
    // basis' structural non-zeros (BasisPattern); upper triangle when K is
    // symmetric (Laplace; p = 2 also symmetric uniform tensors -- counted as
    // the per-element case here).
    const int n = static_cast<int>(nsh), k0 = general ? 0 : 1;
    auto nz = [&](int k, int dof) {
      const int t = dof / (p + 1), a = dof % (p + 1);
      int d = 0, r = t;
      while (r > d) r -= ++d;
      return k == 0 ? true : k == 1 ? r > 0 : k == 2 ? (d - r) > 0 : a > 0;
    };
    double fma_count = 0.0;
    for (int i = 0; i < n; ++i) {
      for (int k = k0; k < 4; ++k) fma_count += nz(k, i) ? (4 - k0) : 0;
      for (int j = general ? 0 : i; j < n; ++j)
        for (int l = k0; l < 4; ++l) fma_count += nz(l, j) ? 1 : 0;
    }
    return nq * (per_point + 2.0 * fma_count);
  }
  // Sum factorisation (kernels_sumfact.cuh): H over (s, a', b', x, y, z),
  // the B-fragment values G (3 FMA each) and the DMMA GEMM (useful, i.e.
  // unpadded, sizes; symmetric paths skip sub-diagonal tile pairs).
  const double ne = ctx->n_eq, nv = p + 1, nve = ne * nv, nt = (p + 1) * (p + 2) / 2.0;
  const double ns = tri_point_count(p), nz = p + 1, dim = nsh * ne;
  const bool elastic = coeff_mode == PI_COEFF_ELASTICITY || coeff_mode == PI_COEFF_ELASTICITY_UNIFORM;
  const double per_point_ne = ne == 1 ? per_point : 2.0 * (21 + 16) + 6 + ne * ne * (elastic ? 60.0 : 200.0);
  const double h_terms = (general && !elastic) ? 16.0 / 9.0 : 1.0;
  const double h = ns * nve * nve * 9.0 * nz * 3.0 * h_terms;
  bool symmetric = coeff_mode == PI_COEFF_LAPLACE || elastic;
  const double g = ns * 3.0 * nve * dim * 3.0 * 2.0 * (symmetric ? sumfact_fragment_fraction(p, ctx->n_eq) : 1.0);
  const double frac = symmetric ? sumfact_sym_fraction(p, ctx->n_eq) : 1.0;
  const double k = nt * 3.0 * ns * dim * nve * 2.0 * frac;
  return nq * per_point_ne + h + g + k;
}

}  // extern "C"
