// include/prism_b200_prismint.hpp -- header-only C++ shim that lets prismint
// (the reference, /root/reference/proj) call the B200 kernels with its own
// types.  Include it from reference code and link libprism_b200.so:
//
//   #include "prismint/integrate_ref.hpp"
//   #include "prism_b200_prismint.hpp"
//   auto mats = prism_b200::run_batch(p, mesh, coeffs);       // kernels.cpp:485 shape
//   auto same = prism_b200::integrate_batch(mesh, coeffs, shapes, rule);
//   auto el   = prism_b200::run_batch(p, mesh, MaterialData{E, nu});  // elasticity, n_eq = 3
//
// Semantics: integrate_generic (integrate_ref.cpp:50-91) per element, in mesh
// order, element-constant coefficients (coefficients_at_point is the
// identity, coefficients.cpp:61-66).  Errors come back as the reference's own
// exception classes (errors.hpp:10-85), InvertedElementError naming the
// global element id base + index like kernels.cpp:158,249.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "prism_b200.h"
#include "prismint/coefficients.hpp"
#include "prismint/errors.hpp"
#include "prismint/geometry.hpp"
#include "prismint/integrate_ref.hpp"
#include "prismint/reference_element.hpp"

namespace prism_b200 {

/// Maps a pi_status to the matching prismint exception.
[[noreturn]] inline void throw_status(pi_status s, const pi_error_info& e) {
  const std::string msg(e.message);
  switch (s) {
    case PI_E_CONFIG: throw prismint::ConfigError(msg);
    case PI_E_DOMAIN: throw prismint::DomainError(msg);
    case PI_E_UNSUPPORTED_DEGREE: throw prismint::UnsupportedDegreeError(msg);
    case PI_E_INVERTED_ELEMENT:
      throw prismint::InvertedElementError(e.element, e.xi[0], e.xi[1], e.xi[2], e.det);
    case PI_E_CAPACITY: throw prismint::CapacityError(msg);
    case PI_E_SHARED_MEMORY: throw prismint::SharedMemoryError(msg);
    case PI_E_CONTRACT: throw prismint::ContractViolation(msg);
    case PI_E_IO: throw prismint::IoError(msg);
    default: throw std::runtime_error("prism_b200: " + msg);
  }
}

inline void check(pi_status s, const pi_error_info& e) {
  if (s != PI_OK) throw_status(s, e);
}

/// RAII context over pi_context_create with the reference's own rule and
/// shape table (the constants run_batch builds, kernels.cpp:493-494).
class Context {
 public:
  Context(const prismint::ShapeTable& shapes, const prismint::QuadratureRule& rule, int n_eq = 1, int device = 0) {
    if (shapes.order_p != rule.order_p || shapes.per_point.size() != rule.points.size())
      throw prismint::ConfigError("prism_b200: shape table and rule disagree");
    const int nq = rule.size(), nsh = shapes.n_shape;
    std::vector<double> pts(3 * nq), tab(static_cast<std::size_t>(nq) * 4 * nsh);
    for (int q = 0; q < nq; ++q) {
      pts[3 * q] = rule.points[q].xi1;
      pts[3 * q + 1] = rule.points[q].xi2;
      pts[3 * q + 2] = rule.points[q].xi3;
      std::memcpy(&tab[static_cast<std::size_t>(q) * 4 * nsh], shapes.per_point[q].data.data(),
                  sizeof(double) * 4 * nsh);
    }
    pi_error_info e{};
    check(pi_context_create(device, rule.order_p, n_eq, nq, nsh, pts.data(), rule.weights.data(), tab.data(),
                            &ctx_, &e),
          e);
    p_ = rule.order_p;
    n_eq_ = n_eq;
    nsh_ = nsh;
  }
  ~Context() { pi_context_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  /// Whole mesh through the host-buffer path; coefficients: one tensor for
  /// all elements, or one per element.
  std::vector<prismint::ElementStiffness> integrate(std::span<const prismint::PrismGeometry> mesh,
                                                    std::span<const prismint::CoefficientTensor> coeffs,
                                                    std::int64_t element_id_base = 0) {
    if (coeffs.empty() || (coeffs.size() != 1 && coeffs.size() != mesh.size()))
      throw prismint::ConfigError("prism_b200: need one coefficient tensor or one per element");
    for (const auto& c : coeffs)
      if (c.n_eq != n_eq_) throw prismint::ConfigError("prism_b200: coefficient n_eq mismatch");
    const int nc = 16 * n_eq_ * n_eq_;
    std::vector<double> cbuf(coeffs.size() * nc);
    for (std::size_t k = 0; k < coeffs.size(); ++k)
      std::memcpy(&cbuf[k * nc], coeffs[k].entries.data(), sizeof(double) * nc);
    const int mode = coeffs.size() == 1 ? PI_COEFF_UNIFORM : PI_COEFF_PER_ELEMENT;
    return run(mesh, mode, cbuf.data(), element_id_base);
  }

  /// Isotropic elasticity (n_eq = 3 context): one material for every
  /// element, or one per element (MaterialData, coefficients.hpp:31-34; the
  /// material input of build_kernel_inputs, kernels.hpp:47-50).  Same result
  /// as integrate_optimized / integrate_generic(elasticity_tensor(mat)).
  std::vector<prismint::ElementStiffness> integrate(std::span<const prismint::PrismGeometry> mesh,
                                                    std::span<const prismint::MaterialData> mats,
                                                    std::int64_t element_id_base = 0) {
    if (n_eq_ != 3) throw prismint::ConfigError("prism_b200: elasticity needs an n_eq = 3 context");
    if (mats.empty() || (mats.size() != 1 && mats.size() != mesh.size()))
      throw prismint::ConfigError("prism_b200: need one material or one per element");
    for (const auto& m : mats) {  // lame_parameters' checks, coefficients.cpp:23-32
      if (m.young_E <= 0.0) throw prismint::DomainError("material: Young modulus must be positive");
      if (m.poisson_nu <= -1.0 || m.poisson_nu > 0.5)
        throw prismint::DomainError("material: Poisson ratio must lie in (-1, 0.5]");
      if (m.poisson_nu == 0.5)
        throw prismint::DomainError("material: nu = 0.5 (incompressible) has no finite Lame lambda");
    }
    std::vector<double> mbuf(2 * mats.size());
    for (std::size_t k = 0; k < mats.size(); ++k) {
      mbuf[2 * k] = mats[k].young_E;
      mbuf[2 * k + 1] = mats[k].poisson_nu;
    }
    return run(mesh, mats.size() == 1 ? PI_COEFF_ELASTICITY_UNIFORM : PI_COEFF_ELASTICITY, mbuf.data(),
               element_id_base);
  }

  /// Stiffness matrices and load vectors F_i = sum_q det w_q f phi_i(x_q)
  /// (scalar weak forms) in one pass over the mesh: f one value per element,
  /// or empty for f_const everywhere (pi_integrate_host_load).
  struct WithLoad {
    std::vector<prismint::ElementStiffness> stiffness;
    std::vector<std::vector<double>> load;
  };
  WithLoad integrate_with_load(std::span<const prismint::PrismGeometry> mesh,
                               std::span<const prismint::CoefficientTensor> coeffs, std::span<const double> f = {},
                               double f_const = 1.0, std::int64_t element_id_base = 0) {
    if (n_eq_ != 1) throw prismint::ConfigError("prism_b200: load vectors need a scalar (n_eq = 1) context");
    if (coeffs.empty() || (coeffs.size() != 1 && coeffs.size() != mesh.size()))
      throw prismint::ConfigError("prism_b200: need one coefficient tensor or one per element");
    if (!f.empty() && f.size() != mesh.size()) throw prismint::ConfigError("prism_b200: need one f per element");
    std::vector<double> cbuf(coeffs.size() * 16);
    for (std::size_t k = 0; k < coeffs.size(); ++k) std::memcpy(&cbuf[k * 16], coeffs[k].entries.data(), 16 * 8);
    const std::size_t n = mesh.size(), kk = static_cast<std::size_t>(nsh_) * nsh_;
    std::vector<double> geom = flat_geometry(mesh), out(kk * n), load(static_cast<std::size_t>(nsh_) * n);
    pi_error_info e{};
    check(pi_integrate_host_load(ctx_, static_cast<std::int64_t>(n), element_id_base, geom.data(),
                                 coeffs.size() == 1 ? PI_COEFF_UNIFORM : PI_COEFF_PER_ELEMENT, cbuf.data(),
                                 f.empty() ? nullptr : f.data(), f_const, out.data(), load.data(), 0, &e),
          e);
    WithLoad r;
    r.stiffness = wrap(out, n, kk);
    r.load.resize(n);
    for (std::size_t i = 0; i < n; ++i) r.load[i].assign(load.begin() + i * nsh_, load.begin() + (i + 1) * nsh_);
    return r;
  }

  pi_context* raw() { return ctx_; }

 private:
  static std::vector<double> flat_geometry(std::span<const prismint::PrismGeometry> mesh) {
    std::vector<double> geom(18 * mesh.size());
    for (std::size_t e = 0; e < mesh.size(); ++e)
      for (int v = 0; v < 6; ++v)
        for (int c = 0; c < 3; ++c) geom[18 * e + 3 * v + c] = mesh[e].vertices[v][c];
    return geom;
  }
  std::vector<prismint::ElementStiffness> run(std::span<const prismint::PrismGeometry> mesh, int mode,
                                              const double* coeff, std::int64_t element_id_base) {
    const std::size_t n = mesh.size();
    std::vector<double> geom = flat_geometry(mesh);
    const std::size_t kk = static_cast<std::size_t>(nsh_) * n_eq_ * nsh_ * n_eq_;
    std::vector<double> out(kk * n);
    pi_error_info e{};
    check(pi_integrate_host(ctx_, static_cast<std::int64_t>(n), element_id_base, geom.data(), mode, coeff,
                            out.data(), 0, &e),
          e);
    return wrap(out, n, kk);
  }
  std::vector<prismint::ElementStiffness> wrap(const std::vector<double>& out, std::size_t n, std::size_t kk) {
    std::vector<prismint::ElementStiffness> res(n);
    for (std::size_t i = 0; i < n; ++i) {
      auto& a = res[i];
      a.order_p = p_;
      a.n_eq = n_eq_;
      a.n_shape = nsh_;
      a.data.assign(out.begin() + i * kk, out.begin() + (i + 1) * kk);
    }
    return res;
  }

  pi_context* ctx_ = nullptr;
  int p_ = 0, n_eq_ = 1, nsh_ = 0;
};

/// integrate_generic for a whole mesh (mesh order), the reference's tables.
inline std::vector<prismint::ElementStiffness> integrate_batch(std::span<const prismint::PrismGeometry> mesh,
                                                               std::span<const prismint::CoefficientTensor> coeffs,
                                                               const prismint::ShapeTable& shapes,
                                                               const prismint::QuadratureRule& rule, int device = 0,
                                                               std::int64_t element_id_base = 0) {
  Context ctx(shapes, rule, coeffs.empty() ? 1 : coeffs.front().n_eq, device);
  return ctx.integrate(mesh, coeffs, element_id_base);
}

/// integrate_generic for a whole mesh over several GPUs: contiguous element
/// ranges, one context and host thread per device (pi_integrate_host_multi);
/// bitwise equal to one device.
inline std::vector<prismint::ElementStiffness> integrate_batch_multi(
    std::span<const prismint::PrismGeometry> mesh, std::span<const prismint::CoefficientTensor> coeffs,
    const prismint::ShapeTable& shapes, const prismint::QuadratureRule& rule, std::span<const int> devices,
    std::int64_t element_id_base = 0) {
  if (devices.empty()) throw prismint::ConfigError("prism_b200: no devices");
  if (coeffs.empty() || (coeffs.size() != 1 && coeffs.size() != mesh.size()))
    throw prismint::ConfigError("prism_b200: need one coefficient tensor or one per element");
  const int n_eq = coeffs.front().n_eq;
  std::vector<std::unique_ptr<Context>> ctx;
  std::vector<pi_context*> raw;
  for (int d : devices) {
    ctx.push_back(std::make_unique<Context>(shapes, rule, n_eq, d));
    raw.push_back(ctx.back()->raw());
  }
  const std::size_t n = mesh.size();
  std::vector<double> geom(18 * n);
  for (std::size_t e = 0; e < n; ++e)
    for (int v = 0; v < 6; ++v)
      for (int c = 0; c < 3; ++c) geom[18 * e + 3 * v + c] = mesh[e].vertices[v][c];
  const int nc = 16 * n_eq * n_eq;
  std::vector<double> cbuf(coeffs.size() * nc);
  for (std::size_t k = 0; k < coeffs.size(); ++k)
    std::memcpy(&cbuf[k * nc], coeffs[k].entries.data(), sizeof(double) * nc);
  const int nsh = shapes.n_shape;
  const std::size_t kk = static_cast<std::size_t>(nsh) * n_eq * nsh * n_eq;
  std::vector<double> out(kk * n);
  pi_error_info e{};
  check(pi_integrate_host_multi(raw.data(), static_cast<int>(raw.size()), static_cast<std::int64_t>(n),
                                element_id_base, geom.data(),
                                coeffs.size() == 1 ? PI_COEFF_UNIFORM : PI_COEFF_PER_ELEMENT, cbuf.data(),
                                out.data(), 0, &e),
        e);
  std::vector<prismint::ElementStiffness> res(n);
  for (std::size_t i = 0; i < n; ++i) {
    res[i].order_p = rule.order_p;
    res[i].n_eq = n_eq;
    res[i].n_shape = nsh;
    res[i].data.assign(out.begin() + i * kk, out.begin() + (i + 1) * kk);
  }
  return res;
}

/// run_batch-shaped entry (kernels.hpp:73-75): builds the rule and table like
/// the reference does, integrates the mesh with one coefficient tensor.
inline std::vector<prismint::ElementStiffness> run_batch(int p, std::span<const prismint::PrismGeometry> mesh,
                                                         const prismint::CoefficientTensor& coeff, int device = 0) {
  if (mesh.empty()) throw prismint::ConfigError("run_batch: empty mesh");
  const prismint::QuadratureRule rule = prismint::prism_quadrature(p);
  const prismint::ShapeTable shapes = prismint::tabulate_shapes(p, rule);
  return integrate_batch(mesh, std::span<const prismint::CoefficientTensor>(&coeff, 1), shapes, rule, device);
}

/// run_batch for the reference's model problem (kernels.hpp:73-75 takes one
/// MaterialData for the mesh): FP64 isotropic elasticity, n_eq = 3, mesh order.
inline std::vector<prismint::ElementStiffness> run_batch(int p, std::span<const prismint::PrismGeometry> mesh,
                                                         const prismint::MaterialData& mat, int device = 0) {
  if (mesh.empty()) throw prismint::ConfigError("run_batch: empty mesh");
  const prismint::QuadratureRule rule = prismint::prism_quadrature(p);
  const prismint::ShapeTable shapes = prismint::tabulate_shapes(p, rule);
  Context ctx(shapes, rule, 3, device);
  return ctx.integrate(mesh, std::span<const prismint::MaterialData>(&mat, 1));
}

}  // namespace prism_b200
