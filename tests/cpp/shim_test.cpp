// C++ drop-in test: the reference's own types and integrate_generic vs the
// B200 kernels through include/prism_b200_prismint.hpp.  Built against the
// reference headers + oracle/_ref (tests/cpp/Makefile); run by
// tests/test_gpu_shim.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <vector>

#include "prism_b200_prismint.hpp"

using namespace prismint;

static double rel_frob(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += a[i] * a[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

int main() {
  int failures = 0;
  const auto mesh = generate_box_mesh(3, 2, 2, 0.2, 31);
  for (int p = 1; p <= 7; ++p) {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    CoefficientTensor lap = CoefficientTensor::zeros(1);
    for (int d = 1; d <= 3; ++d) lap.set(0, 0, d, d, 1.0);
    const auto got = prism_b200::run_batch(p, mesh, lap);
    const QuadCoefficients qc = expand_coefficients(lap, rule);
    double worst = 0;
    for (size_t e = 0; e < mesh.size(); e += (p >= 6 ? 11 : 1)) {
      const ElementStiffness ref = integrate_generic(mesh[e], qc, shapes, rule);
      worst = std::max(worst, rel_frob(ref.data, got[e].data));
    }
    std::printf("p=%d run_batch vs integrate_generic: %.3e\n", p, worst);
    if (!(worst <= 1e-12)) ++failures;
  }
  // per-element coefficient tensors
  {
    const int p = 3;
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    std::vector<CoefficientTensor> cs;
    for (size_t e = 0; e < mesh.size(); ++e) {
      CoefficientTensor c = CoefficientTensor::zeros(1);
      for (int d = 1; d <= 3; ++d) c.set(0, 0, d, d, 1.0 + 0.1 * e);
      c.set(0, 0, 0, 1, 0.3);
      c.set(0, 0, 0, 0, 0.05 * e);
      cs.push_back(c);
    }
    const auto got = prism_b200::integrate_batch(mesh, cs, shapes, rule);
    double worst = 0;
    for (size_t e = 0; e < mesh.size(); ++e) {
      const ElementStiffness ref = integrate_generic(mesh[e], expand_coefficients(cs[e], rule), shapes, rule);
      worst = std::max(worst, rel_frob(ref.data, got[e].data));
    }
    std::printf("per-element coefficients p=3: %.3e\n", worst);
    if (!(worst <= 1e-12)) ++failures;
  }
  // elasticity (the reference's model problem): run_batch(MaterialData) and
  // per-element materials vs integrate_optimized
  for (int p : {1, 2, 4}) {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    const MaterialData mat{2.0, 0.3};
    const auto got = prism_b200::run_batch(p, mesh, mat);
    std::vector<MaterialData> mats;
    for (size_t e = 0; e < mesh.size(); ++e) mats.push_back({1.0 + 0.1 * e, 0.25 + 0.01 * (e % 7)});
    prism_b200::Context ctx(shapes, rule, 3);
    const auto got_pe = ctx.integrate(mesh, std::span<const MaterialData>(mats));
    double worst = 0;
    for (size_t e = 0; e < mesh.size(); e += (p >= 4 ? 5 : 1)) {
      worst = std::max(worst, rel_frob(integrate_optimized(mesh[e], mat, shapes, rule).data, got[e].data));
      worst = std::max(worst, rel_frob(integrate_optimized(mesh[e], mats[e], shapes, rule).data, got_pe[e].data));
    }
    std::printf("p=%d elasticity vs integrate_optimized: %.3e\n", p, worst);
    if (!(worst <= 1e-12)) ++failures;
  }
  // stiffness and load vectors in one pass (Context::integrate_with_load):
  // F = f x column 0 of the c[0][0][0][0] = 1 mass matrix of integrate_generic
  for (int p : {1, 2, 4}) {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    CoefficientTensor lap = CoefficientTensor::zeros(1);
    for (int d = 1; d <= 3; ++d) lap.set(0, 0, d, d, 1.0);
    CoefficientTensor mass = CoefficientTensor::zeros(1);
    mass.set(0, 0, 0, 0, 1.0);
    std::vector<double> f(mesh.size());
    for (size_t e = 0; e < mesh.size(); ++e) f[e] = 0.5 + 0.1 * e;
    prism_b200::Context ctx(shapes, rule);
    const auto r = ctx.integrate_with_load(mesh, std::span<const CoefficientTensor>(&lap, 1), f);
    const QuadCoefficients qm = expand_coefficients(mass, rule), ql = expand_coefficients(lap, rule);
    double worst = 0;
    for (size_t e = 0; e < mesh.size(); e += 3) {
      const ElementStiffness m = integrate_generic(mesh[e], qm, shapes, rule);
      std::vector<double> ref(shapes.n_shape);
      for (int i = 0; i < shapes.n_shape; ++i) ref[i] = f[e] * m.data[static_cast<size_t>(i) * shapes.n_shape];
      worst = std::max(worst, rel_frob(ref, r.load[e]));
      worst = std::max(worst, rel_frob(integrate_generic(mesh[e], ql, shapes, rule).data, r.stiffness[e].data));
    }
    std::printf("p=%d integrate_with_load (K and F) vs integrate_generic: %.3e\n", p, worst);
    if (!(worst <= 1e-12)) ++failures;
  }
  // several contexts (one per device; here twice the same GPU): bitwise equal
  {
    const int p = 4;
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    CoefficientTensor lap = CoefficientTensor::zeros(1);
    for (int d = 1; d <= 3; ++d) lap.set(0, 0, d, d, 1.0);
    const auto one = prism_b200::integrate_batch(mesh, std::span<const CoefficientTensor>(&lap, 1), shapes, rule);
    const int devs[3] = {0, 0, 0};
    const auto multi = prism_b200::integrate_batch_multi(mesh, std::span<const CoefficientTensor>(&lap, 1), shapes,
                                                         rule, std::span<const int>(devs, 3));
    bool same = one.size() == multi.size();
    for (size_t e = 0; same && e < one.size(); ++e) same = one[e].data == multi[e].data;
    std::printf("integrate_batch_multi (3 contexts) bitwise equal: %s\n", same ? "yes" : "NO");
    if (!same) ++failures;
  }
  // error mapping: inverted element with batch offset, table mismatch
  {
    auto bad = generate_box_mesh(2, 2, 1, 0.0);
    std::swap(bad[6].vertices[0], bad[6].vertices[1]);
    const QuadratureRule rule = prism_quadrature(2);
    const ShapeTable shapes = tabulate_shapes(2, rule);
    CoefficientTensor lap = CoefficientTensor::zeros(1);
    for (int d = 1; d <= 3; ++d) lap.set(0, 0, d, d, 1.0);
    try {
      prism_b200::Context ctx(shapes, rule);
      (void)ctx.integrate(bad, std::span<const CoefficientTensor>(&lap, 1), 100);
      std::printf("expected InvertedElementError\n");
      ++failures;
    } catch (const InvertedElementError& e) {
      std::printf("InvertedElementError element=%lld det=%g\n", (long long)e.element(), e.det());
      if (e.element() != 106) ++failures;
    }
    try {
      const QuadratureRule r3 = prism_quadrature(3);
      prism_b200::Context ctx(shapes, r3);
      ++failures;
    } catch (const ConfigError&) {
      std::printf("ConfigError on table mismatch: ok\n");
    }
  }
  std::printf(failures ? "FAILED %d\n" : "ALL OK\n", failures);
  return failures ? 1 : 0;
}
