// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A tiny extern "C" face over the UNMODIFIED reference sources
// (/root/reference/proj/src/{errors,reference_element,geometry,coefficients,
// integrate_ref}.cpp, plus io.cpp when nlohmann json is available), compiled
// together by oracle/Makefile into
// oracle/_ref/libprismint_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.  Nothing here
// re-implements reference arithmetic: every entry point forwards to the
// reference function named in its comment.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <span>
#include <thread>
#include <vector>

#include "prismint/coefficients.hpp"
#ifdef PRISM_REF_IO
#include "prismint/io.hpp"
#endif
#include "prismint/errors.hpp"
#include "prismint/geometry.hpp"
#include "prismint/integrate_ref.hpp"
#include "prismint/reference_element.hpp"

using namespace prismint;

extern "C" {

struct ref_error {
  int code;  // 0 ok, else 1 + errc (errors.hpp:10-19)
  int64_t element;
  double det;
  char message[256];
};

}  // extern "C"

namespace {

int fail(ref_error* err, const Error& e) {
  if (err) {
    err->code = 1 + static_cast<int>(e.code());
    std::strncpy(err->message, e.what(), sizeof(err->message) - 1);
    err->message[sizeof(err->message) - 1] = 0;
    if (auto* inv = dynamic_cast<const InvertedElementError*>(&e)) {
      err->element = inv->element();
      err->det = inv->det();
    }
  }
  return 1 + static_cast<int>(e.code());
}

PrismGeometry geom_from(const double* g) {
  PrismGeometry out;
  for (int v = 0; v < 6; ++v)
    for (int c = 0; c < 3; ++c) out.vertices[v][c] = g[v * 3 + c];
  return out;
}

CoefficientTensor coeff_from(int n_eq, const double* c) {
  CoefficientTensor t = CoefficientTensor::zeros(n_eq);
  for (std::size_t k = 0; k < t.entries.size(); ++k) {
    // CoefficientTensor::set (coefficients.cpp:17-21) keeps the nonzero mask.
    const int jd = k % 4, id = (k / 4) % 4, je = (k / 16) % n_eq, ie = k / (16 * n_eq);
    t.set(ie, je, id, jd, c[k]);
  }
  return t;
}

struct Cache {
  int p = 0;
  QuadratureRule rule;
  ShapeTable shapes;
};

}  // namespace

extern "C" {

int ref_shape_count(int p) { return shape_count(p); }
int ref_quadrature_point_count(int p) { return quadrature_point_count(p); }

// prism_quadrature (reference_element.cpp:175-193): points [nq][3], weights [nq].
int ref_prism_quadrature(int p, double* points, double* weights, ref_error* err) {
  try {
    const QuadratureRule r = prism_quadrature(p);
    for (int q = 0; q < r.size(); ++q) {
      points[3 * q + 0] = r.points[q].xi1;
      points[3 * q + 1] = r.points[q].xi2;
      points[3 * q + 2] = r.points[q].xi3;
      weights[q] = r.weights[q];
    }
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// tabulate_shapes (reference_element.cpp:272-286): table [nq][4][nsh].
int ref_tabulate_shapes(int p, double* table, ref_error* err) {
  try {
    const QuadratureRule r = prism_quadrature(p);
    const ShapeTable t = tabulate_shapes(p, r);
    std::size_t off = 0;
    for (const auto& pv : t.per_point) {
      std::copy(pv.data.begin(), pv.data.end(), table + off);
      off += pv.data.size();
    }
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// gauss_legendre_1d (reference_element.cpp:37-69).
int ref_gauss_legendre(int n, double* x, double* w, ref_error* err) {
  try {
    auto [px, pw] = gauss_legendre_1d(n);
    std::copy(px.begin(), px.end(), x);
    std::copy(pw.begin(), pw.end(), w);
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// triangle_rule (reference_element.cpp:110-173); returns the point count.
int ref_triangle_rule(int degree, double* pts, double* wts, ref_error* err) {
  try {
    auto [p, w] = triangle_rule(degree);
    if (pts) {
      for (std::size_t i = 0; i < p.size(); ++i) {
        pts[2 * i] = p[i][0];
        pts[2 * i + 1] = p[i][1];
        wts[i] = w[i];
      }
    }
    return static_cast<int>(p.size());
  } catch (const Error& e) {
    fail(err, e);
    return -1;
  }
}

// generate_box_mesh (geometry.cpp:134-201): vertices [E][6][3] AoS.
int64_t ref_box_mesh_count(int nx, int ny, int nz) { return 2ll * nx * ny * nz; }
int ref_generate_box_mesh(int nx, int ny, int nz, double distortion, uint64_t seed, double* out,
                          ref_error* err) {
  try {
    const auto mesh = generate_box_mesh(nx, ny, nz, distortion, seed);
    for (std::size_t e = 0; e < mesh.size(); ++e)
      for (int v = 0; v < 6; ++v)
        for (int c = 0; c < 3; ++c) out[(e * 6 + v) * 3 + c] = mesh[e].vertices[v][c];
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// jacobian_terms (geometry.cpp:60-83): det + inv[3][3] (inv[k][i] = dxi_k/dx_i).
int ref_jacobian_terms(const double* geom, const double* xi, double* det, double* inv,
                       int64_t element_id, ref_error* err) {
  try {
    const JacobianTerms jt = jacobian_terms(geom_from(geom), {xi[0], xi[1], xi[2]}, element_id);
    *det = jt.det;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) inv[r * 3 + c] = jt.inv[r][c];
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// integrate_generic (integrate_ref.cpp:50-91) over a batch, element-constant
// coefficients (expand_coefficients, coefficients.cpp:68-76).
//   geom   [n][6][3] AoS
//   coeff  [n][n_eq*n_eq*16] when coeff_per_element, else one [n_eq*n_eq*16] tensor
//   out    [n][dim*dim] canonical (integrate_ref.hpp:14-31)
// n_threads <= 0 uses hardware_concurrency; elements are split round-robin in
// contiguous chunks.  The first error (lowest element index) is reported.
int ref_integrate_generic_batch(int p, int n_eq, int64_t n, const double* geom, const double* coeff,
                                int coeff_per_element, double* out, int64_t element_id_base,
                                int n_threads, ref_error* err) {
  try {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    const int dim = n_eq * shape_count(p);
    const std::size_t kk = static_cast<std::size_t>(dim) * dim;
    const int nc = n_eq * n_eq * 16;
    if (n_threads <= 0) n_threads = std::max(1u, std::thread::hardware_concurrency());
    n_threads = static_cast<int>(std::min<int64_t>(n_threads, std::max<int64_t>(n, 1)));
    std::atomic<int64_t> next{0};
    std::mutex mu;
    int64_t bad = -1;
    ref_error bad_err{};
    const QuadCoefficients shared =
        coeff_per_element ? QuadCoefficients{} : expand_coefficients(coeff_from(n_eq, coeff), rule);
    auto worker = [&]() {
      const int64_t chunk = 16;
      for (;;) {
        const int64_t first = next.fetch_add(chunk);
        if (first >= n) break;
        const int64_t last = std::min(n, first + chunk);
        for (int64_t e = first; e < last; ++e) {
          try {
            const PrismGeometry g = geom_from(geom + e * 18);
            ElementStiffness a;
            if (coeff_per_element) {
              const QuadCoefficients qc = expand_coefficients(coeff_from(n_eq, coeff + e * nc), rule);
              a = integrate_generic(g, qc, shapes, rule, nullptr, element_id_base + e);
            } else {
              a = integrate_generic(g, shared, shapes, rule, nullptr, element_id_base + e);
            }
            std::copy(a.data.begin(), a.data.end(), out + e * kk);
          } catch (const Error& ex) {
            std::lock_guard<std::mutex> lock(mu);
            if (bad < 0 || e < bad) {
              bad = e;
              bad_err = ref_error{};
              fail(&bad_err, ex);
            }
          }
        }
      }
    };
    if (n_threads <= 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < n_threads; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    if (bad >= 0) {
      if (err) *err = bad_err;
      return bad_err.code;
    }
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// integrate_optimized (integrate_ref.cpp:93-130): elasticity, one element.
int ref_integrate_optimized(int p, const double* geom, double young, double nu, double* out,
                            ref_error* err) {
  try {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    const ElementStiffness a = integrate_optimized(geom_from(geom), {young, nu}, shapes, rule);
    std::copy(a.data.begin(), a.data.end(), out);
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// integrate_optimized over a batch with per-element materials [n][2] = (E, nu),
// element-parallel on n_threads (<= 0: hardware_concurrency) -- the
// reference's fastest FP64 elasticity path, used as the CPU baseline.
int ref_integrate_optimized_batch(int p, int64_t n, const double* geom, const double* mats, double* out,
                                  int n_threads, ref_error* err) {
  try {
    const QuadratureRule rule = prism_quadrature(p);
    const ShapeTable shapes = tabulate_shapes(p, rule);
    const int dim = 3 * shape_count(p);
    const std::size_t kk = static_cast<std::size_t>(dim) * dim;
    if (n_threads <= 0) n_threads = std::max(1u, std::thread::hardware_concurrency());
    n_threads = static_cast<int>(std::min<int64_t>(n_threads, std::max<int64_t>(n, 1)));
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    ref_error first_err{};
    std::mutex mu;
    auto worker = [&]() {
      for (;;) {
        const int64_t e = next.fetch_add(1);
        if (e >= n) break;
        try {
          const ElementStiffness a =
              integrate_optimized(geom_from(geom + e * 18), {mats[2 * e], mats[2 * e + 1]}, shapes, rule, e);
          std::copy(a.data.begin(), a.data.end(), out + e * kk);
        } catch (const Error& ex) {
          std::lock_guard<std::mutex> lock(mu);
          if (!failed.exchange(1)) fail(&first_err, ex);
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < n_threads; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    if (failed) {
      if (err) *err = first_err;
      return first_err.code;
    }
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

// elasticity_tensor (coefficients.cpp:40-59): [3*3*16] entries.
int ref_elasticity_tensor(double young, double nu, double* out, ref_error* err) {
  try {
    const CoefficientTensor t = elasticity_tensor({young, nu});
    std::copy(t.entries.begin(), t.entries.end(), out);
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}

#ifdef PRISM_REF_IO
// save_stiffness / load_stiffness (io.cpp:112-168), the PRISTIF1 container.
int ref_save_stiffness(const char* path, int p, int n_eq, const double* k, int64_t element_id, ref_error* err) {
  try {
    ElementStiffness a;
    a.order_p = p;
    a.n_eq = n_eq;
    a.n_shape = shape_count(p);
    a.data.assign(k, k + static_cast<std::size_t>(a.dim()) * a.dim());
    save_stiffness(path, a, element_id);
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}
int ref_load_stiffness(const char* path, double* out, int64_t capacity, int64_t* element_id, int* p, int* n_eq,
                       ref_error* err) {
  try {
    const ElementStiffness a = load_stiffness(path, element_id);
    if (static_cast<int64_t>(a.data.size()) > capacity) return -1;
    std::copy(a.data.begin(), a.data.end(), out);
    *p = a.order_p;
    *n_eq = a.n_eq;
    return 0;
  } catch (const Error& e) {
    return fail(err, e);
  }
}
#endif

}  // extern "C"
