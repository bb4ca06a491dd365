// Synthetic inputs for parity and benchmarks (never timed): the reference's
// seeded box mesh, written straight into the SoA layout the kernels read, and
// seeded per-element convection-diffusion-reaction tensors.
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "pi_internal.hpp"

namespace pib {

// geometry_shape_derivs + jacobian_matrix + cofactor inverse
// (geometry.cpp:32-83); geom_aos is one PrismGeometry [6][3].
bool jacobian_terms(const double* x, const double* xi, double& det, double inv[9]) {
  const double l0 = 1.0 - xi[0] - xi[1], l1 = xi[0], l2 = xi[1];
  const double zm = 0.5 * (1.0 - xi[2]), zp = 0.5 * (1.0 + xi[2]);
  const double dn[3][6] = {{-zm, zm, 0.0, -zp, zp, 0.0},
                           {-zm, 0.0, zm, -zp, 0.0, zp},
                           {-0.5 * l0, -0.5 * l1, -0.5 * l2, 0.5 * l0, 0.5 * l1, 0.5 * l2}};
  double j[3][3];
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int v = 0; v < 6; ++v) s += dn[c][v] * x[v * 3 + i];
      j[i][c] = s;
    }
  const double c00 = j[1][1] * j[2][2] - j[1][2] * j[2][1];
  const double c01 = j[1][2] * j[2][0] - j[1][0] * j[2][2];
  const double c02 = j[1][0] * j[2][1] - j[1][1] * j[2][0];
  det = j[0][0] * c00 + j[0][1] * c01 + j[0][2] * c02;
  if (!(det > 0.0)) return false;
  const double id = 1.0 / det;
  inv[0] = c00 * id;
  inv[1] = (j[0][2] * j[2][1] - j[0][1] * j[2][2]) * id;
  inv[2] = (j[0][1] * j[1][2] - j[0][2] * j[1][1]) * id;
  inv[3] = c01 * id;
  inv[4] = (j[0][0] * j[2][2] - j[0][2] * j[2][0]) * id;
  inv[5] = (j[0][2] * j[1][0] - j[0][0] * j[1][2]) * id;
  inv[6] = c02 * id;
  inv[7] = (j[0][1] * j[2][0] - j[0][0] * j[2][1]) * id;
  inv[8] = (j[0][0] * j[1][1] - j[0][1] * j[1][0]) * id;
  return true;
}

namespace {

// splitmix64 finaliser: counter-based, so element g's draws do not depend on
// how the element range is split across chunks or GPUs.
inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

inline double unit_draw(uint64_t key, int64_t g, int i) {
  const uint64_t z = mix64(key + static_cast<uint64_t>(g) * 16u + static_cast<uint64_t>(i));
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

}  // namespace
}  // namespace pib

extern "C" {

pi_status pi_generate_box_mesh(int nx, int ny, int nz, double distortion, uint64_t seed, int64_t first,
                               int64_t count, int soa, int64_t ld, int validate, double* out,
                               pi_error_info* err) {
  if (nx < 1 || ny < 1 || nz < 1)
    return pib::set_error(err, PI_E_DOMAIN, "generate_box_mesh: all dimensions must be >= 1");
  if (distortion < 0.0 || distortion >= 0.3)
    return pib::set_error(err, PI_E_DOMAIN, "generate_box_mesh: distortion must lie in [0, 0.3)");
  const int64_t total = 2ll * nx * ny * nz;
  if (first < 0 || count < 0 || first + count > total)
    return pib::set_error(err, PI_E_CONTRACT, "generate_box_mesh: range [%lld, %lld) outside [0, %lld)",
                          (long long)first, (long long)(first + count), (long long)total);
  if (soa && ld < count) return pib::set_error(err, PI_E_CONTRACT, "generate_box_mesh: ld < count");

  // Node positions: one mt19937_64 stream, three draws per node in k, j, i
  // order, interior nodes perturbed (geometry.cpp:141-167).
  const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
  const size_t sx = nx + 1, sy = ny + 1;
  std::vector<double> nodes(3 * sx * sy * (nz + 1));
  std::mt19937_64 rng(seed);
  auto su = [&rng]() { return static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5; };
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        double x = i * hx, y = j * hy, z = k * hz;
        const double u0 = su(), u1 = su(), u2 = su();
        if (distortion > 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
          x += distortion * hx * u0;
          y += distortion * hy * u1;
          z += distortion * hz * u2;
        }
        double* dst = &nodes[3 * ((k * sy + j) * sx + i)];
        dst[0] = x;
        dst[1] = y;
        dst[2] = z;
      }

  // Two prisms per cell (geometry.cpp:169-190): element 2c+0 = (n00, n10,
  // n11 | m00, m10, m11), element 2c+1 = (n00, n11, n01 | m00, m11, m01).
  double g[18];
  for (int64_t e = first; e < first + count; ++e) {
    const int64_t cell = e >> 1;
    const int i = static_cast<int>(cell % nx), j = static_cast<int>((cell / nx) % ny),
              k = static_cast<int>(cell / (static_cast<int64_t>(nx) * ny));
    auto node = [&](int di, int dj, int dk) { return &nodes[3 * (((k + dk) * sy + (j + dj)) * sx + (i + di))]; };
    const double* v[6];
    if ((e & 1) == 0) {
      v[0] = node(0, 0, 0); v[1] = node(1, 0, 0); v[2] = node(1, 1, 0);
      v[3] = node(0, 0, 1); v[4] = node(1, 0, 1); v[5] = node(1, 1, 1);
    } else {
      v[0] = node(0, 0, 0); v[1] = node(1, 1, 0); v[2] = node(0, 1, 0);
      v[3] = node(0, 0, 1); v[4] = node(1, 1, 1); v[5] = node(0, 1, 1);
    }
    for (int a = 0; a < 6; ++a) std::memcpy(g + 3 * a, v[a], 3 * sizeof(double));
    const int64_t le = e - first;
    if (soa) {
      for (int c = 0; c < 18; ++c) out[c * ld + le] = g[c];
    } else {
      std::memcpy(out + 18 * le, g, sizeof g);
    }
    if (validate) {
      // Densest rule check (geometry.cpp:192-199).
      static thread_local std::vector<double> pts, wts;
      if (pts.empty()) {
        pts.resize(3 * pib::quad_count(pib::kMaxP));
        wts.resize(pib::quad_count(pib::kMaxP));
        pib::prism_quadrature(pib::kMaxP, pts.data(), wts.data());
      }
      for (int q = 0; q < pib::quad_count(pib::kMaxP); ++q) {
        double det, inv[9];
        if (!pib::jacobian_terms(g, &pts[3 * q], det, inv)) {
          if (err) {
            err->element = e;
            err->det = det;
            std::memcpy(err->xi, &pts[3 * q], sizeof err->xi);
          }
          return pib::set_error(err, PI_E_INVERTED_ELEMENT, "inverted element %lld: det=%g", (long long)e, det);
        }
      }
    }
  }
  return PI_OK;
}

pi_status pi_generate_cdr_coefficients(uint64_t seed, int64_t first, int64_t count, int soa, int64_t ld,
                                       double* out, pi_error_info* err) {
  if (first < 0 || count < 0) return pib::set_error(err, PI_E_CONTRACT, "cdr coefficients: bad range");
  if (soa && ld < count) return pib::set_error(err, PI_E_CONTRACT, "cdr coefficients: ld < count");
  const uint64_t key = pib::mix64(seed ^ 0x43445231ull);  // "CDR1"
  for (int64_t le = 0; le < count; ++le) {
    const int64_t g = first + le;
    double u[10];
    for (int i = 0; i < 10; ++i) u[i] = pib::unit_draw(key, g, i);
    const double lam[3] = {0.5 + 1.5 * u[0], 0.5 + 1.5 * u[1], 0.5 + 1.5 * u[2]};
    // Uniform random rotation from a unit quaternion (Shoemake).
    const double r1 = std::sqrt(1.0 - u[3]), r2 = std::sqrt(u[3]);
    const double t1 = 2.0 * M_PI * u[4], t2 = 2.0 * M_PI * u[5];
    const double qx = r1 * std::sin(t1), qy = r1 * std::cos(t1), qz = r2 * std::sin(t2), qw = r2 * std::cos(t2);
    const double R[3][3] = {
        {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw)},
        {2 * (qx * qy + qz * qw), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw)},
        {2 * (qx * qz - qy * qw), 2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)}};
    double c[16] = {0};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += R[i][k] * lam[k] * R[j][k];
        c[(1 + i) * 4 + (1 + j)] = s;
      }
    for (int d = 0; d < 3; ++d) c[0 * 4 + (1 + d)] = 2.0 * u[6 + d] - 1.0;  // convection b
    c[0] = u[9];                                                           // reaction r
    if (soa) {
      for (int k = 0; k < 16; ++k) out[k * ld + le] = c[k];
    } else {
      std::memcpy(out + 16 * le, c, sizeof c);
    }
  }
  return PI_OK;
}

}  // extern "C"
