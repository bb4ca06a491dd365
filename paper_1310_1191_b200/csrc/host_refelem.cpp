// Host-side per-p constants: the prism quadrature rule and the shape table.
//
// B200 design note: these are one-off, per-p inputs (<= 3.1 MB at p = 7) that
// are uploaded once per context; they are computed here in FP64 with the same
// formulas and operation order as the reference so the device sees the
// identical constants (checked bitwise against the reference in
// tests/test_host.py).
#include <cmath>
#include <cstring>
#include <vector>

#include "pi_internal.hpp"

namespace pib {

int shape_count(int p) { return (p < 1 || p > kMaxP) ? -1 : (p + 1) * (p + 1) * (p + 2) / 2; }

int quad_count(int p) {
  static const int counts[kMaxP + 1] = {0, 6, 18, 48, 80, 150, 231, 336};
  return (p < 1 || p > kMaxP) ? -1 : counts[p];
}

int tri_point_count(int p) {
  static const int counts[kMaxP + 1] = {0, 3, 6, 12, 16, 25, 33, 42};
  return (p < 1 || p > kMaxP) ? -1 : counts[p];
}

// P_k and P_k' by the three-term recurrence (reference_element.cpp:207-228).
void legendre(int k, double x, double& val, double& der) {
  if (k == 0) {
    val = 1.0;
    der = 0.0;
    return;
  }
  double pm1 = 1.0, pk = x;
  for (int i = 2; i <= k; ++i) {
    const double pn = ((2.0 * i - 1.0) * x * pk - (i - 1.0) * pm1) / i;
    pm1 = pk;
    pk = pn;
  }
  const double denom = x * x - 1.0;
  der = std::fabs(denom) > 1e-10 ? k * (x * pk - pm1) / denom
                                 : k * (k + 1.0) / 2.0 * (x > 0 ? 1.0 : (k % 2 == 0 ? -1.0 : 1.0));
  val = pk;
}

// Newton on P_n from the Chebyshev-like guess (reference_element.cpp:37-69).
void gauss_legendre(int n, double* x, double* w) {
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double xi = -std::cos(M_PI * (4.0 * i + 3.0) / (4.0 * n + 2.0));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double v, d;
      legendre(n, xi, v, d);
      dp = d;
      const double dx = v / d;
      xi -= dx;
      if (std::fabs(dx) < 1e-15) {
        legendre(n, xi, v, d);
        dp = d;
        break;
      }
    }
    const double wi = 2.0 / ((1.0 - xi * xi) * dp * dp);
    x[i] = xi;
    w[i] = wi;
    x[n - 1 - i] = -xi;
    w[n - 1 - i] = wi;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

namespace {

struct TriRule {
  std::vector<double> xy, w;
  void centroid(double wt) {
    xy.insert(xy.end(), {1.0 / 3.0, 1.0 / 3.0});
    w.push_back(wt);
  }
  void orbit3(double a, double wt) {
    const double c = 1.0 - 2.0 * a;
    xy.insert(xy.end(), {a, c, a, a, c, a});
    w.insert(w.end(), {wt, wt, wt});
  }
  void orbit6(double a, double b, double wt) {
    const double c = 1.0 - a - b;
    xy.insert(xy.end(), {b, c, c, b, a, c, c, a, a, b, b, a});
    w.insert(w.end(), 6, wt);
  }
};

// Symmetric (Dunavant) triangle rules of degree 2..14, unit-area orbit weights
// scaled by the reference area 1/2 (reference_element.cpp:110-173).
bool triangle_rule(int degree, TriRule& r) {
  const double s = 0.5;
  switch (degree) {
    case 2:
      r.orbit3(1.0 / 6.0, 1.0 / 6.0);
      return true;
    case 4:
      r.orbit3(0.44594849091596488631832925388305, 0.22338158967801146569500700843312 * s);
      r.orbit3(0.09157621350977074345957146340220, 0.10995174365532186763832632490021 * s);
      return true;
    case 6:
      r.orbit3(0.24928674517091042129163855310702, 0.11678627572637936602528961138558 * s);
      r.orbit3(0.06308901449150222834033160287082, 0.05084490637020681692093680910686 * s);
      r.orbit6(0.31035245103378440541660773395655, 0.63650249912139864723014259441205,
               0.08285107561837357519355345642044 * s);
      return true;
    case 8:
      r.centroid(0.14431560767778716825109111048906 * s);
      r.orbit3(0.17056930775176020662229350149146, 0.10321737053471825028179155029212 * s);
      r.orbit3(0.05054722831703097545842355059660, 0.03245849762319808031092592834178 * s);
      r.orbit3(0.45929258829272315602881551449417, 0.09509163426728462479389610438858 * s);
      r.orbit6(0.26311282963463811342178578628464, 0.72849239295540428124100037917606,
               0.02723031417443499426484469007390 * s);
      return true;
    case 10:
      r.centroid(0.090817990382754 * s);
      r.orbit3(0.485577633383657, 0.036725957756467 * s);
      r.orbit3(0.109481575485037, 0.045321059435528 * s);
      r.orbit6(0.141707219414880, 0.307939838764121, 0.072757916845420 * s);
      r.orbit6(0.025003534762686, 0.246672560639903, 0.028327242531057 * s);
      r.orbit6(0.009540815400299, 0.066803251012200, 0.009421666963733 * s);
      return true;
    case 12:
      r.orbit3(0.488217389773805, 0.025731066440455 * s);
      r.orbit3(0.439724392294460, 0.043692544538038 * s);
      r.orbit3(0.271210385012116, 0.062858224217885 * s);
      r.orbit3(0.127576145541586, 0.034796112930709 * s);
      r.orbit3(0.021317350453210, 0.006166261051559 * s);
      r.orbit6(0.115343494534698, 0.275713269685514, 0.040371557766381 * s);
      r.orbit6(0.022838332222257, 0.281325580989940, 0.022356773202303 * s);
      r.orbit6(0.025734050548330, 0.116251915907597, 0.017316231108659 * s);
      return true;
    case 14:
      r.orbit3(0.488963910362179, 0.021883581369429 * s);
      r.orbit3(0.417644719340454, 0.032788353544125 * s);
      r.orbit3(0.273477528308839, 0.051774104507292 * s);
      r.orbit3(0.177205532412543, 0.042162588736993 * s);
      r.orbit3(0.061799883090873, 0.014433699669777 * s);
      r.orbit3(0.019390961248701, 0.004923403602400 * s);
      r.orbit6(0.057124757403648, 0.172266687821356, 0.024665753212564 * s);
      r.orbit6(0.092916249356972, 0.336861459796345, 0.038571510787061 * s);
      r.orbit6(0.014646950055654, 0.298372882136258, 0.014436308113534 * s);
      r.orbit6(0.001268330932872, 0.118974497696957, 0.005010228838501 * s);
      return true;
    default:
      return false;
  }
}

}  // namespace

bool prism_quadrature(int p, double* points, double* weights) {
  if (p < 1 || p > kMaxP) return false;
  TriRule tri;
  if (!triangle_rule(2 * p, tri)) return false;
  double lx[kMaxP + 1], lw[kMaxP + 1];
  gauss_legendre(p + 1, lx, lw);
  const int nt = static_cast<int>(tri.w.size());
  int q = 0;
  for (int iz = 0; iz <= p; ++iz) {  // vertical level outer, triangle index fastest
    for (int it = 0; it < nt; ++it, ++q) {
      points[3 * q + 0] = tri.xy[2 * it];
      points[3 * q + 1] = tri.xy[2 * it + 1];
      points[3 * q + 2] = lx[iz];
      weights[q] = tri.w[it] * lw[iz];
    }
  }
  return true;
}

// Monomial x Legendre basis, dof = tri * (p+1) + k (reference_element.cpp:230-270).
void shape_values(int p, const double* xi, double* out) {
  const int nsh = shape_count(p), nv = p + 1;
  double pow1[kMaxP + 1], pow2[kMaxP + 1], leg[kMaxP + 1], dleg[kMaxP + 1];
  pow1[0] = pow2[0] = 1.0;
  for (int i = 1; i <= p; ++i) {
    pow1[i] = pow1[i - 1] * xi[0];
    pow2[i] = pow2[i - 1] * xi[1];
  }
  for (int k = 0; k < nv; ++k) legendre(k, xi[2], leg[k], dleg[k]);
  int it = 0;
  for (int d = 0; d <= p; ++d) {
    for (int a = 0; a <= d; ++a, ++it) {
      const int b = d - a;
      const double m = pow1[a] * pow2[b];
      const double dm1 = a > 0 ? a * pow1[a - 1] * pow2[b] : 0.0;
      const double dm2 = b > 0 ? b * pow1[a] * pow2[b - 1] : 0.0;
      for (int k = 0; k < nv; ++k) {
        const int dof = it * nv + k;
        out[0 * nsh + dof] = m * leg[k];
        out[1 * nsh + dof] = dm1 * leg[k];
        out[2 * nsh + dof] = dm2 * leg[k];
        out[3 * nsh + dof] = m * dleg[k];
      }
    }
  }
}

}  // namespace pib

extern "C" {

int pi_shape_count(int p) { return pib::shape_count(p); }
int pi_quadrature_point_count(int p) { return pib::quad_count(p); }

pi_status pi_prism_quadrature(int p, double* points, double* weights, pi_error_info* err) {
  if (p < 1 || p > pib::kMaxP)
    return pib::set_error(err, PI_E_DOMAIN, "approximation order p=%d outside supported range [1, 7]", p);
  pib::prism_quadrature(p, points, weights);
  return PI_OK;
}

pi_status pi_tabulate_shapes(int p, const double* points, int n_q, double* table, pi_error_info* err) {
  if (p < 1 || p > pib::kMaxP)
    return pib::set_error(err, PI_E_DOMAIN, "approximation order p=%d outside supported range [1, 7]", p);
  std::vector<double> own;
  if (!points) {
    own.resize(3 * pib::quad_count(p));
    std::vector<double> w(pib::quad_count(p));
    pib::prism_quadrature(p, own.data(), w.data());
    points = own.data();
    n_q = pib::quad_count(p);
  }
  const int nsh = pib::shape_count(p);
  for (int q = 0; q < n_q; ++q) pib::shape_values(p, points + 3 * q, table + static_cast<size_t>(q) * 4 * nsh);
  return PI_OK;
}

}  // extern "C"
