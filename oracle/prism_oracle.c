/* oracle/prism_oracle.c -- TEST INFRASTRUCTURE ONLY (see prism_oracle.h).
 *
 * Scalar C restatement of the reference arithmetic.  Loop orders and
 * expression shapes follow the cited reference lines so that, compiled with
 * -ffp-contract=off, results are bitwise equal to the reference built with its
 * default flags (checked by tests/test_oracle.py).  This is the checker, not
 * the product.
 */
#include "prism_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PO_MAXP 7

int po_shape_count(int p) {
  if (p < 1 || p > PO_MAXP) return -1;
  return (p + 1) * (p + 1) * (p + 2) / 2;
}

int po_quadrature_point_count(int p) {
  static const int counts[PO_MAXP + 1] = {0, 6, 18, 48, 80, 150, 231, 336};
  if (p < 1 || p > PO_MAXP) return -1;
  return counts[p];
}

/* legendre_value_and_derivative, reference_element.cpp:207-228 */
static void legendre(int k, double x, double* val, double* der) {
  if (k == 0) {
    *val = 1.0;
    *der = 0.0;
    return;
  }
  double pm1 = 1.0, p = x;
  for (int i = 2; i <= k; ++i) {
    const double pnew = ((2.0 * i - 1.0) * x * p - (i - 1.0) * pm1) / i;
    pm1 = p;
    p = pnew;
  }
  const double denom = x * x - 1.0;
  if (fabs(denom) > 1e-10) {
    *der = k * (x * p - pm1) / denom;
  } else {
    *der = k * (k + 1.0) / 2.0 * (x > 0 ? 1.0 : (k % 2 == 0 ? -1.0 : 1.0));
  }
  *val = p;
}

/* gauss_legendre_1d, reference_element.cpp:37-69 */
int po_gauss_legendre(int n, double* points, double* weights) {
  if (n < 1) return -1;
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = -cos(M_PI * (4.0 * i + 3.0) / (4.0 * n + 2.0));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double value, deriv;
      legendre(n, x, &value, &deriv);
      dp = deriv;
      const double dx = value / deriv;
      x -= dx;
      if (fabs(dx) < 1e-15) {
        double v2, d2;
        legendre(n, x, &v2, &d2);
        dp = d2;
        break;
      }
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    points[i] = x;
    weights[i] = w;
    points[n - 1 - i] = -x;
    weights[n - 1 - i] = w;
  }
  if (n % 2 == 1) points[n / 2] = 0.0;
  return 0;
}

/* Symmetric-orbit helpers, reference_element.cpp:90-108. */
static int push_centroid(double* pts, double* wts, int n, double w) {
  pts[2 * n] = 1.0 / 3.0;
  pts[2 * n + 1] = 1.0 / 3.0;
  wts[n] = w;
  return n + 1;
}

static int push_orbit3(double* pts, double* wts, int n, double a, double w) {
  const double c = 1.0 - 2.0 * a;
  const double xy[3][2] = {{a, c}, {a, a}, {c, a}};
  for (int k = 0; k < 3; ++k) {
    pts[2 * (n + k)] = xy[k][0];
    pts[2 * (n + k) + 1] = xy[k][1];
    wts[n + k] = w;
  }
  return n + 3;
}

static int push_orbit6(double* pts, double* wts, int n, double a, double b, double w) {
  const double c = 1.0 - a - b;
  const double xy[6][2] = {{b, c}, {c, b}, {a, c}, {c, a}, {a, b}, {b, a}};
  for (int k = 0; k < 6; ++k) {
    pts[2 * (n + k)] = xy[k][0];
    pts[2 * (n + k) + 1] = xy[k][1];
    wts[n + k] = w;
  }
  return n + 6;
}

/* triangle_rule, reference_element.cpp:110-173.  Dunavant orbit data for the
 * unit-area triangle, scaled by the reference area s = 1/2. */
int po_triangle_rule(int degree, double* P, double* W) {
  const double s = 0.5;
  int n = 0;
  switch (degree) {
    case 2:
      n = push_orbit3(P, W, n, 1.0 / 6.0, 1.0 / 6.0);
      break;
    case 4:
      n = push_orbit3(P, W, n, 0.44594849091596488631832925388305, 0.22338158967801146569500700843312 * s);
      n = push_orbit3(P, W, n, 0.09157621350977074345957146340220, 0.10995174365532186763832632490021 * s);
      break;
    case 6:
      n = push_orbit3(P, W, n, 0.24928674517091042129163855310702, 0.11678627572637936602528961138558 * s);
      n = push_orbit3(P, W, n, 0.06308901449150222834033160287082, 0.05084490637020681692093680910686 * s);
      n = push_orbit6(P, W, n, 0.31035245103378440541660773395655, 0.63650249912139864723014259441205,
                      0.08285107561837357519355345642044 * s);
      break;
    case 8:
      n = push_centroid(P, W, n, 0.14431560767778716825109111048906 * s);
      n = push_orbit3(P, W, n, 0.17056930775176020662229350149146, 0.10321737053471825028179155029212 * s);
      n = push_orbit3(P, W, n, 0.05054722831703097545842355059660, 0.03245849762319808031092592834178 * s);
      n = push_orbit3(P, W, n, 0.45929258829272315602881551449417, 0.09509163426728462479389610438858 * s);
      n = push_orbit6(P, W, n, 0.26311282963463811342178578628464, 0.72849239295540428124100037917606,
                      0.02723031417443499426484469007390 * s);
      break;
    case 10:
      n = push_centroid(P, W, n, 0.090817990382754 * s);
      n = push_orbit3(P, W, n, 0.485577633383657, 0.036725957756467 * s);
      n = push_orbit3(P, W, n, 0.109481575485037, 0.045321059435528 * s);
      n = push_orbit6(P, W, n, 0.141707219414880, 0.307939838764121, 0.072757916845420 * s);
      n = push_orbit6(P, W, n, 0.025003534762686, 0.246672560639903, 0.028327242531057 * s);
      n = push_orbit6(P, W, n, 0.009540815400299, 0.066803251012200, 0.009421666963733 * s);
      break;
    case 12:
      n = push_orbit3(P, W, n, 0.488217389773805, 0.025731066440455 * s);
      n = push_orbit3(P, W, n, 0.439724392294460, 0.043692544538038 * s);
      n = push_orbit3(P, W, n, 0.271210385012116, 0.062858224217885 * s);
      n = push_orbit3(P, W, n, 0.127576145541586, 0.034796112930709 * s);
      n = push_orbit3(P, W, n, 0.021317350453210, 0.006166261051559 * s);
      n = push_orbit6(P, W, n, 0.115343494534698, 0.275713269685514, 0.040371557766381 * s);
      n = push_orbit6(P, W, n, 0.022838332222257, 0.281325580989940, 0.022356773202303 * s);
      n = push_orbit6(P, W, n, 0.025734050548330, 0.116251915907597, 0.017316231108659 * s);
      break;
    case 14:
      n = push_orbit3(P, W, n, 0.488963910362179, 0.021883581369429 * s);
      n = push_orbit3(P, W, n, 0.417644719340454, 0.032788353544125 * s);
      n = push_orbit3(P, W, n, 0.273477528308839, 0.051774104507292 * s);
      n = push_orbit3(P, W, n, 0.177205532412543, 0.042162588736993 * s);
      n = push_orbit3(P, W, n, 0.061799883090873, 0.014433699669777 * s);
      n = push_orbit3(P, W, n, 0.019390961248701, 0.004923403602400 * s);
      n = push_orbit6(P, W, n, 0.057124757403648, 0.172266687821356, 0.024665753212564 * s);
      n = push_orbit6(P, W, n, 0.092916249356972, 0.336861459796345, 0.038571510787061 * s);
      n = push_orbit6(P, W, n, 0.014646950055654, 0.298372882136258, 0.014436308113534 * s);
      n = push_orbit6(P, W, n, 0.001268330932872, 0.118974497696957, 0.005010228838501 * s);
      break;
    default:
      return -1;
  }
  return n;
}

/* prism_quadrature, reference_element.cpp:175-193: vertical level outer,
 * triangle index fastest, weight = w_tri * w_line. */
int po_prism_quadrature(int p, double* points, double* weights) {
  if (p < 1 || p > PO_MAXP) return -1;
  double tp[2 * 64], tw[64], lp[16], lw[16];
  const int nt = po_triangle_rule(2 * p, tp, tw);
  po_gauss_legendre(p + 1, lp, lw);
  int q = 0;
  for (int iz = 0; iz < p + 1; ++iz) {
    for (int it = 0; it < nt; ++it) {
      points[3 * q + 0] = tp[2 * it];
      points[3 * q + 1] = tp[2 * it + 1];
      points[3 * q + 2] = lp[iz];
      weights[q] = tw[it] * lw[iz];
      ++q;
    }
  }
  return q;
}

/* shape_values, reference_element.cpp:230-270 (monomials :195-205). */
int po_shape_values(int p, const double* xi, double* out) {
  const int nsh = po_shape_count(p);
  const int nv = p + 1;
  double pow1[PO_MAXP + 1], pow2[PO_MAXP + 1], leg[PO_MAXP + 1], dleg[PO_MAXP + 1];
  pow1[0] = pow2[0] = 1.0;
  for (int i = 1; i <= p; ++i) {
    pow1[i] = pow1[i - 1] * xi[0];
    pow2[i] = pow2[i - 1] * xi[1];
  }
  for (int k = 0; k < nv; ++k) legendre(k, xi[2], &leg[k], &dleg[k]);
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
  return 0;
}

/* tabulate_shapes, reference_element.cpp:272-286 */
int po_tabulate_shapes(int p, double* table) {
  const int nq = po_quadrature_point_count(p), nsh = po_shape_count(p);
  if (nq < 0) return -1;
  double* pts = (double*)malloc(sizeof(double) * 3 * nq);
  double* w = (double*)malloc(sizeof(double) * nq);
  po_prism_quadrature(p, pts, w);
  for (int q = 0; q < nq; ++q) po_shape_values(p, pts + 3 * q, table + (size_t)q * 4 * nsh);
  free(pts);
  free(w);
  return 0;
}

/* geometry_shape_derivs + jacobian_matrix + jacobian_terms,
 * geometry.cpp:32-83.  Returns 1 if det <= 0 (InvertedElementError). */
int po_jacobian_terms(const double* x, const double* xi, double* det_out, double* inv) {
  const double l0 = 1.0 - xi[0] - xi[1];
  const double l1 = xi[0];
  const double l2 = xi[1];
  const double zm = 0.5 * (1.0 - xi[2]);
  const double zp = 0.5 * (1.0 + xi[2]);
  const double dn[3][6] = {{-zm, zm, 0.0, -zp, zp, 0.0},
                           {-zm, 0.0, zm, -zp, 0.0, zp},
                           {-0.5 * l0, -0.5 * l1, -0.5 * l2, 0.5 * l0, 0.5 * l1, 0.5 * l2}};
  double j[3][3];
  for (int i = 0; i < 3; ++i) {
    for (int c = 0; c < 3; ++c) {
      double sum = 0.0;
      for (int v = 0; v < 6; ++v) sum += dn[c][v] * x[v * 3 + i];
      j[i][c] = sum;
    }
  }
  const double c00 = j[1][1] * j[2][2] - j[1][2] * j[2][1];
  const double c01 = j[1][2] * j[2][0] - j[1][0] * j[2][2];
  const double c02 = j[1][0] * j[2][1] - j[1][1] * j[2][0];
  const double det = j[0][0] * c00 + j[0][1] * c01 + j[0][2] * c02;
  *det_out = det;
  if (!(det > 0.0)) return 1;
  const double c10 = j[0][2] * j[2][1] - j[0][1] * j[2][2];
  const double c11 = j[0][0] * j[2][2] - j[0][2] * j[2][0];
  const double c12 = j[0][1] * j[2][0] - j[0][0] * j[2][1];
  const double c20 = j[0][1] * j[1][2] - j[0][2] * j[1][1];
  const double c21 = j[0][2] * j[1][0] - j[0][0] * j[1][2];
  const double c22 = j[0][0] * j[1][1] - j[0][1] * j[1][0];
  const double id = 1.0 / det;
  inv[0] = c00 * id; inv[1] = c10 * id; inv[2] = c20 * id;
  inv[3] = c01 * id; inv[4] = c11 * id; inv[5] = c21 * id;
  inv[6] = c02 * id; inv[7] = c12 * id; inv[8] = c22 * id;
  return 0;
}

/* integrate_generic, integrate_ref.cpp:50-91, with physical_derivatives
 * (geometry.cpp:85-102) and sparse_terms (integrate_ref.cpp:20-34). */
int po_integrate_generic(int p, int n_eq, const double* geom, const double* coeff, double* out,
                         int* bad_point) {
  const int nsh = po_shape_count(p), nq = po_quadrature_point_count(p);
  if (nsh < 0 || n_eq < 1) return -1;
  const int dim = n_eq * nsh;
  double* pts = (double*)malloc(sizeof(double) * 3 * nq);
  double* w = (double*)malloc(sizeof(double) * nq);
  double* phi = (double*)malloc(sizeof(double) * 4 * nsh);
  double* psi = (double*)malloc(sizeof(double) * 4 * nsh);
  int* ti = (int*)malloc(sizeof(int) * 4 * 16 * n_eq * n_eq);
  double* tv = (double*)malloc(sizeof(double) * 16 * n_eq * n_eq);
  po_prism_quadrature(p, pts, w);
  memset(out, 0, sizeof(double) * (size_t)dim * dim);

  /* sparse_terms: (i_D, j_D, i_E, j_E) order, nonzero entries only. */
  int nt = 0;
  for (int id = 0; id < 4; ++id)
    for (int jd = 0; jd < 4; ++jd)
      for (int ie = 0; ie < n_eq; ++ie)
        for (int je = 0; je < n_eq; ++je) {
          const double c = coeff[((ie * n_eq + je) * 4 + id) * 4 + jd];
          if (c != 0.0) {
            ti[4 * nt + 0] = ie; ti[4 * nt + 1] = je; ti[4 * nt + 2] = id; ti[4 * nt + 3] = jd;
            tv[nt++] = c;
          }
        }

  int rc = 0;
  for (int q = 0; q < nq; ++q) {
    double det, inv[9];
    if (po_jacobian_terms(geom, pts + 3 * q, &det, inv)) {
      if (bad_point) *bad_point = q;
      rc = 1;
      break;
    }
    po_shape_values(p, pts + 3 * q, phi);
    for (int dof = 0; dof < nsh; ++dof) psi[dof] = phi[dof];
    for (int i = 0; i < 3; ++i)
      for (int dof = 0; dof < nsh; ++dof) {
        double sum = 0.0;
        for (int k = 0; k < 3; ++k) sum += phi[(k + 1) * nsh + dof] * inv[k * 3 + i];
        psi[(i + 1) * nsh + dof] = sum;
      }
    const double dw = det * w[q];
    for (int i = 0; i < nsh; ++i)
      for (int jj = 0; jj < nsh; ++jj)
        for (int t = 0; t < nt; ++t) {
          const int ie = ti[4 * t], je = ti[4 * t + 1], id = ti[4 * t + 2], jd = ti[4 * t + 3];
          out[(size_t)(i * n_eq + ie) * dim + jj * n_eq + je] +=
              dw * tv[t] * psi[id * nsh + i] * psi[jd * nsh + jj];
        }
  }
  free(pts); free(w); free(phi); free(psi); free(ti); free(tv);
  return rc;
}

int po_load_vector(int p, const double* geom, double f, double* out) {
  const int nsh = po_shape_count(p), nq = po_quadrature_point_count(p);
  if (nsh < 0) return -1;
  double* pts = (double*)malloc(sizeof(double) * 3 * nq);
  double* w = (double*)malloc(sizeof(double) * nq);
  double* phi = (double*)malloc(sizeof(double) * 4 * nsh);
  po_prism_quadrature(p, pts, w);
  memset(out, 0, sizeof(double) * nsh);
  int rc = 0;
  for (int q = 0; q < nq; ++q) {
    double det, inv[9];
    if (po_jacobian_terms(geom, pts + 3 * q, &det, inv)) { rc = 1; break; }
    po_shape_values(p, pts + 3 * q, phi);
    const double dw = det * w[q];
    /* Same expression shape as the mass-matrix column i,0 of integrate_generic:
     * ((dw * f) * phi_i) * phi_0 with phi_0 == 1. */
    for (int i = 0; i < nsh; ++i) out[i] += dw * f * phi[i] * phi[0];
  }
  free(pts); free(w); free(phi);
  return rc;
}

/* ---- std::mt19937_64 (the C++ standard's parameters) ---- */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* signed_unit, geometry.cpp:127-130 */
static double signed_unit(mt64* s) {
  const double u = (double)(mt64_next(s) >> 11) * 0x1.0p-53;
  return u - 0.5;
}

/* generate_box_mesh, geometry.cpp:134-190 */
int po_generate_box_mesh(int nx, int ny, int nz, double distortion, uint64_t seed, double* out) {
  if (nx < 1 || ny < 1 || nz < 1 || distortion < 0.0 || distortion >= 0.3) return -1;
  const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
  const size_t nn = (size_t)(nx + 1) * (ny + 1) * (nz + 1);
  double* nodes = (double*)malloc(sizeof(double) * 3 * nn);
  mt64* rng = (mt64*)malloc(sizeof(mt64));
  mt64_seed(rng, seed);
#define NODE(i, j, k) ((((size_t)(k) * (ny + 1) + (j)) * (nx + 1) + (i)))
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        double pnt[3] = {i * hx, j * hy, k * hz};
        const double u0 = signed_unit(rng), u1 = signed_unit(rng), u2 = signed_unit(rng);
        if (distortion > 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
          pnt[0] += distortion * hx * u0;
          pnt[1] += distortion * hy * u1;
          pnt[2] += distortion * hz * u2;
        }
        memcpy(nodes + 3 * NODE(i, j, k), pnt, sizeof pnt);
      }
  size_t e = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const size_t n00 = NODE(i, j, k), n10 = NODE(i + 1, j, k), n01 = NODE(i, j + 1, k),
                     n11 = NODE(i + 1, j + 1, k), m00 = NODE(i, j, k + 1), m10 = NODE(i + 1, j, k + 1),
                     m01 = NODE(i, j + 1, k + 1), m11 = NODE(i + 1, j + 1, k + 1);
        const size_t a[6] = {n00, n10, n11, m00, m10, m11};
        const size_t b[6] = {n00, n11, n01, m00, m11, m01};
        for (int v = 0; v < 6; ++v) memcpy(out + (e * 6 + v) * 3, nodes + 3 * a[v], 3 * sizeof(double));
        ++e;
        for (int v = 0; v < 6; ++v) memcpy(out + (e * 6 + v) * 3, nodes + 3 * b[v], 3 * sizeof(double));
        ++e;
      }
#undef NODE
  free(nodes);
  free(rng);
  return 0;
}

/* lame_parameters + elasticity_tensor, coefficients.cpp:23-59 */
int po_elasticity_tensor(double young, double nu, double* out) {
  if (young <= 0.0 || nu <= -1.0 || nu >= 0.5) return -1;
  const double mu = young / (2.0 * (1.0 + nu));
  const double lambda = young * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  memset(out, 0, sizeof(double) * 144);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) {
          double c = 0.0;
          if (i == j && k == l) c += lambda;
          if (i == k && j == l) c += mu;
          if (i == l && k == j) c += mu;
          if (c != 0.0) out[((i * 3 + k) * 4 + (j + 1)) * 4 + (l + 1)] = c;
        }
  return 0;
}
