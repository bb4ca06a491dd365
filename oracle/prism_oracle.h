/* oracle/prism_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (prismint) arithmetic on the hot path:
 * quadrature, shape tabulation, Jacobian terms, integrate_generic, and the
 * synthetic box mesh.  Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).  Parity pinned: tests/test_oracle.py
 * checks it against the golden vectors in tests/golden/ (made by running the
 * reference itself, oracle/_ref) and against exact polynomial integrals.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product
 * (paper_1310_1191_b200/) never links it.
 */
#ifndef PRISM_ORACLE_H
#define PRISM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int po_shape_count(int p);            /* reference_element.cpp:19-22 */
int po_quadrature_point_count(int p); /* reference_element.cpp:24-28 */

/* gauss_legendre_1d, reference_element.cpp:37-69 */
int po_gauss_legendre(int n, double* x, double* w);
/* triangle_rule, reference_element.cpp:110-173; returns point count or -1 */
int po_triangle_rule(int degree, double* pts /*[n][2]*/, double* wts);
/* prism_quadrature, reference_element.cpp:175-193; returns nq or -1 */
int po_prism_quadrature(int p, double* points /*[nq][3]*/, double* weights);
/* shape_values / tabulate_shapes, reference_element.cpp:230-286 */
int po_shape_values(int p, const double* xi, double* out /*[4][nsh]*/);
int po_tabulate_shapes(int p, double* table /*[nq][4][nsh]*/);

/* jacobian_terms, geometry.cpp:45-83.  Returns 0, or 1 if det <= 0. */
int po_jacobian_terms(const double* geom /*[6][3]*/, const double* xi, double* det,
                      double* inv /*[3][3]*/);

/* integrate_generic, integrate_ref.cpp:50-91, element-constant coefficients
 * c[n_eq][n_eq][4][4].  out: canonical dense [dim][dim], dim = n_eq*nsh.
 * Returns 0, or 1 (inverted element; *bad_xi_index = quadrature point). */
int po_integrate_generic(int p, int n_eq, const double* geom, const double* coeff, double* out,
                         int* bad_point);

/* Load vector F_i = sum_q dw_q f phi_i(x_q) for constant f (no reference
 * counterpart).  Equals f * M[i][0] of integrate_generic with
 * c[0][0][0][0] = 1, since phi_0 == 1. */
int po_load_vector(int p, const double* geom, double f, double* out /*[nsh]*/);

/* generate_box_mesh, geometry.cpp:123-201 (without the p=7 validation pass).
 * out: [2*nx*ny*nz][6][3]. */
int po_generate_box_mesh(int nx, int ny, int nz, double distortion, uint64_t seed, double* out);

/* elasticity_tensor, coefficients.cpp:23-59; out [3][3][4][4]. */
int po_elasticity_tensor(double young, double nu, double* out);

#ifdef __cplusplus
}
#endif
#endif
