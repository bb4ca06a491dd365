/* include/prism_b200.h -- C ABI of the B200-native prismatic element integrator.
 *
 * The hot path of arXiv 1310.1191 (reference implementation `prismint`,
 * /root/reference/proj): element stiffness matrices (and load vectors) for
 * p = 1..7 prisms, integrated on sm_100a.  Every entry point below names the
 * reference interface it replaces (file:line, relative to proj/).  No C++ or
 * torch types cross this boundary: plain pointers, sizes and status codes.
 *
 * Conventions
 *  - The caller owns every buffer; the library never frees or retains them.
 *  - Device-pointer calls are asynchronous on the given CUDA stream (NULL =
 *    the context's own stream).  Errors raised inside a kernel (inverted
 *    element) surface on pi_check() / any host-buffer call, reporting the
 *    LOWEST offending global element id, like integrate_generic would have
 *    thrown for it first (integrate_ref.cpp:72-75, kernels.cpp:158,249).
 *  - A context is bound to one device and one (p, n_eq), n_eq = 1 (scalar
 *    weak forms) or 3 (systems: elasticity); it is not thread-safe; use one
 *    per device / host thread.
 */
#ifndef PRISM_B200_H
#define PRISM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors prismint::errc order (errors.hpp:10-19) plus CUDA. */
typedef enum {
  PI_OK = 0,
  PI_E_CONFIG = 1,             /* ConfigError */
  PI_E_DOMAIN = 2,             /* DomainError */
  PI_E_UNSUPPORTED_DEGREE = 3, /* UnsupportedDegreeError */
  PI_E_INVERTED_ELEMENT = 4,   /* InvertedElementError(element, xi, det) */
  PI_E_CAPACITY = 5,           /* CapacityError */
  PI_E_SHARED_MEMORY = 6,      /* SharedMemoryError */
  PI_E_CONTRACT = 7,           /* ContractViolation */
  PI_E_IO = 8,                 /* IoError */
  PI_E_CUDA = 9                /* CUDA runtime / launch failure */
} pi_status;

typedef struct {
  int64_t element;   /* global id of the first inverted element, else -1 */
  double det;        /* its Jacobian determinant at xi */
  double xi[3];      /* first failing quadrature point, in rule order */
  int cuda_error;    /* cudaError_t when status == PI_E_CUDA */
  char message[256];
} pi_error_info;

typedef struct pi_context pi_context;

/* Output layouts for stiffness matrices. */
enum {
  PI_OUT_CANONICAL = 0, /* [n_elem][dim][dim] row-major, row = i_dof*n_eq + i_eq
                           (ElementStiffness, integrate_ref.hpp:14-31) */
  PI_OUT_SOA = 1        /* [dim*dim][ld_out]: entry (r,c) of element e at (r*dim+c)*ld_out + e */
};

/* Coefficient modes (CoefficientTensor c[i_E][j_E][i_D][j_D], coefficients.hpp:12-24). */
enum {
  PI_COEFF_LAPLACE = 0,     /* c[0][0][d][d] = 1, d = 1..3 (test_integrate_ref.cpp:72-75); coeff == NULL */
  PI_COEFF_UNIFORM = 1,     /* one HOST tensor [n_eq*n_eq*16] for every element */
  PI_COEFF_PER_ELEMENT = 2, /* DEVICE SoA [n_eq*n_eq*16][ld]; entry k of element e at k*ld + e */
  /* n_eq = 3 isotropic linear elasticity, elasticity_tensor(MaterialData)
   * (coefficients.cpp:40-59) -- the reference's model problem and the material
   * input of its batch API (MaterialData per element, kernels.hpp:47-50): */
  PI_COEFF_ELASTICITY = 3,  /* DEVICE SoA [2][ld]: (young_E, poisson_nu) of element e at e, ld + e */
  PI_COEFF_ELASTICITY_UNIFORM = 4 /* HOST [2]: one (young_E, poisson_nu) for every element */
};

/* Kernel strategy selector (the role KernelVariant plays in planner.hpp:43-56). */
enum {
  PI_VARIANT_AUTO = 0,     /* best measured strategy for (p, n_eq, coefficients) */
  PI_VARIANT_DENSE = 1,    /* per-point B^T (dw C) B accumulation (the reference's loop nest) */
  PI_VARIANT_SUMFACT = 2,  /* tensor-product (sum-factorised) contraction on FP64 DMMA */
  PI_VARIANT_TC32 = 3      /* scalar forms, p = 3..7: FP32-output calls run the sum-factorised
                              contraction on the tcgen05 tensor cores (3xTF32, TMEM accumulators;
                              bound 5e-5, measured ~4e-7); FP64 calls as PI_VARIANT_SUMFACT */
};

/* ---- per-p constants: the product's own restatement of the reference ---- */
int pi_shape_count(int p);            /* shape_count, reference_element.cpp:19-22 */
int pi_quadrature_point_count(int p); /* quadrature_point_count, reference_element.cpp:24-28 */
/* prism_quadrature (reference_element.cpp:175-193): points [n_q][3], weights [n_q]. */
pi_status pi_prism_quadrature(int p, double* points, double* weights, pi_error_info* err);
/* tabulate_shapes (reference_element.cpp:272-286): table [n_q][4][n_shape]. */
pi_status pi_tabulate_shapes(int p, const double* points, int n_q, double* table, pi_error_info* err);

/* ---- synthetic inputs (not timed) ---- */
/* generate_box_mesh (geometry.cpp:134-201) for elements [first, first+count)
 * of the nx*ny*nz box, written as SoA [18][ld] (vertex-major (v*3+c)*ld + e)
 * when soa != 0, else AoS [count][6][3] (PrismGeometry order).  validate != 0
 * runs the reference's p=7 det > 0 check on the produced elements. */
pi_status pi_generate_box_mesh(int nx, int ny, int nz, double distortion, uint64_t seed,
                               int64_t first, int64_t count, int soa, int64_t ld, int validate,
                               double* out, pi_error_info* err);
/* Seeded per-element convection-diffusion-reaction tensors (SURVEY.md 8d,
 * config 3): D = Q diag(l) Q^T (l in U[0.5,2], Q a random rotation) at
 * [1..3][1..3], b in U[-1,1]^3 at [0][1..3], r in U[0,1] at [0][0].  Element
 * g uses its own counter-based stream (seed, g), so any range is
 * reproducible independently.  out: SoA [16][ld] (soa != 0) or AoS [count][16]. */
pi_status pi_generate_cdr_coefficients(uint64_t seed, int64_t first, int64_t count, int soa,
                                       int64_t ld, double* out, pi_error_info* err);

/* ---- contexts ---- */
/* Uploads the per-p constants (the reference's own rule and shape table may be
 * passed, as run_batch does via prism_quadrature/tabulate_shapes,
 * kernels.cpp:493-494); NULL tables => built internally. */
pi_status pi_context_create(int device, int p, int n_eq, int n_q, int n_shape, const double* points,
                            const double* weights, const double* shape_table, pi_context** out,
                            pi_error_info* err);
pi_status pi_context_destroy(pi_context* ctx);
pi_status pi_context_set_variant(pi_context* ctx, int variant, pi_error_info* err);
int pi_context_variant(const pi_context* ctx, int coeff_mode); /* resolved strategy */
void* pi_context_stream(pi_context* ctx);                         /* cudaStream_t */

/* ---- the hot path: device buffers, asynchronous ---- */
/* Batch integrate_generic (integrate_ref.cpp:50-91) over n_elem elements
 * with global ids element_id_base + e; the batch role of run_kernel /
 * run_batch (kernels.hpp:68-75).
 *   geom   device SoA [18][geom_ld]
 *   coeff  see PI_COEFF_*; coeff_ld is the SoA leading dimension
 *   out    device, layout per out_layout (ld_out used by PI_OUT_SOA)
 * Buffers need only element alignment (8 bytes, 4 for float32 output); a
 * 16-byte aligned canonical output lets the kernels store whole element
 * matrices with TMA bulk copies (tests/test_gpu_alignment.py).           */
pi_status pi_integrate(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                       int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld,
                       double* out, int out_layout, int64_t ld_out, void* stream, pi_error_info* err);

/* FP32 variant: K in float32 (half the output bytes;
 * the paper's GPU precision).  Scalar weak forms at p = 2 also compute in
 * FP32 (2x the FP64 FMA rate); the other kernels compute in FP64 and round at
 * the store.  Stated bound: per-element relative Frobenius <= 5e-5 against
 * the FP64 reference (the reference's own f32 tolerance, test_kernels.cpp:41-61). */
pi_status pi_integrate_f32(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                           int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld,
                           float* out, int out_layout, int64_t ld_out, void* stream, pi_error_info* err);

/* Load vectors F_i = sum_q det*w_q * f * phi_i(x_q) (no
 * reference counterpart; equals f times column 0 of the
 * c[0][0][0][0]=1 mass matrix).  f: device [n_elem] per-element constants, or
 * NULL to use f_const.  out: device [n_elem][n_shape]. */
pi_status pi_load_vectors(pi_context* ctx, int64_t n_elem, int64_t element_id_base,
                          const double* geom, int64_t geom_ld, const double* f, double f_const,
                          double* out, void* stream, pi_error_info* err);

/* pi_integrate plus the load vectors in the same call (scalar weak forms,
 * n_eq = 1, FP64): besides K, writes F_i = sum_q det*w_q * f * phi_i(x_q) to
 * load_out (device [n_elem][n_shape]); fused into the stiffness kernel (F
 * from the Jacobians it already forms, no second read of the geometry) or as
 * a second launch, per pi_context_set_load_fusion.  f / f_const as in
 * pi_load_vectors.  Same bound as pi_load_vectors: F equals f times column 0
 * of the c[0][0][0][0] = 1 mass matrix of integrate_generic. */
pi_status pi_integrate_load(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom,
                            int64_t geom_ld, int coeff_mode, const double* coeff, int64_t coeff_ld, double* out,
                            int out_layout, int64_t ld_out, const double* f, double f_const, double* load_out,
                            void* stream, pi_error_info* err);

/* pi_integrate_load strategy: AUTO = fused at p = 1, a second (sum-factorised,
 * geometry re-reading) launch at p >= 2, where the measured fusion overhead on
 * the stiffness kernel exceeds the cost of the extra launch. */
enum { PI_LOAD_AUTO = 0, PI_LOAD_FUSED = 1, PI_LOAD_SEPARATE = 2 };
pi_status pi_context_set_load_fusion(pi_context* ctx, int mode, pi_error_info* err);

/* Waits for the context's outstanding work and reports inverted elements
 * (PI_E_INVERTED_ELEMENT with element/det/xi filled) or CUDA errors. */
pi_status pi_check(pi_context* ctx, pi_error_info* err);

/* ---- end to end: host buffers (the run_batch drop-in, kernels.cpp:485-514) ---- */
/* geom_aos: host [n_elem][6][3] (PrismGeometry order); coeff: host (UNIFORM:
 * one tensor; PER_ELEMENT: AoS [n_elem][16*n_eq*n_eq]); out: host canonical
 * [n_elem][dim][dim].  Streams chunks through device memory with copies
 * overlapped against the kernels; blocks until done.  Pinned host buffers
 * (cudaHostAlloc / cudaHostRegister) reach full PCIe bandwidth.
 * chunk_elems <= 0 picks a chunk from free device memory. */
pi_status pi_integrate_host(pi_context* ctx, int64_t n_elem, int64_t element_id_base,
                            const double* geom_aos, int coeff_mode, const double* coeff, double* out,
                            int64_t chunk_elems, pi_error_info* err);

/* pi_integrate_host plus the load vectors (scalar weak forms; see
 * pi_integrate_load): f host [n_elem] per-element values or NULL (f_const);
 * load_out host [n_elem][n_shape]. */
pi_status pi_integrate_host_load(pi_context* ctx, int64_t n_elem, int64_t element_id_base, const double* geom_aos,
                                 int coeff_mode, const double* coeff, const double* f, double f_const, double* out,
                                 double* load_out, int64_t chunk_elems, pi_error_info* err);

/* ---- stiffness containers (host I/O) ---- */
enum {
  PI_STIFFNESS_PRISTIF1 = 1, /* the reference's single-element f32 container: save_stiffness /
                                load_stiffness (io.cpp:112-168), byte-compatible */
  PI_STIFFNESS_PRISTIF2 = 2  /* FP64 batch container: magic "PRISTIF2", u32 LE header length, JSON
                                header (count, dim, dtype "f64", element_id_base, layout, n_eq,
                                n_shape, p), count x dim x dim LE float64 in mesh order */
};
/* k: host canonical [count][dim][dim]; PRISTIF1 needs count == 1 and stores
 * element_id_base as its element_id. */
pi_status pi_save_stiffness(const char* path, int format, int p, int n_eq, int64_t count,
                            int64_t element_id_base, const double* k, pi_error_info* err);
/* Header of a PRISTIF1 / PRISTIF2 file (any pointer may be NULL). */
pi_status pi_stiffness_info(const char* path, int* format, int* p, int* n_eq, int64_t* count,
                            int64_t* element_id_base, pi_error_info* err);
/* Payload as doubles into out[capacity] (PRISTIF1 widened from f32). */
pi_status pi_load_stiffness(const char* path, double* out, int64_t capacity, pi_error_info* err);

/* Multi-GPU run_batch: the mesh is split into contiguous
 * element ranges [floor(g*n/G), floor((g+1)*n/G)) over the G contexts (one
 * per device; elements are independent, so there is no collective), one
 * host thread per context, each streaming its range through
 * pi_integrate_host.  The output is bitwise identical to a single context.
 * Errors as a single call: the lowest inverted global element id. */
pi_status pi_integrate_host_multi(pi_context* const* ctxs, int n_ctx, int64_t n_elem, int64_t element_id_base,
                                  const double* geom_aos, int coeff_mode, const double* coeff, double* out,
                                  int64_t chunk_elems, pi_error_info* err);

/* Algorithmic work per element: the dense FLOP_alg and the
 * FLOPs the selected strategy actually executes; bytes = K written +
 * geometry read (+ coefficients). */
double pi_flops_dense_per_element(int p, int n_eq, int coeff_mode);
double pi_flops_executed_per_element(const pi_context* ctx, int coeff_mode);
double pi_bytes_per_element(int p, int n_eq, int coeff_mode);

/* Diagnostics: measured FP64 tensor-pipe (DMMA m8n8k4) and FMA-pipe peaks in
 * TFLOP/s on `device` -- the FP64 roofline denominators.  Returns 0 on success. */
int pi_measure_fp64_peak(int device, double* dmma_tflops, double* dfma_tflops);

const char* pi_status_name(pi_status s);
const char* pi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PRISM_B200_H */
