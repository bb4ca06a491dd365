// Internal declarations shared by the host translation units and the CUDA
// dispatch layer.  Not part of the ABI (include/prism_b200.h is).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include "../../include/prism_b200.h"

namespace pib {

constexpr int kMaxP = 7;

int shape_count(int p);
int quad_count(int p);
int tri_point_count(int p);
void legendre(int k, double x, double& val, double& der);
void gauss_legendre(int n, double* x, double* w);
bool prism_quadrature(int p, double* points, double* weights);
void shape_values(int p, const double* xi, double* out);

// Jacobian determinant and inverse at xi (geometry.cpp:32-83), used on the
// host to describe an inverted element the device flagged.
bool jacobian_terms(const double* geom_aos, const double* xi, double& det, double inv[9]);

inline pi_status set_error(pi_error_info* err, pi_status code, const char* fmt, ...) {
  if (err) {
    err->element = -1;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(err->message, sizeof(err->message), fmt, ap);
    va_end(ap);
  }
  return code;
}

}  // namespace pib
