// Host interface of the sum-factorised kernels (kernels_sumfact.cuh), split
// by n_eq into their own translation units (sumfact_ne1.cu, sumfact_ne3.cu)
// so the instantiations compile in parallel.  Internal, not ABI.
#pragma once

#include <vector>

#include <cuda_runtime.h>

#include "kernels_common.cuh"

namespace pib {

struct SumFactTables;

struct SumFactHostTables {
  std::vector<double> xfrag, xplain, yline, tri;
  int ntps = 0;  // row pitch of xplain ([NSP][3][ntps])
};

// True if (p, n_eq) has a sum-factorised instantiation.
bool sumfact_supported(int p, int ne);
// Builds the per-p tables from the caller's rule (points [n_q][3]) and shape
// table ([n_q][4][n_shape], tabulate_shapes order); false if they are not
// the tensor-product prism basis the kernel factorises.
bool sumfact_build(int p, int ne, const double* pts, const double* phi, int n_q, int n_shape, SumFactHostTables& t);
void sumfact_set_attrs(int p, int ne);
// form: SumFactForm; sym: the tensor (hence K) is symmetric.
void sumfact_launch(int p, int ne, int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s);
// Fraction of the (t, t') tile pairs the symmetric path multiplies, and of the
// B-fragment values it forms.
double sumfact_sym_fraction(int p, int ne);
double sumfact_fragment_fraction(int p, int ne);
// Shape numbers of the instantiation: NTILE*8 padded columns, MT*8 padded rows, KSTEPS*4 padded k.
void sumfact_padded_shape(int p, int ne, int& cols, int& rows, int& ksteps4);

}  // namespace pib
