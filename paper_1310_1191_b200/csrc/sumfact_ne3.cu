// Systems with n_eq = 3: general tensors and isotropic elasticity (the
// reference's model problem, integrate_optimized, integrate_ref.cpp:93-130), p = 1..7.
#include "sumfact_host.cuh"

namespace pib {
namespace {
template <int P>
using H3 = SumFactHost<P, 3>;

template <int P>
void launch3(int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
  if (form == kFormElasticity)
    H3<P>::template go<kFormElasticity, true>(a, t, s);
  else if (sym)
    H3<P>::template go<kFormGeneral, true>(a, t, s);
  else
    H3<P>::template go<kFormGeneral, false>(a, t, s);
}
template <int P>
void attrs3() {
  H3<P>::template attr<kFormElasticity, true>();
  H3<P>::template attr_pairs<kFormElasticity>();
  H3<P>::template attr_pairs<kFormGeneral>();
  H3<P>::template attr<kFormGeneral, true>();
  H3<P>::template attr<kFormGeneral, false>();
}
}  // namespace

#define PIB_NE3_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

bool sumfact_ne3_build(int p, const double* pts, const double* phi, int nq, int nsh, SumFactHostTables& t) {
  switch (p) {
#define X(P) case P: return H3<P>::build(pts, phi, nq, nsh, t);
    PIB_NE3_CASES(X)
#undef X
  }
  return false;
}
void sumfact_ne3_attrs(int p) {
  switch (p) {
#define X(P) case P: attrs3<P>(); break;
    PIB_NE3_CASES(X)
#undef X
  }
}
void sumfact_ne3_launch(int p, int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
  switch (p) {
#define X(P) case P: launch3<P>(form, sym, a, t, s); break;
    PIB_NE3_CASES(X)
#undef X
  }
}
double sumfact_ne3_sym_fraction(int p) {
  switch (p) {
#define X(P) case P: return H3<P>::sym_fraction();
    PIB_NE3_CASES(X)
#undef X
  }
  return 1.0;
}
double sumfact_ne3_fragment_fraction(int p) {
  switch (p) {
#define X(P) case P: return H3<P>::fragment_fraction();
    PIB_NE3_CASES(X)
#undef X
  }
  return 1.0;
}
void sumfact_ne3_padded(int p, int& c, int& r, int& k) {
  switch (p) {
#define X(P) case P: H3<P>::padded(c, r, k); break;
    PIB_NE3_CASES(X)
#undef X
  }
}

}  // namespace pib
