// Scalar weak forms (n_eq = 1): Laplace, general and symmetric tensors, p = 2..7.
#include "sumfact_host.cuh"

namespace pib {
namespace {
template <int P>
using H1 = SumFactHost<P, 1>;

template <int P>
void launch1(int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
  if (form == kFormLaplace)
    H1<P>::template go<kFormLaplace, true>(a, t, s);
  else if (sym)
    H1<P>::template go<kFormGeneral, true>(a, t, s);
  else
    H1<P>::template go<kFormGeneral, false>(a, t, s);
}
template <int P>
void attrs1() {
  H1<P>::template attr<kFormLaplace, true>();
  H1<P>::template attr_pairs<kFormLaplace>();
  H1<P>::template attr_pairs<kFormGeneral>();
  H1<P>::template attr<kFormGeneral, true>();
  H1<P>::template attr<kFormGeneral, false>();
}
}  // namespace

#define PIB_NE1_CASES(X) X(2) X(3) X(4) X(5) X(6) X(7)

bool sumfact_ne1_build(int p, const double* pts, const double* phi, int nq, int nsh, SumFactHostTables& t) {
  switch (p) {
#define X(P) case P: return H1<P>::build(pts, phi, nq, nsh, t);
    PIB_NE1_CASES(X)
#undef X
  }
  return false;
}
void sumfact_ne1_attrs(int p) {
  switch (p) {
#define X(P) case P: attrs1<P>(); break;
    PIB_NE1_CASES(X)
#undef X
  }
}
void sumfact_ne1_launch(int p, int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
  switch (p) {
#define X(P) case P: launch1<P>(form, sym, a, t, s); break;
    PIB_NE1_CASES(X)
#undef X
  }
}
double sumfact_ne1_sym_fraction(int p) {
  switch (p) {
#define X(P) case P: return H1<P>::sym_fraction();
    PIB_NE1_CASES(X)
#undef X
  }
  return 1.0;
}
double sumfact_ne1_fragment_fraction(int p) {
  switch (p) {
#define X(P) case P: return H1<P>::fragment_fraction();
    PIB_NE1_CASES(X)
#undef X
  }
  return 1.0;
}
void sumfact_ne1_padded(int p, int& c, int& r, int& k) {
  switch (p) {
#define X(P) case P: H1<P>::padded(c, r, k); break;
    PIB_NE1_CASES(X)
#undef X
  }
}

}  // namespace pib

namespace pib {
bool sumfact_ne3_build(int p, const double* pts, const double* phi, int nq, int nsh, SumFactHostTables& t);
void sumfact_ne3_attrs(int p);
void sumfact_ne3_launch(int p, int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s);
double sumfact_ne3_sym_fraction(int p);
double sumfact_ne3_fragment_fraction(int p);
void sumfact_ne3_padded(int p, int& c, int& r, int& k);

bool sumfact_supported(int p, int ne) { return ne == 1 ? (p >= 2 && p <= 7) : ne == 3 ? (p >= 1 && p <= 7) : false; }
bool sumfact_build(int p, int ne, const double* pts, const double* phi, int nq, int nsh, SumFactHostTables& t) {
  if (!sumfact_supported(p, ne)) return false;
  return ne == 1 ? sumfact_ne1_build(p, pts, phi, nq, nsh, t) : sumfact_ne3_build(p, pts, phi, nq, nsh, t);
}
void sumfact_set_attrs(int p, int ne) { ne == 1 ? sumfact_ne1_attrs(p) : sumfact_ne3_attrs(p); }
void sumfact_launch(int p, int ne, int form, bool sym, const LaunchArgs& a, const SumFactTables& t, cudaStream_t s) {
  if (ne == 1)
    sumfact_ne1_launch(p, form, sym, a, t, s);
  else
    sumfact_ne3_launch(p, form, sym, a, t, s);
}
double sumfact_sym_fraction(int p, int ne) { return ne == 1 ? sumfact_ne1_sym_fraction(p) : sumfact_ne3_sym_fraction(p); }
double sumfact_fragment_fraction(int p, int ne) {
  return ne == 1 ? sumfact_ne1_fragment_fraction(p) : sumfact_ne3_fragment_fraction(p);
}
void sumfact_padded_shape(int p, int ne, int& c, int& r, int& k) {
  ne == 1 ? sumfact_ne1_padded(p, c, r, k) : sumfact_ne3_padded(p, c, r, k);
}
}  // namespace pib
