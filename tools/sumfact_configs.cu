// Prints the launch shape / shared-memory footprint of every sum-factorised
// instantiation (developer tool: nvcc -std=c++17 --expt-relaxed-constexpr).
#include <cstdio>
#include "../paper_1310_1191_b200/csrc/kernels_sumfact.cuh"
using namespace pib;
template <int P, int NE, bool SYM = false>
void show() {
  using C = SumFactConfig<P, NE, SYM>;
  std::printf("p=%d ne=%d sym=%d tmajor=%d threads=%4d warps cons=%2d prod=%d smem=%7.1f KB minb=%d nbuf=%d NTILE=%3d NBLK=%d NAG=%2d NCB=%d MEL=%d MPITCH=%d items/el=%3d acc=%d HB2=%d HS2=%d cons-wavefronts=%d prod-wavefronts=%d\n",
              P, NE, (int)SYM, (int)C::TMAJOR, C::NTHREADS, C::NCW, C::NPW, C::SMEM_BYTES / 1024.0, C::MINB, C::NBUF, C::NTILE, C::NBLK, C::NAG,
              C::NCB, C::MEL, C::MPITCH, C::NITEM, C::WA * C::MT * C::NB * 2, C::HB2, C::HS2, C::hwave_cons(C::HB2, C::HS2), C::hwave_prod(C::HB2, C::HS2));
}
int main() {
  show<2, 1>(); show<3, 1>(); show<4, 1>(); show<5, 1>(); show<6, 1>(); show<7, 1>();
  show<1, 3>(); show<2, 3>(); show<3, 3>(); show<4, 3>(); show<5, 3>(); show<6, 3>(); show<7, 3>();
  show<3, 1, true>(); show<4, 1, true>();
}
