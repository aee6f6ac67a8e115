// launch_fdm_cell.cu - cell local solves, all (dim, n) instantiations.
#include "launch_fdm.cuh"

namespace dgb {

int dispatch_cell_fdm(int d, int n, const FdmArgs& p, const double* hz,
                             const double* hzt, const double* heo, cudaStream_t st) {
  if (d == 1) return oned_fdm(n, false, p, st);
#define X(D, N) if (d == D && n == N) return launch_fdm<D, N, false>(p, hz, hzt, heo, st);
  DG_N_CASES(X, 2)
  DG_N_CASES(X, 3)
#undef X
  return fail(DG_EUNSUPPORTED, "cell fdm: no kernel for dim " + std::to_string(d) +
                                   ", n " + std::to_string(n));
}

}  // namespace dgb
