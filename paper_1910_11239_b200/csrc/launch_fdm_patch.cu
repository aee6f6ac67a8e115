// launch_fdm_patch.cu - vertex-patch local solves, all (dim, n) instantiations.
#include "launch_fdm.cuh"

namespace dgb {

int dispatch_patch_fdm(int d, int n, const FdmArgs& p, const double* hz,
                              const double* hzt, const double* heo, cudaStream_t st) {
#define X(D, N) if (d == D && n == N) return launch_fdm<D, 2 * N, true>(p, hz, hzt, heo, st);
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8)
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) X(3, 7) X(3, 8)
#undef X
  return fail(DG_EUNSUPPORTED, "patch fdm: no kernel for dim " + std::to_string(d) +
                                   ", degree " + std::to_string(n - 1) +
                                   " (vertex patches support k <= 7)");
}

}  // namespace dgb
