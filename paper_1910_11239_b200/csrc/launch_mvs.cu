// launch_mvs.cu - fused restricted-residual + patch-solve launch of one MVS
// colour (mvs_fused.cuh).
#include "launch.h"

#ifdef DGB_EXPERIMENTAL
#include "mvs_fused.cuh"

#include <cstring>

namespace dgb {

template <int N>
static int launch_mvs(const ResArgs& ra, const FdmArgs& fa, const HostRes& h, const double* hz,
                      const double* hzt, const double* heo, cudaStream_t st) {
  if (fa.count <= 0) return DG_OK;
  using SH = MvsShape<N>;
  MvsParams<N> P;  // ~22 KB of tables and scalars in the kernel parameter space
  Res2Params<3, N>& p = P.res;
  p.x = ra.x;
  p.b = ra.b;
  p.r = nullptr;
  p.list = nullptr;
  p.start = 0;
  p.count = 0;
  p.packed = 1;
  p.blocked = 0;
  p.bz0 = p.bnz = 0;
  p.alpha = ra.alpha;
  p.beta = ra.beta;
  p.betap = ra.betap;
  p.geo = ra.geo;
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < N; ++k) {
      p.mats.mass[k * N + i] = h.mass[i * N + k];
      for (int dg = 0; dg < 4; ++dg) p.mats.adiag[dg][k * N + i] = h.adiag[dg * N * N + i * N + k];
    }
  std::memcpy(p.mats.bg0, h.bg, sizeof(p.mats.bg0));
  std::memcpy(p.mats.bg1, h.bg + N, sizeof(p.mats.bg1));
  p.eo = h.eo != nullptr && N % 2 == 0;
  if (p.eo) std::memcpy(p.mats.eo, h.eo, sizeof(p.mats.eo));
  std::memcpy(P.fm.fwd, hz, sizeof(P.fm.fwd));
  std::memcpy(P.fm.bwd, hzt, sizeof(P.fm.bwd));
  P.eo = heo != nullptr;
  if (P.eo) std::memcpy(P.fm.eo, heo, sizeof(P.fm.eo));
  P.x = fa.x;
  P.patches = fa.list;
  P.count = fa.count;
  P.invsum = fa.invsum;
  P.omega = fa.omega;
  const size_t smem = sizeof(double) * SH::SMEM;
  auto k = env_int("DGB_MVS_MINB", 3) >= 3 ? mvs_fused_kernel<N, 3> : mvs_fused_kernel<N, 2>;
  static bool attr = false;
  if (!attr) {
    for (auto kk : {mvs_fused_kernel<N, 3>, mvs_fused_kernel<N, 2>})
      DG_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  k<<<(unsigned)fa.count, SH::NT, smem, st>>>(P);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

bool mvs_fused_supported(int d, int n) { return d == 3 && n == 8; }

// ra: x, b, geometry and SIPG scalars; fa: x, packed patch list of one colour,
// omega, 1 / Lambda-sum table
int dispatch_mvs_fused(int d, int n, const ResArgs& ra, const FdmArgs& fa, const HostRes& h,
                       const double* hz, const double* hzt, const double* heo, cudaStream_t st) {
  if (d == 3 && n == 8) return launch_mvs<8>(ra, fa, h, hz, hzt, heo, st);
  return fail(DG_EUNSUPPORTED, "fused MVS colour: 3D degree 7 only");
}

}  // namespace dgb

#else  // measured slower than the two-launch form: experimental builds only

namespace dgb {
bool mvs_fused_supported(int, int) { return false; }
int dispatch_mvs_fused(int, int, const ResArgs&, const FdmArgs&, const HostRes&, const double*,
                       const double*, const double*, cudaStream_t) {
  return DG_EUNSUPPORTED;
}
}  // namespace dgb

#endif  // DGB_EXPERIMENTAL
