// launch_flow.cu - dataflow AVS kernel (flow.cuh).
#include "launch.h"
#ifdef DGB_EXPERIMENTAL
#include "flow.cuh"

#include <algorithm>
#include <cstring>

namespace dgb {

template <int D, int N>
static int launch_flow(const ResArgs& ra, const FdmArgs& fa, const HostRes& h, const double* hz,
                       const double* hzt, const double* heo, const FlowDev& fd, cudaStream_t st) {
  using S = FlowShape<D, N>;
  constexpr int M = 2 * N;
  const size_t smem = sizeof(double) * S::SMEM;
  auto k = flow_kernel<D, N>;
  static int resident = 0;
  if (!resident) {
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (int rc = resident_ctas(k, S::NT, smem, &resident)) return rc;
  }
  FlowParams<D, N> p;
  Res2Params<D, N>& r = p.res;
  r.x = ra.x;
  r.b = ra.b;
  r.r = ra.r;
  r.list = nullptr;
  r.start = 0;
  r.count = 0;
  r.packed = 0;
  r.blocked = 0;
  r.bz0 = r.bnz = 0;
  r.alpha = ra.alpha;
  r.beta = ra.beta;
  r.betap = ra.betap;
  r.geo = ra.geo;
  for (int i = 0; i < N; ++i)
    for (int kk = 0; kk < N; ++kk) {
      r.mats.mass[kk * N + i] = h.mass[i * N + kk];
      for (int dg = 0; dg < 4; ++dg) r.mats.adiag[dg][kk * N + i] = h.adiag[dg * N * N + i * N + kk];
    }
  std::memcpy(r.mats.bg0, h.bg, sizeof(r.mats.bg0));
  std::memcpy(r.mats.bg1, h.bg + N, sizeof(r.mats.bg1));
  r.eo = h.eo != nullptr && N % 2 == 0;
  if (r.eo) std::memcpy(r.mats.eo, h.eo, sizeof(r.mats.eo));
  Fdm2Params<D, M>& f = p.fdm;
  f.r = fa.r;
  f.x = fa.x;
  f.list = nullptr;
  f.start = 0;
  f.count = 0;
  f.invsum = fa.invsum;
  f.omega = fa.omega;
  f.atomic = 0;
  f.packed = 1;
  f.geo = fa.geo;
  f.direct = env_int("DGB_DIRECT", 1);
  std::memcpy(f.mats.fwd, hz, sizeof(f.mats.fwd));
  std::memcpy(f.mats.bwd, hzt, sizeof(f.mats.bwd));
  f.eo = heo != nullptr;
  if (f.eo) std::memcpy(f.mats.eo, heo, sizeof(f.mats.eo));
  p.tasks = fd.tasks;
  p.succ = fd.succ;
  p.plist = fd.plist;
  p.state = fd.state;
  p.ntasks = fd.ntasks;
  DG_CUDA(cudaMemcpyAsync(fd.state, fd.state_init, sizeof(int) * (4 + 5 * (size_t)fd.ntasks),
                          cudaMemcpyDeviceToDevice, st));
  k<<<(unsigned)std::min<int64_t>(fd.units, resident), S::NT, smem, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

bool flow_shape(int d, int n, int* gp, int* gr) {
#define X(D, N) \
  if (d == D && n == N) { *gp = FlowShape<D, N>::GP; *gr = FlowShape<D, N>::GR; return true; }
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8)
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) X(3, 7) X(3, 8)
#undef X
  return false;
}

int dispatch_flow(int d, int n, const ResArgs& ra, const FdmArgs& fa, const HostRes& h,
                         const double* hz, const double* hzt, const double* heo,
                         const FlowDev& fd, cudaStream_t st) {
#define X(D, N) if (d == D && n == N) return launch_flow<D, N>(ra, fa, h, hz, hzt, heo, fd, st);
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8)
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) X(3, 7) X(3, 8)
#undef X
  return fail(DG_EUNSUPPORTED, "flow: no kernel");
}

}  // namespace dgb

#else  // the dataflow step is a measured-and-rejected variant

namespace dgb {
bool flow_shape(int, int, int*, int*) { return false; }
int dispatch_flow(int, int, const ResArgs&, const FdmArgs&, const HostRes&, const double*,
                  const double*, const double*, const FlowDev&, cudaStream_t) {
  return DG_EUNSUPPORTED;
}
}  // namespace dgb

#endif  // DGB_EXPERIMENTAL

