// launch_fdm_patch.cu - vertex-patch local solves, all (dim, n) instantiations:
// the templated fdm2 kernels up to degree 7 (m <= 16), the generic kernel
// (fdmg.cuh) above.
#include "launch_fdm.cuh"
#include "fdmg.cuh"

namespace dgb {

// largest dynamic shared memory a CTA may opt into on sm_100 (227 KB)
static constexpr size_t kSmemMax = 227 * 1024;

template <int D, int M, bool PATCH>
static int launch_fdmg(const FdmArgs& q, cudaStream_t st) {
  if (q.count <= 0) return DG_OK;
  if (!q.zd || !q.ztd || !q.invsum) return fail(DG_EINVAL, "generic fdm: device tables missing");
  FdmgParams p;
  p.r = q.r;
  p.x = q.x;
  p.list = q.list;
  p.start = q.start;
  p.count = q.count;
  p.invsum = q.invsum;
  p.z = q.zd;
  p.zt = q.ztd;
  p.eo = q.eod;  // null when the level was built without the even/odd tables
  p.omega = q.omega;
  p.atomic = q.atomic;
  p.packed = q.packed;
  p.geo = q.geo;
  if constexpr (D == 2 && M <= 32) {
    // 2D: one warp per patch, 8 patches per CTA (fdmg2_warp_kernel)
    if (env_int("DGB_FDMG2_WARP", 1)) {
      p.pitch = M + 1;
      p.scratch = nullptr;
      const size_t smem2 = sizeof(double) * (size_t)kFdmg2Warps * (M + 1) * M;
      auto k2 = fdmg2_warp_kernel<M, PATCH>;
      static bool attr2 = false;
      if (!attr2 && smem2 > 48 * 1024) {
        DG_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        attr2 = true;
      }
      const int64_t ctas = (q.count + kFdmg2Warps - 1) / kFdmg2Warps;
      k2<<<(unsigned)std::min<int64_t>(ctas, 1 << 20), 32 * kFdmg2Warps, smem2, st>>>(p);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  // shared memory with an odd pitch while the tensor fits, else the level's
  // global scratch (one dense tensor per resident CTA)
  constexpr int64_t rows = (D == 3) ? (int64_t)M * M : M;
  const size_t smem_pad = sizeof(double) * (size_t)(rows * (M + 1));
  const size_t smem_dense = sizeof(double) * (size_t)(rows * M);
  auto k = fdmg_kernel<D, M, PATCH>;
  size_t smem = 0;
  unsigned grid = (unsigned)std::min<int64_t>(q.count, 1 << 20);
  if (smem_pad <= kSmemMax) {
    p.pitch = M + 1;
    p.scratch = nullptr;
    smem = smem_pad;
  } else if (smem_dense <= kSmemMax) {
    p.pitch = M;
    p.scratch = nullptr;
    smem = smem_dense;
  } else {
    if (!q.big_scratch || q.big_slots < 1)
      return fail(DG_EUNSUPPORTED, "generic fdm: no scratch for a subdomain this large");
    p.pitch = M;
    p.scratch = q.big_scratch;
    grid = (unsigned)std::min<int64_t>(q.count, q.big_slots);
  }
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    attr = true;
  }
  k<<<grid, kFdmgThreads, smem, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dispatch_patch_fdm(int d, int n, const FdmArgs& p, const double* hz,
                              const double* hzt, const double* heo, cudaStream_t st) {
  if (d == 1) return oned_fdm(n, true, p, st);
#define X(D, N) if (d == D && n == N) return launch_fdm<D, 2 * N, true>(p, hz, hzt, heo, st);
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8)
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) X(3, 7) X(3, 8)
#undef X
#define X(D, N) if (d == D && n == N) return launch_fdmg<D, 2 * N, true>(p, st);
  X(2, 9) X(2, 10) X(2, 11) X(2, 12) X(2, 13) X(2, 14) X(2, 15) X(2, 16)
  X(3, 9) X(3, 10) X(3, 11) X(3, 12) X(3, 13) X(3, 14) X(3, 15) X(3, 16)
#undef X
  return fail(DG_EUNSUPPORTED, "patch fdm: no kernel for dim " + std::to_string(d) +
                                   ", degree " + std::to_string(n - 1));
}

// bytes of global scratch one resident CTA of the generic kernel needs for a
// (d, n) vertex patch, 0 when the tensor fits in shared memory
size_t patch_fdm_scratch_bytes(int d, int n) {
  const size_t m = 2 * (size_t)n;
  const size_t dense = sizeof(double) * (d == 3 ? m * m * m : m * m);
  return (n > 8 && dense > kSmemMax) ? dense : 0;
}

}  // namespace dgb
