// launch_res.cu - residual kernels (res2.cuh), all (dim, n) instantiations.
#include "launch.h"
#include "res2.cuh"
#include "res3.cuh"
#ifdef DGB_EXPERIMENTAL
#include "res4.cuh"
#endif

#include <algorithm>
#include <cstring>

namespace dgb {

template <int D, int N>
static int launch_residual(const ResArgs& q, const HostRes& h, cudaStream_t st) {
  if (q.count <= 0) return DG_OK;
  constexpr int G = fdm2_groups<D, N>();
  constexpr int NT = G * Lay<D, N>::F;
  Res2Params<D, N> p;
  p.x = q.x;
  p.b = q.b;
  p.r = q.r;
  p.list = q.list;
  p.start = q.start;
  p.count = q.count;
  p.packed = q.packed;
  p.alpha = q.alpha;
  p.beta = q.beta;
  p.betap = q.betap;
  p.geo = q.geo;
  p.blocked = 0;
  p.bz0 = p.bnz = 0;
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < N; ++k) {
      p.mats.mass[k * N + i] = h.mass[i * N + k];
      for (int dg = 0; dg < 4; ++dg) p.mats.adiag[dg][k * N + i] = h.adiag[dg * N * N + i * N + k];
    }
  std::memcpy(p.mats.bg0, h.bg, sizeof(p.mats.bg0));
  std::memcpy(p.mats.bg1, h.bg + N, sizeof(p.mats.bg1));
  p.eo = h.eo != nullptr && N % 2 == 0;
  if (p.eo) std::memcpy(p.mats.eo, h.eo, sizeof(p.mats.eo));
  if constexpr (D == 3) {
    // three-pass residual (res3.cuh) where measured faster than res2
    // (tools/res_sweep.py, ~16.8M dofs, ms res2 / res3): n = 7, 8, 9
    // (0.31 / 0.28 at n = 9) and n = 13..16 (0.32 / 0.24 at n = 16, cfg 4);
    // res2 stays at n = 6 (0.70 / 0.73 on cfg 5) and n = 10..12, where its
    // even/odd split of the interior stiffness wins.  DGB_RES3_HI = 0 / 1
    // forces res2 / res3 for n >= 9.
    constexpr bool PREF = N <= 9 || N >= 13;
    const int hi = env_int("DGB_RES3_HI", -1);
    const bool use = N <= 6 ? env_int("DGB_RES3_LO", 0) != 0
                            : (N <= 8 || (hi < 0 ? PREF : hi != 0));
    if (env_int("DGB_RES3", 1) && use) {
      using S = Res3Shape<N>;
      const size_t smem3 = sizeof(double) * S::SMEM;
      const unsigned grid = (unsigned)((q.count + S::G - 1) / S::G);
      const int minb = env_int("DGB_RES3_MINB", S::MINB);
      // occupancy variants (CTAs per SM the register budget is sized for);
      // the high counts only where the 128-thread CTAs fit them (n <= 8)
      constexpr int HI = N <= 8 ? 8 : 3, MID = N <= 8 ? 6 : 3;
      auto k3 = minb >= HI ? res3_kernel<N, HI>
                           : (minb >= MID ? res3_kernel<N, MID>
                                          : (minb >= 3 ? res3_kernel<N, 3> : res3_kernel<N, 2>));
#ifdef DGB_EXPERIMENTAL
      // batched trace phase (res3b_kernel): measured no faster, opt-in
      if (env_int("DGB_RES3_BATCH", 0))
        k3 = minb >= HI ? res3b_kernel<N, HI>
                        : (minb >= MID ? res3b_kernel<N, MID>
                                       : (minb >= 3 ? res3b_kernel<N, 3> : res3b_kernel<N, 2>));
      if constexpr (N % 2 == 0) {
        // direction-0 rows staged by TMA bulk copies (res3c_kernel, DGB_RES3_TMA)
        if (env_int("DGB_RES3_TMA", 0)) {
          using SC = Res3cShape<N>;
          const size_t smemc = sizeof(double) * SC::SMEM;
          auto kc = minb >= HI ? res3c_kernel<N, HI>
                               : (minb >= MID ? res3c_kernel<N, MID>
                                              : (minb >= 3 ? res3c_kernel<N, 3> : res3c_kernel<N, 2>));
          static bool attrc = false;
          if (!attrc) {
            for (auto kk : {res3c_kernel<N, 2>, res3c_kernel<N, 3>, res3c_kernel<N, MID>,
                            res3c_kernel<N, HI>})
              DG_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smemc));
            attrc = true;
          }
          p.blocked = (S::G == 2 && q.list && q.block_list && q.count % 8 == 0 &&
                       env_int("DGB_RES_BLOCK_LIST", 1)) ? 2 : 0;
          kc<<<grid, S::NT, smemc, st>>>(p);
          DG_CUDA(cudaGetLastError());
          return DG_OK;
        }
      }
#endif
      static bool attr3 = false;
      if (!attr3) {
        for (auto kk : {res3_kernel<N, 2>, res3_kernel<N, 3>, res3_kernel<N, MID>, res3_kernel<N, HI>})
          DG_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
#ifdef DGB_EXPERIMENTAL
        for (auto kk : {res3b_kernel<N, 2>, res3b_kernel<N, 3>, res3b_kernel<N, MID>,
                        res3b_kernel<N, HI>})
          DG_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
#endif
        attr3 = true;
      }
      k3<<<grid, S::NT, smem3, st>>>(p);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
#ifdef DGB_EXPERIMENTAL
  if constexpr (D == 3 && N <= 6) {
    // whole layers: slice-register passes on z-column segments (res4.cuh);
    // measured slower at cfg 5 (0.91 vs 0.66 ms: 12 warps per SM and
    // uncoalesced per-thread slice loads, profiles/r02): opt-in
    const int64_t lc = (int64_t)q.geo.nc[0] * q.geo.nc[1];
    if (!q.list && q.start % lc == 0 && q.count % lc == 0 && env_int("DGB_RES4", 0)) {
      using S4 = Res4Shape<N>;
      const int zl0 = (int)(q.start / lc), nzl = (int)(q.count / lc);
      const int nseg = (nzl + S4::ZC - 1) / S4::ZC;
      const size_t smem4 = sizeof(double) * S4::SMEM;
      auto k4 = res4_kernel<N>;
      static bool attr4 = false;
      if (!attr4) {
        DG_CUDA(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4));
        attr4 = true;
      }
      k4<<<(unsigned)(lc * nseg), S4::NT, smem4, st>>>(p, zl0, nzl);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
#endif
  int64_t ngroups = (q.count + G - 1) / G;
  p.blocked = 0;
  p.bz0 = p.bnz = 0;
  if constexpr (D == 3 && G == 8) {
    // vertex-patch cell lists (the MVS restricted residual): every group of
    // 8 list entries is one patch's 2x2x2 block, in-block traces from shared
    if (q.list && q.block_list && q.count % 8 == 0 && env_int("DGB_RES_BLOCK_LIST", 1))
      p.blocked = 2;
    // whole layers on 2x2x2 cell blocks: half the neighbour traces come from
    // the block's own shared tensors
    const int64_t lc = (int64_t)q.geo.nc[0] * q.geo.nc[1];
    if (!q.list && q.start % lc == 0 && q.count % lc == 0 && env_int("DGB_RES_BLOCK", 1)) {
      p.blocked = 1;
      p.bz0 = q.geo.zb + (int)(q.start / lc);
      p.bnz = (int)(q.count / lc);
      ngroups = (int64_t)((q.geo.nc[0] + 1) / 2) * ((q.geo.nc[1] + 1) / 2) * ((p.bnz + 1) / 2);
    }
  }
#ifdef DGB_EXPERIMENTAL
  if constexpr (D == 3 && N == 6) {
    // narrow pitch (7 / 42): 4 CTAs per SM instead of 3, more bank conflicts
    if (env_int("DGB_RES2_NARROW", 0)) {
      const size_t smemn = sizeof(double) * res2_smem_doubles<D, N, true>();
      auto kn = res2_kernel<D, N, true, 4>;
      DG_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemn));
      kn<<<(unsigned)ngroups, NT, smemn, st>>>(p);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
#endif
  size_t smem = sizeof(double) * res2_smem_doubles<D, N>();
#ifdef DGB_EXPERIMENTAL
  smem += (size_t)env_int("DGB_RES2_PAD", 0);  // occupancy experiment: extra bytes per CTA
#endif
  auto k = res2_kernel<D, N>;
  static size_t attr = 0;
  if (attr < smem) {
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  k<<<(unsigned)ngroups, NT, smem, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dispatch_residual(int d, int n, const ResArgs& p, const HostRes& h,
                             cudaStream_t st) {
  if (d == 1) return oned_residual(n, p, p.oned, st);
#define X(D, N) if (d == D && n == N) return launch_residual<D, N>(p, h, st);
  DG_N_CASES(X, 2)
  DG_N_CASES(X, 3)
#undef X
  return fail(DG_EUNSUPPORTED, "residual: no kernel for dim " + std::to_string(d) +
                                   ", n " + std::to_string(n));
}

}  // namespace dgb
