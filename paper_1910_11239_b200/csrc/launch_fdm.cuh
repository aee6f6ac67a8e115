// launch_fdm.cuh - host launch of the local-solve kernels (fdm2.cuh,
// fdm_mma.cuh); instantiated by launch_fdm_cell.cu / launch_fdm_patch.cu.
#pragma once
#include "launch.h"
#include "fdm2.cuh"
#ifdef DGB_EXPERIMENTAL
#include "fdm2p.cuh"
#endif
#ifdef DGB_EXPERIMENTAL
#include "fdm4.cuh"
#endif
#ifdef DGB_EXPERIMENTAL
#include "fdm3.cuh"
#endif
#ifdef DGB_EXPERIMENTAL
#include "fdm_mma.cuh"
#endif

#ifdef DGB_EXPERIMENTAL
#include "fdm7.cuh"
#endif

#include <algorithm>
#include <cstring>

namespace dgb {

template <int D, int M, bool PATCH>
static int launch_fdm(const FdmArgs& q, const double* hz, const double* hzt, const double* heo,
                      cudaStream_t st) {
  if (q.count <= 0) return DG_OK;
  constexpr int G = fdm2_groups<D, M>();
  Fdm2Params<D, M> p;
  p.r = q.r;
  p.x = q.x;
  p.list = q.list;
  p.start = q.start;
  p.count = q.count;
  p.invsum = q.invsum;
  p.omega = q.omega;
  p.atomic = q.atomic;
  p.packed = q.packed;
  p.geo = q.geo;
  // fwd[k][i] = Z[k][i] (out = Z^T v); bwd[k][i] = Z^T[k][i] (out = Z v)
  std::memcpy(p.mats.fwd, hz, sizeof(p.mats.fwd));
  std::memcpy(p.mats.bwd, hzt, sizeof(p.mats.bwd));
  p.eo = heo != nullptr && M % 2 == 0;
  if (p.eo) std::memcpy(p.mats.eo, heo, sizeof(p.mats.eo));
  p.pv_lo = q.pv_lo;
  p.pv_hi = q.pv_hi;
  p.direct = env_int("DGB_DIRECT", 2);
#ifdef DGB_EXPERIMENTAL
  if constexpr (D == 3 && M % 8 == 0) {
    // fp64 tensor cores (fdm_mma.cuh) for m = 8, 16
    if (!q.cluster && q.zd && q.ztd && env_int("DGB_MMA", 0)) {
      using S = MmaShape<M, PATCH>;
      const size_t smem = sizeof(double) * S::SMEM;
      auto k = fdm_mma_kernel<M, PATCH>;
      static bool attr = false;
      if (!attr) {
        DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
      }
      k<<<(unsigned)((q.count + S::GS - 1) / S::GS), S::NT, smem, st>>>(p, q.zd, q.ztd);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
#endif
#ifdef DGB_EXPERIMENTAL
  if constexpr (D == 3 && M == 16) {
    // tensor cores with the even/odd split (fdm4.cuh)
    // measured at par with the DFMA kernel (cfg 3 solve 0.98 vs 0.95 ms, cfg 4
    // 0.100 vs 0.087 ms; profiles/r02): opt-in
    const int v4 = env_int("DGB_FDM4", 0);
    if (!q.cluster && q.zd && q.ztd && v4) {
      auto k4 = v4 == 2 ? fdm4_kernel<PATCH, 3> : fdm4_kernel<PATCH, 4>;
      const size_t smem4 = sizeof(double) * Fdm4Lay<PATCH>::SZ;
      static bool attr4[3] = {false, false, false};
      if (!attr4[v4 & 3 ? (v4 == 2) : 0]) {
        DG_CUDA(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4));
        attr4[v4 == 2] = true;
      }
      k4<<<(unsigned)q.count, Fdm4Lay<PATCH>::NT, smem4, st>>>(p, q.zd, q.ztd, p.eo ? q.eod : nullptr);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
#endif
  const int64_t ngroups = (q.count + G - 1) / G;
#ifdef DGB_EXPERIMENTAL
  if (!q.atomic && !q.cluster && env_int("DGB_FDM", 2) == 5) {
    using S5 = Fdm5Shape<D, M, PATCH>;
    const size_t smem5 = sizeof(double) * S5::SMEM;
    auto k5 = fdm5_kernel<D, M, PATCH>;
    static int resident = 0;
    if (!resident) {
      DG_CUDA(cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem5));
      if (int rc = resident_ctas(k5, S5::NT, smem5, &resident)) return rc;
    }
    k5<<<(unsigned)std::min<int64_t>(ngroups, resident), S5::NT, smem5, st>>>(p, ngroups);
    DG_CUDA(cudaGetLastError());
    return DG_OK;
  }
#endif
  const size_t smem = sizeof(double) * fdm2_smem_doubles<D, M>();
#ifdef DGB_EXPERIMENTAL
  if constexpr (PATCH) {
    if (q.cluster) {
      auto kc = cluster_kernel<D, M>;
      static bool attr_c = false;
      if (!attr_c) {
        DG_CUDA(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_c = true;
      }
      kc<<<(unsigned)ngroups, G * Lay<D, M>::F, smem, st>>>(p);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  if (!q.cluster && env_int("DGB_FDM", 2) == 6) {
    auto k6 = fdm6_kernel<D, M, PATCH>;
    static int resident = 0, nsm = 0;
    if (!resident) {
      DG_CUDA(cudaFuncSetAttribute(k6, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (int rc = resident_ctas(k6, G * Lay<D, M>::F, smem, &resident)) return rc;
      int dev = 0;
      DG_CUDA(cudaGetDevice(&dev));
      DG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    k6<<<(unsigned)std::min<int64_t>(ngroups, resident), G * Lay<D, M>::F, smem, st>>>(
        p, ngroups, env_int("DGB_STAGGER", 2000), nsm);
    DG_CUDA(cudaGetLastError());
    return DG_OK;
  }
#endif
  if constexpr ((Rows<D, M, PATCH>::N % 2) == 0) {
    // the bulk reduce-add is an element-wise atomic fp64 add at L2, so the
    // bulk path also serves overlapping subdomains (atomic accumulation)
#ifdef DGB_EXPERIMENTAL
    // v3 (fdm3.cuh): persistent, double-buffered, in place on the staged cells
    if constexpr (PATCH && D == 3 && (M / 2) % 2 == 0) {
      if (p.direct == 2 && !q.cluster && env_int("DGB_FDM3", 0)) {
        using S3 = Fdm3Shape<D, M>;
        constexpr int MB = fdm2_min_ctas<D, M>(true);
        const int v3 = env_int("DGB_FDM3", 0);
        auto k3 = v3 == 2 ? fdm3_kernel<D, M, (MB > 1 ? MB - 1 : 1)> : fdm3_kernel<D, M, MB>;
        const size_t smem3 = sizeof(double) * S3::SMEM;
        static int resident3[3] = {0, 0, 0};
        if (!resident3[v3 & 1]) {
          DG_CUDA(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
          if (int rc = resident_ctas(k3, S3::NT, smem3, &resident3[v3 & 1])) return rc;
        }
        const int resident3v = resident3[v3 & 1];
        const int64_t ng3 = (q.count + S3::G - 1) / S3::G;
        k3<<<(unsigned)std::min<int64_t>(ng3, resident3v), S3::NT, smem3, st>>>(p, ng3);
        DG_CUDA(cudaGetLastError());
        return DG_OK;
      }
    }
#endif
#ifdef DGB_EXPERIMENTAL
    // persistent, with the next group's cells prefetched (fdm2p.cuh): measured
    // 2x slower at cfg 5 (3.9 vs 1.8 ms: spills at 3 CTAs/SM, the digit
    // switch compiled to register-indexed constant loads, doubled x write-back)
    if constexpr (Rows<D, M, PATCH>::N % 8 != 0) {
      const int vp = env_int("DGB_FDM2P", 0);
      if (p.direct == 2 && !q.cluster && q.counter && vp) {
        using SP = Fdm2pShape<D, M, PATCH>;
        auto kp = vp == 2 ? fdm2p_kernel<D, M, PATCH, 2> : fdm2p_kernel<D, M, PATCH, 3>;
        const size_t smemp = sizeof(double) * SP::SMEM;
        static int residentp_[2] = {0, 0};
        int& residentp = residentp_[vp == 2];
        if (!residentp) {
          DG_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemp));
          if (int rc = resident_ctas(kp, SP::NT, smemp, &residentp)) return rc;
        }
        const int64_t ngp = (q.count + SP::G - 1) / SP::G;
        DG_CUDA(cudaMemsetAsync(q.counter, 0, sizeof(int), st));
        kp<<<(unsigned)std::min<int64_t>(ngp, residentp), SP::NT, smemp, st>>>(p, ngp, q.counter);
        DG_CUDA(cudaGetLastError());
        return DG_OK;
      }
    }
#endif
#ifdef DGB_EXPERIMENTAL
    if constexpr (PATCH && D == 3 && M == 12) {
      // two fibers per thread (fdm7.cuh): measured slower (2.43 vs 1.79 ms at
      // cfg 5 with two CTAs of 288 threads per SM, 4.24 ms with one), opt-in
      const int v7 = env_int("DGB_FDM7", 0);
      if (v7 && p.direct == 2 && (!q.atomic || env_int("DGB_BULK_ATOMIC", 1)) && !q.cluster) {
        using S7 = Fdm7Shape<M>;
        auto k7 = v7 == 1 ? fdm7_kernel<M, 96> : fdm7_kernel<M, 128>;
        const size_t smem7 = sizeof(double) * S7::SMEM;
        static bool attr7[2] = {false, false};
        if (!attr7[v7 == 1]) {
          DG_CUDA(cudaFuncSetAttribute(k7, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem7));
          DG_CUDA(cudaFuncSetAttribute(k7, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
          attr7[v7 == 1] = true;
        }
        k7<<<(unsigned)((q.count + S7::G - 1) / S7::G), S7::NT, smem7, st>>>(p);
        DG_CUDA(cudaGetLastError());
        return DG_OK;
      }
    }
#endif
    if (p.direct == 2 && (!q.atomic || env_int("DGB_BULK_ATOMIC", 1)) && !q.cluster) {
      auto kb = fdm2_kernel<D, M, PATCH, true>;
      static bool attr_b = false;
      if (!attr_b) {
        DG_CUDA(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_b = true;
      }
      kb<<<(unsigned)ngroups, G * Lay<D, M>::F, smem, st>>>(p);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  auto k = fdm2_kernel<D, M, PATCH>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  k<<<(unsigned)ngroups, G * Lay<D, M>::F, smem, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

}  // namespace dgb
