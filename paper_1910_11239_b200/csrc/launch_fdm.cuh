// launch_fdm.cuh - host launch of the local-solve kernels (fdm2.cuh,
// fdm_mma.cuh); instantiated by launch_fdm_cell.cu / launch_fdm_patch.cu.
#pragma once
#include "launch.h"
#include "fdm2.cuh"
#ifdef DGB_EXPERIMENTAL
#include "fibermap.h"
#include "fdm3.cuh"
#endif
#ifdef DGB_EXPERIMENTAL
#include "fdm_mma.cuh"
#endif

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>

namespace dgb {

#ifdef DGB_EXPERIMENTAL
// fibermap.h maps of the bulk kernel's three pass kinds, built and uploaded
// once per kernel shape by fdm_prepare_maps (dg_level_create: never inside a
// graph capture); launches before that run in the natural order
template <int D, int M, bool PATCH>
static std::atomic<const uint32_t*>& fdm_maps_slot() {
  static std::atomic<const uint32_t*> slot{nullptr};
  return slot;
}

template <int D, int M, bool PATCH>
static void fdm_prepare_maps() {
  static std::once_flag once;
  std::call_once(once, [] {
    using L = Lay<D, M>;
    using R = Rows<D, M, PATCH>;
    constexpr int G = fdm2_groups<D, M>();
    constexpr int F = L::F;
    constexpr int N = R::N;
    constexpr int NEc = (D == 3) ? N * N * N : N * N;
    constexpr int GSZ = fdm_gstride<D, M, G>();
    constexpr int H = PATCH ? 2 : 1;
    // dense 16-byte rows: mapped where the rows are not a power-of-two number
    // of chunks (those use the rotated chunk order of fdm2.cuh instead)
    constexpr int NB = (N % 8 == 0) ? 0 : H;
    std::vector<uint32_t> all;
    for (int kind = 0; kind < 3; ++kind) {
      const int t = kind == 0 ? 0 : (kind == 1 ? std::min(1, D - 1) : D - 1);
      std::vector<FiberItem> items;
      for (int g = 0; g < G; ++g)
        for (int f = 0; f < F; ++f) {
          FiberItem it;
          it.code = (uint32_t)g << 16 | (uint32_t)f;
          it.a = (g * GSZ + L::sbase(t, f)) % 16;
          it.b[0] = it.b[1] = 0;
          if (kind == 0) {
            int slot0 = 0, goff = 0;
            fiber_rows<D, M, PATCH>(f, slot0, goff);
            for (int h = 0; h < NB; ++h)
              it.b[h] = ((g * GSZ + dense_off<NEc>(slot0 + h) + goff) / 2) % 8;
          }
          items.push_back(it);
        }
      std::vector<uint32_t> m = fibermap_build(items, kind == 0 ? NB : 0);
      if (kind == 2 && fdm_interleave<D, G>()) {
        // keep the interleaved order when the builder does not beat it
        std::vector<FiberItem> il(items.size());
        for (int tid = 0; tid < G * F; ++tid) il[tid] = items[(tid % G) * F + tid / G];
        std::vector<FiberItem> got(items.size());
        for (size_t i = 0; i < m.size(); ++i) got[i] = items[(m[i] >> 16) * F + (m[i] & 0xffff)];
        if (fibermap_cost(il, 0) <= fibermap_cost(got, 0))
          for (size_t i = 0; i < m.size(); ++i) m[i] = il[i].code;
      }
      all.insert(all.end(), m.begin(), m.end());
    }
    uint32_t* d = nullptr;
    if (cudaMalloc(&d, all.size() * sizeof(uint32_t)) != cudaSuccess) return;
    // the pageable copy may still be in flight on the legacy stream when
    // cudaMemcpy returns; a later capture on a blocking stream would then
    // inherit an implicit dependency and be invalidated: wait for it here
    if (cudaMemcpy(d, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(d);
      return;
    }
    fdm_maps_slot<D, M, PATCH>().store(d);
  });
}

#endif  // DGB_EXPERIMENTAL

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
  p.maps = nullptr;
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
    if (p.direct == 2 && (!q.atomic || env_int("DGB_BULK_ATOMIC", 1)) && !q.cluster) {
#ifdef DGB_EXPERIMENTAL
      if (env_int("DGB_FIBERMAP", 0)) p.maps = fdm_maps_slot<D, M, PATCH>().load();
#endif
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
