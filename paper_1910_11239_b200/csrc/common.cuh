// common.cuh - geometry, tensor layout and index helpers shared by the
// sm_100a kernels of the Schwarz smoothing step.
//
// Index conventions follow the reference exactly (bit-exact maps):
//  - cell id c = sum_t c_t N_t^(t-1), direction 1 fastest (mesh.py:105-112);
//  - dof = cell * n^d + sum_t i_t n^(t-1) (dgop.py:70-103);
//  - patch j <-> interior vertex v in [1, N_t-1]^d, v_1 fastest
//    (mesh.py:297-326); patch cell for offset s: v_t - 1 + s_t;
//  - boundary digit per direction: bit 0 = left face on the boundary,
//    bit 1 = right face (fastdiag.py:349-369, 535-566).
#pragma once
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace dgb {

// division by a runtime constant d >= 1 for 0 <= n < 2^31 (round-up method)
struct FastDiv {
  uint32_t d, m, s;
  __host__ void init(uint32_t div) {
    d = div;
    s = 0;
    while ((1u << s) < div) ++s;
    const uint64_t one = 1;
    m = (uint32_t)(((one << 32) * ((one << s) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint64_t t = __umulhi(n, m);
    return (uint32_t)((t + n) >> s);
  }
};

struct Geo {
  int nc[3];       // global cells per direction (1 for unused directions)
  int zb;          // first stored layer (global index) along the last direction
  int zn;          // stored layers
  FastDiv fc[3];   // division by nc[t]
  FastDiv fv[3];   // division by nc[t] - 1 (patch vertex span)
};

// packed global coordinates of list entries: 3D x | y << 10 | z << 20
// (<= 1024 cells per direction), 2D x | y << 15 (<= 32768); dg_level_create
// rejects larger levels
constexpr int kPackMax3 = 1024;
constexpr int kPackMax2 = 32768;
__host__ __device__ __forceinline__ int32_t pack3(int a, int b, int c) {
  return a | (b << 10) | (c << 20);
}
__host__ __device__ __forceinline__ int32_t pack_d(int d, int a, int b, int c) {
  return d == 3 ? pack3(a, b, c) : (a | (b << 15));
}
template <int D>
__host__ __device__ __forceinline__ void unpack_d(int e, int* v) {
  if (D == 3) {
    v[0] = e & 1023;
    v[1] = (e >> 10) & 1023;
    v[2] = (e >> 20) & 1023;
  } else {
    v[0] = e & 32767;
    v[1] = (e >> 15) & 32767;
    v[2] = 0;
  }
}

template <int D, int N>
struct Lay {
  static constexpr int P = (N % 2 == 0) ? N + 1 : N;          // padded pitch
  static constexpr int F = (D == 3) ? N * N : N;               // fibers / tensor
  static constexpr int SZ = (D == 3) ? P * N * N : P * N;      // padded doubles
  static constexpr int NE = (D == 3) ? N * N * N : N * N;      // elements
  __host__ __device__ __forceinline__ static int sstride(int t) {
    return t == 0 ? 1 : (t == 1 ? P : P * N);
  }
  __host__ __device__ __forceinline__ static int gstride(int t) {
    return t == 0 ? 1 : (t == 1 ? N : N * N);
  }
  // shared-memory base offset of fiber f (0 <= f < F) along direction t
  __host__ __device__ __forceinline__ static int sbase(int t, int f) {
    if (D == 2) return t == 0 ? f * P : f;
    const int a = f % N, b = f / N;
    if (t == 0) return a * P + b * P * N;
    if (t == 1) return a + b * P * N;
    return a + b * P;
  }
  // canonical (unpadded) base offset of fiber f along t
  __host__ __device__ __forceinline__ static int gbase(int t, int f) {
    if (D == 2) return t == 0 ? f * N : f;
    const int a = f % N, b = f / N;
    if (t == 0) return a * N + b * N * N;
    if (t == 1) return a + b * N * N;
    return a + b * N;
  }
};

// subdomains per CTA: a whole number of warps, 128..512 threads if possible
template <int D, int M>
__host__ __device__ constexpr int fdm2_groups() {
  constexpr int F = Lay<D, M>::F;
#ifdef FDM_G12
  if (D == 3 && M == 12) return FDM_G12;
#endif
#ifdef FDM_G8
  if (D == 3 && M == 8) return FDM_G8;
#endif
  for (int g = 1; g <= 32; ++g)
    if ((g * F) % 32 == 0 && g * F >= 128 && g * F <= 512) return g;
  return F >= 128 ? 1 : (128 + F - 1) / F;
}

// local cell id -> global multi-index
template <int D>
__device__ __forceinline__ void cell_multi(const Geo& g, int cell, int* c) {
  const uint32_t q0 = g.fc[0].div((uint32_t)cell);
  c[0] = cell - (int)q0 * g.nc[0];
  if (D == 2) {
    c[1] = (int)q0 + g.zb;
  } else {
    const uint32_t q1 = g.fc[1].div(q0);
    c[1] = (int)q0 - (int)q1 * g.nc[1];
    c[2] = (int)q1 + g.zb;
  }
}

// DGB_CHECKS builds (__graft_entry__.build with DGB_CHECKS=1, the in-repo
// stand-in for compute-sanitizer, which this GPU pool does not allow): every
// cell a kernel addresses through cell_local is checked against the stored
// window; a violation prints the site and traps (the launch then fails)
#ifdef DGB_CHECKS
#define DG_DEVICE_CHECK(cond, msg)                                                  \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("DGB_CHECKS: %s (%s:%d) block %d thread %d\n", msg, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                    \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define DG_DEVICE_CHECK(cond, msg) \
  do {                             \
  } while (0)
#endif

// global multi-index -> local cell id
template <int D>
__device__ __forceinline__ int cell_local(const Geo& g, const int* c) {
  DG_DEVICE_CHECK(c[0] >= 0 && c[0] < g.nc[0] && (D == 2 || (c[1] >= 0 && c[1] < g.nc[1])) &&
                      c[D - 1] >= g.zb && c[D - 1] < g.zb + g.zn,
                  "cell outside the stored window");
  if (D == 2) return c[0] + g.nc[0] * (c[1] - g.zb);
  return c[0] + g.nc[0] * (c[1] + g.nc[1] * (c[2] - g.zb));
}

// subdomain id -> (per-direction digit, base cell multi-index).  Patch ids
// are global patch numbers j, or packed vertex coordinates when `packed`;
// cell ids are local cell ids, or packed global cell coordinates.
template <int D, bool PATCH>
__device__ __forceinline__ void subdomain_info(const Geo& g, int id, bool packed, int* digit,
                                               int* base) {
  if (PATCH) {
    int v[3] = {1, 1, 1};
    if (packed) {
      unpack_d<D>(id, v);
    } else {
      uint32_t rem = (uint32_t)id;
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const uint32_t q = g.fv[t].div(rem);
        v[t] = 1 + (int)(rem - q * (uint32_t)(g.nc[t] - 1));
        rem = q;
      }
    }
#pragma unroll
    for (int t = 0; t < D; ++t) {
      digit[t] = (v[t] == 1 ? 1 : 0) | (v[t] == g.nc[t] - 1 ? 2 : 0);
      base[t] = v[t] - 1;
    }
  } else {
    if (packed) {
      unpack_d<D>(id, base);
    } else {
      cell_multi<D>(g, id, base);
    }
#pragma unroll
    for (int t = 0; t < D; ++t)
      digit[t] = (base[t] == 0 ? 1 : 0) | (base[t] == g.nc[t] - 1 ? 2 : 0);
  }
}

// R_j gather map (local dof indices) of a patch list
struct MapParams {
  const int32_t* list;
  int64_t count;
  int64_t* out;
  int m, n, d;
  Geo geo;
};

__global__ void gather_map_kernel(MapParams p);

}  // namespace dgb
