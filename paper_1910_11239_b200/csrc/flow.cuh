// flow.cuh - the whole additive vertex-patch smoothing step (AVS) as one
// persistent, dependency-driven ("dataflow") kernel.
//
// Colour-by-colour launches stream the whole level through HBM once per
// colour (16 x ~0.6 GB at cfg 5) because a colour touches every z-layer.  Here
// the step is cut into tasks:
//   R(z)    residual r = b - A x on cell layer z            (res_group)
//   P(b, c) patches of colour c whose vertex layer lies in z-block b (fdm_group)
// sequenced so that a few neighbouring z-blocks are in flight at any time
// (colour skew between consecutive blocks), which keeps their cells resident
// in the 126 MB L2.  Every task carries the list of earlier tasks it conflicts
// with (built on the host, transitively reduced):
//   - P after P: different colours touching a common cell layer (the
//     reference's colour order per DoF is preserved: ascending colours);
//   - P after R: the patch reads r of, or writes x read by, the residual.
// CTAs claim work items (task, unit) in sequence order from a global counter,
// wait (acquire loads) until the dependencies have completed all their units,
// run the unit, and publish completion (fence + atomic add).  An item only
// waits on items earlier in the sequence, all claimed by running CTAs, so the
// schedule cannot deadlock.  Per DoF the additions happen in the same order as
// in the colour-by-colour launches, so the result is bit-identical to them.
#pragma once
#include "fdm2.cuh"
#include "res2.cuh"

namespace dgb {

constexpr int FLOW_MAX_DEPS = 12;

struct FlowTask {
  int type;            // 0 = residual layer, 1 = patch block x colour
  int units;           // work units (groups of cells / patches)
  int64_t first_item;  // index of the task's first work item
  int64_t start;       // residual: first local cell; patch: offset into plist
  int64_t count;       // cells / patches
  int ndeps;
  int deps[FLOW_MAX_DEPS];
};

template <int D, int N>
struct FlowParams {
  Res2Params<D, N> res;
  Fdm2Params<D, 2 * N> fdm;
  const FlowTask* tasks;
  const int32_t* item_task;
  const int32_t* plist;  // packed patch vertex coordinates, concatenated per task
  int64_t nitems;
  unsigned* ctrl;        // [0] next item, [1 + t] completed units of task t
};

template <int D, int N>
struct FlowShape {
  static constexpr int M = 2 * N;
  static constexpr int GP = fdm2_groups<D, M>();
  static constexpr int NT = GP * Lay<D, M>::F;
  static constexpr int GR = NT / Lay<D, N>::F;  // cells per residual unit
  static constexpr int SMEM_R = 3 * GR * Lay<D, N>::SZ;
  static constexpr int SMEM_P = GP * Lay<D, M>::SZ;
  static constexpr int SMEM = SMEM_R > SMEM_P ? SMEM_R : SMEM_P;
  // keep the merged residual + patch code at the register budget of the
  // standalone kernels (~64 regs) so that 3 CTAs share an SM
  static constexpr int MIN_CTAS = NT <= 256 ? 4 : 3;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int D, int N>
__global__ void __launch_bounds__(FlowShape<D, N>::NT, FlowShape<D, N>::MIN_CTAS)
flow_kernel(const __grid_constant__ FlowParams<D, N> p) {
  using S = FlowShape<D, N>;
  extern __shared__ double sm[];
  __shared__ int64_t s_item;
  for (;;) {
    if (threadIdx.x == 0) s_item = (int64_t)atomicAdd(p.ctrl, 1u);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= p.nitems) break;
    const int t = p.item_task[item];
    const FlowTask* T = p.tasks + t;
    if (threadIdx.x == 0) {
      const int nd = T->ndeps;
      for (int i = 0; i < nd; ++i) {
        const int dd = T->deps[i];
        const unsigned need = (unsigned)p.tasks[dd].units;
        while (ld_acquire(p.ctrl + 1 + dd) < need) __nanosleep(64);
      }
    }
    __syncthreads();
    const int64_t unit = item - T->first_item;
    if (T->type == 0) {
      res_group<D, N, S::GR>(p.res, nullptr, 0, T->start, T->count, unit, sm);
    } else {
      fdm_group<D, S::M, true, S::GP>(p.fdm, p.plist + T->start, 1, 0, T->count, unit, sm, true);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(p.ctrl + 1 + t, 1u);
    }
  }
}

}  // namespace dgb
