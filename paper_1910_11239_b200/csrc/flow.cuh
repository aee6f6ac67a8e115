// flow.cuh - the whole additive vertex-patch smoothing step (AVS) as one
// persistent, dependency-driven ("dataflow") kernel with a ready queue.
//
// Colour-by-colour launches stream the whole level through HBM once per
// colour (16 x ~0.6 GB at cfg 5) because every colour touches every z-layer.
// Here the step is cut into tasks
//   R(z)    residual r = b - A x on cell layer z            (res_group)
//   P(b, c) patches of colour c whose vertex layer lies in z-block b (fdm_group)
// with dependencies built on the host (transitively reduced):
//   - P after P: different colours touching a common cell layer (every DoF
//     keeps the reference's ascending colour order, so the result is
//     bit-identical to the colour launches);
//   - P after R: the patch reads r of, or writes x read by, the residual;
//   - locality edges P(b, 0) <- P(b-1, lag): block b starts its colours only
//     when block b-1 is `lag` colours in, so only a few z-blocks (and their
//     cells) are live at a time and stay resident in the 126 MB L2.
// Scheduling is push-based: a task whose last unit completes decrements the
// pending counts of its successors and appends every newly ready one to a
// global FIFO.  CTAs claim units of the task at the queue head (atomic claim
// counters), so no CTA ever waits on a specific task -- an idle CTA only polls
// the queue -- and the schedule cannot deadlock.
#pragma once
#include "fdm2.cuh"
#include "res2.cuh"

namespace dgb {

struct FlowTask {
  int type;       // 0 = residual layer, 1 = patch block x colour
  int units;      // work units (groups of cells / patches)
  int64_t start;  // residual: first local cell; patch: offset into plist
  int64_t count;  // cells / patches
  int succ_off;   // successors: succ[succ_off .. succ_off + nsucc)
  int nsucc;
};

// per-launch scheduler state (reset from a host-built image before each step)
struct FlowState {
  int head;       // queue head (first entry that may still have units)
  int tail;       // queue entries allocated
  int finished;   // completed tasks
  int pad;
  // followed by: pending[nt], claimed[nt], done[nt], queue[nt], valid[nt]
};

template <int D, int N>
struct FlowParams {
  Res2Params<D, N> res;
  Fdm2Params<D, 2 * N> fdm;
  const FlowTask* tasks;
  const int32_t* succ;
  const int32_t* plist;  // packed patch vertex coordinates, concatenated per task
  int* state;            // FlowState + 5 * ntasks ints
  int ntasks;
};

template <int D, int N>
struct FlowShape {
  static constexpr int M = 2 * N;
  static constexpr int GP = fdm2_groups<D, M>();
  static constexpr int NT = GP * Lay<D, M>::F;
  static constexpr int GR = NT / Lay<D, N>::F;  // cells per residual unit
  static constexpr int SMEM_R = res_smem_doubles<D, N, GR>();
  static constexpr int SMEM_P = GP * fdm_gstride<D, M, GP>();
  static constexpr int SMEM = SMEM_R > SMEM_P ? SMEM_R : SMEM_P;
  // keep the merged residual + patch code at the register budget of the
  // standalone kernels so that 3-4 CTAs share an SM
  static constexpr int MIN_CTAS = NT <= 256 ? 4 : 3;
};

__device__ __forceinline__ int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int D, int N>
__global__ void __launch_bounds__(FlowShape<D, N>::NT, FlowShape<D, N>::MIN_CTAS)
flow_kernel(const __grid_constant__ FlowParams<D, N> p) {
  using S = FlowShape<D, N>;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_task, s_unit;
  const int nt = p.ntasks;
  int* st = p.state;
  int* pending = st + 4;
  int* claimed = pending + nt;
  int* done = claimed + nt;
  int* queue = done + nt;
  int* valid = queue + nt;
  for (;;) {
    if (threadIdx.x == 0) {
      int task = -1, unit = 0;
      for (;;) {
        const int h = ld_acquire_i(st + 0);
        if (h < ld_acquire_i(st + 1)) {
          while (!ld_acquire_i(valid + h)) __nanosleep(32);
          const int t = queue[h];
          const int u = atomicAdd(claimed + t, 1);
          if (u < p.tasks[t].units) {
            task = t;
            unit = u;
            break;
          }
          atomicCAS(st + 0, h, h + 1);  // head task fully claimed: advance
          continue;
        }
        if (ld_acquire_i(st + 2) >= nt) break;  // everything done
        __nanosleep(128);
      }
      s_task = task;
      s_unit = unit;
    }
    __syncthreads();
    const int t = s_task;
    const int unit = s_unit;
    if (t < 0) break;
    const FlowTask T = p.tasks[t];
    if (T.type == 0) {
      res_group<D, N, S::GR>(p.res, nullptr, 0, T.start, T.count, unit, sm);
    } else {
      fdm_group<D, S::M, true, S::GP>(p.fdm, p.plist + T.start, 1, 0, T.count, unit, sm, true);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(done + t, 1) == T.units - 1) {  // last unit of the task
        __threadfence();
        for (int i = 0; i < T.nsucc; ++i) {
          const int s = p.succ[T.succ_off + i];
          if (atomicSub(pending + s, 1) == 1) {  // successor became ready
            const int pos = atomicAdd(st + 1, 1);
            queue[pos] = s;
            __threadfence();
            st_release_i(valid + pos, 1);
          }
        }
        __threadfence();
        atomicAdd(st + 2, 1);
      }
    }
  }
}

}  // namespace dgb
