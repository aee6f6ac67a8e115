// fdm2p.cuh - the bulk (TMA) local-solve kernel of fdm2.cuh, persistent with
// the next group's cells prefetched.
//
// Same arithmetic, layout and passes as fdm_group<..., BULK = true> (the
// padded tensor per subdomain, dense staging overlaid, first / last pass on
// the dense rows, bulk fp64 reduce-add of omega y).  ncu of the one-shot
// kernel at cfg 5 (profiles/r02) has 11% of its stall samples on the bulk
// loads' mbarrier: every CTA starts by waiting for its own cells.  Here each
// CTA keeps two tensor buffers and walks groups handed out by a global
// counter (in launch order, so the groups in flight stay a thin slab whose
// r and x live in L2 -- a static blockIdx stride lets CTAs drift apart and
// doubled the DRAM traffic of the persistent fdm3 variant); after the first
// pass of group i it issues the cell copies of group i+1 into the other
// buffer, whose reduce-adds of group i-1 have been read by then.
#pragma once
#include "fdm2.cuh"

namespace dgb {

template <int D, int M, bool PATCH>
struct Fdm2pShape {
  using R = Rows<D, M, PATCH>;
  static constexpr int G = fdm2_groups<D, M>();
  static constexpr int F = Lay<D, M>::F;
  static constexpr int NT = G * F;
  static constexpr int GSZ = fdm_gstride<D, M, G>();
  static constexpr int BUF = G * GSZ;
  static constexpr int SMEM = 2 * BUF;
};

template <int D, int M, bool PATCH>
__device__ __forceinline__ void fdm2p_info(const Fdm2Params<D, M>& p, int64_t grp, int tid,
                                           int (*si)[8], int64_t (*sc)[Rows<D, M, PATCH>::SLOTS]) {
  using S = Fdm2pShape<D, M, PATCH>;
  using R = Rows<D, M, PATCH>;
  constexpr int N = R::N;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  if (tid < S::G) {
    const int64_t idx = grp * S::G + tid;
    int* inf = si[tid];
    inf[7] = idx < p.count;
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    if (inf[7]) {
      const int id = p.list ? p.list[idx] : (int)(p.start + idx);
      subdomain_info<D, PATCH>(p.geo, id, p.packed != 0, digit, base);
    }
    int cls = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
#pragma unroll
    for (int t = 0; t < 3; ++t) inf[t] = digit[t];
    inf[6] = cls;
#pragma unroll
    for (int s = 0; s < R::SLOTS; ++s) {
      int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
      if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
      sc[tid][s] = inf[7] ? (int64_t)cell_local<D>(p.geo, c) * NEc : 0;
    }
  }
}

template <int D, int M, bool PATCH>
__device__ __forceinline__ void fdm2p_load(const Fdm2Params<D, M>& p, int lane, const int (*si)[8],
                                           const int64_t (*sc)[Rows<D, M, PATCH>::SLOTS],
                                           double* buf, uint64_t* bar) {
  using S = Fdm2pShape<D, M, PATCH>;
  using R = Rows<D, M, PATCH>;
  constexpr int N = R::N;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  if (lane == 0) {
    unsigned bytes = 0;
    for (int gg = 0; gg < S::G; ++gg)
      if (si[gg][7]) bytes += R::SLOTS * NEc * 8;
    mbar_expect_tx(bar, bytes);
  }
  __syncwarp();
  for (int l = lane; l < S::G * R::SLOTS; l += 32) {
    const int gg = l / R::SLOTS, sl = l - gg * R::SLOTS;
    if (si[gg][7]) bulk_load(buf + gg * S::GSZ + dense_off<NEc>(sl), p.r + sc[gg][sl], NEc * 8, bar);
  }
}

template <int D, int M, bool PATCH, int MINB = 3>
__global__ void __launch_bounds__(Fdm2pShape<D, M, PATCH>::NT, MINB)
fdm2p_kernel(const __grid_constant__ Fdm2Params<D, M> p, int64_t ngroups, int* counter) {
  using S = Fdm2pShape<D, M, PATCH>;
  using L = Lay<D, M>;
  using R = Rows<D, M, PATCH>;
  constexpr int N = R::N, G = S::G, F = S::F, GSZ = S::GSZ;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  constexpr int H = PATCH ? 2 : 1;
  static_assert(N % 2 == 0 && N % 8 != 0, "dense rows of 16-byte chunks, unrotated");
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_info[2][G][8];
  __shared__ int64_t s_cell[2][G][R::SLOTS];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int64_t s_grp[2];
  const int tid = threadIdx.x;
  const int g = tid / F, f = tid - (tid / F) * F;
  constexpr bool IL = fdm_interleave<D, G>();
  const int gi = IL ? tid % G : g, fi = IL ? tid / G : f;
  int slot0 = 0, goff = 0;
  fiber_rows<D, M, PATCH>(f, slot0, goff);
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    s_grp[0] = atomicAdd(counter, 1);
  }
  __syncthreads();
  if (s_grp[0] >= ngroups) return;
  fdm2p_info<D, M, PATCH>(p, s_grp[0], tid, s_info[0], s_cell[0]);
  __syncthreads();
  if (tid < 32) fdm2p_load<D, M, PATCH>(p, tid, s_info[0], s_cell[0], sm, &s_bar[0]);
  for (int it = 0;; ++it) {
    const int b = it & 1;
    double* base = sm + b * S::BUF;
    if (tid == 0) s_grp[b ^ 1] = atomicAdd(counter, 1);  // the next group (read after a barrier)
    const bool active = s_info[b][g][7];
    const int* dg = s_info[b][g];
    double* buf = base + g * GSZ;
    mbar_wait(&s_bar[b], (it >> 1) & 1);
    // pass 1: Z^T along direction 0 from the dense rows
    double v[M], o[M];
    if (active) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const double* src = buf + dense_off<NEc>(slot0 + h) + goff;
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          const double2 t = *reinterpret_cast<const double2*>(src + i);
          v[h * N + i] = t.x;
          v[h * N + i + 1] = t.y;
        }
      }
      fdm_matvec<M, true>(p.mats, p.eo, dg[0], v, o);
    }
    __syncthreads();  // dense rows read; s_grp[b^1] visible
    const int64_t nxt = s_grp[b ^ 1];
    if (active) {
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) buf[sb + k] = o[k];
    }
    // the next group's subdomain info (its buffer's previous info was last
    // read by the reduce-adds of group i-1, issued by warp 0 before this point)
    if (nxt < ngroups) fdm2p_info<D, M, PATCH>(p, nxt, tid, s_info[b ^ 1], s_cell[b ^ 1]);
    __syncthreads();
    if (tid < 32 && nxt < ngroups) {
      // the other buffer: the reduce-adds of group i-1 (same lanes) must
      // have finished reading it before new cells land there
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      fdm2p_load<D, M, PATCH>(p, tid, s_info[b ^ 1], s_cell[b ^ 1], sm + (b ^ 1) * S::BUF,
                              &s_bar[b ^ 1]);
    }
    // forward contractions with Z^T, directions 1 .. D-2
#pragma unroll
    for (int t = 1; t < D - 1; ++t) {
      if (active) fdm_fiber<M, true>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
      __syncthreads();
    }
    // fused direction D-1
    if (s_info[b][gi][7]) {
      constexpr int t = D - 1;
      const int* dgi = s_info[b][gi];
      double* bufi = base + gi * GSZ;
      const int sb = L::sbase(t, fi), ss = L::sstride(t);
      const double* inv = p.invsum + (int64_t)dgi[6] * L::NE + L::gbase(t, fi);
      double w[M], q[M];
#pragma unroll
      for (int k = 0; k < M; ++k) w[k] = bufi[sb + k * ss];
      fdm_matvec<M, true>(p.mats, p.eo, dgi[t], w, q);
#pragma unroll
      for (int k = 0; k < M; ++k) q[k] *= __ldg(inv + k * L::gstride(t));
      fdm_matvec<M, false>(p.mats, p.eo, dgi[t], q, w);
#pragma unroll
      for (int k = 0; k < M; ++k) bufi[sb + k * ss] = w[k];
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < D - 2; ++s) {
      const int t = D - 2 - s;
      if (active) fdm_fiber<M, false>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
      __syncthreads();
    }
    // last pass: Z along direction 0, omega y densely over the tensor
    if (active) {
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = buf[sb + k];
      fdm_matvec<M, false>(p.mats, p.eo, dg[0], v, o);
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        double* dst = buf + dense_off<NEc>(slot0 + h) + goff;
#pragma unroll
        for (int i = 0; i < N; i += 2)
          *reinterpret_cast<double2*>(dst + i) =
              make_double2(__dmul_rn(p.omega, o[h * N + i]), __dmul_rn(p.omega, o[h * N + i + 1]));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < 32) {
      bool any = false;
      for (int l = tid; l < G * R::SLOTS; l += 32) {
        const int gg = l / R::SLOTS, sl = l - gg * R::SLOTS;
        if (s_info[b][gg][7]) {
          bulk_red_add(p.x + s_cell[b][gg][sl], base + gg * GSZ + dense_off<NEc>(sl), NEc * 8);
          any = true;
        }
      }
      if (any) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (nxt >= ngroups) break;
  }
  if (tid < 32) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace dgb
