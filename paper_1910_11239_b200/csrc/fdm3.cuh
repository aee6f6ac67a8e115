// fdm3.cuh - vertex-patch fast-diagonalisation solves, v3: persistent CTAs,
// double-buffered TMA staging, contractions in place on the staged cells.
//
// Same arithmetic as fdm2 (x += omega Z Lambda^-1 Z^T R_j r per patch,
// fastdiag.py:602-628; even/odd split of the interior digit, constant-bank
// matrices), reorganised around the two costs the ncu profile of fdm2 shows
// at cfg 5 (profiles/r02): warps waiting for their own patch's bulk loads
// (SYNCS TRYWAIT, 11% of stall samples) and the barriers around the dense <->
// padded re-layout of the first and last pass.
//  - the 2^d cells of R_j r stay where the bulk copies put them (cell-major,
//    one n^d block per cell) and every pass contracts its fibers in place
//    there: a fiber along t is two n-long pieces in the cells s and s + 2^t
//    of the patch, so there is no padded tensor and no re-layout pass; the
//    last pass leaves omega * y in the same cells, from where the TMA
//    engine's fp64 bulk reduce-add sends them into x;
//  - that halves the shared memory per patch, which pays for a second
//    staging buffer: each CTA is persistent, and while it contracts group i
//    the bulk copies of group i+1 land in the other buffer (issued after the
//    second pass, once the reduce-add of group i-1 has finished reading it);
//  - one mbarrier per buffer, phase = iteration parity.
#pragma once
#include "fdm2.cuh"

namespace dgb {

template <int D, int M>
struct Fdm3Shape {
  static constexpr int N = M / 2;                           // cell n
  static constexpr int NEc = (D == 3) ? N * N * N : N * N;   // doubles per cell
  static constexpr int SLOTS = 1 << D;
  static constexpr int G = fdm2_groups<D, M>();              // patches per group
  static constexpr int F = Lay<D, M>::F;                     // fibers per patch
  static constexpr int NT = G * F;
  // cell s of a patch at s * (NEc + 2): the 16-byte skew per cell spreads the
  // rows of neighbouring cells over the bank groups and keeps 16-byte alignment
  __host__ __device__ static constexpr int doff(int s) { return s * (NEc + 2); }
  // patch stride == 8 (mod 16) doubles: the fused pass interleaves the G = 2
  // patches over consecutive lanes (fdm_interleave), which then hit distinct banks
  static constexpr int PSZ0 = SLOTS * (NEc + 2);
  static constexpr int PSZ = PSZ0 + ((8 - PSZ0 % 16) + 16) % 16;  // doubles per patch
  static constexpr int BUF = G * PSZ;                        // doubles per buffer
  static constexpr int SMEM = 2 * BUF;                       // two buffers
};

// shared offsets of the two halves of fiber f along t (patch-local), and the
// element stride inside a half
template <int D, int M>
__device__ __forceinline__ void fdm3_fiber(int t, int f, int& a0, int& a1, int& stride) {
  using S = Fdm3Shape<D, M>;
  constexpr int N = S::N;
  const int a = (D == 3) ? f % M : f, b = (D == 3) ? f / M : 0;
  int s = 0, base = 0;
  if (D == 3) {
    if (t == 0) {        // (j1, j2) = (a, b)
      s = 2 * (a / N) + 4 * (b / N);
      base = (a % N) * N + (b % N) * N * N;
      stride = 1;
    } else if (t == 1) {  // (j0, j2) = (a, b)
      s = (a / N) + 4 * (b / N);
      base = (a % N) + (b % N) * N * N;
      stride = N;
    } else {              // (j0, j1) = (a, b)
      s = (a / N) + 2 * (b / N);
      base = (a % N) + (b % N) * N;
      stride = N * N;
    }
  } else {
    if (t == 0) {        // j1 = a
      s = 2 * (a / N);
      base = (a % N) * N;
      stride = 1;
    } else {              // j0 = a
      s = a / N;
      base = a % N;
      stride = N;
    }
  }
  a0 = S::doff(s) + base;
  a1 = S::doff(s + (1 << t)) + base;
}

// the two halves of a fiber: shared <-> registers (rows of even n as 16-byte
// vectors: patch offsets are even by construction)
template <int N, int T>
__device__ __forceinline__ void fdm3_get(const double* pb, int a0, int a1, int st, double* v) {
  if constexpr (T == 0 && N % 2 == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 2) {
      const double2 x0 = *reinterpret_cast<const double2*>(pb + a0 + k);
      const double2 x1 = *reinterpret_cast<const double2*>(pb + a1 + k);
      v[k] = x0.x, v[k + 1] = x0.y, v[N + k] = x1.x, v[N + k + 1] = x1.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      v[k] = pb[a0 + k * st];
      v[N + k] = pb[a1 + k * st];
    }
  }
}
template <int N, int T>
__device__ __forceinline__ void fdm3_put(double* pb, int a0, int a1, int st, const double* o) {
  if constexpr (T == 0 && N % 2 == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 2) {
      *reinterpret_cast<double2*>(pb + a0 + k) = make_double2(o[k], o[k + 1]);
      *reinterpret_cast<double2*>(pb + a1 + k) = make_double2(o[N + k], o[N + k + 1]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      pb[a0 + k * st] = o[k];
      pb[a1 + k * st] = o[N + k];
    }
  }
}

template <int D, int M, int T, bool FWD>
__device__ __forceinline__ void fdm3_pass(const Fdm2Params<D, M>& p, int digit, double* pb, int f) {
  constexpr int N = M / 2;
  int a0, a1, st;
  fdm3_fiber<D, M>(T, f, a0, a1, st);
  double v[M], o[M];
  fdm3_get<N, T>(pb, a0, a1, st, v);
  fdm_matvec<M, FWD>(p.mats, p.eo, digit, v, o);
  fdm3_put<N, T>(pb, a0, a1, st, o);
}

// subdomain info of group `grp` into si[G][8] / sc[G][SLOTS] (threads < G)
template <int D, int M>
__device__ __forceinline__ void fdm3_info(const Fdm2Params<D, M>& p, int64_t grp, int tid,
                                          int (*si)[8], int64_t (*sc)[1 << D]) {
  using S = Fdm3Shape<D, M>;
  if (tid < S::G) {
    const int64_t idx = grp * S::G + tid;
    int* inf = si[tid];
    inf[7] = idx < p.count;
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    if (inf[7]) {
      const int id = p.list ? p.list[idx] : (int)(p.start + idx);
      subdomain_info<D, true>(p.geo, id, p.packed != 0, digit, base);
    }
    int cls = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
#pragma unroll
    for (int t = 0; t < 3; ++t) inf[t] = digit[t];
    inf[6] = cls;
#pragma unroll
    for (int s = 0; s < S::SLOTS; ++s) {
      int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
      sc[tid][s] = inf[7] ? (int64_t)cell_local<D>(p.geo, c) * S::NEc : 0;
    }
  }
}

// lanes of warp 0 issue the group's cell copies into `buf` (one per lane),
// lane 0 arms the barrier with the byte count first
template <int D, int M>
__device__ __forceinline__ void fdm3_load(const Fdm2Params<D, M>& p, int lane, const int (*si)[8],
                                          const int64_t (*sc)[1 << D], double* buf,
                                          uint64_t* bar) {
  using S = Fdm3Shape<D, M>;
  if (lane == 0) {
    unsigned bytes = 0;
    for (int g = 0; g < S::G; ++g)
      if (si[g][7]) bytes += S::SLOTS * S::NEc * 8;
    mbar_expect_tx(bar, bytes);
  }
  __syncwarp();
  for (int l = lane; l < S::G * S::SLOTS; l += 32) {
    const int g = l / S::SLOTS, s = l - g * S::SLOTS;
    if (si[g][7]) bulk_load(buf + g * S::PSZ + S::doff(s), p.r + sc[g][s], S::NEc * 8, bar);
  }
}

template <int D, int M, int MINB>
__global__ void __launch_bounds__(Fdm3Shape<D, M>::NT, MINB)
fdm3_kernel(const __grid_constant__ Fdm2Params<D, M> p, int64_t ngroups) {
  using S = Fdm3Shape<D, M>;
  using L = Lay<D, M>;
  constexpr int G = S::G, F = S::F, N = S::N;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_info[2][G][8];
  __shared__ int64_t s_cell[2][G][S::SLOTS];
  __shared__ __align__(8) uint64_t s_bar[2];
  const int tid = threadIdx.x;
  const int g = tid / F, f = tid - (tid / F) * F;
  constexpr bool IL = fdm_interleave<D, G>();
  const int gi = IL ? tid % G : g, fi = IL ? tid / G : f;
  int64_t grp = blockIdx.x;
  if (grp >= ngroups) return;
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  fdm3_info<D, M>(p, grp, tid, s_info[0], s_cell[0]);
  __syncthreads();
  if (tid < 32) fdm3_load<D, M>(p, tid, s_info[0], s_cell[0], sm, &s_bar[0]);
  for (int it = 0; grp < ngroups; ++it, grp += gridDim.x) {
    const int b = it & 1;
    double* buf = sm + b * S::BUF;
    const int64_t nxt = grp + gridDim.x;
    // the next group's subdomain info (its copies are issued after pass 2)
    fdm3_info<D, M>(p, nxt, tid, s_info[b ^ 1], s_cell[b ^ 1]);
    mbar_wait(&s_bar[b], (it >> 1) & 1);
    const int* dg = s_info[b][g];
    const bool active = dg[7];
    double* pb = buf + g * S::PSZ;
    // forward contractions along 0 .. D-2 (in place, own fiber: the first
    // needs no barrier between its reads and writes)
    if (active) fdm3_pass<D, M, 0, true>(p, dg[0], pb, f);
    __syncthreads();
    if constexpr (D == 3) {
      if (active) fdm3_pass<D, M, 1, true>(p, dg[1], pb, f);
      __syncthreads();
    }
    // prefetch: the buffer of the next group was last read by the
    // reduce-adds of the previous iteration (same lanes: wait for them)
    if (tid < 32 && nxt < ngroups) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      fdm3_load<D, M>(p, tid, s_info[b ^ 1], s_cell[b ^ 1], sm + (b ^ 1) * S::BUF, &s_bar[b ^ 1]);
    }
    // fused: Z^T along D-1, 1/Lambda-sum, Z along D-1 (subdomains interleaved)
    {
      const int* dgi = s_info[b][gi];
      if (dgi[7]) {
        constexpr int t = D - 1;
        double* pbi = buf + gi * S::PSZ;
        int a0, a1, st;
        fdm3_fiber<D, M>(t, fi, a0, a1, st);
        const double* inv = p.invsum + (int64_t)dgi[6] * L::NE + L::gbase(t, fi);
        double v[M], o[M];
        fdm3_get<N, t>(pbi, a0, a1, st, v);
        fdm_matvec<M, true>(p.mats, p.eo, dgi[t], v, o);
#pragma unroll
        for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * L::gstride(t));
        fdm_matvec<M, false>(p.mats, p.eo, dgi[t], o, v);
        fdm3_put<N, t>(pbi, a0, a1, st, v);
      }
    }
    __syncthreads();
    if constexpr (D == 3) {
      if (active) fdm3_pass<D, M, 1, false>(p, dg[1], pb, f);
      __syncthreads();
    }
    // last backward contraction, scaled by omega, in place
    if (active) {
      int a0, a1, st;
      fdm3_fiber<D, M>(0, f, a0, a1, st);
      double v[M], o[M];
      fdm3_get<N, 0>(pb, a0, a1, st, v);
      fdm_matvec<M, false>(p.mats, p.eo, dg[0], v, o);
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = __dmul_rn(p.omega, o[k]);
      fdm3_put<N, 0>(pb, a0, a1, st, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < 32) {  // omega y -> x by bulk fp64 reduce-add (tracked by this lane's group)
      bool any = false;
      for (int l = tid; l < G * S::SLOTS; l += 32) {
        const int gg = l / S::SLOTS, s = l - gg * S::SLOTS;
        if (s_info[b][gg][7]) {
          bulk_red_add(p.x + s_cell[b][gg][s], buf + gg * S::PSZ + S::doff(s), S::NEc * 8);
          any = true;
        }
      }
      if (any) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      __syncwarp();  // lanes < G rewrite this buffer's s_info next iteration
    }
  }
  if (tid < 32) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace dgb
