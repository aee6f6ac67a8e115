// res3.cuh - SIPG residual r = b - A x in 3D with three contraction passes.
//
// Same operator as res2.cuh (dgop.py:762-788, Kronecker-sum form of SURVEY
// App. A.5), regrouped so that every pass reads each tensor once:
//   a = G_0 x,   b = M_0 x                       (pass t = 0, row in registers)
//   c = M_1 a + G_1 b,   d = M_1 b               (pass t = 1, in place)
//   A x = M_2 c + G_2 d                          (pass t = 2, written to global)
// = M_2 M_1 G_0 x + M_2 G_1 M_0 x + G_2 M_1 M_0 x.
// G_1 and G_2 act on mass-transformed data, so their face couplings need the
// neighbour traces transformed the same way: the four face scalars per
// transverse position (R_all = beta' x_R[0], R_hi = alpha x_R[0] + beta bg0.x_R,
// L_all = beta x_L[n-1], L_lo = alpha x_L[n-1] + beta' bg1.x_L) are computed
// raw into small 2D fields and the transverse masses are applied to those
// fields (2D work, n^2 per field).  Shared traffic per cell: 8 tensor
// accesses per DoF (res2: 18), 7 tensor contractions (res2: 8).
#pragma once
#include "res2.cuh"

namespace dgb {

// the right-hand side fiber of the last pass is prefetched across the barrier
// for n > RES3_BPRE_MIN (16 more live registers in pass 1)
#ifndef RES3_BPRE_MIN
#define RES3_BPRE_MIN 6
#endif

template <int N>
struct Res3Shape {
  using L = Lay<3, N>;
  static constexpr int G = fdm2_groups<3, N>();
  static constexpr int F = N * N;
  static constexpr int NT = G * F;
  // face fields: rows of N at an odd pitch NP (the row-wise M_0 transform
  // reads a row per thread: a pitch of N = 8 or 16 doubles put every thread
  // of a half-warp on the same bank, 40% of the kernel's shared wavefronts)
  static constexpr int NP = N | 1;
  static constexpr int FP = N * NP;                  // one face field
  static constexpr int CS = 2 * L::SZ + 8 * FP;      // A, B tensors + F1[4], F2[4] fields
  static constexpr int SMEM = G * CS;                // doubles
  // CTAs per SM the register budget is sized for (launch_res.cu: DGB_RES3_MINB).
  // n = 8 (128-thread CTAs): 6 -> 80 registers, no spills (cfg 3 residual
  // 1.35 -> 1.29 ms; 8 CTAs / 64 registers spill and lose); n = 7 (147
  // threads) and n >= 9 keep 2 (n = 7 at 6: 0.25 -> 0.44 ms)
  static constexpr int MINB = N == 8 ? 6 : 2;
};

// the four face scalars of a fiber along t (zero where the neighbour is absent)
template <int N>
__device__ __forceinline__ void face_scalars(const Res2Params<3, N>& p, const double* xr,
                                             const double* xl, int gs, double (&fq)[4]) {
  fq[0] = fq[1] = fq[2] = fq[3] = 0.0;
  if (xr) {
    double v[N];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = __ldg(xr + k * gs);
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg0[k], v[k], g);
    fq[0] = p.betap * v[0];
    fq[1] = p.alpha * v[0] + p.beta * g;
  }
  asm volatile("" ::: "memory");  // one neighbour fiber live at a time (registers)
  if (xl) {
    double v[N];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = __ldg(xl + k * gs);
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg1[k], v[k], g);
    fq[2] = p.beta * v[N - 1];
    fq[3] = p.alpha * v[N - 1] + p.betap * g;
  }
}

// o += face couplings of the four scalars along the fiber
template <int N>
__device__ __forceinline__ void add_faces(const Res2Params<3, N>& p, const double (&fq)[4],
                                          double (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) o[i] = fma(p.mats.bg1[i], fq[0], fma(p.mats.bg0[i], fq[2], o[i]));
  o[N - 1] += fq[1];
  o[0] += fq[3];
}

template <int N>
__device__ __forceinline__ void res_adiag(const Res2Params<3, N>& p, int digit,
                                          const double (&v)[N], double (&o)[N]) {
  if constexpr (N % 2 == 0) {
    if (p.eo && digit == 0) {
      matvec_cs<N>(p.mats.eo[2], p.mats.eo[3], v, o);
      return;
    }
  }
  matvec_digit<N>(p.mats.adiag, digit, v, o);
}

template <int N>
__device__ __forceinline__ void mass3(const Res2Params<3, N>& p, const double (&v)[N],
                                      double (&o)[N]) {
  res_mass<3, N>(p, v, o);
}

// passes t = 1, 2 and the face-field transforms (after pass 0 and a barrier)
template <int N, class Sink>
__device__ __forceinline__ void res3_tail_to(const Res2Params<3, N>& p, bool active, int f, int fa,
                                             int fb, const int (&dig)[3], int64_t cb, double* A,
                                             double* B, double* F1, double* F2, Sink sink) {
  using S = Res3Shape<N>;
  using L = Lay<3, N>;
  constexpr int F = S::F;
  constexpr int FP = S::FP, NP = S::NP;
  // ---- M_0 along i0 of the face fields, rows F1[q][i2][.] and F2[q][i1][.]
  if (active) {
    for (int w = f; w < 8 * N; w += F) {  // in place, one thread per row
      double* row = F1 + (w / N) * FP + (w % N) * NP;
      double v[N], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = row[j];
      mass3<N>(p, v, o);
#pragma unroll
      for (int j = 0; j < N; ++j) row[j] = o[j];
    }
  }
  __syncthreads();
  // ---- pass t = 1 at (i0, i2) = (fa, fb); M_1 along i1 of the F2 columns
  double bq[N];
  if (active) {
    for (int w = f; w < 4 * N; w += F) {  // F2 column (q, i0): in place
      double* col = F2 + (w / N) * FP + (w % N);
      double v[N], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = col[j * NP];
      mass3<N>(p, v, o);
#pragma unroll
      for (int j = 0; j < N; ++j) col[j * NP] = o[j];
    }
    const int sb = L::sbase(1, f), ss = L::sstride(1);
    double v[N], o[N], t[N];
    double fq[4];  // faces along t = 1, transformed by M_0
#pragma unroll
    for (int q = 0; q < 4; ++q) fq[q] = F1[q * FP + fb * NP + fa];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = B[sb + k * ss];
    res_adiag<N>(p, dig[1], v, t);  // G_1 b
    add_faces<N>(p, fq, t);
    mass3<N>(p, v, o);        // d = M_1 b
#pragma unroll
    for (int k = 0; k < N; ++k) B[sb + k * ss] = o[k];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = A[sb + k * ss];
    mass3<N>(p, v, o);        // c = M_1 a + G_1 b
#pragma unroll
    for (int k = 0; k < N; ++k) A[sb + k * ss] = o[k] + t[k];
    // right-hand side along the t = 2 fiber (i0, i1) = (fa, fb), prefetched
    // across the barrier (n <= 6: loaded in the last pass, fewer registers)
    if (N > RES3_BPRE_MIN && p.b) {
#pragma unroll
      for (int k = 0; k < N; ++k) bq[k] = __ldg(p.b + cb + fa + N * fb + N * N * k);
    }
  }
  __syncthreads();
  // ---- pass t = 2 at (i0, i1) = (fa, fb); faces transformed by M_1 along i1
  if (active) {
    const int sb = L::sbase(2, f), ss = L::sstride(2);
    double v[N], o[N], t[N];
    double fq[4];  // faces along t = 2, transformed by M_0 and M_1
#pragma unroll
    for (int q = 0; q < 4; ++q) fq[q] = F2[q * FP + fb * NP + fa];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = B[sb + k * ss];
    res_adiag<N>(p, dig[2], v, t);  // G_2 d
    add_faces<N>(p, fq, t);
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = A[sb + k * ss];
    mass3<N>(p, v, o);        // M_2 c
    if (N <= RES3_BPRE_MIN && p.b) {
#pragma unroll
      for (int k = 0; k < N; ++k) bq[k] = __ldg(p.b + cb + fa + N * fb + N * N * k);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double ax = o[k] + t[k];
      sink(k, p.b ? bq[k] - ax : ax);  // entry (i0, i1, i2) = (fa, fb, k) of the cell
    }
  }
}

// ... with r = b - A x (or A x) written to global memory
template <int N>
__device__ __forceinline__ void res3_tail(const Res2Params<3, N>& p, bool active, int f, int fa,
                                          int fb, const int (&dig)[3], int64_t cb, double* A,
                                          double* B, double* F1, double* F2) {
  double* r = p.r + cb + fa + N * fb;
  res3_tail_to<N>(p, active, f, fa, fb, dig, cb, A, B, F1, F2,
                  [&](int k, double v) { r[N * N * k] = v; });
}

// pass t = 0 of one cell (own row from global memory, the two direction-0
// neighbour rows) and the raw face fields of directions 1 and 2
template <int N>
__device__ __forceinline__ void res3_pass0(const Res2Params<3, N>& p, bool active, int f, int fa,
                                           int fb, const int (&c)[3], const int (&dig)[3],
                                           int64_t cb, double* A, double* B, double* F1,
                                           double* F2) {
  using S = Res3Shape<N>;
  using L = Lay<3, N>;
  constexpr int NE = L::NE;
  constexpr int FP = S::FP, NP = S::NP;
  auto nbr = [&](int t, int dir) -> const double* {  // neighbour cell data or null
    if (dir > 0 ? (dig[t] & 2) : (dig[t] & 1)) return nullptr;
    int nb[3] = {c[0], c[1], c[2]};
    nb[t] += dir;
    return p.x + (int64_t)cell_local<3>(p.geo, nb) * NE;
  };
  // ---- pass t = 0: own row (i1, i2) = (fa, fb) from global; raw face fields
  if (active) {
    double v[N], o[N];
    row_load_reg<N>(v, p.x + cb + f * N);
    double fq[4] = {0.0, 0.0, 0.0, 0.0};
    {
      const double* r = nbr(0, +1);
      const double* l = nbr(0, -1);
      if (r) {
        double w[N];
        row_load_reg<N>(w, r + f * N);
        double gg = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) gg = fma(p.mats.bg0[k], w[k], gg);
        fq[0] = p.betap * w[0];
        fq[1] = p.alpha * w[0] + p.beta * gg;
      }
      asm volatile("" ::: "memory");
      if (l) {
        double w[N];
        row_load_reg<N>(w, l + f * N);
        double gg = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) gg = fma(p.mats.bg1[k], w[k], gg);
        fq[2] = p.beta * w[N - 1];
        fq[3] = p.alpha * w[N - 1] + p.betap * gg;
      }
    }
    res_adiag<N>(p, dig[0], v, o);
    add_faces<N>(p, fq, o);
    const int sb = L::sbase(0, f);
#pragma unroll
    for (int k = 0; k < N; ++k) A[sb + k] = o[k];
    mass3<N>(p, v, o);
#pragma unroll
    for (int k = 0; k < N; ++k) B[sb + k] = o[k];
    asm volatile("" ::: "memory");
    // faces along t = 1 at (i0, i2) = (fa, fb): fibers stride n
    {
      const double* r = nbr(1, +1);
      const double* l = nbr(1, -1);
      const int gb = fa + N * N * fb;
      face_scalars<N>(p, r ? r + gb : nullptr, l ? l + gb : nullptr, N, fq);
#pragma unroll
      for (int q = 0; q < 4; ++q) F1[q * FP + fb * NP + fa] = fq[q];
    }
    asm volatile("" ::: "memory");
    // faces along t = 2 at (i0, i1) = (fa, fb): fibers stride n^2
    {
      const double* r = nbr(2, +1);
      const double* l = nbr(2, -1);
      const int gb = fa + N * fb;
      face_scalars<N>(p, r ? r + gb : nullptr, l ? l + gb : nullptr, N * N, fq);
#pragma unroll
      for (int q = 0; q < 4; ++q) F2[q * FP + fb * NP + fa] = fq[q];
    }
  }
}

template <int N, int MINB>
__global__ void __launch_bounds__(Res3Shape<N>::NT, MINB)
res3_kernel(const __grid_constant__ Res2Params<3, N> p) {
  using S = Res3Shape<N>;
  using L = Lay<3, N>;
  constexpr int G = S::G, F = S::F, NE = L::NE;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_cell[G];
  __shared__ int s_c[G][3];
  const int tid = threadIdx.x;
  if (tid < G)
    s_cell[tid] = res_cell<3>(p.geo, p.list, p.packed, p.start, p.count,
                              (int64_t)blockIdx.x * G + tid, s_c[tid]);
  __syncthreads();
  const int g = tid / F, f = tid - g * F;
  const int cell = s_cell[g];
  const bool active = cell >= 0;
  int c[3] = {s_c[g][0], s_c[g][1], s_c[g][2]};
  int dig[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) dig[t] = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
  double* A = sm + g * S::CS;
  double* B = A + L::SZ;
  double* F1 = B + L::SZ;      // F1[q][i2][i0]: faces along t = 1
  double* F2 = F1 + 4 * S::FP;  // F2[q][i1][i0]: faces along t = 2
  constexpr int FP = S::FP, NP = S::NP;
  const int fa = f % N, fb = f / N;
  const int64_t cb = (int64_t)(active ? cell : 0) * NE;
  res3_pass0<N>(p, active, f, fa, fb, c, dig, cb, A, B, F1, F2);
  __syncthreads();
  res3_tail<N>(p, active, f, fa, fb, dig, cb, A, B, F1, F2);
}

#ifdef DGB_EXPERIMENTAL
// ---------------------------------------------------------------------------
// res3b: the same three passes with a batched trace phase.  ncu of res3 at
// cfg 3 / cfg 4 (profiles/r01_v7/ncu_cfg34_after): 41% / 33% of the stall
// samples are long-scoreboard waits at 19 / 15 active warps per SM -- each
// thread walked its six neighbour fibers one after another (one fiber live
// at a time for the register budget), seven dependent round trips to L2 per
// thread.  Here the neighbour loads come first, NB faces per batch issued
// back to back without branches (an absent neighbour reads the own cell and
// its scalars are zeroed afterwards), so a thread has NB*N loads in flight
// and 6/NB round trips; the own row rides in the first batch.  Arithmetic
// and summation order are those of res3_kernel (bitwise equal, tested).
// Measured (r02, kbench): cfg 3 residual 1.291 -> 1.324 ms, cfg 4 0.2411 ->
// 0.2445 ms: no gain, the round trips were not the limiter; opt-in
// (DGB_RES3_BATCH=1 in DGB_EXPERIMENTAL builds).
// ---------------------------------------------------------------------------
template <int N>
__host__ __device__ constexpr int res3b_batch() {
  return N <= 8 ? 3 : 2;
}

// face fc = 2 t + side (side 0: +e_t neighbour, 1: -e_t) of fiber (fa, fb)
template <int N>
__device__ __forceinline__ void nbr_fiber_load(double (&w)[N], const double* cellp, int t, int fa,
                                               int fb) {
  if (t == 0) {
    row_load_reg<N>(w, cellp + (fa + N * fb) * N);
  } else {
    const int gb = t == 1 ? fa + N * N * fb : fa + N * fb;
    const int gs = t == 1 ? N : N * N;
#pragma unroll
    for (int k = 0; k < N; ++k) w[k] = __ldg(cellp + gb + k * gs);
  }
}

template <int N, int MINB>
__global__ void __launch_bounds__(Res3Shape<N>::NT, MINB)
res3b_kernel(const __grid_constant__ Res2Params<3, N> p) {
  using S = Res3Shape<N>;
  using L = Lay<3, N>;
  constexpr int G = S::G, F = S::F, NE = L::NE;
  constexpr int NB = res3b_batch<N>();
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_cell[G];
  __shared__ int s_c[G][3];
  const int tid = threadIdx.x;
  if (tid < G)
    s_cell[tid] = res_cell<3>(p.geo, p.list, p.packed, p.start, p.count,
                              (int64_t)blockIdx.x * G + tid, s_c[tid]);
  __syncthreads();
  const int g = tid / F, f = tid - g * F;
  const int cell = s_cell[g];
  const bool active = cell >= 0;
  int c[3] = {s_c[g][0], s_c[g][1], s_c[g][2]};
  int dig[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) dig[t] = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
  double* A = sm + g * S::CS;
  double* B = A + L::SZ;
  double* F1 = B + L::SZ;      // F1[q][i2][i0]: faces along t = 1
  double* F2 = F1 + 4 * S::FP;  // F2[q][i1][i0]: faces along t = 2
  constexpr int FP = S::FP, NP = S::NP;
  const int fa = f % N, fb = f / N;
  const int64_t cb = (int64_t)(active ? cell : 0) * NE;
  double fq0[4] = {0.0, 0.0, 0.0, 0.0};
  double v[N];
  if (active) {
    // ---- trace phase: the six neighbour fibers of this thread, NB per batch
    row_load_reg<N>(v, p.x + cb + f * N);
#pragma unroll
    for (int b0 = 0; b0 < 6; b0 += NB) {
      double w[NB][N];
      bool have[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int fc = b0 + j, t = fc >> 1, side = fc & 1;
        have[j] = side == 0 ? !(dig[t] & 2) : !(dig[t] & 1);
        int nb[3] = {c[0], c[1], c[2]};
        nb[t] += have[j] ? (side == 0 ? 1 : -1) : 0;
        nbr_fiber_load<N>(w[j], p.x + (int64_t)cell_local<3>(p.geo, nb) * NE, t, fa, fb);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int fc = b0 + j, t = fc >> 1, side = fc & 1;
        double gg = 0.0, qa, qh;
        if (side == 0) {
#pragma unroll
          for (int k = 0; k < N; ++k) gg = fma(p.mats.bg0[k], w[j][k], gg);
          qa = p.betap * w[j][0];
          qh = p.alpha * w[j][0] + p.beta * gg;
        } else {
#pragma unroll
          for (int k = 0; k < N; ++k) gg = fma(p.mats.bg1[k], w[j][k], gg);
          qa = p.beta * w[j][N - 1];
          qh = p.alpha * w[j][N - 1] + p.betap * gg;
        }
        qa = have[j] ? qa : 0.0;
        qh = have[j] ? qh : 0.0;
        if (t == 0) {
          fq0[2 * side] = qa;
          fq0[2 * side + 1] = qh;
        } else {
          double* Ft = t == 1 ? F1 : F2;
          Ft[(2 * side) * FP + fb * NP + fa] = qa;
          Ft[(2 * side + 1) * FP + fb * NP + fa] = qh;
        }
      }
    }
    // ---- pass t = 0 on the own row (i1, i2) = (fa, fb)
    double o[N];
    res_adiag<N>(p, dig[0], v, o);
    add_faces<N>(p, fq0, o);
    const int sb = L::sbase(0, f);
#pragma unroll
    for (int k = 0; k < N; ++k) A[sb + k] = o[k];
    mass3<N>(p, v, o);
#pragma unroll
    for (int k = 0; k < N; ++k) B[sb + k] = o[k];
  }
  __syncthreads();
  res3_tail<N>(p, active, f, fa, fb, dig, cb, A, B, F1, F2);
}

// ---------------------------------------------------------------------------
// res3c: res3b with the direction-0 rows staged by the TMA engine.  ncu of
// res3b at cfg 3 (profiles/r02/ncu_cfg3_res3b_*): the LSU data pipe is the
// limiter (l1tex__data_pipe_lsu_wavefronts 86% of peak, half of it global
// accesses), and 6.2 L1 tag requests per LDG -- a thread's own row and the
// rows of its two direction-0 neighbours are n contiguous doubles per
// thread, so one 16-byte load instruction of a warp touches 16 (n = 8) or
// 32 (n = 16) lines.  Here the own cell and the two direction-0 neighbour
// cells arrive densely in shared memory by cp.async.bulk (no LSU wavefronts)
// and each thread reads its rows with conflict-free 16-byte accesses
// (rotated chunks for 64 / 128-byte rows, dense_row_load).  Staging aliases
// the tensors: own -> B, left -> A, right -> an extra n^3 doubles; a barrier
// separates the row reads from the pass-0 stores.  In patch-list mode with
// two cells per CTA (x-adjacent slots of a patch block) each cell's in-pair
// neighbour is the partner's own staging.  Even n only (16-byte bulk sizes).
// Arithmetic and summation order are those of res3_kernel (bitwise equal).
// Measured (r02, kbench): cfg 3 residual 1.291 -> 1.294 ms, cfg 4 0.2415 ->
// 0.2727 ms, n = 6 (cfg 5) 0.80 -> 0.85 ms: the wavefronts saved on the LSU
// pipe are spent by the bulk copies on the same shared-memory banks and the
// CTA still waits for its own copies; opt-in (DGB_RES3_TMA=1, experimental).
// ---------------------------------------------------------------------------
template <int N>
struct Res3cShape {
  using S = Res3Shape<N>;
  static constexpr int CS = S::CS + Lay<3, N>::NE;  // + right-neighbour staging
  static constexpr int SMEM = S::G * CS;
};

// row f (n doubles at src) of a dense cell in shared memory -> registers
template <int N>
__device__ __forceinline__ void dense_row_load(double (&v)[N], const double* src, int f) {
  if constexpr (N % 8 == 0) {
    double2 w[N / 2];
    const int rot = row_rot<N>(f);
#pragma unroll
    for (int j = 0; j < N / 2; ++j)
      w[j] = *reinterpret_cast<const double2*>(src + 2 * ((j + rot) & (N / 2 - 1)));
    rotate_chunks<N / 2>(w, (N / 2 - rot) & (N / 2 - 1));
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      v[2 * j] = w[j].x;
      v[2 * j + 1] = w[j].y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(src + i);
      v[i] = t.x;
      v[i + 1] = t.y;
    }
  }
}

template <int N, int MINB>
__global__ void __launch_bounds__(Res3Shape<N>::NT, MINB)
res3c_kernel(const __grid_constant__ Res2Params<3, N> p) {
  static_assert(N % 2 == 0, "bulk staging needs 16-byte rows");
  using S = Res3Shape<N>;
  using SC = Res3cShape<N>;
  using L = Lay<3, N>;
  constexpr int G = S::G, F = S::F, NE = L::NE;
  constexpr int NB = N <= 8 ? 4 : 2;  // direction-1/2 faces per load batch
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_cell[G];
  __shared__ int s_c[G][3];
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  // pair mode: the CTA's two cells are x-neighbours of one patch block
  const bool pair = G == 2 && p.blocked == 2;
  if (tid == 0) mbar_init(&s_bar, 3 * G);
  if (tid < G)
    s_cell[tid] = res_cell<3>(p.geo, p.list, p.packed, p.start, p.count,
                              (int64_t)blockIdx.x * G + tid, s_c[tid]);
  __syncthreads();
  if (tid < 3 * G) {
    // lane = (cell gg, which): 0 own -> B, 1 left -> A, 2 right -> extra
    const int gg = tid / 3, which = tid - 3 * gg;
    const int cl = s_cell[gg];
    int nb[3] = {s_c[gg][0], s_c[gg][1], s_c[gg][2]};
    bool want = cl >= 0;
    if (which == 1) want = want && nb[0] > 0 && !(pair && gg == 1);
    if (which == 2) want = want && nb[0] < p.geo.nc[0] - 1 && !(pair && gg == 0);
    nb[0] += which == 1 ? -1 : (which == 2 ? 1 : 0);
    double* base = sm + gg * SC::CS;
    double* dst = which == 0 ? base + L::SZ : (which == 1 ? base : base + S::CS);
    mbar_expect_tx(&s_bar, want ? NE * 8u : 0u);
    if (want) bulk_load(dst, p.x + (int64_t)cell_local<3>(p.geo, nb) * NE, NE * 8, &s_bar);
  }
  const int g = tid / F, f = tid - g * F;
  const int cell = s_cell[g];
  const bool active = cell >= 0;
  int c[3] = {s_c[g][0], s_c[g][1], s_c[g][2]};
  int dig[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) dig[t] = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
  double* A = sm + g * SC::CS;
  double* B = A + L::SZ;
  double* F1 = B + L::SZ;      // F1[q][i2][i0]: faces along t = 1
  double* F2 = F1 + 4 * S::FP;  // F2[q][i1][i0]: faces along t = 2
  double* XR = A + S::CS;      // right-neighbour staging
  constexpr int FP = S::FP, NP = S::NP;
  const int fa = f % N, fb = f / N;
  const int64_t cb = (int64_t)(active ? cell : 0) * NE;
  double fq0[4] = {0.0, 0.0, 0.0, 0.0};
  double v[N];
  if (active) {
    // ---- faces along t = 1, 2 from global fibers (coalesced), NB per batch,
    //      in flight while the bulk copies land
#pragma unroll
    for (int b0 = 2; b0 < 6; b0 += NB) {
      double w[NB][N];
      bool have[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int fc = b0 + j, t = fc >> 1, side = fc & 1;
        have[j] = side == 0 ? !(dig[t] & 2) : !(dig[t] & 1);
        int nb[3] = {c[0], c[1], c[2]};
        nb[t] += have[j] ? (side == 0 ? 1 : -1) : 0;
        nbr_fiber_load<N>(w[j], p.x + (int64_t)cell_local<3>(p.geo, nb) * NE, t, fa, fb);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int fc = b0 + j, t = fc >> 1, side = fc & 1;
        double gg = 0.0, qa, qh;
        if (side == 0) {
#pragma unroll
          for (int k = 0; k < N; ++k) gg = fma(p.mats.bg0[k], w[j][k], gg);
          qa = p.betap * w[j][0];
          qh = p.alpha * w[j][0] + p.beta * gg;
        } else {
#pragma unroll
          for (int k = 0; k < N; ++k) gg = fma(p.mats.bg1[k], w[j][k], gg);
          qa = p.beta * w[j][N - 1];
          qh = p.alpha * w[j][N - 1] + p.betap * gg;
        }
        double* Ft = t == 1 ? F1 : F2;
        Ft[(2 * side) * FP + fb * NP + fa] = have[j] ? qa : 0.0;
        Ft[(2 * side + 1) * FP + fb * NP + fa] = have[j] ? qh : 0.0;
      }
    }
  }
  mbar_wait(&s_bar, 0);
  if (active) {
    // ---- direction-0 rows from the dense staging
    dense_row_load<N>(v, B + f * N, f);
    if (!(dig[0] & 2)) {
      const double* src = (pair && g == 0) ? sm + SC::CS + L::SZ : XR;  // partner's own cell
      double w[N];
      dense_row_load<N>(w, src + f * N, f);
      double gg = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) gg = fma(p.mats.bg0[k], w[k], gg);
      fq0[0] = p.betap * w[0];
      fq0[1] = p.alpha * w[0] + p.beta * gg;
    }
    if (!(dig[0] & 1)) {
      const double* src = (pair && g == 1) ? sm + L::SZ : A;
      double w[N];
      dense_row_load<N>(w, src + f * N, f);
      double gg = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) gg = fma(p.mats.bg1[k], w[k], gg);
      fq0[2] = p.beta * w[N - 1];
      fq0[3] = p.alpha * w[N - 1] + p.betap * gg;
    }
  }
  __syncthreads();  // every staged row is in registers before A / B are written
  if (active) {
    // ---- pass t = 0 on the own row (i1, i2) = (fa, fb)
    double o[N];
    res_adiag<N>(p, dig[0], v, o);
    add_faces<N>(p, fq0, o);
    const int sb = L::sbase(0, f);
#pragma unroll
    for (int k = 0; k < N; ++k) A[sb + k] = o[k];
    mass3<N>(p, v, o);
#pragma unroll
    for (int k = 0; k < N; ++k) B[sb + k] = o[k];
  }
  __syncthreads();
  res3_tail<N>(p, active, f, fa, fb, dig, cb, A, B, F1, F2);
}
#endif  // DGB_EXPERIMENTAL

}  // namespace dgb
