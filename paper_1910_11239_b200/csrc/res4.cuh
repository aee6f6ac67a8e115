// res4.cuh - SIPG residual r = b - A x in 3D for n <= 6, v4: slice-register
// passes on z-columns of cells.
//
// Same operator as res2/res3 (dgop.py:762-788, Kronecker-sum form of SURVEY
// App. A.5), grouped as A x = M_2 P + G_2 Q with the slice-wise 2D operators
//   P = M_1 G_0 x + G_1 M_0 x,   Q = M_1 M_0 x
// (G_t = A_diag(digit_t) along t plus the rank-2 couplings to the neighbours
// across the faces normal to t).  A thread owns one i2-slice (n x n values)
// of one cell, so the contractions along directions 0 and 1 run in its
// registers (the n rows, then the n columns of the slice); only the
// direction-2 contraction needs other threads' data.  ncu of res2 at cfg 5
// (profiles/r02) shows it bound by latency and shared-memory traffic
// (18 accesses per DoF, 5 barrier phases, 46% issue); here a DoF costs 2
// thread-private and 2+2 shared accesses and the CTA has one barrier.
//
// CTA = a column segment of up to ZC cells along z at fixed (x, y), plus the
// cell below and above it (halo: only their Q, whose face traces the
// direction-2 couplings of the end cells need).  Phase A (thread = (cell,
// slice)): G_0 x and M_0 x row by row (the direction-0 couplings from the x
// neighbours' rows of the same slice, loaded from global memory), stored in
// the thread's own P / Q slots; then column by column P = M_1 (G_0 x) +
// A_1 (M_0 x) + the direction-1 couplings (face traces of M_0 x of the y
// neighbours, computed from their slice in global memory) and Q = M_1 M_0 x,
// in place.  Phase B (thread = direction-2 fiber of a cell): r = b - (M_2 P +
// A_2 Q + couplings), the couplings from the neighbour cells' Q fibers in
// shared memory, written straight to global memory (coalesced along i0 + n i1).
#pragma once
#include "res3.cuh"

namespace dgb {

template <int N>
struct Res4Shape {
  static constexpr int ZC = 16;                 // cells per column segment
  static constexpr int CELLS = ZC + 2;          // + halo below / above
  // slot (slice) pitch: odd, so the 8-byte accesses of 16 consecutive slots
  // (phase A: each thread its own slot) fall in 16 distinct banks
  static constexpr int SPITCH = (N * N) | 1;
  static constexpr int CP = N * SPITCH;         // cell pitch
  static constexpr int NT = 128;
  static constexpr int SMEM = 2 * CELLS * CP;   // P and Q (doubles)
};

// dir-t face scalars (R_all, R_hi, L_all, L_lo) from the neighbours' traces:
// right neighbour value v and derivative dg (bg0 . x_R), left value v, dg (bg1 . x_L)
template <int N>
__device__ __forceinline__ void fq_right(const Res2Params<3, N>& p, double v, double dg, double& all,
                                         double& hi) {
  all = p.betap * v;
  hi = p.alpha * v + p.beta * dg;
}
template <int N>
__device__ __forceinline__ void fq_left(const Res2Params<3, N>& p, double v, double dg, double& all,
                                        double& lo) {
  all = p.beta * v;
  lo = p.alpha * v + p.betap * dg;
}

template <int N>
__device__ __forceinline__ void row_store_sh(double* s, const double (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) s[i] = v[i];
}

template <int N>
__global__ void __launch_bounds__(Res4Shape<N>::NT, 3)
res4_kernel(const __grid_constant__ Res2Params<3, N> p, int zl0, int nzl) {
  using S = Res4Shape<N>;
  constexpr int NN = N * N, NE = N * N * N;
  extern __shared__ __align__(16) double sm[];
  double* SP_ = sm;                       // P slots
  double* SQ = sm + S::CELLS * S::CP;     // Q slots
  const int tid = threadIdx.x;
  const Geo& geo = p.geo;
  // CTA -> (cx, cy, segment)
  const int nseg = (nzl + S::ZC - 1) / S::ZC;
  int rem = blockIdx.x;
  const int cx = rem % geo.nc[0];
  rem /= geo.nc[0];
  const int cy = rem % geo.nc[1];
  const int seg = rem / geo.nc[1];
  if (seg >= nseg) return;
  const int lz0 = zl0 + seg * S::ZC;                 // first local layer of the segment
  const int nz = min(S::ZC, zl0 + nzl - lz0);        // cells of the segment
  const int nzg = geo.nc[2];
  const int64_t lc = (int64_t)geo.nc[0] * geo.nc[1];
  const int64_t col = (int64_t)cx + (int64_t)geo.nc[0] * cy;
  const int d0 = (cx == 0 ? 1 : 0) | (cx == geo.nc[0] - 1 ? 2 : 0);
  const int d1 = (cy == 0 ? 1 : 0) | (cy == geo.nc[1] - 1 ? 2 : 0);

  // ---------------- phase A: thread = (cell ci in 0..nz+1, slice i2)
  if (tid < S::CELLS * N) {
    const int ci = tid / N, i2 = tid - ci * N;
    const int lz = lz0 - 1 + ci;                     // local layer of this cell
    const int gz = geo.zb + lz;
    const bool halo = ci == 0 || ci == nz + 1;
    const bool exists = ci <= nz + 1 && lz >= 0 && lz < geo.zn && gz >= 0 && gz < nzg;
    if (exists) {
      const double* xs = p.x + (col + lc * lz) * NE + i2 * NN;   // own slice
      double* ps = SP_ + ci * S::CP + i2 * S::SPITCH;
      double* qs = SQ + ci * S::CP + i2 * S::SPITCH;
      // direction-1 face scalars per column i0 (non-halo cells only)
      double f1[4][N];
#pragma unroll
      for (int j = 0; j < N; ++j) f1[0][j] = f1[1][j] = f1[2][j] = f1[3][j] = 0.0;
      if (!halo) {
        if (!(d1 & 2)) {  // y neighbour above: value row X_N[0][:], deriv sum_k bg0[k] X_N[k][:]
          const double* ns = xs + geo.nc[0] * NE;
          double v[N], dg[N], tv[N], td[N];
#pragma unroll
          for (int j = 0; j < N; ++j) {
            v[j] = __ldg(ns + j);
            dg[j] = p.mats.bg0[0] * v[j];
          }
#pragma unroll
          for (int k = 1; k < N; ++k)
#pragma unroll
            for (int j = 0; j < N; ++j) dg[j] = fma(p.mats.bg0[k], __ldg(ns + k * N + j), dg[j]);
          res_mass<3, N>(p, v, tv);
          res_mass<3, N>(p, dg, td);
#pragma unroll
          for (int j = 0; j < N; ++j) fq_right<N>(p, tv[j], td[j], f1[0][j], f1[1][j]);
        }
        if (!(d1 & 1)) {  // below: value row X_S[n-1][:], deriv sum_k bg1[k] X_S[k][:]
          const double* ss = xs - geo.nc[0] * NE;
          double v[N], dg[N], tv[N], td[N];
#pragma unroll
          for (int j = 0; j < N; ++j) {
            v[j] = __ldg(ss + (N - 1) * N + j);
            dg[j] = p.mats.bg1[N - 1] * v[j];
          }
#pragma unroll
          for (int k = 0; k < N - 1; ++k)
#pragma unroll
            for (int j = 0; j < N; ++j) dg[j] = fma(p.mats.bg1[k], __ldg(ss + k * N + j), dg[j]);
          res_mass<3, N>(p, v, tv);
          res_mass<3, N>(p, dg, td);
#pragma unroll
          for (int j = 0; j < N; ++j) fq_left<N>(p, tv[j], td[j], f1[2][j], f1[3][j]);
        }
      }
      // rows: G_0 x -> P slot, M_0 x -> Q slot
#pragma unroll
      for (int i1 = 0; i1 < N; ++i1) {
        double v[N], t[N];
        row_load_reg<N>(v, xs + i1 * N);
        res_mass<3, N>(p, v, t);
        row_store_sh<N>(qs + i1 * N, t);
        if (!halo) {
          double fq[4] = {0.0, 0.0, 0.0, 0.0};
          if (!(d0 & 2)) {  // x neighbour right: its row (i1, i2)
            double w[N];
            row_load_reg<N>(w, xs + NE + i1 * N);
            double dg = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) dg = fma(p.mats.bg0[k], w[k], dg);
            fq_right<N>(p, w[0], dg, fq[0], fq[1]);
          }
          if (!(d0 & 1)) {
            double w[N];
            row_load_reg<N>(w, xs - NE + i1 * N);
            double dg = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) dg = fma(p.mats.bg1[k], w[k], dg);
            fq_left<N>(p, w[N - 1], dg, fq[2], fq[3]);
          }
          res_adiag<N>(p, d0, v, t);
          add_faces<N>(p, fq, t);
          row_store_sh<N>(ps + i1 * N, t);
        }
      }
      // columns i0: P = M_1 G + A_1 T + faces_1, Q = M_1 T (in place; own slots only)
#pragma unroll
      for (int i0 = 0; i0 < N; ++i0) {
        double tc[N], o[N];
#pragma unroll
        for (int i1 = 0; i1 < N; ++i1) tc[i1] = qs[i0 + N * i1];
        res_mass<3, N>(p, tc, o);
#pragma unroll
        for (int i1 = 0; i1 < N; ++i1) qs[i0 + N * i1] = o[i1];
        if (!halo) {
          double gc[N], a[N];
#pragma unroll
          for (int i1 = 0; i1 < N; ++i1) gc[i1] = ps[i0 + N * i1];
          res_mass<3, N>(p, gc, o);
          res_adiag<N>(p, d1, tc, a);
          const double fq[4] = {f1[0][i0], f1[1][i0], f1[2][i0], f1[3][i0]};
          add_faces<N>(p, fq, a);
#pragma unroll
          for (int i1 = 0; i1 < N; ++i1) ps[i0 + N * i1] = o[i1] + a[i1];
        }
      }
    }
  }
  __syncthreads();
  // ---------------- phase B: thread = direction-2 fiber (i0, i1) of cell ci in 1..nz
  for (int it = tid; it < nz * NN; it += S::NT) {
    const int c = it / NN, f = it - c * NN;
    const int ci = c + 1;
    const int lz = lz0 + c;
    const int gz = geo.zb + lz;
    const int d2 = (gz == 0 ? 1 : 0) | (gz == nzg - 1 ? 2 : 0);
    const int i0 = f % N, i1 = f / N;
    const double* pc = SP_ + ci * S::CP + i0 + N * i1;
    const double* qc = SQ + ci * S::CP + i0 + N * i1;
    double pv[N], qv[N], o[N], a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      pv[k] = pc[k * S::SPITCH];
      qv[k] = qc[k * S::SPITCH];
    }
    double fq[4] = {0.0, 0.0, 0.0, 0.0};
    if (!(d2 & 2)) {  // cell above: its Q fiber (value at k = 0, derivative bg0 . Q)
      const double* qu = qc + S::CP;
      double dg = 0.0, v0 = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double w = qu[k * S::SPITCH];
        if (k == 0) v0 = w;
        dg = fma(p.mats.bg0[k], w, dg);
      }
      fq_right<N>(p, v0, dg, fq[0], fq[1]);
    }
    if (!(d2 & 1)) {  // below: value at k = n-1, derivative bg1 . Q
      const double* qd = qc - S::CP;
      double dg = 0.0, v1 = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double w = qd[k * S::SPITCH];
        if (k == N - 1) v1 = w;
        dg = fma(p.mats.bg1[k], w, dg);
      }
      fq_left<N>(p, v1, dg, fq[2], fq[3]);
    }
    res_mass<3, N>(p, pv, o);
    res_adiag<N>(p, d2, qv, a);
    add_faces<N>(p, fq, a);
    const int64_t gb = (col + lc * lz) * NE + i0 + N * i1;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double ax = o[k] + a[k];
      p.r[gb + k * NN] = p.b ? __ldg(p.b + gb + k * NN) - ax : ax;
    }
  }
}

}  // namespace dgb
