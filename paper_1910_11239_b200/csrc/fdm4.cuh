// fdm4.cuh - fast-diagonalisation solves on the fp64 tensor cores with the
// even/odd split, for 3D subdomains of 1D size 16 (vertex patches of Q7,
// cfg 3; cells of Q15, cfg 4).
//
// x += omega Z Lambda^-1 Z^T R r (fastdiag.py:457-496, 602-628).  Each of the
// six contractions of the 16^3 tensor is a small GEMM on DMMA.8x8x4
// (mma.sync m8n8k4 f64).  On an interior direction (digit 0) the 1D pencil
// is symmetric, its eigenvectors are even / odd (tables.device_tables), and
// the contraction splits into two 8x8 blocks on the folded fibers
// u_k = v_k + v_{15-k}, w_k = v_k - v_{15-k} (forward) or is unfolded as
// out_i = e_i + q_i, out_{15-i} = e_i - q_i (backward): the 8x8 blocks tile
// m8n8k4 exactly, so the tensor cores do half the work of the dense 16x16
// contraction (fdm_mma.cuh, measured slower than DFMA in round 1 for want of
// this split).  Boundary digits keep the dense 16x16 matrices.
//
// Shared layout: the tensor T(i3, i2, i1) (i1 = direction 0) is unpadded,
// 16 doubles per row, with an XOR swizzle of the column within the row,
// i1 ^ SW[(i2 + i3) & 3], SW = {0, 8, 4, 12}: the 8-byte fragment loads of
// every direction (lane q -> k = 4 kk + q, lane g -> row or column) and the
// 16-byte result stores all hit distinct banks, and T is 32 KB.  The cells of
// R_j r arrive densely (cell-major) by one TMA bulk copy each; the first
// contraction reads them there (with the k order 2q + kk, so a lane's two
// k-values are one 16-byte load) and writes T after a barrier; the last
// contraction reads T and writes omega * y back densely, from where fp64
// bulk reduce-adds send whole cells into x.  8 warps per subdomain, each
// owning 4 units of 8 fibers per pass.
#pragma once
#include "fdm2.cuh"

namespace dgb {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool PATCH>
struct Fdm4Lay {
  static constexpr int N = PATCH ? 8 : 16;   // cell n
  static constexpr int NEc = N * N * N;
  static constexpr int SLOTS = PATCH ? 8 : 1;
  static constexpr int SZ = 4096;            // the swizzled tensor = the dense staging
  static constexpr int NT = 256;             // 8 warps
  // dense (cell-major) offset of element (i3, i2, 8 h) of the 16^3 tensor
  __device__ __forceinline__ static int dense(int i3, int i2, int h) {
    if (PATCH) {
      const int s = h + 2 * (i2 >> 3) + 4 * (i3 >> 3);
      return s * NEc + (i2 & 7) * 8 + (i3 & 7) * 64;
    }
    return i2 * 16 + i3 * 256 + 8 * h;
  }
};

__device__ __forceinline__ int sw4(int i2, int i3) { return (0xC480 >> (4 * ((i2 + i3) & 3))) & 15; }
__device__ __forceinline__ int tz(int i3, int i2, int i1) { return i3 * 256 + i2 * 16 + (i1 ^ sw4(i2, i3)); }

// k order of a fragment: STD = 4 kk + q (padded-free swizzled tensor),
// PAIR = 2q + kk (+8 for the upper half; dense rows, one 16-byte load)
template <bool PAIR>
__device__ __forceinline__ int kidx(int kk, int q) {
  return PAIR ? 2 * q + (kk & 1) + 8 * (kk >> 1) : 4 * kk + q;
}

// fragments of S (S[a][k] = src[k * ld + a], the k-outer table storage):
// lane (g, q) of k-step kk holds S[8 ta + g][kidx(kk, q)] -- the A operand of
// D = S X and, for the row passes, the B operand of D = X S^T
struct Frag8 {
  double v[2];
};
struct Frag16 {
  double v[2][4];
};
template <bool PAIR>
__device__ __forceinline__ void load_frag8(Frag8& f, const double* __restrict__ src, int lane) {
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) f.v[kk] = __ldg(src + kidx<PAIR>(kk, q) * 8 + g);
}
template <bool PAIR>
__device__ __forceinline__ void load_frag16(Frag16& f, const double* __restrict__ src, int lane) {
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int ta = 0; ta < 2; ++ta)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) f.v[ta][kk] = __ldg(src + kidx<PAIR>(kk, q) * 16 + 8 * ta + g);
}

// ---- columns: unit u of direction t = 1 / 2 is 8 columns, element (k, n) --
// For t = 1: (i3, i2, i1) = (o, k, j0 + n), for t = 2: (k, o, j0 + n).  The
// swizzle index (k + o) & 3 of the lane's k = 4 kk + q does not depend on kk,
// so each lane's addresses are a few per-unit offsets plus multiples of 4 ks.
struct ColUnit {
  int base;  // element (0, 0) without swizzle: o * (t == 1 ? 256 : 16) + j0
  int ks;    // k stride: 16 (t = 1) or 256 (t = 2)
  int o, j0;
  __device__ __forceinline__ ColUnit(int t, int u) {
    o = u >> 1;
    j0 = (u & 1) * 8;
    ks = t == 1 ? 16 : 256;
    base = o * (t == 1 ? 256 : 16);
  }
  // element (k, n) for a k with (k + o) & 3 == sidx
  __device__ __forceinline__ int at(int k, int n) const {
    return base + k * ks + ((j0 + n) ^ sw4(k, o));
  }
};

// lane offsets of a unit: loads of k = 4 kk + q (lo), of 15 - k (hi) and
// of 8 + k (kk-step = 4 ks); stores of rows g, 8 + g, 15 - g at columns 2q
struct ColLane {
  int lo, hi, st_g, st_hi;
  __device__ __forceinline__ ColLane(const ColUnit& c, int g, int q) {
    lo = c.at(q, g);
    hi = c.at(15 - q, g);
    st_g = c.at(g, 2 * q);
    st_hi = c.at(15 - g, 2 * q);
  }
};

__device__ __forceinline__ void col_fwd_eo2(double* T, const ColUnit (&c)[2], const Frag8& E,
                                            const Frag8& O, int lane) {
  const int g = lane >> 2, q = lane & 3;
  const ColLane l0(c[0], g, q), l1(c[1], g, q);
  double ce[2][2] = {}, co[2][2] = {};
  double x[2][2][2];  // [unit][kk][lo/hi]
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    x[0][kk][0] = T[l0.lo + 4 * kk * c[0].ks];
    x[0][kk][1] = T[l0.hi - 4 * kk * c[0].ks];
    x[1][kk][0] = T[l1.lo + 4 * kk * c[1].ks];
    x[1][kk][1] = T[l1.hi - 4 * kk * c[1].ks];
  }
#pragma unroll
  for (int kk = 0; kk < 2; ++kk)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      dmma(ce[u][0], ce[u][1], E.v[kk], x[u][kk][0] + x[u][kk][1]);
      dmma(co[u][0], co[u][1], O.v[kk], x[u][kk][0] - x[u][kk][1]);
    }
  __syncwarp();
  *reinterpret_cast<double2*>(&T[l0.st_g]) = make_double2(ce[0][0], ce[0][1]);
  *reinterpret_cast<double2*>(&T[l0.st_g + 8 * c[0].ks]) = make_double2(co[0][0], co[0][1]);
  *reinterpret_cast<double2*>(&T[l1.st_g]) = make_double2(ce[1][0], ce[1][1]);
  *reinterpret_cast<double2*>(&T[l1.st_g + 8 * c[1].ks]) = make_double2(co[1][0], co[1][1]);
}

__device__ __forceinline__ void col_bwd_eo2(double* T, const ColUnit (&c)[2], const Frag8& Et,
                                            const Frag8& Ot, int lane) {
  const int g = lane >> 2, q = lane & 3;
  const ColLane l0(c[0], g, q), l1(c[1], g, q);
  double e[2][2] = {}, o[2][2] = {};
  double x[2][2][2];  // [unit][kk][even/odd]
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    x[0][kk][0] = T[l0.lo + 4 * kk * c[0].ks];
    x[0][kk][1] = T[l0.lo + (4 * kk + 8) * c[0].ks];
    x[1][kk][0] = T[l1.lo + 4 * kk * c[1].ks];
    x[1][kk][1] = T[l1.lo + (4 * kk + 8) * c[1].ks];
  }
#pragma unroll
  for (int kk = 0; kk < 2; ++kk)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      dmma(e[u][0], e[u][1], Et.v[kk], x[u][kk][0]);
      dmma(o[u][0], o[u][1], Ot.v[kk], x[u][kk][1]);
    }
  __syncwarp();
  *reinterpret_cast<double2*>(&T[l0.st_g]) = make_double2(e[0][0] + o[0][0], e[0][1] + o[0][1]);
  *reinterpret_cast<double2*>(&T[l0.st_hi]) = make_double2(e[0][0] - o[0][0], e[0][1] - o[0][1]);
  *reinterpret_cast<double2*>(&T[l1.st_g]) = make_double2(e[1][0] + o[1][0], e[1][1] + o[1][1]);
  *reinterpret_cast<double2*>(&T[l1.st_hi]) = make_double2(e[1][0] - o[1][0], e[1][1] - o[1][1]);
}

__device__ __forceinline__ void col_dense(double* T, const ColUnit& c, const Frag16& S, int lane) {
  const int g = lane >> 2, q = lane & 3;
  const ColLane l(c, g, q);
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double b[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) b[kk] = T[l.lo + 4 * kk * c.ks];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    dmma(d[0][0], d[0][1], S.v[0][kk], b[kk]);
    dmma(d[1][0], d[1][1], S.v[1][kk], b[kk]);
  }
  __syncwarp();
  *reinterpret_cast<double2*>(&T[l.st_g]) = make_double2(d[0][0], d[0][1]);
  *reinterpret_cast<double2*>(&T[l.st_g + 8 * c.ks]) = make_double2(d[1][0], d[1][1]);
}

// ---- rows (direction 0): D[r][a] = sum_k X(r, k) S[a][k] ------------------
// Results as two 16-byte chunks: columns ca, ca+1 and cb, cb+1 of the row.
struct RowOut {
  double c[4];
  int ca, cb;
};

// pass 1 (forward, dense cell rows lo / hi = columns 0..7 / 8..15, PAIR order)
__device__ __forceinline__ RowOut row_fwd_eo(const double* lo, const double* hi, const Frag8& E,
                                             const Frag8& O, int lane) {
  const int q = lane & 3;
  const double2 a = *reinterpret_cast<const double2*>(lo + 2 * q);       // x[2q], x[2q+1]
  const double2 b = *reinterpret_cast<const double2*>(hi + 6 - 2 * q);   // x[14-2q], x[15-2q]
  double ce[2] = {0.0, 0.0}, co[2] = {0.0, 0.0};
  dmma(ce[0], ce[1], a.x + b.y, E.v[0]);   // k = 2q: x[k] + x[15-k]
  dmma(co[0], co[1], a.x - b.y, O.v[0]);
  dmma(ce[0], ce[1], a.y + b.x, E.v[1]);   // k = 2q+1
  dmma(co[0], co[1], a.y - b.x, O.v[1]);
  return {{ce[0], ce[1], co[0], co[1]}, 2 * q, 8 + 2 * q};
}
__device__ __forceinline__ RowOut row_fwd_dense(const double* lo, const double* hi,
                                                const Frag16& S, int lane) {
  const int q = lane & 3;
  const double2 a = *reinterpret_cast<const double2*>(lo + 2 * q);   // k = 2q, 2q+1
  const double2 b = *reinterpret_cast<const double2*>(hi + 2 * q);   // k = 8+2q, 9+2q
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const double av[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    dmma(d[0][0], d[0][1], av[kk], S.v[0][kk]);
    dmma(d[1][0], d[1][1], av[kk], S.v[1][kk]);
  }
  return {{d[0][0], d[0][1], d[1][0], d[1][1]}, 2 * q, 8 + 2 * q};
}

// pass 5 (backward times omega, swizzled row (i3, i2) of T, STD order)
__device__ __forceinline__ RowOut row_bwd_eo(const double* T, int i3, int i2, const Frag8& Et,
                                             const Frag8& Ot, int lane, double scale) {
  const int q = lane & 3;
  double e[2] = {0.0, 0.0}, o[2] = {0.0, 0.0};
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const int k = 4 * kk + q;
    dmma(e[0], e[1], T[tz(i3, i2, k)], Et.v[kk]);
    dmma(o[0], o[1], T[tz(i3, i2, 8 + k)], Ot.v[kk]);
  }
  // out_i = e_i + q_i (i = 2q, 2q+1), out_{15-i} = e_i - q_i at 14-2q, 15-2q
  return {{__dmul_rn(scale, e[0] + o[0]), __dmul_rn(scale, e[1] + o[1]),
           __dmul_rn(scale, e[1] - o[1]), __dmul_rn(scale, e[0] - o[0])},
          2 * q, 14 - 2 * q};
}
__device__ __forceinline__ RowOut row_bwd_dense(const double* T, int i3, int i2, const Frag16& S,
                                                int lane, double scale) {
  const int q = lane & 3;
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const double a = T[tz(i3, i2, 4 * kk + q)];
    dmma(d[0][0], d[0][1], a, S.v[0][kk]);
    dmma(d[1][0], d[1][1], a, S.v[1][kk]);
  }
  return {{__dmul_rn(scale, d[0][0]), __dmul_rn(scale, d[0][1]), __dmul_rn(scale, d[1][0]),
           __dmul_rn(scale, d[1][1])},
          2 * q, 8 + 2 * q};
}

template <bool FWD>
__device__ __forceinline__ void fdm4_cols(double* T, const double* zd, const double* ztd,
                                          const double* eod, bool eo, int t, int digit, int warp,
                                          int lane) {
  if (eo) {
    Frag8 A, B;
    load_frag8<false>(A, eod + (FWD ? 0 : 2) * 64, lane);
    load_frag8<false>(B, eod + (FWD ? 1 : 3) * 64, lane);
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      const ColUnit c[2] = {ColUnit(t, 4 * warp + j), ColUnit(t, 4 * warp + j + 1)};
      if (FWD) col_fwd_eo2(T, c, A, B, lane);
      else col_bwd_eo2(T, c, A, B, lane);
    }
  } else {
    // dense: fwd out = Z^T v (S[a][k] = Z[k][a] = zd[k*16+a]); bwd out = Z v (ztd)
    Frag16 S;
    load_frag16<false>(S, (FWD ? zd : ztd) + digit * 256, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) col_dense(T, ColUnit(t, 4 * warp + j), S, lane);
  }
}

// pass 3: Z^T, 1/Lambda, Z along direction 2 on this warp's own columns
// (the 1/Lambda values of a lane are loaded before the forward products)
template <bool EO>
__device__ __forceinline__ void fdm4_pass3(double* T, const double* zd, const double* ztd,
                                           const double* eod, const double* inv, int dg2,
                                           int warp, int lane) {
  const int g = lane >> 2, q = lane & 3;
  auto inv_of = [&](const ColUnit& c, double2 (&iv)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h)  // rows a = 8h + g, columns 2q, 2q+1
      iv[h] = __ldg(reinterpret_cast<const double2*>(inv + (8 * h + g) * 256 + c.o * 16 + c.j0 + 2 * q));
  };
  auto scale = [&](const ColUnit& c, const double2 (&iv)[2]) {
    const ColLane l(c, g, q);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // own values written by the forward step
      double2* tp = reinterpret_cast<double2*>(&T[l.st_g + 8 * h * c.ks]);
      const double2 v = *tp;
      *tp = make_double2(v.x * iv[h].x, v.y * iv[h].y);
    }
  };
  if constexpr (EO) {
    Frag8 E, O, Et, Ot;
    load_frag8<false>(E, eod + 0 * 64, lane);
    load_frag8<false>(O, eod + 1 * 64, lane);
    load_frag8<false>(Et, eod + 2 * 64, lane);
    load_frag8<false>(Ot, eod + 3 * 64, lane);
#pragma unroll 1
    for (int j = 0; j < 4; j += 2) {
      const ColUnit c[2] = {ColUnit(2, 4 * warp + j), ColUnit(2, 4 * warp + j + 1)};
      double2 iv[2][2];
      inv_of(c[0], iv[0]);
      inv_of(c[1], iv[1]);
      col_fwd_eo2(T, c, E, O, lane);
      scale(c[0], iv[0]);
      scale(c[1], iv[1]);
      __syncwarp();
      col_bwd_eo2(T, c, Et, Ot, lane);
      __syncwarp();
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const ColUnit c(2, 4 * warp + j);
      double2 iv[2];
      inv_of(c, iv);
      {
        Frag16 S;
        load_frag16<false>(S, zd + dg2 * 256, lane);
        col_dense(T, c, S, lane);
      }
      scale(c, iv);
      __syncwarp();
      {
        Frag16 St;
        load_frag16<false>(St, ztd + dg2 * 256, lane);
        col_dense(T, c, St, lane);
      }
      __syncwarp();
    }
  }
}

template <bool PATCH, bool EO>
__device__ __forceinline__ void fdm4_pass1(const double* T, const double* zd, const double* eod,
                                           int dg0, int warp, int lane, RowOut (&out)[4]) {
  using L = Fdm4Lay<PATCH>;
  const int g = lane >> 2;
  if constexpr (EO) {
    Frag8 E, O;
    load_frag8<true>(E, eod + 0 * 64, lane);
    load_frag8<true>(O, eod + 1 * 64, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * (4 * warp + j) + g, i3 = r >> 4, i2 = r & 15;
      out[j] = row_fwd_eo(T + L::dense(i3, i2, 0), T + L::dense(i3, i2, 1), E, O, lane);
    }
  } else {
    Frag16 S;
    load_frag16<true>(S, zd + dg0 * 256, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * (4 * warp + j) + g, i3 = r >> 4, i2 = r & 15;
      out[j] = row_fwd_dense(T + L::dense(i3, i2, 0), T + L::dense(i3, i2, 1), S, lane);
    }
  }
}

template <bool EO>
__device__ __forceinline__ void fdm4_pass5(const double* T, const double* ztd, const double* eod,
                                           int dg0, int warp, int lane, double omega,
                                           RowOut (&out)[4]) {
  const int g = lane >> 2;
  if constexpr (EO) {
    Frag8 Et, Ot;
    load_frag8<false>(Et, eod + 2 * 64, lane);
    load_frag8<false>(Ot, eod + 3 * 64, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * (4 * warp + j) + g;
      out[j] = row_bwd_eo(T, r >> 4, r & 15, Et, Ot, lane, omega);
    }
  } else {
    Frag16 St;
    load_frag16<false>(St, ztd + dg0 * 256, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * (4 * warp + j) + g;
      out[j] = row_bwd_dense(T, r >> 4, r & 15, St, lane, omega);
    }
  }
}

template <bool PATCH, int MINB = 4>
__global__ void __launch_bounds__(256, MINB)
fdm4_kernel(const __grid_constant__ Fdm2Params<3, 16> p, const double* __restrict__ zd,
            const double* __restrict__ ztd, const double* __restrict__ eod) {
  using L = Fdm4Lay<PATCH>;
  extern __shared__ __align__(16) double T[];
  __shared__ int s_info[8];
  __shared__ int64_t s_cell[L::SLOTS];
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2;
  if (tid == 0) {
    const int64_t idx = blockIdx.x;
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    const int id = p.list ? p.list[idx] : (int)(p.start + idx);
    subdomain_info<3, PATCH>(p.geo, id, p.packed != 0, digit, base);
    for (int t = 0; t < 3; ++t) s_info[t] = digit[t];
    s_info[6] = digit[0] + 4 * digit[1] + 16 * digit[2];
    for (int s = 0; s < L::SLOTS; ++s) {
      int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
      if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
      s_cell[s] = (int64_t)cell_local<3>(p.geo, c) * L::NEc;
    }
    mbar_init(&s_bar, 1);
  }
  __syncthreads();
  if (warp == 0) {  // R_j r: one bulk copy per cell, densely
    if (lane == 0) mbar_expect_tx(&s_bar, L::SLOTS * L::NEc * 8);
    __syncwarp();
    if (lane < L::SLOTS) bulk_load(T + lane * L::NEc, p.r + s_cell[lane], L::NEc * 8, &s_bar);
  }
  const int dg0 = s_info[0], dg1 = s_info[1], dg2 = s_info[2], cls = s_info[6];
  const bool eo0 = p.eo && dg0 == 0 && eod, eo1 = p.eo && dg1 == 0 && eod,
             eo2 = p.eo && dg2 == 0 && eod;
  mbar_wait(&s_bar, 0);
  // ---- pass 1: Z^T along direction 0, dense rows -> registers -> swizzled T
  RowOut out[4];
  if (eo0) fdm4_pass1<PATCH, true>(T, zd, eod, dg0, warp, lane, out);
  else fdm4_pass1<PATCH, false>(T, zd, eod, dg0, warp, lane, out);
  __syncthreads();  // every dense row read before T overwrites them
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = 8 * (4 * warp + j) + g, i3 = r >> 4, i2 = r & 15;
    *reinterpret_cast<double2*>(&T[tz(i3, i2, out[j].ca)]) = make_double2(out[j].c[0], out[j].c[1]);
    *reinterpret_cast<double2*>(&T[tz(i3, i2, out[j].cb)]) = make_double2(out[j].c[2], out[j].c[3]);
  }
  __syncthreads();
  // ---- pass 2: Z^T along direction 1
  fdm4_cols<true>(T, zd, ztd, eod, eo1, 1, dg1, warp, lane);
  __syncthreads();
  // ---- pass 3: Z^T, 1/Lambda, Z along direction 2 on this warp's columns
  {
    const double* inv = p.invsum + (int64_t)cls * 4096;
    if (eo2) fdm4_pass3<true>(T, zd, ztd, eod, inv, dg2, warp, lane);
    else fdm4_pass3<false>(T, zd, ztd, eod, inv, dg2, warp, lane);
  }
  __syncthreads();
  // ---- pass 4: Z along direction 1
  fdm4_cols<false>(T, zd, ztd, eod, eo1, 1, dg1, warp, lane);
  __syncthreads();
  // ---- pass 5: Z along direction 0, times omega: swizzled T -> dense cell rows
  if (eo0) fdm4_pass5<true>(T, ztd, eod, dg0, warp, lane, p.omega, out);
  else fdm4_pass5<false>(T, ztd, eod, dg0, warp, lane, p.omega, out);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = 8 * (4 * warp + j) + g, i3 = r >> 4, i2 = r & 15;
    double* lo = T + L::dense(i3, i2, 0);
    double* hi = T + L::dense(i3, i2, 1);
    const int ca = out[j].ca, cb = out[j].cb;
    *reinterpret_cast<double2*>((ca < 8 ? lo + ca : hi + ca - 8)) = make_double2(out[j].c[0], out[j].c[1]);
    *reinterpret_cast<double2*>((cb < 8 ? lo + cb : hi + cb - 8)) = make_double2(out[j].c[2], out[j].c[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0 && lane < L::SLOTS) {  // omega y -> x: one fp64 bulk reduce-add per cell
    bulk_red_add(p.x + s_cell[lane], T + lane * L::NEc, L::NEc * 8);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

}  // namespace dgb
