// fdm_mma.cuh - fast-diagonalisation solves on the fp64 tensor cores
// (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) for 3D subdomains whose 1D size
// m is a multiple of 8 (patches m = 8, 16; cells n = 8, 16).
//
// x += omega * Z Lambda^-1 Z^T R r (fastdiag.py:457-496, 602-628).  Each
// contraction of the m^3 tensor along one direction is a small GEMM:
//   t = 2:  out[a][c]     = sum_k S[a][k] T[k][c]        (c = (i2,i1))
//   t = 1:  out[i3][a][j] = sum_k S[a][k] T[i3][k][j]
//   t = 0:  out[r][a]     = sum_k T[r][k] S[a][k]        (r = (i3,i2))
// S = Z^T (forward) or Z (backward) of the direction's boundary digit.  S is
// the A operand for t = 1, 2 and (as S^T) the B operand for t = 0; for an
// 8x4 tile both need lane value S[a0 + g][k0 + q] (g = lane/4, q = lane%4).
// Every warp owns whole output column (t = 1, 2) or row (t = 0) blocks across
// all of K, so each contraction runs in place in one shared tensor buffer.
// Strides: row 4 mod 16, plane 8 mod 16 doubles -> the 8-byte fragment loads
// and 16-byte C stores are bank-conflict free for all three directions.
// After the last forward contraction (t = 2) each warp scales its own columns
// by 1/Lambda and immediately runs the backward t = 2 contraction on them.
#pragma once
#include "fdm2.cuh"

#ifndef MMA_U
#define MMA_U 2
#endif

namespace dgb {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int M>
struct MmaLay {
  static_assert(M % 8 == 0, "tensor-core path needs m % 8 == 0");
  static constexpr int S2 = M + ((4 - (M % 16)) % 16 + 16) % 16;            // row stride = 4 mod 16
  static constexpr int S3r = M * S2;
  static constexpr int S3 = S3r + ((8 - (S3r % 16)) % 16 + 16) % 16;       // plane stride = 8 mod 16
  static constexpr int SZ = M * S3;                                        // doubles per tensor
  __device__ __forceinline__ static int at(int i3, int i2, int i1) { return i3 * S3 + i2 * S2 + i1; }
};

template <int M, bool PATCH>
struct MmaShape {
  static constexpr int WPS = (M == 16) ? 8 : 2;     // warps per subdomain
  static constexpr int GS = (M == 16) ? 1 : 2;      // subdomains per CTA
  static constexpr int NT = 32 * WPS * GS;
  static constexpr int N = PATCH ? M / 2 : M;
  static constexpr int SMEM = GS * MmaLay<M>::SZ;   // doubles
};

// S fragments for all (a0, k0) tiles: frag[(a0/8) * (M/4) + k0/4]
template <int M>
__device__ __forceinline__ void load_sfrag(const double* __restrict__ S, int lane,
                                           double (&fr)[(M / 8) * (M / 4)]) {
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int ta = 0; ta < M / 8; ++ta)
#pragma unroll
    for (int tk = 0; tk < M / 4; ++tk) fr[ta * (M / 4) + tk] = __ldg(S + (ta * 8 + g) * M + tk * 4 + q);
}

// contraction along t = 2 for the column blocks [cb0, cb0 + ncb) of this warp;
// optional fused scale-by-invsum + backward contraction with S2nd
template <int M, bool FUSED>
__device__ __forceinline__ void mma_dir2(double* T, const double (&fr)[(M / 8) * (M / 4)],
                                         const double (&fr2)[(M / 8) * (M / 4)],
                                         const double* __restrict__ inv, int lane, int cb0,
                                         int ncb) {
  using L = MmaLay<M>;
  constexpr int U = MMA_U;  // column blocks in flight per warp
  const int g = lane >> 2, q = lane & 3;
  for (int cbu = cb0; cbu < cb0 + ncb; cbu += U) {
    int i2[U], j0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) i2[u] = (cbu + u) / (M / 8), j0[u] = ((cbu + u) % (M / 8)) * 8;
    double c[U][M / 8][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ta = 0; ta < M / 8; ++ta) c[u][ta][0] = c[u][ta][1] = 0.0;
#pragma unroll
    for (int tk = 0; tk < M / 4; ++tk) {
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = T[L::at(tk * 4 + q, i2[u], j0[u] + g)];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ta = 0; ta < M / 8; ++ta) dmma884(c[u][ta][0], c[u][ta][1], fr[ta * (M / 4) + tk], b[u]);
    }
    __syncwarp();
    if (FUSED) {
      // scale rows a (eigen index along t = 2) by 1/Lambda, then the backward
      // contraction along t = 2 on the same columns
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ta = 0; ta < M / 8; ++ta) {
          const int a = ta * 8 + g;
          const int e = a * M * M + i2[u] * M + j0[u] + 2 * q;
          const double2 iv = __ldg(reinterpret_cast<const double2*>(inv + e));
          *reinterpret_cast<double2*>(&T[L::at(a, i2[u], j0[u] + 2 * q)]) =
              make_double2(c[u][ta][0] * iv.x, c[u][ta][1] * iv.y);
          c[u][ta][0] = c[u][ta][1] = 0.0;
        }
      __syncwarp();
#pragma unroll
      for (int tk = 0; tk < M / 4; ++tk) {
        double b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = T[L::at(tk * 4 + q, i2[u], j0[u] + g)];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int ta = 0; ta < M / 8; ++ta) dmma884(c[u][ta][0], c[u][ta][1], fr2[ta * (M / 4) + tk], b[u]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ta = 0; ta < M / 8; ++ta)
        *reinterpret_cast<double2*>(&T[L::at(ta * 8 + g, i2[u], j0[u] + 2 * q)]) =
            make_double2(c[u][ta][0], c[u][ta][1]);
    __syncwarp();
  }
}

// contraction along t = 1 for the (i3, column block) units [u0, u0 + nu)
template <int M>
__device__ __forceinline__ void mma_dir1(double* T, const double (&fr)[(M / 8) * (M / 4)],
                                         int lane, int u0, int nu) {
  using L = MmaLay<M>;
  constexpr int U = MMA_U;
  const int g = lane >> 2, q = lane & 3;
  for (int uu = u0; uu < u0 + nu; uu += U) {
    int i3[U], j0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) i3[u] = (uu + u) / (M / 8), j0[u] = ((uu + u) % (M / 8)) * 8;
    double c[U][M / 8][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ta = 0; ta < M / 8; ++ta) c[u][ta][0] = c[u][ta][1] = 0.0;
#pragma unroll
    for (int tk = 0; tk < M / 4; ++tk) {
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = T[L::at(i3[u], tk * 4 + q, j0[u] + g)];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ta = 0; ta < M / 8; ++ta) dmma884(c[u][ta][0], c[u][ta][1], fr[ta * (M / 4) + tk], b[u]);
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ta = 0; ta < M / 8; ++ta)
        *reinterpret_cast<double2*>(&T[L::at(i3[u], ta * 8 + g, j0[u] + 2 * q)]) =
            make_double2(c[u][ta][0], c[u][ta][1]);
    __syncwarp();
  }
}

// contraction along t = 0 for the row blocks [rb0, rb0 + nrb) (rows r = (i3,i2))
template <int M>
__device__ __forceinline__ void mma_dir0(double* T, const double (&fr)[(M / 8) * (M / 4)],
                                         int lane, int rb0, int nrb) {
  using L = MmaLay<M>;
  constexpr int U = MMA_U;
  const int g = lane >> 2, q = lane & 3;
  for (int rbu = rb0; rbu < rb0 + nrb; rbu += U) {
    int i3[U], i2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = (rbu + u) * 8 + g;  // this lane's A row
      i3[u] = r / M, i2[u] = r % M;
    }
    double c[U][M / 8][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int tn = 0; tn < M / 8; ++tn) c[u][tn][0] = c[u][tn][1] = 0.0;
#pragma unroll
    for (int tk = 0; tk < M / 4; ++tk) {
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = T[L::at(i3[u], i2[u], tk * 4 + q)];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int tn = 0; tn < M / 8; ++tn) dmma884(c[u][tn][0], c[u][tn][1], a[u], fr[tn * (M / 4) + tk]);
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int tn = 0; tn < M / 8; ++tn)
        *reinterpret_cast<double2*>(&T[L::at(i3[u], i2[u], tn * 8 + 2 * q)]) =
            make_double2(c[u][tn][0], c[u][tn][1]);
    __syncwarp();
  }
}

template <int M, bool PATCH>
__global__ void __launch_bounds__(MmaShape<M, PATCH>::NT)
fdm_mma_kernel(const __grid_constant__ Fdm2Params<3, M> p, const double* __restrict__ zg,
               const double* __restrict__ ztg) {
  // zg / ztg: device copies of Z and Z^T per digit (row-major M x M)
  using S = MmaShape<M, PATCH>;
  using L = MmaLay<M>;
  using R = Rows<3, M, PATCH>;
  constexpr int N = S::N, GS = S::GS, NT = S::NT;
  constexpr int NEc = N * N * N;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_info[GS][8];
  __shared__ int64_t s_cell[GS][R::SLOTS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < GS) {
    const int64_t idx = (int64_t)blockIdx.x * GS + tid;
    int* inf = s_info[tid];
    inf[7] = idx < p.count;
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    if (inf[7]) {
      const int id = p.list ? p.list[idx] : (int)(p.start + idx);
      subdomain_info<3, PATCH>(p.geo, id, p.packed != 0, digit, base);
    }
    for (int t = 0; t < 3; ++t) inf[t] = digit[t];
    inf[6] = digit[0] + 4 * digit[1] + 16 * digit[2];
    for (int s = 0; s < R::SLOTS; ++s) {
      int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
      if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
      s_cell[tid][s] = (int64_t)cell_local<3>(p.geo, c) * NEc;
    }
  }
  __syncthreads();
  // gather cell rows into the strided tensor
  for (int row = tid; row < GS * R::RPS; row += NT) {
    const int gg = row / R::RPS;
    if (!s_info[gg][7]) continue;
    const int rr = row - gg * R::RPS;
    const int slot = rr / R::RPC, w = rr - slot * R::RPC;
    const int i1 = w % N, i2 = w / N;
    const int s0 = slot & 1, s1 = (slot >> 1) & 1, s2 = (slot >> 2) & 1;
    double* dst = sm + gg * L::SZ + L::at(s2 * N + i2, s1 * N + i1, s0 * N);
    row_load<N>(dst, p.r + s_cell[gg][slot] + w * N);
  }
  __syncthreads();
  const int sub = warp / S::WPS, wl = warp % S::WPS;
  const bool active = s_info[sub][7];
  double* T = sm + sub * L::SZ;
  const int* dg = s_info[sub];
  constexpr int BLK = M * M / 8;            // column / row blocks per direction
  constexpr int PER = BLK / S::WPS;         // blocks per warp
  double fr[(M / 8) * (M / 4)], fr2[(M / 8) * (M / 4)];
  // forward: Z^T along t = 0, 1
  if (active) {
    load_sfrag<M>(ztg + dg[0] * M * M, lane, fr);
    mma_dir0<M>(T, fr, lane, wl * PER, PER);
  }
  __syncthreads();
  if (active) {
    load_sfrag<M>(ztg + dg[1] * M * M, lane, fr);
    mma_dir1<M>(T, fr, lane, wl * PER, PER);
  }
  __syncthreads();
  // t = 2: Z^T, scale by 1/Lambda, Z (fused per warp column block)
  if (active) {
    load_sfrag<M>(ztg + dg[2] * M * M, lane, fr);
    load_sfrag<M>(zg + dg[2] * M * M, lane, fr2);
    mma_dir2<M, true>(T, fr, fr2, p.invsum + (int64_t)dg[6] * M * M * M, lane, wl * PER, PER);
  }
  __syncthreads();
  // backward: Z along t = 1, 0
  if (active) {
    load_sfrag<M>(zg + dg[1] * M * M, lane, fr);
    mma_dir1<M>(T, fr, lane, wl * PER, PER);
  }
  __syncthreads();
  if (active) {
    load_sfrag<M>(zg + dg[0] * M * M, lane, fr);
    mma_dir0<M>(T, fr, lane, wl * PER, PER);
  }
  __syncthreads();
  // x += omega * y, whole cell rows
  for (int row = tid; row < GS * R::RPS; row += NT) {
    const int gg = row / R::RPS;
    if (!s_info[gg][7]) continue;
    const int rr = row - gg * R::RPS;
    const int slot = rr / R::RPC, w = rr - slot * R::RPC;
    const int i1 = w % N, i2 = w / N;
    const int s0 = slot & 1, s1 = (slot >> 1) & 1, s2 = (slot >> 2) & 1;
    const double* y = sm + gg * L::SZ + L::at(s2 * N + i2, s1 * N + i1, s0 * N);
    double* dst = p.x + s_cell[gg][slot] + w * N;
    if (p.atomic) row_red<N>(dst, y, p.omega);
    else row_update<N>(dst, y, p.omega, false);
  }
}

}  // namespace dgb
