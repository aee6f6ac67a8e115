// dist_op.cu - SIPG operator on multilinear (distorted) cells, SURVEY 8(f)
// row 3 (reference: dgop._volume_apply / _faces_apply non-Cartesian
// branches, dgop.py:432-481, 583-759; geometry dgop.py:277-374).
//
// 2D (all degrees) and 3D k <= 4 run dist_apply_reg_kernel: one thread per
// cell with everything in registers (below).  3D k = 5 runs dist_apply_kernel:
// 1-8 cells per CTA, all tensors of the cells in shared memory:
//  - volume: the d reference gradients at the n^d Gauss points by
//    sum-factorised contractions (values / derivative tables per direction,
//    shared prefixes), the symmetric metric detJ J^-1 J^-T w per point
//    (host-precomputed), and the adjoint contractions back to the nodes;
//  - faces: for each of the 2d faces the cell evaluates the value and the
//    full reference gradient of itself and (interior faces) of its
//    neighbour at the face Gauss points, forms the SIPG face moments with the
//    per-point penalty and normal-derivative factors, and adds only its own
//    side's contribution -- every interior face is evaluated by both of its
//    cells, so the kernel needs no atomics and no face colouring;
//  - out = A u, or out = b - A u.
// Index conventions: nodes canonical (direction 1 fastest); face fields
// [q_t2][q_t1] with t1 < t2 the transverse directions; the host geometry is
// in the reference's reversed layouts (first direction slowest).
#include "launch.h"

namespace dgb {

using DistArgs = dg_dist_args_t;  // include/dgmg_b200.h; ctypes mirror in distorted.py

template <int N>
struct DistTabs {
  double V[N * N], Dg[N * N], bv[2][N], bg[2][N];
};

template <int D, int N>
struct DistParams {
  const double* u;
  const double* b;
  double* out;
  const double* metric;
  const double* faces[3];
  const double* bnd[6];
  int n;
  DistTabs<N> tab;
};

// out[e] (+)= sum_j M(o, j) in[e | i_dir = j] over G consecutive N^K tensors
// (dir 0 fastest); M(o, j) = TR ? M[j*N + o] : M[o*N + j].  Ends with a barrier.
template <int K, int N, bool TR, bool ACC, int G = 1>
__device__ __forceinline__ void contract(double* out, const double* in, int dir, const double* M) {
  constexpr int TOT = G * (K == 3 ? N * N * N : (K == 2 ? N * N : N));
  const int stride = dir == 0 ? 1 : (dir == 1 ? N : N * N);
  for (int e = threadIdx.x; e < TOT; e += blockDim.x) {
    const int o = (e / stride) % N;
    const int base = e - o * stride;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(TR ? M[j * N + o] : M[o * N + j], in[base + j * stride], s);
    out[e] = ACC ? out[e] + s : s;
  }
  __syncthreads();
}

// canonical element index of cell-local nodes: (transverse e = i_t1 + N i_t2, i_tau)
template <int D, int N>
__device__ __forceinline__ int elem(int tau, int e, int i) {
  if (D == 2) {
    const int it = e;  // the one transverse direction
    return tau == 1 ? i + N * it : it + N * i;
  }
  const int a = e % N, b = e / N;  // i_t1, i_t2 (t1 < t2)
  if (tau == 1) return i + N * a + N * N * b;
  if (tau == 2) return a + N * i + N * N * b;
  return a + N * b + N * N * i;
}

// traces along tau at side p of G cells: tv = sum_i bv_p[i] X, tg = sum_i bg_p[i] X
template <int D, int N, int G>
__device__ __forceinline__ void traces(const DistTabs<N>& T, const double* X, int tau, int p,
                                       double* tv, double* tg) {
  constexpr int FT = D == 3 ? N * N : N;
  constexpr int ND = D == 3 ? N * N * N : N * N;
  for (int x = threadIdx.x; x < G * FT; x += blockDim.x) {
    const int g = x / FT, e = x - g * FT;
    double sv = 0.0, sg = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double v = X[g * ND + elem<D, N>(tau, e, i)];
      sv = fma(T.bv[p][i], v, sv);
      sg = fma(T.bg[p][i], v, sg);
    }
    tv[x] = sv;
    tg[x] = sg;
  }
  __syncthreads();
}

// value and the d reference gradients at the face points from the traces;
// G[t] for t = 0..D-1 (direction t+1): normal for t+1 == tau
template <int D, int N, int G>
__device__ __forceinline__ void face_values(const DistTabs<N>& T, const double* tv,
                                            const double* tg, int tau, double* val, double* G0,
                                            double* G1, double* G2, double* tmp) {
  double* Gd[3] = {G0, G1, G2};
  if (D == 2) {
    const int tt = tau == 1 ? 1 : 0;  // transverse direction index (0-based)
    contract<1, N, false, false, G>(val, tv, 0, T.V);
    contract<1, N, false, false, G>(Gd[tt], tv, 0, T.Dg);
    contract<1, N, false, false, G>(Gd[tau - 1], tg, 0, T.V);
    return;
  }
  const int t1 = tau == 1 ? 1 : 0, t2 = tau == 3 ? 1 : 2;  // 0-based transverse dirs
  contract<2, N, false, false, G>(tmp, tv, 0, T.V);         // V along t1
  contract<2, N, false, false, G>(val, tmp, 1, T.V);        // V along t2
  contract<2, N, false, false, G>(Gd[t2], tmp, 1, T.Dg);    // d/d t2
  contract<2, N, false, false, G>(tmp, tv, 0, T.Dg);        // D along t1
  contract<2, N, false, false, G>(Gd[t1], tmp, 1, T.V);     // d/d t1
  contract<2, N, false, false, G>(tmp, tg, 0, T.V);
  contract<2, N, false, false, G>(Gd[tau - 1], tmp, 1, T.V);  // normal
}

// adjoint: acc[node] += bv_p (x) (V^T V^T val + tangential adjoints of M_t)
//                     + bg_p (x) V^T V^T M_tau
template <int D, int N, int G>
__device__ __forceinline__ void face_scatter(const DistTabs<N>& T, double* acc, int tau, int p,
                                             double* mval, double* M0, double* M1, double* M2,
                                             double* tv, double* tg, double* tmp) {
  double* Mm[3] = {M0, M1, M2};
  constexpr int FT = D == 3 ? N * N : N;
  if (D == 2) {
    const int tt = tau == 1 ? 1 : 0;
    contract<1, N, true, false, G>(tv, mval, 0, T.V);
    contract<1, N, true, true, G>(tv, Mm[tt], 0, T.Dg);
    contract<1, N, true, false, G>(tg, Mm[tau - 1], 0, T.V);
  } else {
    const int t1 = tau == 1 ? 1 : 0, t2 = tau == 3 ? 1 : 2;
    // tv = V1^T V2^T mval + V1^T D2^T M_t2 + D1^T V2^T M_t1;  tg = V1^T V2^T M_tau
    contract<2, N, true, false, G>(tmp, mval, 1, T.V);
    contract<2, N, true, true, G>(tmp, Mm[t2], 1, T.Dg);
    contract<2, N, true, false, G>(tv, tmp, 0, T.V);
    contract<2, N, true, false, G>(tmp, Mm[t1], 1, T.V);
    contract<2, N, true, true, G>(tv, tmp, 0, T.Dg);
    contract<2, N, true, false, G>(tmp, Mm[tau - 1], 1, T.V);
    contract<2, N, true, false, G>(tg, tmp, 0, T.V);
  }
  constexpr int ND = D == 3 ? N * N * N : N * N;
  for (int xx = threadIdx.x; xx < G * ND; xx += blockDim.x) {
    const int g = xx / ND, x = xx - g * ND;
    int i, e;  // decompose x into (transverse e, i_tau)
    if (D == 2) {
      const int i1 = x % N, i2 = x / N;
      i = tau == 1 ? i1 : i2;
      e = tau == 1 ? i2 : i1;
    } else {
      const int i1 = x % N, i2 = (x / N) % N, i3 = x / (N * N);
      if (tau == 1) { i = i1; e = i2 + N * i3; }
      else if (tau == 2) { i = i2; e = i1 + N * i3; }
      else { i = i3; e = i1 + N * i2; }
    }
    acc[xx] += T.bv[p][i] * tv[g * FT + e] + T.bg[p][i] * tg[g * FT + e];
  }
  __syncthreads();
}

// cells per CTA: a few small cells share the 128 threads
template <int D, int N>
__host__ __device__ constexpr int dist_cells() {
  constexpr int ND = D == 3 ? N * N * N : N * N;
  return ND > 64 ? 1 : (128 / ND > 8 ? 8 : 128 / ND);
}

// shared doubles of dist_apply_kernel; large cells alias the face-phase
// buffers with the volume-phase ones (see the kernel)
template <int D, int N>
__host__ __device__ constexpr bool dist_alias() {
  constexpr size_t ND = D == 3 ? N * N * N : N * N, FT = D == 3 ? N * N : N;
  return N >= 7 && sizeof(double) * dist_cells<D, N>() * (7 * ND + 19 * FT) > 160 * 1024;
}
template <int D, int N>
__host__ __device__ constexpr size_t dist_smem_doubles() {
  constexpr size_t ND = D == 3 ? N * N * N : N * N, FT = D == 3 ? N * N : N;
  return dist_cells<D, N>() * (dist_alias<D, N>() ? 6 * ND : 7 * ND + 19 * FT);
}

template <int D, int N>
__global__ void __launch_bounds__(128) dist_apply_kernel(const __grid_constant__ DistParams<D, N> P,
                                                         int64_t ncells) {
  constexpr int G = dist_cells<D, N>();
  constexpr int ND = D == 3 ? N * N * N : N * N;
  constexpr int FT = D == 3 ? N * N : N;
  constexpr int S = D == 3 ? 6 : 3;
  extern __shared__ __align__(16) double sm[];
  // seven cell tensors plus the face scratch; for large cells (dist_alias)
  // the face phase reuses the volume phase's dead buffers: the neighbour
  // copy NB lives in A and the 19 face fields in B, E, F (19 n^(d-1) <= 3 n^d
  // for n >= 7), which lets 3D n = 16 fit in 192 KB
  constexpr bool AL = dist_alias<D, N>();
  double* U = sm;
  double* A = U + G * ND;
  double* C = A + G * ND;
  double* B = C + G * ND;
  double* E = B + G * ND;
  double* F = E + G * ND;
  double* NB = AL ? A : F + G * ND;
  double* fs = AL ? B : NB + G * ND;  // face scratch: 19 fields of G * FT
  __shared__ int s_c[G][3];
  __shared__ int s_ok[G];
  const int n = P.n;
  const int64_t cell0 = (int64_t)blockIdx.x * G;
  if (threadIdx.x < G) {
    const int64_t cell = cell0 + threadIdx.x;
    s_ok[threadIdx.x] = cell < ncells;
    int64_t r = cell < ncells ? cell : 0;
    for (int t = 0; t < 3; ++t) {
      s_c[threadIdx.x][t] = t < D ? (int)(r % n) : 0;
      r /= n;
    }
  }
  const DistTabs<N>& T = P.tab;
  for (int x = threadIdx.x; x < G * ND; x += blockDim.x) {
    const int64_t cell = cell0 + x / ND;
    U[x] = cell < ncells ? P.u[cell * ND + x % ND] : 0.0;
  }
  __syncthreads();
  // ---------------- volume
  if (D == 3) {
    contract<3, N, false, false, G>(A, U, 0, T.V);
    contract<3, N, false, false, G>(B, U, 0, T.Dg);
    contract<3, N, false, false, G>(C, A, 1, T.V);    // x12vv
    contract<3, N, false, false, G>(E, B, 1, T.V);    // x12dv
    contract<3, N, false, false, G>(F, A, 1, T.Dg);   // x12vd
    contract<3, N, false, false, G>(A, E, 2, T.V);    // g1
    contract<3, N, false, false, G>(B, F, 2, T.V);    // g2
    contract<3, N, false, false, G>(E, C, 2, T.Dg);   // g3
    for (int x = threadIdx.x; x < G * ND; x += blockDim.x) {
      const int g = x / ND, e = x - g * ND;
      const int q1 = e % N, q2 = (e / N) % N, q3 = e / (N * N);
      const int64_t cell = s_ok[g] ? cell0 + g : 0;
      const double* gm = P.metric + (cell * ND + q1 * N * N + q2 * N + q3) * S;  // reversed
      const double a1 = A[x], a2 = B[x], a3 = E[x];
      A[x] = gm[0] * a1 + gm[3] * a2 + gm[4] * a3;
      B[x] = gm[3] * a1 + gm[1] * a2 + gm[5] * a3;
      E[x] = gm[4] * a1 + gm[5] * a2 + gm[2] * a3;
    }
    __syncthreads();
    contract<3, N, true, false, G>(C, A, 2, T.V);     // s3_1
    contract<3, N, true, false, G>(F, B, 2, T.V);     // s3_2
    contract<3, N, true, false, G>(A, E, 2, T.Dg);    // s3_3
    contract<3, N, true, false, G>(B, C, 1, T.V);     // s2_1
    contract<3, N, true, false, G>(E, F, 1, T.Dg);    // s2_23 = D^T s3_2
    contract<3, N, true, true, G>(E, A, 1, T.V);      //        + V^T s3_3
    contract<3, N, true, false, G>(C, B, 0, T.Dg);
    contract<3, N, true, true, G>(C, E, 0, T.V);
  } else {
    contract<2, N, false, false, G>(A, U, 0, T.V);    // x1v
    contract<2, N, false, false, G>(B, U, 0, T.Dg);   // x1d
    contract<2, N, false, false, G>(E, B, 1, T.V);    // g1
    contract<2, N, false, false, G>(F, A, 1, T.Dg);   // g2
    for (int x = threadIdx.x; x < G * ND; x += blockDim.x) {
      const int g = x / ND, e = x - g * ND;
      const int q1 = e % N, q2 = e / N;
      const int64_t cell = s_ok[g] ? cell0 + g : 0;
      const double* gm = P.metric + (cell * ND + q1 * N + q2) * S;
      const double a1 = E[x], a2 = F[x];
      E[x] = gm[0] * a1 + gm[2] * a2;
      F[x] = gm[2] * a1 + gm[1] * a2;
    }
    __syncthreads();
    contract<2, N, true, false, G>(A, E, 1, T.V);
    contract<2, N, true, false, G>(B, F, 1, T.Dg);
    contract<2, N, true, false, G>(C, A, 0, T.Dg);
    contract<2, N, true, true, G>(C, B, 0, T.V);
  }
  // ---------------- faces
  constexpr int GF = G * FT;
  double* tvo = fs;            double* tgo = fs + GF;
  double* tvn = fs + 2 * GF;   double* tgn = fs + 3 * GF;
  double* vo = fs + 4 * GF;    double* go[3] = {fs + 5 * GF, fs + 6 * GF, fs + 7 * GF};
  double* vn = fs + 8 * GF;    double* gn[3] = {fs + 9 * GF, fs + 10 * GF, fs + 11 * GF};
  double* mv = fs + 12 * GF;   double* mm[3] = {fs + 13 * GF, fs + 14 * GF, fs + 15 * GF};
  double* tmp = fs + 16 * GF;  double* sv = fs + 17 * GF;  double* sg = fs + 18 * GF;
  for (int tau = 1; tau <= D; ++tau) {
    const int t0 = tau - 1;
    for (int p = 0; p < 2; ++p) {
      traces<D, N, G>(T, U, tau, p, tvo, tgo);
      face_values<D, N, G>(T, tvo, tgo, tau, vo, go[0], go[1], go[2], tmp);
      // neighbours across this face (zeros where the face is on the boundary)
      for (int x = threadIdx.x; x < G * ND; x += blockDim.x) {
        const int g = x / ND;
        const int* c = s_c[g];
        const bool bnd = !s_ok[g] || (p == 0 ? c[t0] == 0 : c[t0] == n - 1);
        double v = 0.0;
        if (!bnd) {
          int64_t nid = 0;
          for (int t = D - 1; t >= 0; --t) nid = nid * n + c[t] + (t == t0 ? (p == 1 ? 1 : -1) : 0);
          v = P.u[nid * ND + x % ND];
        }
        NB[x] = v;
      }
      __syncthreads();
      traces<D, N, G>(T, NB, tau, 1 - p, tvn, tgn);
      face_values<D, N, G>(T, tvn, tgn, tau, vn, gn[0], gn[1], gn[2], tmp);
      // face moments at the points, own side only
      for (int x = threadIdx.x; x < GF; x += blockDim.x) {
        const int g = x / FT, e = x - g * FT;
        const int* c = s_c[g];
        const bool boundary = p == 0 ? c[t0] == 0 : c[t0] == n - 1;
        const int gi = D == 3 ? (e % N) * N + e / N : e;  // reversed face-point index
        int64_t f = 0;  // face index in the reference's slab order (first direction slowest)
        if (boundary) {
          for (int t = D - 1; t >= 0; --t)
            if (t != t0) f = f * n + c[t];
          const double* gg = P.bnd[2 * t0 + p] + (f * FT + gi) * (1 + D);
          double m = vo[x] * gg[0];
          for (int t = 0; t < D; ++t) m -= go[t][x] * gg[1 + t];
          mv[x] = s_ok[g] ? m : 0.0;
          for (int t = 0; t < D; ++t) mm[t][x] = s_ok[g] ? -vo[x] * gg[1 + t] : 0.0;
        } else {
          for (int t = D - 1; t >= 0; --t)
            f = f * (t == t0 ? n - 1 : n) + c[t] - (t == t0 && p == 0 ? 1 : 0);
          const double* gg = P.faces[t0] + (f * FT + gi) * (1 + 2 * D);
          const bool left = p == 1;
          const double vp = left ? vo[x] : vn[x], vmn = left ? vn[x] : vo[x];
          const double jump = vp - vmn;
          double m = jump * gg[0];
          for (int t = 0; t < D; ++t) {
            const double gp = left ? go[t][x] : gn[t][x];
            const double gm = left ? gn[t][x] : go[t][x];
            m -= gp * gg[1 + t] + gm * gg[1 + D + t];
          }
          mv[x] = s_ok[g] ? (left ? m : -m) : 0.0;
          for (int t = 0; t < D; ++t)
            mm[t][x] = s_ok[g] ? -jump * gg[(left ? 1 : 1 + D) + t] : 0.0;
        }
      }
      __syncthreads();
      face_scatter<D, N, G>(T, C, tau, p, mv, mm[0], mm[1], mm[2], sv, sg, tmp);
    }
  }
  for (int x = threadIdx.x; x < G * ND; x += blockDim.x) {
    const int64_t cell = cell0 + x / ND;
    if (cell < ncells) {
      const int64_t gx = cell * ND + x % ND;
      P.out[gx] = P.b ? P.b[gx] - C[x] : C[x];
    }
  }
}

// ---------------------------------------------------------------------------
// Register variant (2D all degrees, 3D k <= 4; dist_reg_ok): one thread per
// cell, the cell's nodes, quadrature values and face fields in registers
// (every index is a compile-time constant after unrolling; from 2D n = 6 /
// 3D n = 4 the surplus spills to L1-resident local memory and still beats
// the shared kernel), the basis tables in the constant bank (kernel
// parameters), no shared memory and no barriers.  Same arithmetic as
// dist_apply_kernel, term for term.

template <int K, int N, int DIR, bool TR, bool ACC>
__device__ __forceinline__ void rcon(double* out, const double* in, const double* M) {
  constexpr int TOT = K == 3 ? N * N * N : (K == 2 ? N * N : N);
  constexpr int stride = DIR == 0 ? 1 : (DIR == 1 ? N : N * N);
#pragma unroll
  for (int e = 0; e < TOT; ++e) {
    const int o = (e / stride) % N;
    const int base = e - o * stride;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(TR ? M[j * N + o] : M[o * N + j], in[base + j * stride], s);
    out[e] = ACC ? out[e] + s : s;
  }
}

template <int CNT>
__device__ __forceinline__ void rload(double* dst, const double* __restrict__ src) {
  if constexpr (CNT % 2 == 0) {  // 16-byte aligned: CNT even, base 256-byte aligned
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int i = 0; i < CNT / 2; ++i) {
      const double2 v = __ldg(s2 + i);
      dst[2 * i] = v.x;
      dst[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < CNT; ++i) dst[i] = __ldg(src + i);
  }
}

template <int D, int N, int TAU>
__device__ __forceinline__ void rtraces(const double* bv, const double* bg, const double* X,
                                        double* tv, double* tg) {
  constexpr int FT = D == 3 ? N * N : N;
#pragma unroll
  for (int e = 0; e < FT; ++e) {
    double sv = 0.0, sg = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double v = X[elem<D, N>(TAU, e, i)];
      sv = fma(bv[i], v, sv);
      sg = fma(bg[i], v, sg);
    }
    tv[e] = sv;
    tg[e] = sg;
  }
}

template <int D, int N, int TAU>
__device__ __forceinline__ void rface_values(const DistTabs<N>& T, const double* tv,
                                             const double* tg, double* val,
                                             double (*Gd)[D == 3 ? N * N : N]) {
  if constexpr (D == 2) {
    constexpr int tt = TAU == 1 ? 1 : 0;
    rcon<1, N, 0, false, false>(val, tv, T.V);
    rcon<1, N, 0, false, false>(Gd[tt], tv, T.Dg);
    rcon<1, N, 0, false, false>(Gd[TAU - 1], tg, T.V);
  } else {
    constexpr int t1 = TAU == 1 ? 1 : 0, t2 = TAU == 3 ? 1 : 2;
    double tmp[N * N];
    rcon<2, N, 0, false, false>(tmp, tv, T.V);
    rcon<2, N, 1, false, false>(val, tmp, T.V);
    rcon<2, N, 1, false, false>(Gd[t2], tmp, T.Dg);
    rcon<2, N, 0, false, false>(tmp, tv, T.Dg);
    rcon<2, N, 1, false, false>(Gd[t1], tmp, T.V);
    rcon<2, N, 0, false, false>(tmp, tg, T.V);
    rcon<2, N, 1, false, false>(Gd[TAU - 1], tmp, T.V);
  }
}

template <int D, int N, int TAU, int PS>
__device__ __forceinline__ void rface_scatter(const DistTabs<N>& T, double* C, const double* mval,
                                              double (*Mm)[D == 3 ? N * N : N]) {
  constexpr int FT = D == 3 ? N * N : N;
  constexpr int ND = D == 3 ? N * N * N : N * N;
  double sv[FT], sg[FT];
  if constexpr (D == 2) {
    constexpr int tt = TAU == 1 ? 1 : 0;
    rcon<1, N, 0, true, false>(sv, mval, T.V);
    rcon<1, N, 0, true, true>(sv, Mm[tt], T.Dg);
    rcon<1, N, 0, true, false>(sg, Mm[TAU - 1], T.V);
  } else {
    constexpr int t1 = TAU == 1 ? 1 : 0, t2 = TAU == 3 ? 1 : 2;
    double tmp[FT];
    rcon<2, N, 1, true, false>(tmp, mval, T.V);
    rcon<2, N, 1, true, true>(tmp, Mm[t2], T.Dg);
    rcon<2, N, 0, true, false>(sv, tmp, T.V);
    rcon<2, N, 1, true, false>(tmp, Mm[t1], T.V);
    rcon<2, N, 0, true, true>(sv, tmp, T.Dg);
    rcon<2, N, 1, true, false>(tmp, Mm[TAU - 1], T.V);
    rcon<2, N, 0, true, false>(sg, tmp, T.V);
  }
#pragma unroll
  for (int x = 0; x < ND; ++x) {
    int i, e;
    if constexpr (D == 2) {
      const int i1 = x % N, i2 = x / N;
      i = TAU == 1 ? i1 : i2;
      e = TAU == 1 ? i2 : i1;
    } else {
      const int i1 = x % N, i2 = (x / N) % N, i3 = x / (N * N);
      if (TAU == 1) { i = i1; e = i2 + N * i3; }
      else if (TAU == 2) { i = i2; e = i1 + N * i3; }
      else { i = i3; e = i1 + N * i2; }
    }
    C[x] += T.bv[PS][i] * sv[e] + T.bg[PS][i] * sg[e];
  }
}

// one face of the cell (direction TAU, side PS): own side's moments, scattered into C
template <int D, int N, int TAU, int PS>
__device__ __forceinline__ void rface(const DistParams<D, N>& P, const double* U, double* C,
                                      const int* c) {
  constexpr int ND = D == 3 ? N * N * N : N * N;
  constexpr int FT = D == 3 ? N * N : N;
  constexpr int t0 = TAU - 1;
  const DistTabs<N>& T = P.tab;
  const int n = P.n;
  double tv[FT], tg[FT], vo[FT], go[D][FT];
  rtraces<D, N, TAU>(T.bv[PS], T.bg[PS], U, tv, tg);
  rface_values<D, N, TAU>(T, tv, tg, vo, go);
  double mv[FT], mm[D][FT];
  const bool boundary = PS == 0 ? c[t0] == 0 : c[t0] == n - 1;
  if (boundary) {
    int64_t f = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t)
      if (t != t0) f = f * n + c[t];
    const double* gb = P.bnd[2 * t0 + PS] + f * FT * (1 + D);
#pragma unroll
    for (int e = 0; e < FT; ++e) {
      const int gi = D == 3 ? (e % N) * N + e / N : e;
      const double* gg = gb + gi * (1 + D);
      double m = vo[e] * __ldg(gg);
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const double w = __ldg(gg + 1 + t);
        m -= go[t][e] * w;
        mm[t][e] = -vo[e] * w;
      }
      mv[e] = m;
    }
  } else {
    int64_t nid = 0, f = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t) {
      nid = nid * n + c[t] + (t == t0 ? (PS == 1 ? 1 : -1) : 0);
      f = f * (t == t0 ? n - 1 : n) + c[t] - (t == t0 && PS == 0 ? 1 : 0);
    }
    double NB[ND];
    rload<ND>(NB, P.u + nid * ND);
    double tvn[FT], tgn[FT], vn[FT], gn[D][FT];
    rtraces<D, N, TAU>(T.bv[1 - PS], T.bg[1 - PS], NB, tvn, tgn);
    rface_values<D, N, TAU>(T, tvn, tgn, vn, gn);
    const double* gf = P.faces[t0] + f * FT * (1 + 2 * D);
    constexpr bool left = PS == 1;
#pragma unroll
    for (int e = 0; e < FT; ++e) {
      const int gi = D == 3 ? (e % N) * N + e / N : e;
      const double* gg = gf + gi * (1 + 2 * D);
      const double vp = left ? vo[e] : vn[e], vmn = left ? vn[e] : vo[e];
      const double jump = vp - vmn;
      double m = jump * __ldg(gg);
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const double gp = left ? go[t][e] : gn[t][e];
        const double gm = left ? gn[t][e] : go[t][e];
        m -= gp * __ldg(gg + 1 + t) + gm * __ldg(gg + 1 + D + t);
      }
      mv[e] = left ? m : -m;
#pragma unroll
      for (int t = 0; t < D; ++t) mm[t][e] = -jump * __ldg(gg + (left ? 1 : 1 + D) + t);
    }
  }
  rface_scatter<D, N, TAU, PS>(T, C, mv, mm);
}

// the register kernel wins even where it spills (2D n = 6..8, 3D n = 4, 5:
// local-memory spills stay in L1); only at 3D n = 6 is the shared kernel faster
template <int D, int N>
__host__ __device__ constexpr bool dist_reg_ok() {
  return (D == 2 && N <= 8) || (D == 3 && N <= 5);
}

// CTAs per SM the register budget targets (176 -> 168 registers at 2D n = 4: 3 CTAs, not 2)
template <int D, int N>
__host__ __device__ constexpr int dist_reg_minb() {
  return D == 2 ? (N == 2 ? 8 : N == 3 ? 5 : N == 4 ? 3 : 2) : (N == 2 ? 4 : 1);
}

template <int D, int N>
__global__ void __launch_bounds__(128, dist_reg_minb<D, N>())
    dist_apply_reg_kernel(const __grid_constant__ DistParams<D, N> P, int64_t ncells) {
  constexpr int ND = D == 3 ? N * N * N : N * N;
  constexpr int S = D == 3 ? 6 : 3;
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= ncells) return;
  const DistTabs<N>& T = P.tab;
  int c[3];
  {
    int64_t r = cell;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      c[t] = t < D ? (int)(r % P.n) : 0;
      r /= P.n;
    }
  }
  double U[ND], C[ND];
  rload<ND>(U, P.u + cell * ND);
  {  // volume
    double g[D][ND];
    if constexpr (D == 3) {
      double A[ND], B[ND], X[ND];
      rcon<3, N, 0, false, false>(A, U, T.V);
      rcon<3, N, 0, false, false>(B, U, T.Dg);
      rcon<3, N, 1, false, false>(X, B, T.V);   // x12dv
      rcon<3, N, 2, false, false>(g[0], X, T.V);
      rcon<3, N, 1, false, false>(X, A, T.Dg);  // x12vd
      rcon<3, N, 2, false, false>(g[1], X, T.V);
      rcon<3, N, 1, false, false>(X, A, T.V);   // x12vv
      rcon<3, N, 2, false, false>(g[2], X, T.Dg);
    } else {
      double A[ND], B[ND];
      rcon<2, N, 0, false, false>(A, U, T.V);
      rcon<2, N, 0, false, false>(B, U, T.Dg);
      rcon<2, N, 1, false, false>(g[0], B, T.V);
      rcon<2, N, 1, false, false>(g[1], A, T.Dg);
    }
    const double* gmc = P.metric + cell * ND * S;
#pragma unroll
    for (int e = 0; e < (D == 3 ? ND : 0); ++e) {
      if constexpr (D == 3) {
        const int q1 = e % N, q2 = (e / N) % N, q3 = e / (N * N);
        const double2* m2 = reinterpret_cast<const double2*>(gmc + (q1 * N * N + q2 * N + q3) * S);
        const double2 m01 = __ldg(m2), m23 = __ldg(m2 + 1), m45 = __ldg(m2 + 2);  // reversed
        const double a1 = g[0][e], a2 = g[1][e], a3 = g[2][e];
        g[0][e] = m01.x * a1 + m23.y * a2 + m45.x * a3;
        g[1][e] = m23.y * a1 + m01.y * a2 + m45.y * a3;
        g[2][e] = m45.x * a1 + m45.y * a2 + m23.x * a3;
      }
    }
    if constexpr (D == 2) {  // whole-cell metric block: 16-byte loads (2D is faster so)
      double gm[ND * S];
      rload<ND * S>(gm, gmc);
#pragma unroll
      for (int e = 0; e < ND; ++e) {
        const int q1 = e % N, q2 = e / N;
        const double* m = gm + (q1 * N + q2) * S;
        const double a1 = g[0][e], a2 = g[1][e];
        g[0][e] = m[0] * a1 + m[2] * a2;
        g[1][e] = m[2] * a1 + m[1] * a2;
      }
    }
    if constexpr (D == 3) {
      double A[ND], B[ND], X[ND];
      rcon<3, N, 2, true, false>(A, g[0], T.V);   // s3_1
      rcon<3, N, 1, true, false>(B, A, T.V);      // s2_1
      rcon<3, N, 2, true, false>(A, g[1], T.V);   // s3_2
      rcon<3, N, 1, true, false>(X, A, T.Dg);
      rcon<3, N, 2, true, false>(A, g[2], T.Dg);  // s3_3
      rcon<3, N, 1, true, true>(X, A, T.V);       // s2_23
      rcon<3, N, 0, true, false>(C, B, T.Dg);
      rcon<3, N, 0, true, true>(C, X, T.V);
    } else {
      double A[ND], B[ND];
      rcon<2, N, 1, true, false>(A, g[0], T.V);
      rcon<2, N, 1, true, false>(B, g[1], T.Dg);
      rcon<2, N, 0, true, false>(C, A, T.Dg);
      rcon<2, N, 0, true, true>(C, B, T.V);
    }
  }
  rface<D, N, 1, 0>(P, U, C, c);
  rface<D, N, 1, 1>(P, U, C, c);
  rface<D, N, 2, 0>(P, U, C, c);
  rface<D, N, 2, 1>(P, U, C, c);
  if constexpr (D == 3) {
    rface<D, N, 3, 0>(P, U, C, c);
    rface<D, N, 3, 1>(P, U, C, c);
  }
  double* o = P.out + cell * ND;
  if (P.b) {
    double B[ND];
    rload<ND>(B, P.b + cell * ND);
#pragma unroll
    for (int x = 0; x < ND; ++x) C[x] = B[x] - C[x];
  }
  if constexpr (ND % 2 == 0) {
#pragma unroll
    for (int x = 0; x < ND; x += 2) reinterpret_cast<double2*>(o)[x / 2] = make_double2(C[x], C[x + 1]);
  } else {
#pragma unroll
    for (int x = 0; x < ND; ++x) o[x] = C[x];
  }
}

// Surrogate cell solves on multilinear levels (fastdiag.py:381-436, 457-496):
// x_c += omega (Z_d x .. x Z_1) diag(1/Lambda_c) (Z_d^T x .. x Z_1^T) r_c with
// per-cell 1D eigenbases Z_t (global memory, staged in shared memory); small
// cells are batched G per 128-thread CTA like the operator kernel.
template <int D, int N, int G, bool TR>
__device__ __forceinline__ void contract_cells(double* out, const double* in, int dir,
                                               const double* Zs, int t) {
  constexpr int ND = D == 3 ? N * N * N : N * N;
  const int stride = dir == 0 ? 1 : (dir == 1 ? N : N * N);
  for (int e = threadIdx.x; e < G * ND; e += blockDim.x) {
    const double* M = Zs + ((e / ND) * D + t) * N * N;
    const int o = (e / stride) % N;
    const int base = e - o * stride;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(TR ? M[j * N + o] : M[o * N + j], in[base + j * stride], s);
    out[e] = s;
  }
  __syncthreads();
}

template <int D, int N>
__global__ void __launch_bounds__(128)
    dist_cell_fdm_kernel(const double* __restrict__ r, double* __restrict__ x,
                         const double* __restrict__ Z, const double* __restrict__ inv,
                         const int32_t* __restrict__ list, int64_t nitems, int64_t ncells,
                         double omega) {
  constexpr int G = dist_cells<D, N>();
  constexpr int ND = D == 3 ? N * N * N : N * N;
  extern __shared__ __align__(16) double sm[];
  double* T0 = sm;
  double* T1 = T0 + G * ND;
  double* Zs = T1 + G * ND;
  __shared__ int64_t s_cell[G];
  const int64_t i0 = (int64_t)blockIdx.x * G;
  if (threadIdx.x < G) {
    const int64_t it = i0 + threadIdx.x;
    s_cell[threadIdx.x] = it < nitems ? (list ? (int64_t)list[it] : it) : -1;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D * N * N; e += blockDim.x) {
    const int g = e / (D * N * N), q = e - g * D * N * N, t = q / (N * N);
    const int64_t cell = s_cell[g];
    Zs[e] = cell >= 0 ? Z[((int64_t)t * ncells + cell) * N * N + q - t * N * N] : 0.0;
  }
  for (int e = threadIdx.x; e < G * ND; e += blockDim.x) {
    const int64_t cell = s_cell[e / ND];
    T0[e] = cell >= 0 ? r[cell * ND + e % ND] : 0.0;
  }
  __syncthreads();
  double* a = T0;
  double* b = T1;
  for (int t = 0; t < D; ++t) {  // forward: Z^T along each direction
    contract_cells<D, N, G, true>(b, a, t, Zs, t);
    double* s = a; a = b; b = s;
  }
  for (int e = threadIdx.x; e < G * ND; e += blockDim.x) {  // 1/Lambda, reversed index
    const int64_t cell = s_cell[e / ND];
    const int el = e % ND;
    int ri;
    if (D == 3) ri = (el % N) * N * N + ((el / N) % N) * N + el / (N * N);
    else ri = (el % N) * N + el / N;
    a[e] *= cell >= 0 ? inv[cell * ND + ri] : 0.0;
  }
  __syncthreads();
  for (int t = D - 1; t >= 0; --t) {  // backward: Z along each direction
    contract_cells<D, N, G, false>(b, a, t, Zs, t);
    double* s = a; a = b; b = s;
  }
  for (int e = threadIdx.x; e < G * ND; e += blockDim.x) {
    const int64_t cell = s_cell[e / ND];
    if (cell >= 0) x[cell * ND + e % ND] = fma(omega, a[e], x[cell * ND + e % ND]);
  }
}

// register variant (2D k <= 6, 3D k <= 3): one thread per cell, r_c, the d eigenbases
// and the intermediate tensors in registers; no shared memory, no barriers
template <int D, int N>
__host__ __device__ constexpr bool dist_fdm_reg_ok() {
  return (D == 2 && N <= 7) || (D == 3 && N <= 4);
}

template <int D, int N>
__global__ void __launch_bounds__(128)
    dist_cell_fdm_reg_kernel(const double* __restrict__ r, double* __restrict__ x,
                             const double* __restrict__ Z, const double* __restrict__ inv,
                             const int32_t* __restrict__ list, int64_t nitems, int64_t ncells,
                             double omega) {
  constexpr int ND = D == 3 ? N * N * N : N * N;
  constexpr int NN = N * N;
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= nitems) return;
  const int64_t cell = list ? (int64_t)list[it] : it;
  double a[ND], b[ND], Z0[NN], Z1[NN], Z2[D == 3 ? NN : 1];
  rload<NN>(Z0, Z + cell * NN);
  rload<NN>(Z1, Z + (ncells + cell) * NN);
  if constexpr (D == 3) rload<NN>(Z2, Z + (2 * ncells + cell) * NN);
  rload<ND>(a, r + cell * ND);
  rcon<D, N, 0, true, false>(b, a, Z0);  // forward: Z^T along each direction
  rcon<D, N, 1, true, false>(a, b, Z1);
  double* f = a;
  if constexpr (D == 3) {
    rcon<D, N, 2, true, false>(b, a, Z2);
    f = b;
  }
  double lam[ND];
  rload<ND>(lam, inv + cell * ND);
#pragma unroll
  for (int el = 0; el < ND; ++el) {  // 1/Lambda, reversed index
    const int ri = D == 3 ? (el % N) * N * N + ((el / N) % N) * N + el / (N * N)
                          : (el % N) * N + el / N;
    f[el] *= lam[ri];
  }
  if constexpr (D == 3) {  // backward: Z along each direction
    rcon<D, N, 2, false, false>(a, b, Z2);
    rcon<D, N, 1, false, false>(b, a, Z1);
    rcon<D, N, 0, false, false>(a, b, Z0);
  } else {
    rcon<D, N, 1, false, false>(b, a, Z1);
    rcon<D, N, 0, false, false>(a, b, Z0);
  }
  double xv[ND];
  rload<ND>(xv, x + cell * ND);
  double* o = x + cell * ND;
  if constexpr (ND % 2 == 0) {
#pragma unroll
    for (int e = 0; e < ND; e += 2)
      reinterpret_cast<double2*>(o)[e / 2] =
          make_double2(fma(omega, a[e], xv[e]), fma(omega, a[e + 1], xv[e + 1]));
  } else {
#pragma unroll
    for (int e = 0; e < ND; ++e) o[e] = fma(omega, a[e], xv[e]);
  }
}

template <int D, int N>
static int launch_dist(const DistArgs& a, const double* u, const double* b, double* out,
                       cudaStream_t st) {
  DistParams<D, N> P;
  P.u = u;
  P.b = b;
  P.out = out;
  P.metric = a.metric;
  for (int t = 0; t < 3; ++t) P.faces[t] = a.faces[t];
  for (int t = 0; t < 6; ++t) P.bnd[t] = a.bnd[t];
  P.n = a.ncells_dim;
  for (int q = 0; q < N * N; ++q) {
    P.tab.V[q] = a.vals[q];
    P.tab.Dg[q] = a.grads[q];
  }
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < N; ++i) {
      P.tab.bv[p][i] = a.bv[p * N + i];
      P.tab.bg[p][i] = a.bg[p * N + i];
    }
  int64_t ncells = 1;
  for (int t = 0; t < D; ++t) ncells *= a.ncells_dim;
  if constexpr (dist_reg_ok<D, N>()) {
    if (env_int("DGB_DIST_REG", 1) != 0) {
      dist_apply_reg_kernel<D, N><<<(unsigned)((ncells + 127) / 128), 128, 0, st>>>(P, ncells);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  constexpr int G = dist_cells<D, N>();
  const size_t smem = sizeof(double) * dist_smem_doubles<D, N>();
  auto k = dist_apply_kernel<D, N>;
  if (smem > 48 * 1024)
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)((ncells + G - 1) / G), 128, smem, st>>>(P, ncells);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

template <int D, int N>
static int launch_cell_fdm(const double* r, double* x, const double* z, const double* inv,
                           const int32_t* cells, int64_t nb, int64_t ncells, double omega,
                           cudaStream_t st) {
  if constexpr (dist_fdm_reg_ok<D, N>()) {
    if (env_int("DGB_DIST_REG", 1) != 0) {
      dist_cell_fdm_reg_kernel<D, N><<<(unsigned)((nb + 127) / 128), 128, 0, st>>>(
          r, x, z, inv, cells, nb, ncells, omega);
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  constexpr int G = dist_cells<D, N>();
  constexpr int ND = D == 3 ? N * N * N : N * N;
  const size_t smem = sizeof(double) * G * (2 * (size_t)ND + D * N * N);
  auto k = dist_cell_fdm_kernel<D, N>;
  if (smem > 48 * 1024)
    DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)((nb + G - 1) / G), 128, smem, st>>>(r, x, z, inv, cells, nb, ncells, omega);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

}  // namespace dgb

extern "C" int dg_dist_apply(const dg_dist_args_t* args, const double* u, const double* b,
                             double* out, void* stream) {
  using namespace dgb;
  if (!args || !u || !out) return fail(DG_EINVAL, "null argument");
  const DistArgs& a = *args;
  const int n = a.degree + 1;
  cudaStream_t st = (cudaStream_t)stream;
#define DG_DCASE(D, NN) \
  if (a.dim == D && n == NN) return launch_dist<D, NN>(a, u, b, out, st);
  DG_N_CASES(DG_DCASE, 2)
  DG_N_CASES(DG_DCASE, 3)
#undef DG_DCASE
  return fail(DG_EUNSUPPORTED, "distorted operator: dim 2 or 3, degree 1..15");
}

extern "C" int dg_dist_cell_fdm(int dim, int degree, int64_t ncells, const double* z,
                                const double* inv, const double* r, double* x, double omega,
                                const int32_t* cells, int64_t n_cells, void* stream) {
  using namespace dgb;
  if (!z || !inv || !r || !x || (cells && n_cells < 0)) return fail(DG_EINVAL, "bad argument");
  if (r == x) return fail(DG_EINVAL, "cell solve: r must not alias x");
  const int n = degree + 1;
  const int64_t nb = cells ? n_cells : ncells;
  if (nb == 0) return DG_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define DG_FCASE(D, NN) \
  if (dim == D && n == NN) return launch_cell_fdm<D, NN>(r, x, z, inv, cells, nb, ncells, omega, st);
  DG_N_CASES(DG_FCASE, 2)
  DG_N_CASES(DG_FCASE, 3)
#undef DG_FCASE
  return fail(DG_EUNSUPPORTED, "surrogate cell solve: dim 2 or 3, degree 1..15");
}
