// kernels.cuh - sm_100a kernels of the fp64 Schwarz smoothing step.
//
// Three kernel families replace the reference's numpy hot loops:
//
//  residual_kernel  r = b - A x  (dgop.residual, dgop.py:782-788).  The SIPG
//                   operator on a uniform Cartesian level is the Kronecker sum
//                   A = sum_t M x .. x A_g^(t) x .. x M with A_g^(t)
//                   block-tridiagonal: cell blocks A_diag(digit) and the rank-2
//                   face coupling a_pm (polybasis.py:247-302; equal to the
//                   quadrature form of dgop.py:432-759 on Cartesian levels).
//                   Per cell: G_t = A_diag ._t x_c + rank-2 neighbour terms,
//                   then the transversal masses (8 contractions in 3D).
//  fdm_kernel       x += omega Z Lambda^-1 Z^T R r for cells or vertex
//                   patches (fastdiag.py:457-496, 602-628): gather, d forward
//                   contractions with Z^T, scale by 1/Lambda-sum, d backward
//                   contractions with Z, scatter-add.
//  gather_map_kernel the R_j index map (fastdiag.py:546-582), bit-exact.
//
// Tensors are staged in shared memory in canonical order (direction 1
// fastest) with an odd row pitch P so that fibers along direction 1 are
// bank-conflict free for 8-byte accesses.  Each thread owns one fiber of the
// contracted direction and applies the n x n matrix with DFMA.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dgb {

struct Geo {
  int nc[3];   // global cells per direction (1 for unused directions)
  int zb;      // first stored layer (global index) along the last direction
  int zn;      // stored layers
};

template <int D, int N>
struct Lay {
  static constexpr int P = (N % 2 == 0) ? N + 1 : N;          // padded pitch
  static constexpr int F = (D == 3) ? N * N : N;               // fibers / tensor
  static constexpr int SZ = (D == 3) ? P * N * N : P * N;      // padded doubles
  static constexpr int NE = (D == 3) ? N * N * N : N * N;      // elements
  __device__ __forceinline__ static int sstride(int t) {
    return t == 0 ? 1 : (t == 1 ? P : P * N);
  }
  __device__ __forceinline__ static int gstride(int t) {
    return t == 0 ? 1 : (t == 1 ? N : N * N);
  }
  // shared-memory base offset of fiber f (0 <= f < F) along direction t
  __device__ __forceinline__ static int sbase(int t, int f) {
    if (D == 2) return t == 0 ? f * P : f;
    const int a = f % N, b = f / N;
    if (t == 0) return a * P + b * P * N;
    if (t == 1) return a + b * P * N;
    return a + b * P;
  }
  // canonical (unpadded) base offset of fiber f along t
  __device__ __forceinline__ static int gbase(int t, int f) {
    if (D == 2) return t == 0 ? f * N : f;
    const int a = f % N, b = f / N;
    if (t == 0) return a * N + b * N * N;
    if (t == 1) return a + b * N * N;
    return a + b * N;
  }
  __device__ __forceinline__ static int smem_of(int e) {
    if (D == 2) return (e % N) + P * (e / N);
    return (e % N) + P * ((e / N) % N) + P * N * (e / (N * N));
  }
};

// groups (subdomains) per CTA so that a CTA has >= ~128 threads
__host__ __device__ constexpr int groups_for(int F) {
  return F >= 96 ? 1 : (128 + F - 1) / F;
}

// out_i (+)= sum_k S[i*N+k] in_k along one fiber
template <int N, bool ACC>
__device__ __forceinline__ void fiber_apply(const double* __restrict__ S,
                                            const double* in, double* out,
                                            int base, int stride) {
  double v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = in[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(S[i * N + k], v[k], s);
    if (ACC) out[base + i * stride] += s;
    else out[base + i * stride] = s;
  }
}

// ----------------------------------------------------------------------------
// residual / operator apply
// ----------------------------------------------------------------------------
struct ResParams {
  const double* x;       // local vector
  const double* b;       // nullptr -> v = A x
  double* r;             // output
  const int32_t* list;   // local cell ids or nullptr (contiguous range)
  int64_t start;         // first local cell id when list == nullptr
  int64_t count;         // cells
  const double* mass;    // n*n
  const double* adiag;   // 4*n*n
  const double* bg;      // 2*n
  double alpha, beta, betap;
  Geo geo;
};

template <int D>
__device__ __forceinline__ void cell_multi(const Geo& g, int cell, int* c) {
  c[0] = cell % g.nc[0];
  if (D == 2) {
    c[1] = cell / g.nc[0] + g.zb;
  } else {
    c[1] = (cell / g.nc[0]) % g.nc[1];
    c[2] = cell / (g.nc[0] * g.nc[1]) + g.zb;
  }
}

template <int D>
__device__ __forceinline__ int cell_local(const Geo& g, const int* c) {
  if (D == 2) return c[0] + g.nc[0] * (c[1] - g.zb);
  return c[0] + g.nc[0] * (c[1] + g.nc[1] * (c[2] - g.zb));
}

// G_t = A_diag(digit) ._t X + rank-2 neighbour couplings, one fiber
template <int D, int N>
__device__ __forceinline__ void stiff_fiber(const ResParams& p, int t, int f,
                                            const int* c, const double* X,
                                            double* GB, const double* sA,
                                            const double* sBg) {
  using L = Lay<D, N>;
  const int sb = L::sbase(t, f), ss = L::sstride(t);
  const int digit = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
  const double* A = sA + digit * N * N;
  double v[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = X[sb + k * ss];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(A[i * N + k], v[k], s);
    o[i] = s;
  }
  const int gb = L::gbase(t, f), gs = L::gstride(t);
  int nb[3] = {c[0], c[1], D == 3 ? c[2] : 0};
  if (!(digit & 2)) {  // right neighbour: a_pm x_R
    nb[t] = c[t] + 1;
    const double* xr = p.x + (int64_t)cell_local<D>(p.geo, nb) * L::NE + gb;
    const double v0 = __ldg(xr);
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(sBg[k], __ldg(xr + k * gs), g);
    const double fall = p.betap * v0;
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = fma(sBg[N + i], fall, o[i]);
    o[N - 1] += p.alpha * v0 + p.beta * g;
    nb[t] = c[t];
  }
  if (!(digit & 1)) {  // left neighbour: a_pm^T x_L
    nb[t] = c[t] - 1;
    const double* xl = p.x + (int64_t)cell_local<D>(p.geo, nb) * L::NE + gb;
    const double v1 = __ldg(xl + (N - 1) * gs);
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(sBg[N + k], __ldg(xl + k * gs), g);
    const double fall = p.beta * v1;
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = fma(sBg[i], fall, o[i]);
    o[0] += p.alpha * v1 + p.betap * g;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) GB[sb + i * ss] = o[i];
}

template <int D, int N>
__host__ __device__ constexpr int res_smem_doubles() {
  return 5 * N * N + 2 * N + 4 * groups_for(Lay<D, N>::F) * Lay<D, N>::SZ;
}

template <int D, int N>
__global__ void __launch_bounds__(groups_for(Lay<D, N>::F) * Lay<D, N>::F)
residual_kernel(ResParams p) {
  using L = Lay<D, N>;
  constexpr int G = groups_for(L::F);
  extern __shared__ double sm[];
  double* sM = sm;                 // N*N mass
  double* sA = sM + N * N;         // 4*N*N stiffness per digit
  double* sBg = sA + 4 * N * N;    // 2N
  double* bufs = sBg + 2 * N;
  const int tid = threadIdx.x;
  for (int i = tid; i < 5 * N * N; i += G * L::F)
    sM[i] = i < N * N ? p.mass[i] : p.adiag[i - N * N];
  for (int i = tid; i < 2 * N; i += G * L::F) sBg[i] = p.bg[i];

  const int g = tid / L::F, f = tid % L::F;
  const int64_t idx = (int64_t)blockIdx.x * G + g;
  const bool active = idx < p.count;
  const int cell = active ? (p.list ? p.list[idx] : (int)(p.start + idx)) : 0;
  int c[3] = {0, 0, 0};
  cell_multi<D>(p.geo, cell, c);
  double* X = bufs + g * L::SZ;
  double* GB = X + G * L::SZ;
  double* H = GB + G * L::SZ;
  double* OUT = H + G * L::SZ;
  const double* xc = p.x + (int64_t)cell * L::NE;
  if (active)
    for (int e = f; e < L::NE; e += L::F) X[L::smem_of(e)] = xc[e];
  __syncthreads();
  if (D == 2) {
    if (active) stiff_fiber<D, N>(p, 0, f, c, X, GB, sA, sBg);
    __syncthreads();
    if (active) fiber_apply<N, false>(sM, GB, OUT, L::sbase(1, f), L::sstride(1));
    __syncthreads();
    if (active) stiff_fiber<D, N>(p, 1, f, c, X, GB, sA, sBg);
    __syncthreads();
    if (active) fiber_apply<N, true>(sM, GB, OUT, L::sbase(0, f), L::sstride(0));
    __syncthreads();
  } else {
    // T1 + T2 = M_3 (M_2 G_1 + M_1 G_2);  T3 = M_1 M_2 G_3
    if (active) stiff_fiber<D, N>(p, 0, f, c, X, GB, sA, sBg);
    __syncthreads();
    if (active) fiber_apply<N, false>(sM, GB, H, L::sbase(1, f), L::sstride(1));
    __syncthreads();
    if (active) stiff_fiber<D, N>(p, 1, f, c, X, GB, sA, sBg);
    __syncthreads();
    if (active) fiber_apply<N, true>(sM, GB, H, L::sbase(0, f), L::sstride(0));
    __syncthreads();
    if (active) fiber_apply<N, false>(sM, H, OUT, L::sbase(2, f), L::sstride(2));
    __syncthreads();
    if (active) stiff_fiber<D, N>(p, 2, f, c, X, GB, sA, sBg);
    __syncthreads();
    if (active) fiber_apply<N, false>(sM, GB, H, L::sbase(1, f), L::sstride(1));
    __syncthreads();
    if (active) fiber_apply<N, true>(sM, H, OUT, L::sbase(0, f), L::sstride(0));
    __syncthreads();
  }
  if (active) {
    double* rc = p.r + (int64_t)cell * L::NE;
    if (p.b) {
      const double* bc = p.b + (int64_t)cell * L::NE;
      for (int e = f; e < L::NE; e += L::F) rc[e] = bc[e] - OUT[L::smem_of(e)];
    } else {
      for (int e = f; e < L::NE; e += L::F) rc[e] = OUT[L::smem_of(e)];
    }
  }
}

// ----------------------------------------------------------------------------
// fast-diagonalisation solves (cells and vertex patches)
// ----------------------------------------------------------------------------
struct FdmParams {
  const double* r;
  double* x;
  const int32_t* list;   // cell: local ids; patch: global patch ids; or nullptr
  int64_t start;
  int64_t count;
  const double* z;       // 4*m*m
  const double* zt;      // 4*m*m
  const double* invsum;  // 4^d * m^d
  double omega;
  int atomic;
  Geo geo;
};

// subdomain -> (per-direction digit, base cell multi-index)
template <int D, bool PATCH>
__device__ __forceinline__ void subdomain_info(const Geo& g, int id, int* digit,
                                               int* base) {
  if (PATCH) {
    int rem = id;
#pragma unroll
    for (int t = 0; t < D; ++t) {
      const int span = g.nc[t] - 1;
      const int v = 1 + rem % span;
      rem /= span;
      digit[t] = (v == 1 ? 1 : 0) | (v == g.nc[t] - 1 ? 2 : 0);
      base[t] = v - 1;
    }
  } else {
    cell_multi<D>(g, id, base);
#pragma unroll
    for (int t = 0; t < D; ++t)
      digit[t] = (base[t] == 0 ? 1 : 0) | (base[t] == g.nc[t] - 1 ? 2 : 0);
  }
}

// canonical subdomain element e -> local dof index
template <int D, int M, bool PATCH>
__device__ __forceinline__ int64_t sub_dof(const Geo& g, const int* base, int e) {
  constexpr int N = PATCH ? M / 2 : M;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  int q[3] = {e % M, (e / M) % M, D == 3 ? e / (M * M) : 0};
  int c[3] = {base[0], base[1], D == 3 ? base[2] : 0};
  int off = 0, mul = 1;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const int s = PATCH ? q[t] / N : 0;
    const int i = PATCH ? q[t] % N : q[t];
    c[t] += s;
    off += i * mul;
    mul *= N;
  }
  return (int64_t)cell_local<D>(g, c) * NEc + off;
}

template <int D, int M>
__host__ __device__ constexpr int fdm_smem_doubles() {
  return 8 * M * M + 2 * groups_for(Lay<D, M>::F) * Lay<D, M>::SZ;
}

template <int D, int M, bool PATCH>
__global__ void __launch_bounds__(groups_for(Lay<D, M>::F) * Lay<D, M>::F)
fdm_kernel(FdmParams p) {
  using L = Lay<D, M>;
  constexpr int G = groups_for(L::F);
  extern __shared__ double sm[];
  double* sZ = sm;               // 4*M*M
  double* sZt = sZ + 4 * M * M;  // 4*M*M
  double* bufs = sZt + 4 * M * M;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * M * M; i += G * L::F) {
    sZ[i] = p.z[i];
    sZt[i] = p.zt[i];
  }
  const int g = tid / L::F, f = tid % L::F;
  const int64_t idx = (int64_t)blockIdx.x * G + g;
  const bool active = idx < p.count;
  const int id = active ? (p.list ? p.list[idx] : (int)(p.start + idx)) : 0;
  int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
  if (active) subdomain_info<D, PATCH>(p.geo, id, digit, base);
  int cls = 0;
#pragma unroll
  for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
  double* A = bufs + g * L::SZ;
  double* B = A + G * L::SZ;
  if (active)
    for (int e = f; e < L::NE; e += L::F)
      A[L::smem_of(e)] = p.r[sub_dof<D, M, PATCH>(p.geo, base, e)];
  __syncthreads();
  // forward: y = (Z^T x .. x Z^T) r, direction 1 first (_tensor.py:59-78)
#pragma unroll
  for (int t = 0; t < D; ++t) {
    if (active)
      fiber_apply<M, false>(sZt + digit[t] * M * M, (t & 1) ? B : A,
                            (t & 1) ? A : B, L::sbase(t, f), L::sstride(t));
    __syncthreads();
  }
  double* Y = (D & 1) ? B : A;
  double* W = (D & 1) ? A : B;
  if (active) {
    const double* inv = p.invsum + (int64_t)cls * L::NE;
    for (int e = f; e < L::NE; e += L::F) Y[L::smem_of(e)] *= inv[e];
  }
  __syncthreads();
  // backward: x = (Z x .. x Z) y, direction d first (_tensor.py:81-97)
#pragma unroll
  for (int s = 0; s < D; ++s) {
    const int t = D - 1 - s;
    if (active)
      fiber_apply<M, false>(sZ + digit[t] * M * M, (s & 1) ? W : Y,
                            (s & 1) ? Y : W, L::sbase(t, f), L::sstride(t));
    __syncthreads();
  }
  const double* R = (D & 1) ? W : Y;
  if (active) {
    for (int e = f; e < L::NE; e += L::F) {
      const int64_t gi = sub_dof<D, M, PATCH>(p.geo, base, e);
      const double u = p.omega * R[L::smem_of(e)];
      if (p.atomic) atomicAdd(p.x + gi, u);
      else p.x[gi] += u;
    }
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
