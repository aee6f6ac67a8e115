// fdmg.cuh - fast-diagonalisation solves for large subdomains (generic path).
//
// x += omega * Z Lambda^-1 Z^T R_j r for vertex patches of degree k >= 8
// (m = 2(k+1) = 18 .. 32 per direction; fastdiag.py:510-634 handles any m)
// and for the whole-level "patch" of the coarse solver (multigrid.py: on a
// Cartesian level the operator is a Kronecker sum of global 1D matrices, so
// one fast diagonalisation with the global 1D eigenpairs is an exact solve).
// The templated fdm2 kernels keep Z in the kernel parameter space (<= 16^2
// entries per digit); here the matrices are too large for that and are read
// from global memory (L1-resident, warp-uniform addresses), one CTA works on
// one subdomain, its threads loop over the fibers, and the m^d tensor lives
// in shared memory (pitch m+1) while it fits (m <= 30 in 3D) or in a
// per-CTA slice of a global scratch buffer (3D m = 32: 256 KB).
// The interior digit takes the even/odd split (half blocks from global
// memory).  Throughput is not the point of this path (no bulk copies, one
// CTA per patch); parity with the reference at every degree is.
#pragma once
#include "common.cuh"
#include "fdm2.cuh"

namespace dgb {

struct FdmgParams {
  const double* r;
  double* x;
  const int32_t* list;
  int64_t start;
  int64_t count;
  const double* invsum;  // [class][m^d], canonical patch order
  const double* z;       // [digit][k*m + i] = Z[k][i]   (out = Z^T v)
  const double* zt;      // [digit][k*m + i] = Z[i][k]   (out = Z v)
  const double* eo;      // even/odd halves of the interior digit (4 x (m/2)^2) or nullptr
  double omega;
  int atomic;
  int packed;
  int pitch;        // doubles between rows of the tensor
  double* scratch;  // per-CTA tensors in global memory, or nullptr (shared memory)
  Geo geo;
};

constexpr int kFdmgThreads = 256;

// o_i = sum_k S[k*M + i] v_k with S in global memory (every lane reads the
// same addresses: one L1 transaction per 16-byte load)
template <int M>
__device__ __forceinline__ void matvec_g(const double* __restrict__ S, const double (&v)[M],
                                         double (&o)[M]) {
  const double2* S2 = reinterpret_cast<const double2*>(S);
#pragma unroll
  for (int i = 0; i < M; i += 2) {
    const double2 a = __ldg(S2 + i / 2);
    o[i] = a.x * v[0];
    o[i + 1] = a.y * v[0];
  }
#pragma unroll
  for (int k = 1; k < M; ++k) {
#pragma unroll
    for (int i = 0; i < M; i += 2) {
      const double2 a = __ldg(S2 + (k * M + i) / 2);
      o[i] = fma(a.x, v[k], o[i]);
      o[i + 1] = fma(a.y, v[k], o[i + 1]);
    }
  }
}

// even/odd forms of the interior digit (fdm2.cuh matvec_eo_fwd / _bwd) with
// the half blocks in global memory: half the FMAs and half the loads
template <int M>
__device__ __forceinline__ void matvec_eo_fwd_g(const double* __restrict__ E,
                                                const double* __restrict__ O,
                                                const double (&v)[M], double (&o)[M]) {
  constexpr int H = M / 2;
  double u[H], w[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    u[i] = v[i] + v[M - 1 - i];
    w[i] = v[i] - v[M - 1 - i];
  }
#pragma unroll
  for (int r = 0; r < H; ++r) {
    o[r] = __ldg(E + r) * u[0];
    o[H + r] = __ldg(O + r) * w[0];
  }
#pragma unroll
  for (int k = 1; k < H; ++k) {
#pragma unroll
    for (int r = 0; r < H; ++r) {
      o[r] = fma(__ldg(E + k * H + r), u[k], o[r]);
      o[H + r] = fma(__ldg(O + k * H + r), w[k], o[H + r]);
    }
  }
}

template <int M>
__device__ __forceinline__ void matvec_eo_bwd_g(const double* __restrict__ Et,
                                                const double* __restrict__ Ot,
                                                const double (&v)[M], double (&o)[M]) {
  constexpr int H = M / 2;
  double e[H], q[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = __ldg(Et + i) * v[0];
    q[i] = __ldg(Ot + i) * v[H];
  }
#pragma unroll
  for (int k = 1; k < H; ++k) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      e[i] = fma(__ldg(Et + k * H + i), v[k], e[i]);
      q[i] = fma(__ldg(Ot + k * H + i), v[H + k], q[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    o[i] = e[i] + q[i];
    o[M - 1 - i] = e[i] - q[i];
  }
}

template <int M, bool FWD>
__device__ __forceinline__ void fdmg_matvec(const FdmgParams& p, int digit, const double (&v)[M],
                                            double (&o)[M]) {
  constexpr int HH = (M / 2) * (M / 2);
  if (p.eo && digit == 0) {
    if (FWD) matvec_eo_fwd_g<M>(p.eo, p.eo + HH, v, o);
    else matvec_eo_bwd_g<M>(p.eo + 2 * HH, p.eo + 3 * HH, v, o);
    return;
  }
  matvec_g<M>((FWD ? p.z : p.zt) + (int64_t)digit * M * M, v, o);
}

template <int D, int M, bool PATCH>
__global__ void __launch_bounds__(kFdmgThreads)
fdmg_kernel(const FdmgParams p) {
  static_assert(M % 2 == 0, "even subdomain size");
  constexpr int N = PATCH ? M / 2 : M;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  constexpr int NE = (D == 3) ? M * M * M : M * M;
  constexpr int F = (D == 3) ? M * M : M;
  constexpr int RPC = (D == 3) ? N * N : N;
  constexpr int SLOTS = PATCH ? (1 << D) : 1;
  constexpr int NT = kFdmgThreads;
  extern __shared__ __align__(16) double sm[];
  const int P = p.pitch;
  const int PM = P * M;
  double* T = p.scratch ? p.scratch + (int64_t)blockIdx.x * ((D == 3) ? (int64_t)PM * M : PM) : sm;
  const int tid = threadIdx.x;
  auto sstride = [&](int t) { return t == 0 ? 1 : (t == 1 ? P : PM); };
  auto sbase = [&](int t, int f) {
    if (D == 2) return t == 0 ? f * P : f;
    const int a = f % M, b = f / M;
    return t == 0 ? a * P + b * PM : (t == 1 ? a + b * PM : a + b * P);
  };
  for (int64_t idx = blockIdx.x; idx < p.count; idx += gridDim.x) {
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    subdomain_info<D, PATCH>(p.geo, p.list ? p.list[idx] : (int)(p.start + idx), p.packed != 0,
                             digit, base);
    int cls = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
    // gather R_j r, one cell row per thread iteration
    for (int rr = tid; rr < SLOTS * RPC; rr += NT) {
      const int slot = rr / RPC, w = rr - slot * RPC;
      const int i1 = (D == 3) ? w % N : w, i2 = (D == 3) ? w / N : 0;
      const int s0 = slot & 1, s1 = (slot >> 1) & 1, s2 = (slot >> 2) & 1;
      int c[3] = {base[0] + s0, base[1] + s1, base[2] + s2};
      const double* src = p.r + (int64_t)cell_local<D>(p.geo, c) * NEc + w * N;
      double* dst = T + s0 * N + P * (s1 * N + i1) + (D == 3 ? PM * (s2 * N + i2) : 0);
#pragma unroll 4
      for (int i = 0; i < N; ++i) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    // forward contractions with Z^T along 0 .. D-1
#pragma unroll 1
    for (int t = 0; t < D; ++t) {
      const int ss = sstride(t);
      for (int f = tid; f < F; f += NT) {
        const int sb = sbase(t, f);
        double v[M], o[M];
#pragma unroll
        for (int k = 0; k < M; ++k) v[k] = T[sb + k * ss];
        fdmg_matvec<M, true>(p, digit[t], v, o);
        if (t == D - 1) {
          // scale by 1 / (lambda_1 + .. + lambda_d) on the last forward pass
          const int a = (D == 3) ? f % M : f, b = (D == 3) ? f / M : 0;
          const double* inv = p.invsum + (int64_t)cls * NE +
                              ((D == 3) ? a + M * b : a);
          constexpr int gs = (D == 3) ? M * M : M;
#pragma unroll
          for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * gs);
        }
#pragma unroll
        for (int k = 0; k < M; ++k) T[sb + k * ss] = o[k];
      }
      __syncthreads();
    }
    // backward contractions with Z along D-1 .. 0
#pragma unroll 1
    for (int t = D - 1; t >= 0; --t) {
      const int ss = sstride(t);
      for (int f = tid; f < F; f += NT) {
        const int sb = sbase(t, f);
        double v[M], o[M];
#pragma unroll
        for (int k = 0; k < M; ++k) v[k] = T[sb + k * ss];
        fdmg_matvec<M, false>(p, digit[t], v, o);
#pragma unroll
        for (int k = 0; k < M; ++k) T[sb + k * ss] = o[k];
      }
      __syncthreads();
    }
    // x += omega R_j^T y
    for (int rr = tid; rr < SLOTS * RPC; rr += NT) {
      const int slot = rr / RPC, w = rr - slot * RPC;
      const int i1 = (D == 3) ? w % N : w, i2 = (D == 3) ? w / N : 0;
      const int s0 = slot & 1, s1 = (slot >> 1) & 1, s2 = (slot >> 2) & 1;
      int c[3] = {base[0] + s0, base[1] + s1, base[2] + s2};
      double* dst = p.x + (int64_t)cell_local<D>(p.geo, c) * NEc + w * N;
      const double* src = T + s0 * N + P * (s1 * N + i1) + (D == 3 ? PM * (s2 * N + i2) : 0);
      if (p.atomic) {
#pragma unroll 4
        for (int i = 0; i < N; ++i) atomicAdd(dst + i, p.omega * src[i]);
      } else {
#pragma unroll 4
        for (int i = 0; i < N; ++i) dst[i] = xupd(dst[i], p.omega, src[i]);
      }
    }
    __syncthreads();  // the tensor is refilled by the next subdomain
  }
}

// 2D: a patch has only m <= 32 fibers per direction, so one warp owns one
// patch (lane = fiber, __syncwarp between the passes) and a CTA of 8 warps
// works on 8 patches at once, each with its own padded tensor in shared
// memory (m (m+1) doubles).  Same passes and arithmetic as fdmg_kernel<2, m>.
constexpr int kFdmg2Warps = 8;

template <int M, bool PATCH>
__global__ void __launch_bounds__(32 * kFdmg2Warps)
fdmg2_warp_kernel(const FdmgParams p) {
  static_assert(M % 2 == 0 && M <= 32, "one fiber per lane");
  constexpr int D = 2;
  constexpr int N = PATCH ? M / 2 : M;
  constexpr int NEc = N * N, NE = M * M;
  constexpr int SLOTS = PATCH ? 4 : 1;
  constexpr int P = M + 1;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* T = sm + warp * (P * M);
  const int64_t nw = (int64_t)gridDim.x * kFdmg2Warps;
  for (int64_t idx = (int64_t)blockIdx.x * kFdmg2Warps + warp; idx < p.count; idx += nw) {
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    subdomain_info<D, PATCH>(p.geo, p.list ? p.list[idx] : (int)(p.start + idx), p.packed != 0,
                             digit, base);
    const int cls = digit[1] * 4 + digit[0];
    // gather: row w of cell slot -> T[(s1 N + w) P + s0 N ..]
    for (int rr = lane; rr < SLOTS * N; rr += 32) {
      const int slot = rr / N, w = rr - slot * N;
      const int s0 = slot & 1, s1 = (slot >> 1) & 1;
      int c[3] = {base[0] + s0, base[1] + s1, 0};
      const double* src = p.r + (int64_t)cell_local<D>(p.geo, c) * NEc + w * N;
      double* dst = T + s0 * N + P * (s1 * N + w);
#pragma unroll 4
      for (int i = 0; i < N; ++i) dst[i] = __ldg(src + i);
    }
    __syncwarp();
    double v[M], o[M];
    if (lane < M) {  // Z^T along direction 0: fiber = row `lane`
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = T[lane * P + k];
      fdmg_matvec<M, true>(p, digit[0], v, o);
#pragma unroll
      for (int k = 0; k < M; ++k) T[lane * P + k] = o[k];
    }
    __syncwarp();
    if (lane < M) {  // Z^T along direction 1, 1 / (lambda_0 + lambda_1), Z along direction 1
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = T[lane + k * P];
      fdmg_matvec<M, true>(p, digit[1], v, o);
      const double* inv = p.invsum + (int64_t)cls * NE + lane;
#pragma unroll
      for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * M);
      fdmg_matvec<M, false>(p, digit[1], o, v);
#pragma unroll
      for (int k = 0; k < M; ++k) T[lane + k * P] = v[k];
    }
    __syncwarp();
    if (lane < M) {  // Z along direction 0
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = T[lane * P + k];
      fdmg_matvec<M, false>(p, digit[0], v, o);
#pragma unroll
      for (int k = 0; k < M; ++k) T[lane * P + k] = o[k];
    }
    __syncwarp();
    for (int rr = lane; rr < SLOTS * N; rr += 32) {
      const int slot = rr / N, w = rr - slot * N;
      const int s0 = slot & 1, s1 = (slot >> 1) & 1;
      int c[3] = {base[0] + s0, base[1] + s1, 0};
      double* dst = p.x + (int64_t)cell_local<D>(p.geo, c) * NEc + w * N;
      const double* src = T + s0 * N + P * (s1 * N + w);
      if (p.atomic) {
#pragma unroll 4
        for (int i = 0; i < N; ++i) atomicAdd(dst + i, p.omega * src[i]);
      } else {
#pragma unroll 4
        for (int i = 0; i < N; ++i) dst[i] = xupd(dst[i], p.omega, src[i]);
      }
    }
    __syncwarp();
  }
}

}  // namespace dgb
