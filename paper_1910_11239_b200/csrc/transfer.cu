// transfer.cu - nested-level DG transfers between a coarse level and its
// uniform refinement (reference: dgmg.multigrid.LevelTransfer,
// multigrid.py:58-130; 1D embeddings build_transfer, multigrid.py:51-55).
//
// Prolongation embeds the degree-k polynomial of every coarse cell into its
// 2^d children: child s gets (E^{s_d} (x) ... (x) E^{s_1}) x_c with
// E^s[i,j] = phi_j((x_i + s)/2).  Stacking E^0 over E^1 gives one 2n x n
// matrix E per direction, so the 2^d children of a coarse cell are exactly a
// (2n)^d tensor in the patch layout (p = sum_t (s_t n + i_t)(2n)^(t-1)) and
// the transfer is d sum-factorised contractions that expand one direction
// from n to 2n each (2+4+8 = 14 n^4 FMAs per 3D cell instead of the
// reference's 8 separate 3-pass child chains, 24 n^4).  Restriction is the
// exact adjoint (E^T per direction, fine -> coarse, multigrid.py:110-130).
//
// Kernel layout: CPB coarse cells per CTA; one thread per fiber of the
// contracted direction; E lives in the kernel parameter space (constant
// bank); the last prolongation pass writes the fine rows (or adds them to
// the fine vector, fusing the V-cycle's `x += P e`, multigrid.py:340-341)
// straight from registers, and the first restriction pass reads the fine
// rows straight from global memory.  The transfers are HBM-bound: 8 B per
// fine dof + 8 B per coarse dof (+8 B per fine dof for the accumulate read).
#include "launch.h"
#include "fdm2.cuh"  // TMA bulk-copy / mbarrier helpers

// the D == 1 branches return early; the rest of each kernel is unreachable there
#pragma nv_diag_suppress 128

namespace dgb {

template <int N>
struct EPar {
  double e[2 * N * N];   // row o (0 <= o < 2N) of the stacked E: e[o*N + j]
  double et[2 * N * N];  // E^T, et[j*2N + o]: the expanding contractions run
                         // k-outer so each LDCU.128 feeds two outputs in load order
};

// out[o] = sum_j E[o][j] a[j], o < 2N (k-outer over j)
template <int N>
__device__ __forceinline__ void expand(const EPar<N>& E, const double (&a)[N],
                                       double (&out)[2 * N]) {
#pragma unroll
  for (int o = 0; o < 2 * N; ++o) out[o] = E.et[o] * a[0];
#pragma unroll
  for (int j = 1; j < N; ++j)
#pragma unroll
    for (int o = 0; o < 2 * N; ++o) out[o] = fma(E.et[j * 2 * N + o], a[j], out[o]);
}

struct TGeo {
  int nc[3];      // coarse cells per direction (1 for unused)
  int64_t ncells; // coarse cells
  FastDiv f0, f1; // division by nc[0], nc[1]
};

template <int D, int N>
struct TLay {
  static constexpr int M = 2 * N;
  static constexpr int PA = N | 1;       // padded pitch of the coarse cell rows
  static constexpr int PB = M + 1;       // pitch of the first-expanded tensor
  // region 1: coarse cell (prolong) then the (M,M,N) tensor; region 2: (M,N,N)
  static constexpr int R1 = D == 3 ? (M * M * N > PA * N * N ? M * M * N : PA * N * N)
                                   : (D == 2 ? PA * N : N);
  static constexpr int R2 = D == 3 ? PB * N * N : (D == 2 ? PB * N : 0);
  static constexpr int PER_CELL = R1 + R2;
  static constexpr int LAST_FIBERS = D == 3 ? M * M : (D == 2 ? M : 1);
  static constexpr int CPB = LAST_FIBERS >= 128 ? 1 : 128 / LAST_FIBERS;
  static constexpr int THREADS = LAST_FIBERS * CPB >= 256 ? 256
                                 : ((LAST_FIBERS * CPB + 31) / 32) * 32;
  static constexpr size_t SMEM = sizeof(double) * (size_t)PER_CELL * CPB;
  // CTAs per SM the register budget is sized for (<= ~96 registers per thread):
  // the kernels are latency/HBM-bound and need the warps more than the ILP
  // (n > 8: the fibers need more registers and shared memory limits the CTAs)
  static constexpr int MINB = (D >= 2 && N <= 8 && 65536 / (THREADS * 96) > 0) ? 65536 / (THREADS * 96) : 1;
};

// run body(e) for e in [0, cnt): a single guarded iteration when the
// compile-time bound fits the CTA (no loop, so the compiler cannot hoist the
// constant-bank matrix loads of every pass into the uniform register file)
template <int MAXCNT, int THREADS, class F>
__device__ __forceinline__ void for_fibers(int cnt, F&& body) {
  if constexpr (MAXCNT <= THREADS) {
    if ((int)threadIdx.x < cnt) body((int)threadIdx.x);
  } else {
    for (int e = threadIdx.x; e < cnt; e += THREADS) body(e);
  }
}

template <int D>
__device__ __forceinline__ void coarse_multi(const TGeo& g, int64_t c, int* m) {
  const uint32_t q0 = g.f0.div((uint32_t)c);
  m[0] = (int)c - (int)q0 * g.nc[0];
  if (D == 1) return;
  if (D == 2) { m[1] = (int)q0; return; }
  const uint32_t q1 = g.f1.div(q0);
  m[1] = (int)q0 - (int)q1 * g.nc[1];
  m[2] = (int)q1;
}

// fine dof of output position (o0, o1, o2) (o_t in [0, 2N)) of coarse cell c
template <int D, int N>
__device__ __forceinline__ int64_t fine_index(const TGeo& g, const int* c, int o0, int o1,
                                              int o2) {
  const int s0 = o0 >= N, s1 = o1 >= N, s2 = o2 >= N;
  int64_t cell = 2 * c[0] + s0;
  int64_t node = o0 - s0 * N;
  if (D >= 2) {
    cell += (int64_t)(2 * g.nc[0]) * (2 * c[1] + s1);
    node += N * (o1 - s1 * N);
  }
  if (D == 3) {
    cell += (int64_t)(2 * g.nc[0]) * (2 * g.nc[1]) * (2 * c[2] + s2);
    node += N * N * (o2 - s2 * N);
  }
  constexpr int ND = D == 3 ? N * N * N : (D == 2 ? N * N : N);
  return cell * ND + node;
}

template <int D, int N, bool ADD>
__global__ void __launch_bounds__(TLay<D, N>::THREADS, TLay<D, N>::MINB)
    prolong_kernel(const __grid_constant__ EPar<N> E, const double* __restrict__ xc,
                   double* __restrict__ xf, TGeo g) {
  using L = TLay<D, N>;
  constexpr int M = L::M;
  constexpr int ND = D == 3 ? N * N * N : (D == 2 ? N * N : N);
  extern __shared__ double sm[];
  const int64_t c0 = (int64_t)blockIdx.x * L::CPB;
  const int ncell = (int)(g.ncells - c0 < (int64_t)L::CPB ? g.ncells - c0 : (int64_t)L::CPB);
  double* r1 = sm;
  double* r2 = sm + L::R1 * L::CPB;

  if (D == 1) {
    for (int f = threadIdx.x; f < ncell; f += blockDim.x) {
      const int64_t cc = c0 + f;
      double a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = xc[cc * N + j];
      int cm[3] = {(int)cc, 0, 0};
      double ex[M];
      expand<N>(E, a, ex);
#pragma unroll
      for (int o = 0; o < M; ++o) {
        const double s = ex[o];
        const int64_t idx = fine_index<D, N>(g, cm, o, 0, 0);
        xf[idx] = ADD ? xf[idx] + s : s;
      }
    }
    return;
  }

  // stage the CPB coarse cells (contiguous in the canonical layout)
  for_fibers<L::CPB * ND, L::THREADS>(ncell * ND, [&](int e) {
    const int cl = e / ND, q = e - cl * ND;
    const int row = q / N, i0 = q - row * N;
    r1[cl * L::R1 + row * L::PA + i0] = xc[c0 * ND + e];
  });
  __syncthreads();

  // pass 0: expand direction 1 (rows of N -> rows of M), region 1 -> region 2
  constexpr int F0 = D == 3 ? N * N : N;
  for_fibers<L::CPB * F0, L::THREADS>(ncell * F0, [&](int e) {
    const int cl = e / F0, f = e - cl * F0;
    const double* in = r1 + cl * L::R1 + f * L::PA;
    double a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = in[j];
    double* out = r2 + cl * L::R2 + f * L::PB;
    double ex[M];
    expand<N>(E, a, ex);
#pragma unroll
    for (int o = 0; o < M; ++o) {
      const double s = ex[o];
      out[o] = s;
    }
  });
  __syncthreads();

  if (D == 2) {
    // pass 1: expand direction 2 from region 2, write the fine rows
    for_fibers<L::CPB * M, L::THREADS>(ncell * M, [&](int e) {
      const int cl = e / M, o0 = e - cl * M;
      const double* in = r2 + cl * L::R2 + o0;
      double a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = in[j * L::PB];
      int cm[3];
      coarse_multi<D>(g, c0 + cl, cm);
      double ex[M];
      expand<N>(E, a, ex);
#pragma unroll
      for (int o1 = 0; o1 < M; ++o1) {
        const double s = ex[o1];
        const int64_t idx = fine_index<D, N>(g, cm, o0, o1, 0);
        xf[idx] = ADD ? xf[idx] + s : s;
      }
    });
    return;
  }

  // pass 1 (3D): expand direction 2, region 2 (M,N,N; pitch PB) -> region 1 (M,M,N)
  for_fibers<L::CPB * M * N, L::THREADS>(ncell * M * N, [&](int e) {
    const int cl = e / (M * N), f = e - cl * (M * N);
    const int o0 = f % M, i2 = f / M;
    const double* in = r2 + cl * L::R2 + o0 + L::PB * N * i2;
    double a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = in[j * L::PB];
    double* out = r1 + cl * L::R1 + o0 + M * M * i2;
    double ex[M];
    expand<N>(E, a, ex);
#pragma unroll
    for (int o1 = 0; o1 < M; ++o1) {
      const double s = ex[o1];
      out[o1 * M] = s;
    }
  });
  __syncthreads();

  // pass 2 (3D): expand direction 3 and write the fine rows
  for_fibers<L::CPB * M * M, L::THREADS>(ncell * M * M, [&](int e) {
    const int cl = e / (M * M), f = e - cl * (M * M);
    const int o0 = f % M, o1 = f / M;
    const double* in = r1 + cl * L::R1 + f;
    double a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = in[j * M * M];
    int cm[3];
    coarse_multi<D>(g, c0 + cl, cm);
    double ex[M];
    expand<N>(E, a, ex);
#pragma unroll
    for (int o2 = 0; o2 < M; ++o2) {
      const double s = ex[o2];
      const int64_t idx = fine_index<D, N>(g, cm, o0, o1, o2);
      xf[idx] = ADD ? xf[idx] + s : s;
    }
  });
}

template <int D, int N>
__global__ void __launch_bounds__(TLay<D, N>::THREADS, TLay<D, N>::MINB)
    restrict_kernel(const __grid_constant__ EPar<N> E, const double* __restrict__ xf,
                    double* __restrict__ xc, TGeo g) {
  using L = TLay<D, N>;
  constexpr int M = L::M;
  constexpr int ND = D == 3 ? N * N * N : (D == 2 ? N * N : N);
  extern __shared__ double sm[];
  const int64_t c0 = (int64_t)blockIdx.x * L::CPB;
  const int ncell = (int)(g.ncells - c0 < (int64_t)L::CPB ? g.ncells - c0 : (int64_t)L::CPB);
  double* r1 = sm;
  double* r2 = sm + L::R1 * L::CPB;

  if (D == 1) {
    for (int f = threadIdx.x; f < ncell; f += blockDim.x) {
      const int64_t cc = c0 + f;
      int cm[3] = {(int)cc, 0, 0};
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = xf[fine_index<D, N>(g, cm, o, 0, 0)];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        xc[cc * N + j] = s;
      }
    }
    return;
  }

  if (D == 3) {
    // pass 2^T: contract direction 3 reading the fine rows, -> region 1 (M,M,N)
    for_fibers<L::CPB * M * M, L::THREADS>(ncell * M * M, [&](int e) {
      const int cl = e / (M * M), f = e - cl * (M * M);
      const int o0 = f % M, o1 = f / M;
      int cm[3];
      coarse_multi<D>(g, c0 + cl, cm);
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = xf[fine_index<D, N>(g, cm, o0, o1, o)];
      double* out = r1 + cl * L::R1 + f;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * M * M] = s;
      }
    });
    __syncthreads();
    // pass 1^T: contract direction 2, region 1 -> region 2 (M,N,N; pitch PB)
    for_fibers<L::CPB * M * N, L::THREADS>(ncell * M * N, [&](int e) {
      const int cl = e / (M * N), f = e - cl * (M * N);
      const int o0 = f % M, j2 = f / M;
      const double* in = r1 + cl * L::R1 + o0 + M * M * j2;
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = in[o * M];
      double* out = r2 + cl * L::R2 + o0 + L::PB * N * j2;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * L::PB] = s;
      }
    });
  } else {
    // pass 1^T (2D): contract direction 2 reading the fine rows -> region 2 (M,N)
    for_fibers<L::CPB * M, L::THREADS>(ncell * M, [&](int e) {
      const int cl = e / M, o0 = e - cl * M;
      int cm[3];
      coarse_multi<D>(g, c0 + cl, cm);
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = xf[fine_index<D, N>(g, cm, o0, o, 0)];
      double* out = r2 + cl * L::R2 + o0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * L::PB] = s;
      }
    });
  }
  __syncthreads();

  // pass 0^T: contract direction 1, region 2 -> coarse rows (staged in region 1)
  constexpr int F0 = D == 3 ? N * N : N;
  for_fibers<L::CPB * F0, L::THREADS>(ncell * F0, [&](int e) {
    const int cl = e / F0, f = e - cl * F0;
    const double* in = r2 + cl * L::R2 + f * L::PB;
    double a[M];
#pragma unroll
    for (int o = 0; o < M; ++o) a[o] = in[o];
    double* out = r1 + cl * L::R1 + f * L::PA;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
      out[j] = s;
    }
  });
  __syncthreads();
  for_fibers<L::CPB * ND, L::THREADS>(ncell * ND, [&](int e) {
    const int cl = e / ND, q = e - cl * ND;
    const int row = q / N, i0 = q - row * N;
    xc[c0 * ND + e] = r1[cl * L::R1 + row * L::PA + i0];
  });
}

// ---------------------------------------------------------------------------
// TMA variants (n even, n <= 8): the 2^d child cells of a coarse cell are
// staged densely in shared memory (one slot of n^d doubles per child, 2-double
// skew per slot) and move as whole cells through the bulk-copy engine:
// prolongation stores them (or reduce-adds them into x, the fused V-cycle
// correction) with cp.async.bulk / cp.reduce.async.bulk .add.f64, restriction
// loads them with cp.async.bulk completing on an mbarrier.  Every fine cell is
// one 1728-byte (Q5) contiguous transfer instead of 48-byte row fragments
// from the LSU.
// ---------------------------------------------------------------------------
template <int D, int N>
struct TBulk {
  using L = TLay<D, N>;
  static constexpr int ND = D == 3 ? N * N * N : N * N;
  static constexpr int SL = 1 << D;                 // child slots
  static constexpr int ST = SL * (ND + 2);          // dense child staging
  static constexpr int PER_CELL = L::R1 + L::R2 + ST;
  static constexpr size_t SMEM = sizeof(double) * (size_t)PER_CELL * L::CPB;
  __device__ __forceinline__ static int slot_off(int s) { return s * (ND + 2); }
};

__device__ __forceinline__ void bulk_store(double* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}

// global id of child slot s (bit t = s_t) of coarse cell cm
template <int D>
__device__ __forceinline__ int64_t child_cell(const TGeo& g, const int* cm, int s) {
  int64_t cell = 2 * cm[0] + (s & 1);
  if (D >= 2) cell += (int64_t)(2 * g.nc[0]) * (2 * cm[1] + ((s >> 1) & 1));
  if (D == 3) cell += (int64_t)(2 * g.nc[0]) * (2 * g.nc[1]) * (2 * cm[2] + ((s >> 2) & 1));
  return cell;
}

// staging offset (slot + node) of output position (o0, o1, o2)
template <int D, int N>
__device__ __forceinline__ int stage_index(int o0, int o1, int o2) {
  const int s0 = o0 >= N, s1 = o1 >= N, s2 = o2 >= N;
  const int slot = s0 | (D >= 2 ? s1 << 1 : 0) | (D == 3 ? s2 << 2 : 0);
  int node = o0 - s0 * N;
  if (D >= 2) node += N * (o1 - s1 * N);
  if (D == 3) node += N * N * (o2 - s2 * N);
  return TBulk<D, N>::slot_off(slot) + node;
}

template <int D, int N, bool ADD>
__global__ void __launch_bounds__(TLay<D, N>::THREADS, TLay<D, N>::MINB)
    prolong_bulk_kernel(const __grid_constant__ EPar<N> E, const double* __restrict__ xc,
                        double* __restrict__ xf, TGeo g) {
  using L = TLay<D, N>;
  using B = TBulk<D, N>;
  constexpr int M = L::M, ND = B::ND;
  extern __shared__ __align__(16) double sm[];
  const int64_t c0 = (int64_t)blockIdx.x * L::CPB;
  const int ncell = (int)(g.ncells - c0 < (int64_t)L::CPB ? g.ncells - c0 : (int64_t)L::CPB);
  double* r1 = sm;
  double* r2 = sm + L::R1 * L::CPB;
  double* st = r2 + L::R2 * L::CPB;
  for_fibers<L::CPB * ND, L::THREADS>(ncell * ND, [&](int e) {
    const int cl = e / ND, q = e - cl * ND;
    const int row = q / N, i0 = q - row * N;
    r1[cl * L::R1 + row * L::PA + i0] = xc[c0 * ND + e];
  });
  __syncthreads();
  constexpr int F0 = D == 3 ? N * N : N;
  for_fibers<L::CPB * F0, L::THREADS>(ncell * F0, [&](int e) {
    const int cl = e / F0, f = e - cl * F0;
    const double* in = r1 + cl * L::R1 + f * L::PA;
    double a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = in[j];
    double* out = r2 + cl * L::R2 + f * L::PB;
    double ex[M];
    expand<N>(E, a, ex);
#pragma unroll
    for (int o = 0; o < M; ++o) {
      const double s = ex[o];
      out[o] = s;
    }
  });
  __syncthreads();
  if constexpr (D == 2) {
    for_fibers<L::CPB * M, L::THREADS>(ncell * M, [&](int e) {
      const int cl = e / M, o0 = e - cl * M;
      const double* in = r2 + cl * L::R2 + o0;
      double a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = in[j * L::PB];
      double* so = st + cl * B::ST;
      double ex[M];
      expand<N>(E, a, ex);
#pragma unroll
      for (int o1 = 0; o1 < M; ++o1) {
        const double s = ex[o1];
        so[stage_index<D, N>(o0, o1, 0)] = s;
      }
    });
  } else {
    for_fibers<L::CPB * M * N, L::THREADS>(ncell * M * N, [&](int e) {
      const int cl = e / (M * N), f = e - cl * (M * N);
      const int o0 = f % M, i2 = f / M;
      const double* in = r2 + cl * L::R2 + o0 + L::PB * N * i2;
      double a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = in[j * L::PB];
      double* out = r1 + cl * L::R1 + o0 + M * M * i2;
      double ex[M];
      expand<N>(E, a, ex);
#pragma unroll
      for (int o1 = 0; o1 < M; ++o1) {
        const double s = ex[o1];
        out[o1 * M] = s;
      }
    });
    __syncthreads();
    for_fibers<L::CPB * M * M, L::THREADS>(ncell * M * M, [&](int e) {
      const int cl = e / (M * M), f = e - cl * (M * M);
      const int o0 = f % M, o1 = f / M;
      const double* in = r1 + cl * L::R1 + f;
      double a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = in[j * M * M];
      double* so = st + cl * B::ST;
      double ex[M];
      expand<N>(E, a, ex);
#pragma unroll
      for (int o2 = 0; o2 < M; ++o2) {
        const double s = ex[o2];
        so[stage_index<D, N>(o0, o1, o2)] = s;
      }
    });
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    bool any = false;
    for (int l = threadIdx.x; l < ncell * B::SL; l += 32) {
      const int cl = l / B::SL, sl = l - cl * B::SL;
      int cm[3];
      coarse_multi<D>(g, c0 + cl, cm);
      double* dst = xf + child_cell<D>(g, cm, sl) * ND;
      const double* src = st + cl * B::ST + B::slot_off(sl);
      if (ADD) bulk_red_add(dst, src, ND * 8);
      else bulk_store(dst, src, ND * 8);
      any = true;
    }
    if (any) {
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
}

template <int D, int N>
__global__ void __launch_bounds__(TLay<D, N>::THREADS, TLay<D, N>::MINB)
    restrict_bulk_kernel(const __grid_constant__ EPar<N> E, const double* __restrict__ xf,
                         double* __restrict__ xc, TGeo g) {
  using L = TLay<D, N>;
  using B = TBulk<D, N>;
  constexpr int M = L::M, ND = B::ND;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t c0 = (int64_t)blockIdx.x * L::CPB;
  const int ncell = (int)(g.ncells - c0 < (int64_t)L::CPB ? g.ncells - c0 : (int64_t)L::CPB);
  double* r1 = sm;
  double* r2 = sm + L::R1 * L::CPB;
  double* st = r2 + L::R2 * L::CPB;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (unsigned)(ncell * B::SL * ND * 8));
    }
    __syncwarp();
    for (int l = threadIdx.x; l < ncell * B::SL; l += 32) {
      const int cl = l / B::SL, sl = l - cl * B::SL;
      int cm[3];
      coarse_multi<D>(g, c0 + cl, cm);
      bulk_load(st + cl * B::ST + B::slot_off(sl), xf + child_cell<D>(g, cm, sl) * ND, ND * 8,
                &bar);
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  if constexpr (D == 3) {
    for_fibers<L::CPB * M * M, L::THREADS>(ncell * M * M, [&](int e) {
      const int cl = e / (M * M), f = e - cl * (M * M);
      const int o0 = f % M, o1 = f / M;
      const double* si = st + cl * B::ST;
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = si[stage_index<D, N>(o0, o1, o)];
      double* out = r1 + cl * L::R1 + f;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * M * M] = s;
      }
    });
    __syncthreads();
    for_fibers<L::CPB * M * N, L::THREADS>(ncell * M * N, [&](int e) {
      const int cl = e / (M * N), f = e - cl * (M * N);
      const int o0 = f % M, j2 = f / M;
      const double* in = r1 + cl * L::R1 + o0 + M * M * j2;
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = in[o * M];
      double* out = r2 + cl * L::R2 + o0 + L::PB * N * j2;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * L::PB] = s;
      }
    });
  } else {
    for_fibers<L::CPB * M, L::THREADS>(ncell * M, [&](int e) {
      const int cl = e / M, o0 = e - cl * M;
      const double* si = st + cl * B::ST;
      double a[M];
#pragma unroll
      for (int o = 0; o < M; ++o) a[o] = si[stage_index<D, N>(o0, o, 0)];
      double* out = r2 + cl * L::R2 + o0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
        out[j * L::PB] = s;
      }
    });
  }
  __syncthreads();
  constexpr int F0 = D == 3 ? N * N : N;
  for_fibers<L::CPB * F0, L::THREADS>(ncell * F0, [&](int e) {
    const int cl = e / F0, f = e - cl * F0;
    const double* in = r2 + cl * L::R2 + f * L::PB;
    double a[M];
#pragma unroll
    for (int o = 0; o < M; ++o) a[o] = in[o];
    double* out = r1 + cl * L::R1 + f * L::PA;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int o = 0; o < M; ++o) s = fma(E.e[o * N + j], a[o], s);
      out[j] = s;
    }
  });
  __syncthreads();
  for_fibers<L::CPB * ND, L::THREADS>(ncell * ND, [&](int e) {
    const int cl = e / ND, q = e - cl * ND;
    const int row = q / N, i0 = q - row * N;
    xc[c0 * ND + e] = r1[cl * L::R1 + row * L::PA + i0];
  });
}

template <int D, int N>
static int launch_transfer(int dir, int accumulate, const double* e0, const double* e1,
                           const TGeo& g, const double* src, double* dst, cudaStream_t st) {
  using L = TLay<D, N>;
  EPar<N> E;
  for (int o = 0; o < N; ++o)
    for (int j = 0; j < N; ++j) {
      E.e[o * N + j] = e0[o * N + j];
      E.e[(o + N) * N + j] = e1[o * N + j];
      E.et[j * 2 * N + o] = e0[o * N + j];
      E.et[j * 2 * N + o + N] = e1[o * N + j];
    }
  const int64_t blocks = (g.ncells + L::CPB - 1) / L::CPB;
  if (blocks == 0) return DG_OK;
  if constexpr (D >= 2 && N % 2 == 0 && N <= 8) {
    // measured at Q5 32^3 -> 64^3: bulk prolongate 0.114 ms (plain stores
    // 0.115), bulk prolongate-accumulate 0.161 ms (load-add-store 0.191);
    // restriction reads faster through the LSU (0.098 vs 0.105 ms bulk)
    // the bulk copies need 16-byte aligned cell rows: a misaligned view takes
    // the LSU kernels below instead of faulting
    const bool al16 = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
    if (al16 && env_int("DGB_TRANSFER_BULK", 1) && (dir == 0 || env_int("DGB_RESTRICT_BULK", 0))) {
      const size_t sm = TBulk<D, N>::SMEM;
      if (dir == 0) {
        auto k = accumulate ? prolong_bulk_kernel<D, N, true> : prolong_bulk_kernel<D, N, false>;
        DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k<<<(unsigned)blocks, L::THREADS, sm, st>>>(E, src, dst, g);
      } else {
        auto k = restrict_bulk_kernel<D, N>;
        DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k<<<(unsigned)blocks, L::THREADS, sm, st>>>(E, src, dst, g);
      }
      DG_CUDA(cudaGetLastError());
      return DG_OK;
    }
  }
  const size_t smem = D == 1 ? 0 : L::SMEM;
  if (dir == 0) {
    auto k = accumulate ? prolong_kernel<D, N, true> : prolong_kernel<D, N, false>;
    if (smem > 48 * 1024)
      DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)blocks, L::THREADS, smem, st>>>(E, src, dst, g);
  } else {
    auto k = restrict_kernel<D, N>;
    if (smem > 48 * 1024)
      DG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)blocks, L::THREADS, smem, st>>>(E, src, dst, g);
  }
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

static int transfer(int dir, int dim, int degree, const int* coarse_cells, const double* e0,
                    const double* e1, const double* src, double* dst, int accumulate,
                    void* stream) {
  if (!coarse_cells || !e0 || !e1 || !src || !dst) return fail(DG_EINVAL, "null argument");
  if (dim < 1 || dim > 3) return fail(DG_EINVAL, "dim must be 1, 2 or 3");
  if (src == dst) return fail(DG_EINVAL, "transfer: source and destination alias");
  TGeo g;
  g.ncells = 1;
  for (int t = 0; t < 3; ++t) {
    g.nc[t] = t < dim ? coarse_cells[t] : 1;
    if (g.nc[t] < 1 || g.nc[t] > (1 << 20)) return fail(DG_EINVAL, "bad coarse cell count");
    g.ncells *= g.nc[t];
  }
  g.f0.init((uint32_t)g.nc[0]);
  g.f1.init((uint32_t)g.nc[1]);
  const int n = degree + 1;
  cudaStream_t st = (cudaStream_t)stream;
#define DG_TCASE(D, NN) \
  if (dim == D && n == NN) return launch_transfer<D, NN>(dir, accumulate, e0, e1, g, src, dst, st);
  DG_N_CASES(DG_TCASE, 1)
  DG_N_CASES(DG_TCASE, 2)
  DG_N_CASES(DG_TCASE, 3)
#undef DG_TCASE
  return fail(DG_EUNSUPPORTED, "transfer: degree " + std::to_string(degree) +
                                   " has no compiled kernel (1 <= k <= 15)");
}

}  // namespace dgb

extern "C" {

int dg_prolongate(int dim, int degree, const int* coarse_cells, const double* e0,
                  const double* e1, const double* xc, double* xf, int accumulate,
                  void* stream) {
  return dgb::transfer(0, dim, degree, coarse_cells, e0, e1, xc, xf, accumulate, stream);
}

int dg_restrict(int dim, int degree, const int* coarse_cells, const double* e0,
                const double* e1, const double* xf, double* xc, void* stream) {
  return dgb::transfer(1, dim, degree, coarse_cells, e0, e1, xf, xc, 0, stream);
}

}  // extern "C"
