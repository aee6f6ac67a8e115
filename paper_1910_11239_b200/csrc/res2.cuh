// res2.cuh - SIPG residual r = b - A x, v2 (constant-operand DFMA).
//
// dgop.residual / apply_operator (dgop.py:762-788) on a uniform Cartesian
// level in Kronecker-sum form:
//   A x |_c = sum_t (x)_{s != t} M_s  G_t,
//   G_t = A_diag(digit_t) ._t x_c + a_pm ._t x_{c+e_t} + a_pm^T ._t x_{c-e_t},
// with a_pm = alpha e_{n-1} e_0^T + beta e_{n-1} bg0^T + beta' bg1 e_0^T
// (polybasis.py:278-284; bv0 = e_0, bv1 = e_{n-1} on GL nodes).
//
// The 1D matrices (M, A_diag per digit) and the basis derivatives live in the
// kernel parameter space, so the DFMAs take their matrix operand from the
// constant bank.  Per cell three shared buffers X, A, B and five phases
// (3D; 8 contractions):
//   1: A = G_0(X) [fibers t=0],  B = G_1(X) [t=1]
//   2: A <- M A   [t=1],         B <- M B   [t=0]
//   3: A <- M (A + B) [t=2],     B = G_2(X) [t=2]     (same fiber: no race)
//   4: B <- M B   [t=1]
//   5: A <- A + M B [t=0]; then r = b - A (coalesced)
#pragma once
#include "common.cuh"
#include "fdm2.cuh"

namespace dgb {

template <int N>
struct ResMats {
  double mass[N * N];      // stored transposed (matvec_t): mass[k][i] = M[i][k]
  double adiag[4][N * N];  // transposed A_diag per digit
  double bg0[N];
  double bg1[N];
  // centro-symmetric halves (k-outer P^T, Q^T) of M and A_diag(0)
  double eo[4][(N / 2) * (N / 2)];
};

template <int D, int N>
struct Res2Params {
  const double* x;
  const double* b;  // nullptr: v = A x
  double* r;
  const int32_t* list;
  int64_t start;
  int64_t count;
  double alpha, beta, betap;
  int packed;   // list entries are packed global cell coordinates (pack3)
  int eo;       // mass and interior stiffness on the even/odd path
  int blocked;  // 1: range mode on 2x2x2 cell blocks (G = 8), layers [bz0, bz0 + bnz);
                // 2: list mode whose consecutive groups of 8 cells are 2x2x2
                //    blocks in slot order dx + 2 dy + 4 dz (vertex-patch cells)
  int bz0, bnz;
  Geo geo;
  ResMats<N> mats;
};

// Shared tensor layout of the residual (the padded Lay) and the thread ->
// (cell, fiber) map per contraction direction.  (Interleaving the cells of a
// CTA across consecutive threads makes all three directions bank-conflict
// free but scatters the neighbour-trace loads and row stores over 8 cells;
// measured slower.)
template <int D, int N, int G, bool NARROW = false>
struct RLay {
  using L = Lay<D, N>;
  static constexpr int F = L::F;
  // 3D n = 6 (cfg 5): row pitch 9 and plane pitch 54 instead of 7 / 42 make
  // the direction-1 fibers bank-conflict free as well (shared wavefronts per
  // cell group 504 -> 396, the residual is L1/shared-pipe bound); the
  // direction-2 fibers stay 2-way (no straight layout frees all three)
  static constexpr bool WIDE = (D == 3 && N == 6 && !NARROW);
  static constexpr int P = WIDE ? 9 : L::P;
  static constexpr int Q = WIDE ? 54 : L::P * N;
  static constexpr int GS = (D == 3) ? Q * N : L::SZ;
  __device__ __forceinline__ static int sstride(int t) {
    if (D == 2) return L::sstride(t);
    return t == 0 ? 1 : (t == 1 ? P : Q);
  }
  __device__ __forceinline__ static int sbase(int t, int f) {
    if (D == 2) return L::sbase(t, f);
    const int a = f % N, b = f / N;
    if (t == 0) return a * P + b * Q;
    if (t == 1) return a + b * Q;
    return a + b * P;
  }
  // shared offset of cell row w (direction-0 fiber w = i1 + n i2)
  __device__ __forceinline__ static int row(int w) { return sbase(0, w); }
  __device__ __forceinline__ static void who(int, int tid, int& g, int& f) {
    g = tid / F;
    f = tid - g * F;
  }
};

// cell of work item idx: local id (or -1) and global multi-index
template <int D>
__device__ __forceinline__ int res_cell(const Geo& geo, const int32_t* list, int packed,
                                        int64_t start, int64_t count, int64_t idx, int* c) {
  c[0] = c[1] = c[2] = 0;
  if (idx >= count) return -1;
  if (list) {
    const int e = list[idx];
    if (packed) {
      unpack_d<D>(e, c);
      return cell_local<D>(geo, c);
    }
    cell_multi<D>(geo, e, c);
    return e;
  }
  const int cell = (int)(start + idx);
  cell_multi<D>(geo, cell, c);
  return cell;
}

// face scalars of the global neighbour fiber f along t on side `right`
// (a_pm x_R: hi = alpha x_R[0] + beta bg0.x_R, all = beta' x_R[0];
//  a_pm^T x_L: hi = alpha x_L[n-1] + beta' bg1.x_L, all = beta x_L[n-1])
template <int D, int N>
__device__ __forceinline__ void face_pair(const Res2Params<D, N>& p, int t, int f, const int* c,
                                          bool right, double& hi, double& all) {
  using L = Lay<D, N>;
  int nb[3] = {c[0], c[1], D == 3 ? c[2] : 0};
  nb[t] += right ? 1 : -1;
  const double* q = p.x + (int64_t)cell_local<D>(p.geo, nb) * L::NE + L::gbase(t, f);
  double xv[N];
  if (t == 0) {
    row_load_reg<N>(xv, q);
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) xv[k] = __ldg(q + k * L::gstride(t));
  }
  double g = 0.0;
  if (right) {
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg0[k], xv[k], g);
    all = p.betap * xv[0];
    hi = p.alpha * xv[0] + p.beta * g;
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg1[k], xv[k], g);
    all = p.beta * xv[N - 1];
    hi = p.alpha * xv[N - 1] + p.betap * g;
  }
}

// G_t fiber: A_diag(digit) along t plus the rank-2 neighbour couplings.  The
// neighbour fibers are reduced to their face value and normal derivative
// before the own fiber is loaded, so at most one fiber-sized array of
// neighbour data is live (register budget at n = 16).  `pre` (blocked mode)
// carries the out-of-block side's scalars, loaded at kernel start.
struct FacePre {
  int side;  // -1 none, 0 left, 1 right
  double hi, all;
};

template <int D, int N, class LY>
__device__ __forceinline__ void stiff2_fiber(const Res2Params<D, N>& p, int t, int f,
                                             const int* c, const double* X, double* out,
                                             const double* XR = nullptr,
                                             const double* XL = nullptr,
                                             FacePre pre = FacePre{-1, 0.0, 0.0}) {
  using L = Lay<D, N>;
  const int sb = LY::sbase(t, f), ss = LY::sstride(t);
  const int digit = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
  const int gb = L::gbase(t, f), gs = L::gstride(t);
  int nb[3] = {c[0], c[1], D == 3 ? c[2] : 0};
  double r_hi = 0.0, r_all = 0.0, l_lo = 0.0, l_all = 0.0;
  if (pre.side == 1) {
    r_hi = pre.hi, r_all = pre.all;
  } else if (pre.side == 0) {
    l_lo = pre.hi, l_all = pre.all;
  }
  if (!(digit & 2) && pre.side != 1) {  // a_pm x_R: value and normal derivative at the shared face
    double xr[N];
    if (XR) {  // neighbour tensor of the same CTA block (shared memory)
#pragma unroll
      for (int k = 0; k < N; ++k) xr[k] = XR[sb + k * ss];
    } else {
      nb[t] = c[t] + 1;
      const double* q = p.x + (int64_t)cell_local<D>(p.geo, nb) * L::NE + gb;
      if (t == 0) {
        row_load_reg<N>(xr, q);  // a cell row: 16-byte loads for even n
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) xr[k] = __ldg(q + k * gs);
      }
    }
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg0[k], xr[k], g);
    r_all = p.betap * xr[0];
    r_hi = p.alpha * xr[0] + p.beta * g;
  }
  if (!(digit & 1) && pre.side != 0) {  // a_pm^T x_L
    double xl[N];
    if (XL) {
#pragma unroll
      for (int k = 0; k < N; ++k) xl[k] = XL[sb + k * ss];
    } else {
      nb[t] = c[t] - 1;
      const double* q = p.x + (int64_t)cell_local<D>(p.geo, nb) * L::NE + gb;
      if (t == 0) {
        row_load_reg<N>(xl, q);
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) xl[k] = __ldg(q + k * gs);
      }
    }
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) g = fma(p.mats.bg1[k], xl[k], g);
    l_all = p.beta * xl[N - 1];
    l_lo = p.alpha * xl[N - 1] + p.betap * g;
  }
  double v[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = X[sb + k * ss];
  if constexpr (N % 2 == 0) {
    if (p.eo && digit == 0) matvec_cs<N>(p.mats.eo[2], p.mats.eo[3], v, o);
    else matvec_digit<N>(p.mats.adiag, digit, v, o);
  } else {
    matvec_digit<N>(p.mats.adiag, digit, v, o);
  }
  if (!(digit & 2)) {
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = fma(p.mats.bg1[i], r_all, o[i]);
    o[N - 1] += r_hi;
  }
  if (!(digit & 1)) {
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = fma(p.mats.bg0[i], l_all, o[i]);
    o[0] += l_lo;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) out[sb + i * ss] = o[i];
}

template <int D, int N>
__device__ __forceinline__ void res_mass(const Res2Params<D, N>& p, const double (&v)[N],
                                         double (&o)[N]) {
  if constexpr (N % 2 == 0) {
    if (p.eo) {
      matvec_cs<N>(p.mats.eo[0], p.mats.eo[1], v, o);
      return;
    }
  }
  matvec_t<N>(p.mats.mass, v, o);
}

// buf <- M buf along t (in place), optionally adding `add` first
template <int D, int N, bool ADD, class LY>
__device__ __forceinline__ void mass_fiber(const Res2Params<D, N>& p, int t, int f, double* buf,
                                           const double* add) {
  const int sb = LY::sbase(t, f), ss = LY::sstride(t);
  double v[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = ADD ? buf[sb + k * ss] + add[sb + k * ss] : buf[sb + k * ss];
  res_mass<D, N>(p, v, o);
#pragma unroll
  for (int k = 0; k < N; ++k) buf[sb + k * ss] = o[k];
}

// one group of G cells (work items grp*G .. grp*G+G-1 of the list/range);
// all NT = G*F threads of the CTA take part; `sm` holds res_smem_doubles doubles.
template <int D, int N, int G, bool NARROW = false>
__device__ __forceinline__ void res_group(const Res2Params<D, N>& p, const int32_t* list,
                                          int packed, int64_t start, int64_t count, int64_t grp,
                                          double* sm) {
  using L = Lay<D, N>;
  constexpr int F = L::F;
  constexpr int NT = G * F;
  __shared__ int s_cell[G];
  __shared__ int s_c[G][3];
  const int tid = threadIdx.x;
  constexpr bool BLK = (D == 3 && G == 8);
  const bool range_blocked = BLK && p.blocked == 1 && !list;
  const bool blocked = range_blocked || (BLK && p.blocked == 2 && list);
  if (tid < G) {
    if (range_blocked) {
      // CTA = 2x2x2 cell block; group g = dx + 2 dy + 4 dz
      const int nbx = (p.geo.nc[0] + 1) >> 1, nby = (p.geo.nc[1] + 1) >> 1;
      const int64_t bxy = (int64_t)nbx * nby;
      const int bz = (int)(grp / bxy), rem = (int)(grp - bz * bxy);
      const int by = rem / nbx, bx = rem - by * nbx;
      int* c = s_c[tid];
      c[0] = 2 * bx + (tid & 1);
      c[1] = 2 * by + ((tid >> 1) & 1);
      c[2] = p.bz0 + 2 * bz + (tid >> 2);
      const bool in = c[0] < p.geo.nc[0] && c[1] < p.geo.nc[1] && c[2] < p.bz0 + p.bnz;
      s_cell[tid] = in ? cell_local<D>(p.geo, c) : -1;
    } else {
      s_cell[tid] = res_cell<D>(p.geo, list, packed, start, count, grp * G + tid, s_c[tid]);
    }
  }
  __syncthreads();
  using LY = RLay<D, N, G, NARROW>;
  constexpr int GS = LY::GS;
  constexpr int RPC = (D == 3) ? N * N : N;  // rows per cell
  for (int row = tid; row < G * RPC; row += NT) {
    const int gg = row / RPC, w = row - gg * RPC;
    const int cell = s_cell[gg];
    if (cell < 0) continue;
    row_load<N>(sm + gg * GS + LY::row(w), p.x + (int64_t)cell * L::NE + w * N);
  }
  // blocked mode: every cell has one out-of-block face per direction (the
  // side away from its block partner), whose neighbour fiber comes from
  // global memory; those loads are issued here, behind the block's row
  // loads, so their latency overlaps the barrier instead of the phases
  // (measured: cfg 2, n = 4, residual 0.042 -> 0.037 ms; n = 6 loses, 0.663 ->
  // 0.693 ms at cfg 5, so it stays off there)
  FacePre pre0{-1, 0.0, 0.0}, pre1{-1, 0.0, 0.0}, pre2{-1, 0.0, 0.0};
  if constexpr (D == 3 && G == 8 && N <= 4) {
    if (blocked) {
      const int g0 = tid / Lay<D, N>::F, f0 = tid - g0 * Lay<D, N>::F;
      const int* cc = s_c[g0];
#pragma unroll
      for (int t = 0; t < D; ++t) {
        FacePre& pr = t == 0 ? pre0 : (t == 1 ? pre1 : pre2);
        const bool right = (g0 >> t) & 1;  // high cell of the pair: +e_t is outside
        const bool at_bnd = right ? cc[t] == p.geo.nc[t] - 1 : cc[t] == 0;
        pr.side = (s_cell[g0] < 0 || at_bnd) ? -1 : (right ? 1 : 0);
        if (pr.side >= 0) face_pair<D, N>(p, t, f0, cc, right, pr.hi, pr.all);
      }
    }
  }
  // thread -> (cell, fiber) per direction
  int gt[3], ft[3];
#pragma unroll
  for (int t = 0; t < D; ++t) LY::who(t, tid, gt[t], ft[t]);
  auto X = [&](int t) { return sm + gt[t] * GS; };
  auto A = [&](int t) { return sm + (G + gt[t]) * GS; };
  auto B = [&](int t) { return sm + (2 * G + gt[t]) * GS; };
  auto act = [&](int t) { return s_cell[gt[t]] >= 0; };
  // in-block neighbour tensors along t (blocked mode): right if bit t of g is 0
  auto nbr = [&](int t, bool right) -> const double* {
    if (!blocked) return nullptr;
    const int g = gt[t];
    const bool hi = (g >> t) & 1;
    if (right == hi) return nullptr;
    const int gn = g ^ (1 << t);
    return s_cell[gn] >= 0 ? sm + gn * GS : nullptr;
  };
  __syncthreads();
  if (act(0))
    stiff2_fiber<D, N, LY>(p, 0, ft[0], s_c[gt[0]], X(0), A(0), nbr(0, true), nbr(0, false), pre0);
  if (act(1))
    stiff2_fiber<D, N, LY>(p, 1, ft[1], s_c[gt[1]], X(1), B(1), nbr(1, true), nbr(1, false), pre1);
  __syncthreads();
  if (act(1)) mass_fiber<D, N, false, LY>(p, 1, ft[1], A(1), nullptr);
  if (act(0)) mass_fiber<D, N, false, LY>(p, 0, ft[0], B(0), nullptr);
  __syncthreads();
  // each thread's last fiber (t = 0) is a whole cell row, so the final
  // contraction writes r = b - A x straight to global memory; b is
  // prefetched into registers one phase earlier
  const int cell0 = s_cell[gt[0]];
  const int64_t gi = (int64_t)(cell0 >= 0 ? cell0 : 0) * L::NE + ft[0] * N;
  double bv[N];
  if (D == 3) {
    if (act(2)) {
      mass_fiber<D, N, true, LY>(p, 2, ft[2], A(2), B(2));  // A = M_2 (M_1 G_0 + M_0 G_1)
      stiff2_fiber<D, N, LY>(p, 2, ft[2], s_c[gt[2]], X(2), B(2), nbr(2, true),
                             nbr(2, false), pre2);                 // B = G_2
    }
    __syncthreads();
    if (act(0) && p.b) row_load_reg<N>(bv, p.b + gi);
    if (act(1)) mass_fiber<D, N, false, LY>(p, 1, ft[1], B(1), nullptr);
    __syncthreads();
    if (act(0)) {  // r = b - (A + M_0 B), row ft[0]
      const int sb = LY::sbase(0, ft[0]);
      const double* Bs = B(0);
      const double* As = A(0);
      double v[N], o[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = Bs[sb + k];
      res_mass<D, N>(p, v, o);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double ax = As[sb + k] + o[k];
        o[k] = p.b ? bv[k] - ax : ax;
      }
      row_store<N>(p.r + gi, o);
    }
  } else {
    if (act(0) && p.b) row_load_reg<N>(bv, p.b + gi);
    // 2D: A x = M_1 G_0 + M_0 G_1 = A + B, row ft[0]
    if (act(0)) {
      const int sb = LY::sbase(0, ft[0]);
      const double* Bs = B(0);
      const double* As = A(0);
      double o[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double ax = As[sb + k] + Bs[sb + k];
        o[k] = p.b ? bv[k] - ax : ax;
      }
      row_store<N>(p.r + gi, o);
    }
  }
}

template <int D, int N, bool NARROW = false, int MINB = 0>
__global__ void __launch_bounds__(fdm2_groups<D, N>() * Lay<D, N>::F, MINB)
res2_kernel(const __grid_constant__ Res2Params<D, N> p) {
  extern __shared__ __align__(16) double sm[];
  res_group<D, N, fdm2_groups<D, N>(), NARROW>(p, p.list, p.packed, p.start, p.count, blockIdx.x,
                                               sm);
}


template <int D, int N, int G, bool NARROW = false>
__host__ __device__ constexpr int res_smem_doubles() {
  return 3 * G * RLay<D, N, G, NARROW>::GS;
}

template <int D, int N, bool NARROW = false>
__host__ __device__ constexpr int res2_smem_doubles() {
  return res_smem_doubles<D, N, fdm2_groups<D, N>(), NARROW>();
}

}  // namespace dgb
