// fdm2.cuh - fast-diagonalisation solves, v2 (constant-operand DFMA).
//
// x += omega * Z Lambda^-1 Z^T R r for cells or vertex patches
// (fastdiag.py:457-496, 602-628).  Design:
//  - the 1D eigenvector matrices Z, Z^T of the four boundary digits travel in
//    the kernel's parameter space (__grid_constant__); the matvec runs k-outer
//    over a transposed-stored matrix so each LDCU.128 feeds two DFMAs with
//    their constant operand and the tensor is the only shared-memory traffic;
//  - one tensor buffer per subdomain: each thread owns one fiber of the
//    contracted direction, reads it to registers, writes the result back in
//    place (fibers of one direction partition the tensor);
//  - the last forward contraction, the 1/Lambda-sum scaling and the first
//    backward contraction act on the same fiber and are fused (2d-1 passes);
//  - gather / scatter move whole cell rows (n contiguous doubles of one
//    cell, 16-byte vectors when n is even) so index math is per row, not per
//    element; a patch row lands at (s0 n, s1 n + i1, s2 n + i2) of the patch
//    tensor (fastdiag.py:546-557); the update is a vectorised
//    load-add-store (write-disjoint colours) or fp64 RED reductions when the
//    caller asks for overlap-safe accumulation (measured: RED costs ~0.1 ms
//    per cfg-5 colour at L2, so the disjoint path avoids it);
//  - several subdomains per CTA so that the CTA is a whole number of warps.
#pragma once
#include "common.cuh"

namespace dgb {

template <int M>
struct FdmMats {
  double fwd[4][M * M];  // Z per digit, row-major: fwd[k][i] = Z[k][i] -> out = Z^T v
  double bwd[4][M * M];  // Z^T per digit, row-major: bwd[k][i] = Z[i][k] -> out = Z v
  // even/odd halves of the interior digit (tables.py device_tables):
  // [0] top-even (k-outer fwd), [1] top-odd, [2] top-even^T, [3] top-odd^T
  double eo[4][(M / 2) * (M / 2)];
};

template <int D, int M>
struct Fdm2Params {
  const double* r;
  double* x;
  const int32_t* list;
  int64_t start;
  int64_t count;
  const double* invsum;
  double omega;
  int atomic;   // overlapping subdomains: fp64 reductions instead of load-add-store
  int packed;   // list entries are packed global coordinates (pack3)
  int eo;       // interior digit uses the even/odd halves
  int pv_lo, pv_hi;  // cluster mode: patch vertices v_d outside are skipped
  int direct;   // first/last contraction straight from/to global rows (no gather/scatter pass)
  Geo geo;
  FdmMats<M> mats;
};

// out_i = sum_k St[k*M+i] v_k  (k outer: constants consumed in load order)
template <int M>
__device__ __forceinline__ void matvec_t(const double* __restrict__ St, const double (&v)[M],
                                         double (&o)[M]) {
#pragma unroll
  for (int i = 0; i < M; ++i) o[i] = St[i] * v[0];
#pragma unroll
  for (int k = 1; k < M; ++k) {
#pragma unroll
    for (int i = 0; i < M; ++i) o[i] = fma(St[k * M + i], v[k], o[i]);
  }
}

// compile-time matrix addresses for each digit (warp-uniform in practice)
template <int M>
__device__ __forceinline__ void matvec_digit(const double (&S)[4][M * M], int digit,
                                             const double (&v)[M], double (&o)[M]) {
  switch (digit) {
    case 0: matvec_t<M>(S[0], v, o); break;
    case 1: matvec_t<M>(S[1], v, o); break;
    case 2: matvec_t<M>(S[2], v, o); break;
    default: matvec_t<M>(S[3], v, o); break;
  }
}

// even/odd split of an interior-digit contraction (half the FMAs):
// forward  y_even = E^T u, y_odd = O^T w  with u = v_i + v_{m-1-i}, w = v_i - v_{m-1-i}
// backward x_i = e_i + o_i, x_{m-1-i} = e_i - o_i, e = E y_even, o = O y_odd
template <int M>
__device__ __forceinline__ void matvec_eo_fwd(const double* __restrict__ E,
                                              const double* __restrict__ O, const double (&v)[M],
                                              double (&o)[M]) {
  constexpr int H = M / 2;
  double u[H], w[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    u[i] = v[i] + v[M - 1 - i];
    w[i] = v[i] - v[M - 1 - i];
  }
#pragma unroll
  for (int r = 0; r < H; ++r) {
    o[r] = E[r] * u[0];
    o[H + r] = O[r] * w[0];
  }
#pragma unroll
  for (int k = 1; k < H; ++k) {
#pragma unroll
    for (int r = 0; r < H; ++r) {
      o[r] = fma(E[k * H + r], u[k], o[r]);
      o[H + r] = fma(O[k * H + r], w[k], o[H + r]);
    }
  }
}

template <int M>
__device__ __forceinline__ void matvec_eo_bwd(const double* __restrict__ Et,
                                              const double* __restrict__ Ot, const double (&v)[M],
                                              double (&o)[M]) {
  constexpr int H = M / 2;
  double e[H], q[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = Et[i] * v[0];
    q[i] = Ot[i] * v[H];
  }
#pragma unroll
  for (int k = 1; k < H; ++k) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      e[i] = fma(Et[k * H + i], v[k], e[i]);
      q[i] = fma(Ot[k * H + i], v[H + k], q[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    o[i] = e[i] + q[i];
    o[M - 1 - i] = e[i] - q[i];
  }
}

// centro-symmetric matrix (stored as k-outer P^T, Q^T halves): y = A v
template <int M>
__device__ __forceinline__ void matvec_cs(const double* __restrict__ Pt,
                                          const double* __restrict__ Qt, const double (&v)[M],
                                          double (&o)[M]) {
  constexpr int H = M / 2;
  double u[H], w[H], s[H], d[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    u[i] = v[i] + v[M - 1 - i];
    w[i] = v[i] - v[M - 1 - i];
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    s[i] = Pt[i] * u[0];
    d[i] = Qt[i] * w[0];
  }
#pragma unroll
  for (int k = 1; k < H; ++k) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      s[i] = fma(Pt[k * H + i], u[k], s[i]);
      d[i] = fma(Qt[k * H + i], w[k], d[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    o[i] = s[i] + d[i];
    o[M - 1 - i] = s[i] - d[i];
  }
}

// FDM contractions with the interior digit on the even/odd path
template <int M, bool FWD>
__device__ __forceinline__ void fdm_matvec(const FdmMats<M>& m, int eo, int digit,
                                           const double (&v)[M], double (&o)[M]) {
  if constexpr (M % 2 == 0) {
    if (eo && digit == 0) {
      if (FWD) matvec_eo_fwd<M>(m.eo[0], m.eo[1], v, o);
      else matvec_eo_bwd<M>(m.eo[2], m.eo[3], v, o);
      return;
    }
  }
  matvec_digit<M>(FWD ? m.fwd : m.bwd, digit, v, o);
}

template <int M, bool FWD>
__device__ __forceinline__ void fdm_fiber(const FdmMats<M>& m, int eo, int digit, double* buf,
                                          int base, int stride) {
  double v[M], o[M];
#pragma unroll
  for (int k = 0; k < M; ++k) v[k] = buf[base + k * stride];
  fdm_matvec<M, FWD>(m, eo, digit, v, o);
#pragma unroll
  for (int k = 0; k < M; ++k) buf[base + k * stride] = o[k];
}

template <int M>
__device__ __forceinline__ void fiber_inplace(const double (&S)[4][M * M], int digit, double* buf,
                                              int base, int stride) {
  double v[M], o[M];
#pragma unroll
  for (int k = 0; k < M; ++k) v[k] = buf[base + k * stride];
  matvec_digit<M>(S, digit, v, o);
#pragma unroll
  for (int k = 0; k < M; ++k) buf[base + k * stride] = o[k];
}

// x + omega * y with two roundings: the same value the fp64 reduction paths
// (RED.ADD, bulk reduce-add) produce, so every update path is bitwise equal
__device__ __forceinline__ double xupd(double x, double omega, double y) {
  return __dadd_rn(x, __dmul_rn(omega, y));
}

// one row of N doubles: global <-> shared
template <int N>
__device__ __forceinline__ void row_load(double* __restrict__ s, const double* __restrict__ g) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(g + i));
      s[i] = v.x;
      s[i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) s[i] = __ldg(g + i);
  }
}

template <int N>
__device__ __forceinline__ void row_update(double* __restrict__ g, const double* __restrict__ s,
                                           double omega, bool atomic) {
  if (atomic) {
#pragma unroll
    for (int i = 0; i < N; ++i) atomicAdd(g + i, omega * s[i]);
    return;
  }
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      double2 v = *reinterpret_cast<const double2*>(g + i);
      v.x = xupd(v.x, omega, s[i]);
      v.y = xupd(v.y, omega, s[i + 1]);
      *reinterpret_cast<double2*>(g + i) = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = xupd(g[i], omega, s[i]);
  }
}

// L2-coherent variants (ld.global.cg) for data written by other CTAs of the
// same kernel (dataflow kernel)
template <int N>
__device__ __forceinline__ void row_load_cg(double* __restrict__ s, const double* __restrict__ g) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(g + i));
      s[i] = v.x;
      s[i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) s[i] = __ldcg(g + i);
  }
}

template <int N>
__device__ __forceinline__ void row_update_cg(double* __restrict__ g, const double* __restrict__ s,
                                              double omega) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      double2 v = __ldcg(reinterpret_cast<const double2*>(g + i));
      v.x = xupd(v.x, omega, s[i]);
      v.y = xupd(v.y, omega, s[i + 1]);
      __stcg(reinterpret_cast<double2*>(g + i), v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) __stcg(g + i, xupd(__ldcg(g + i), omega, s[i]));
  }
}

// x[row] += omega * y as fp64 reductions at L2 (RED.E.ADD.F64, no load
// latency on the SM).  Correct for overlapping subdomains too; within one
// launch of a colour every DoF is hit once, so the result is deterministic.
template <int N>
__device__ __forceinline__ void row_red(double* __restrict__ g, const double* __restrict__ s,
                                        double omega) {
#pragma unroll
  for (int i = 0; i < N; ++i) atomicAdd(g + i, omega * s[i]);
}

template <int N>
__device__ __forceinline__ void row_load_reg(double (&v)[N], const double* __restrict__ g) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(g + i));
      v[i] = t.x;
      v[i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = __ldg(g + i);
  }
}

template <int N>
__device__ __forceinline__ void row_store(double* __restrict__ g, const double (&v)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) *reinterpret_cast<double2*>(g + i) = make_double2(v[i], v[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = v[i];
  }
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// Direction-0 fiber f of a subdomain as global cell rows: the fiber is the
// row (j1 % N, j2 % N) of the cell slots h + 2 (j1 / N) + 4 (j2 / N), h = 0, 1
// (patches), or one row of the single cell.  goff = row offset in the cell.
template <int D, int M, bool PATCH>
__host__ __device__ __forceinline__ void fiber_rows(int f, int& slot0, int& goff) {
  constexpr int N = PATCH ? M / 2 : M;
  const int j1 = (D == 3) ? f % M : f, j2 = (D == 3) ? f / M : 0;
  if (PATCH) {
    slot0 = 2 * (j1 / N) + ((D == 3) ? 4 * (j2 / N) : 0);
    goff = ((j1 % N) + ((D == 3) ? N * (j2 % N) : 0)) * N;
  } else {
    slot0 = 0;
    goff = (j1 + ((D == 3) ? N * j2 : 0)) * N;
  }
}

template <int N, int M>
__device__ __forceinline__ void rows_to_reg(double (&v)[M], int h, const double* __restrict__ g,
                                            bool coherent) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 t = coherent ? __ldcg(reinterpret_cast<const double2*>(g + i))
                                 : __ldg(reinterpret_cast<const double2*>(g + i));
      v[h * N + i] = t.x;
      v[h * N + i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[h * N + i] = coherent ? __ldcg(g + i) : __ldg(g + i);
  }
}

template <int N, int M>
__device__ __forceinline__ void reg_update(double* __restrict__ g, const double (&o)[M], int h,
                                           double omega, int atomic, bool coherent) {
  if (atomic) {
#pragma unroll
    for (int i = 0; i < N; ++i) atomicAdd(g + i, omega * o[h * N + i]);
    return;
  }
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      double2 t = coherent ? __ldcg(reinterpret_cast<const double2*>(g + i))
                           : *reinterpret_cast<const double2*>(g + i);
      t.x = xupd(t.x, omega, o[h * N + i]);
      t.y = xupd(t.y, omega, o[h * N + i + 1]);
      if (coherent) __stcg(reinterpret_cast<double2*>(g + i), t);
      else *reinterpret_cast<double2*>(g + i) = t;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double t = coherent ? __ldcg(g + i) : g[i];
      if (coherent) __stcg(g + i, xupd(t, omega, o[h * N + i]));
      else g[i] = xupd(t, omega, o[h * N + i]);
    }
  }
}

// rows of a subdomain: (cell slot, i1, i2) -> (global offset, shared offset)
template <int D, int M, bool PATCH>
struct Rows {
  static constexpr int N = PATCH ? M / 2 : M;
  static constexpr int RPC = (D == 3) ? N * N : N;      // rows per cell
  static constexpr int SLOTS = PATCH ? (1 << D) : 1;     // cells per subdomain
  static constexpr int RPS = SLOTS * RPC;                // rows per subdomain
  __device__ __forceinline__ static void map(int rr, int& slot, int& goff, int& soff) {
    using L = Lay<D, M>;
    slot = rr / RPC;
    const int w = rr - slot * RPC;
    goff = w * N;
    const int i1 = (D == 3) ? w % N : w;
    const int i2 = (D == 3) ? w / N : 0;
    const int s0 = slot & 1, s1 = (slot >> 1) & 1, s2 = (slot >> 2) & 1;
    soff = s0 * N + L::P * (s1 * N + i1) + (D == 3 ? L::P * M * (s2 * N + i2) : 0);
  }
};

// bulk copies through the TMA engine (no LSU wavefronts on the SM):
// global -> shared completing on an mbarrier, and shared -> global fp64
// reduce-add tracked by a bulk group
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_red_add(double* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                   gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}

// Dense cell rows of 8 or 16 doubles (64 / 128 bytes) put the 16-byte
// accesses of a quarter-warp (8 consecutive rows) into the same bank group.
// Each thread therefore starts its row at chunk row_rot (distinct bank
// groups across the quarter-warp) and the chunk registers are rotated with a
// log-depth select network, so the register array stays statically indexed.
template <int N>
__device__ __forceinline__ int row_rot(int f) {
  return N == 16 ? (f & 7) : ((f >> 1) & 3);  // N = 8: rows pair up in a bank group
}
// w[j] <- w[(j + r) % C] for 0 <= r < C (C a power of two)
template <int C>
__device__ __forceinline__ void rotate_chunks(double2 (&w)[C], int r) {
#pragma unroll
  for (int b = 1; b < C; b <<= 1) {
    const bool on = (r & b) != 0;
    double2 t[C];
#pragma unroll
    for (int j = 0; j < C; ++j) t[j] = w[(j + b) % C];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      w[j].x = on ? t[j].x : w[j].x;
      w[j].y = on ? t[j].y : w[j].y;
    }
  }
}

// shared offset of cell slot s in the dense (bulk-staged) layout: the small
// skew keeps the 16-byte row accesses of a quarter-warp that straddles two
// cells in distinct bank groups (fits: 8 cells + 8 doubles <= tensor size)
template <int NEc>
__host__ __device__ constexpr int dense_off(int s) {
  return s * NEc + 4 * ((s + 2) >> 2);
}

template <int D, int G>
__host__ __device__ constexpr bool fdm_interleave() {
  return D == 3 && G > 1 && 16 % G == 0;
}

// doubles between the G subdomain tensors of a CTA: == 16/G (mod 16) when
// the fused pass interleaves the subdomains, so that its 16 threads of a
// half-warp (16/G fibers x G subdomains) hit 16 distinct 8-byte banks
template <int D, int M, int G>
__host__ __device__ constexpr int fdm_gstride() {
  constexpr int SZ = Lay<D, M>::SZ;
  if (!fdm_interleave<D, G>()) return SZ;
  return SZ + ((16 / G - SZ % 16) % 16 + 16) % 16;
}

// one group of G subdomains (work items grp*G .. grp*G+G-1); all G*F threads
// of the CTA take part; `sm` holds G*fdm_gstride doubles.  `coherent` reads r and x
// through L2 only (ld.cg) for use inside a kernel where other CTAs write them.
template <int D, int M, bool PATCH, int G, bool BULK = false>
__device__ __forceinline__ void fdm_group(const Fdm2Params<D, M>& p, const int32_t* list,
                                          int packed, int64_t start, int64_t count, int64_t grp,
                                          double* sm, bool coherent, int delta = -1) {
  using L = Lay<D, M>;
  using R = Rows<D, M, PATCH>;
  constexpr int N = R::N;
  constexpr int NEc = (D == 3) ? N * N * N : N * N;
  constexpr int F = L::F;
  constexpr int NT = G * F;
  __shared__ int s_info[G][8];            // digit[3], cls, active
  __shared__ int64_t s_cell[G][R::SLOTS];  // dof offset of each cell of the subdomain
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  if constexpr (BULK) {
    // prologue of the bulk path: the lanes of warp 0 take one (subdomain,
    // cell) each, compute its offset and issue its copy at once; one CTA
    // barrier.  (ncu r02, cfg 5: a quarter of the stall samples sat in the
    // old prologue -- subdomain info by G threads, a barrier, the copies, a
    // second barrier -- before the copies' own latency.)
    if (tid < 32) {
      if (tid == 0) {
        mbar_init(&s_bar, 1);
        const int64_t left = count - grp * G;
        const int nact = left < G ? (int)left : G;
        mbar_expect_tx(&s_bar, (unsigned)(nact * R::SLOTS * NEc * 8));
      }
      __syncwarp();
      for (int l = tid; l < G * R::SLOTS; l += 32) {
        const int gg = l / R::SLOTS, sl = l - gg * R::SLOTS;
        const int64_t idx = grp * G + gg;
        const bool act = idx < count;
        int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
        if (act) subdomain_info<D, PATCH>(p.geo, list ? list[idx] : (int)(start + idx), packed != 0,
                                          digit, base);
        if (sl == 0) {
          int* inf = s_info[gg];
          int cls = 0;
#pragma unroll
          for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
#pragma unroll
          for (int t = 0; t < 3; ++t) inf[t] = digit[t];
          inf[6] = cls;
          inf[7] = act;
        }
        int c[3] = {base[0] + (sl & 1), base[1] + ((sl >> 1) & 1), base[2] + ((sl >> 2) & 1)};
        if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
        const int64_t off = act ? (int64_t)cell_local<D>(p.geo, c) * NEc : 0;
        s_cell[gg][sl] = off;
        if (act) bulk_load(sm + gg * fdm_gstride<D, M, G>() + dense_off<NEc>(sl), p.r + off, NEc * 8, &s_bar);
      }
    }
  } else if (tid < G) {
    const int64_t idx = grp * G + tid;
    int* inf = s_info[tid];
    inf[7] = idx < count;
    int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
    if (inf[7]) {
      int id = list ? list[idx] : (int)(start + idx);
      if (PATCH && delta >= 0) {
        // cluster mode: list holds packed base vertices of 2^d-patch clusters
        int v[3];
        unpack_d<D>(id, v);
        bool ok = true;
#pragma unroll
        for (int t = 0; t < D; ++t) {
          v[t] += (delta >> t) & 1;
          ok = ok && v[t] >= 1 && v[t] <= p.geo.nc[t] - 1;
        }
        ok = ok && v[D - 1] >= p.pv_lo && v[D - 1] <= p.pv_hi;
        inf[7] = ok;
        id = pack_d(D, v[0], v[1], D == 3 ? v[2] : 0);
      }
      if (inf[7]) subdomain_info<D, PATCH>(p.geo, id, packed != 0, digit, base);
    }
    int cls = 0;
#pragma unroll
    for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
#pragma unroll
    for (int t = 0; t < 3; ++t) inf[t] = digit[t];
    inf[6] = cls;
#pragma unroll
    for (int s = 0; s < R::SLOTS; ++s) {
      int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
      if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
      s_cell[tid][s] = inf[7] ? (int64_t)cell_local<D>(p.geo, c) * NEc : 0;
    }
  }
  __syncthreads();
  const int g = tid / F, f = tid - (tid / F) * F;
  const bool active = s_info[g][7];
  const int* dg = s_info[g];
  constexpr int GSZ = fdm_gstride<D, M, G>();
  double* buf = sm + g * GSZ;
  constexpr int H = PATCH ? 2 : 1;  // cell rows per direction-0 fiber
  int slot0 = 0, goff = 0;
  fiber_rows<D, M, PATCH>(f, slot0, goff);
  // bulk mode: the cells of R_j r arrive densely (cell-major) in the tensor
  // buffers by TMA bulk copies, and omega * R_j^T y leaves by bulk fp64
  // reduce-add; the SM's load/store pipe only sees shared memory
  // (caller guarantees: NEc even, not coherent, not atomic, no cluster delta)
  static_assert(!BULK || dense_off<NEc>(R::SLOTS - 1) + NEc <= GSZ, "dense staging fits");
  if constexpr (BULK) {
    mbar_wait(&s_bar, 0);  // the copies issued in the prologue
    double v[M], o[M];
    if (active) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const double* src = buf + dense_off<NEc>(slot0 + h) + goff;
        if constexpr (N % 8 == 0) {
          // rows of 64 / 128 bytes: the quarter-warp's 16-byte accesses start
          // in rotated chunks (distinct bank groups), registers rotated back
          double2 w[N / 2];
          const int rot = row_rot<N>(f);
#pragma unroll
          for (int j = 0; j < N / 2; ++j)
            w[j] = *reinterpret_cast<const double2*>(src + 2 * ((j + rot) & (N / 2 - 1)));
          rotate_chunks<N / 2>(w, (N / 2 - rot) & (N / 2 - 1));
#pragma unroll
          for (int j = 0; j < N / 2; ++j) {
            v[h * N + 2 * j] = w[j].x;
            v[h * N + 2 * j + 1] = w[j].y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            const double2 t = *reinterpret_cast<const double2*>(src + i);
            v[h * N + i] = t.x;
            v[h * N + i + 1] = t.y;
          }
        }
      }
      fdm_matvec<M, true>(p.mats, p.eo, dg[0], v, o);
    }
    __syncthreads();  // all dense rows read before the padded tensor overwrites them
    if (active) {
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) buf[sb + k] = o[k];
    }
    __syncthreads();
  } else if (p.direct) {
    // first forward contraction (direction 0) straight from the global rows of R_j r
    if (active) {
      double v[M], o[M];
#pragma unroll
      for (int h = 0; h < H; ++h) rows_to_reg<N, M>(v, h, p.r + s_cell[g][slot0 + h] + goff, coherent);
      fdm_matvec<M, true>(p.mats, p.eo, dg[0], v, o);
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) buf[sb + k] = o[k];
    }
    __syncthreads();
  } else {
    // gather R_j r, one cell row per thread iteration
    for (int row = tid; row < G * R::RPS; row += NT) {
      const int gg = row / R::RPS;
      if (!s_info[gg][7]) continue;
      int slot, go, soff;
      R::map(row - gg * R::RPS, slot, go, soff);
      if (coherent) row_load_cg<N>(sm + gg * GSZ + soff, p.r + s_cell[gg][slot] + go);
      else row_load<N>(sm + gg * GSZ + soff, p.r + s_cell[gg][slot] + go);
    }
    __syncthreads();
    if (active) fdm_fiber<M, true>(p.mats, p.eo, dg[0], buf, L::sbase(0, f), L::sstride(0));
    __syncthreads();
  }
  // forward contractions with Z^T, directions 1 .. D-2
#pragma unroll
  for (int t = 1; t < D - 1; ++t) {
    if (active) fdm_fiber<M, true>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
    __syncthreads();
  }
  // fused: Z^T along D-1, scale by 1/Lambda-sum, Z along D-1.  In 3D the
  // threads take the G subdomains interleaved here (with the group stride of
  // fdm_gstride the half-warp accesses of this strided pass are conflict free)
  {
    constexpr bool IL = fdm_interleave<D, G>();
    const int gi = IL ? tid % G : g, fi = IL ? tid / G : f;
    if (s_info[gi][7]) {
      constexpr int t = D - 1;
      const int* dgi = s_info[gi];
      double* bufi = sm + gi * GSZ;
      const int sb = L::sbase(t, fi), ss = L::sstride(t);
      const double* inv = p.invsum + (int64_t)dgi[6] * L::NE + L::gbase(t, fi);
      double v[M], o[M];
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = bufi[sb + k * ss];
      fdm_matvec<M, true>(p.mats, p.eo, dgi[t], v, o);
#pragma unroll
      for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * L::gstride(t));
      fdm_matvec<M, false>(p.mats, p.eo, dgi[t], o, v);
#pragma unroll
      for (int k = 0; k < M; ++k) bufi[sb + k * ss] = v[k];
    }
  }
  __syncthreads();
  // backward contractions with Z, directions D-2 .. 1
#pragma unroll
  for (int s = 0; s < D - 2; ++s) {
    const int t = D - 2 - s;
    if (active) fdm_fiber<M, false>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
    __syncthreads();
  }
  if constexpr (BULK) {
    // last backward contraction (direction 0); omega * y rows written densely
    // over the tensor, then reduce-added into x by the TMA engine
    double v[M], o[M];
    if (active) {
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = buf[sb + k];
      fdm_matvec<M, false>(p.mats, p.eo, dg[0], v, o);
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        double* dst = buf + dense_off<NEc>(slot0 + h) + goff;
        if constexpr (N % 8 == 0) {
          double2 w[N / 2];
#pragma unroll
          for (int j = 0; j < N / 2; ++j)
            w[j] = make_double2(__dmul_rn(p.omega, o[h * N + 2 * j]),
                                __dmul_rn(p.omega, o[h * N + 2 * j + 1]));
          const int rot = row_rot<N>(f);
          rotate_chunks<N / 2>(w, rot);
#pragma unroll
          for (int j = 0; j < N / 2; ++j)
            *reinterpret_cast<double2*>(dst + 2 * ((j + rot) & (N / 2 - 1))) = w[j];
        } else {
#pragma unroll
          for (int i = 0; i < N; i += 2)
            *reinterpret_cast<double2*>(dst + i) =
                make_double2(__dmul_rn(p.omega, o[h * N + i]), __dmul_rn(p.omega, o[h * N + i + 1]));
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < 32) {  // one reduce per lane; each lane waits for its own group
      bool any = false;
      for (int l = tid; l < G * R::SLOTS; l += 32) {
        const int gg = l / R::SLOTS, sl = l - gg * R::SLOTS;
        if (s_info[gg][7]) {
          bulk_red_add(p.x + s_cell[gg][sl], sm + gg * GSZ + dense_off<NEc>(sl), NEc * 8);
          any = true;
        }
      }
      if (any) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    return;
  }
  if (p.direct) {
    // last backward contraction (direction 0) and x += omega R_j^T y from registers
    if (active) {
      double v[M], o[M];
      const int sb = L::sbase(0, f);
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = buf[sb + k];
      fdm_matvec<M, false>(p.mats, p.eo, dg[0], v, o);
#pragma unroll
      for (int h = 0; h < H; ++h)
        reg_update<N, M>(p.x + s_cell[g][slot0 + h] + goff, o, h, p.omega, p.atomic, coherent);
    }
    return;
  }
  if (active) fdm_fiber<M, false>(p.mats, p.eo, dg[0], buf, L::sbase(0, f), L::sstride(0));
  __syncthreads();
  // scatter-add omega * R_j^T y, one cell row per thread iteration
  for (int row = tid; row < G * R::RPS; row += NT) {
    const int gg = row / R::RPS;
    if (!s_info[gg][7]) continue;
    int slot, go, soff;
    R::map(row - gg * R::RPS, slot, go, soff);
    if (p.atomic) row_red<N>(p.x + s_cell[gg][slot] + go, sm + gg * GSZ + soff, p.omega);
    else if (coherent) row_update_cg<N>(p.x + s_cell[gg][slot] + go, sm + gg * GSZ + soff, p.omega);
    else row_update<N>(p.x + s_cell[gg][slot] + go, sm + gg * GSZ + soff, p.omega, false);
  }
}

// bulk variant: register budget of 56 per thread (4 CTAs of 288 threads per SM;
// 5 CTAs would mean 40 registers and ~1 KB of spills per thread at m = 12)
#ifndef FDM_BULK_REGS
#define FDM_BULK_REGS 56
#endif
#ifndef FDM_BULK_REGS_M16
#define FDM_BULK_REGS_M16 80
#endif
// (m >= 14: v[m], o[m] alone are 56-64 registers -- 56 would spill ~350 B per
// thread; 80 gives 3 CTAs of 256 threads without spills)
template <int M>
__host__ __device__ constexpr int fdm2_bulk_regs() {
  return M >= 14 ? FDM_BULK_REGS_M16 : FDM_BULK_REGS;
}
template <int D, int M>
__host__ __device__ constexpr int fdm2_min_ctas(bool bulk) {
  return bulk ? (65536 / (fdm2_groups<D, M>() * Lay<D, M>::F * fdm2_bulk_regs<M>()) > 0
                     ? 65536 / (fdm2_groups<D, M>() * Lay<D, M>::F * fdm2_bulk_regs<M>())
                     : 1)
              : 0;  // 0: no minimum (ptxas default heuristics)
}

template <int D, int M, bool PATCH, bool BULK = false>
__global__ void __launch_bounds__(fdm2_groups<D, M>() * Lay<D, M>::F, fdm2_min_ctas<D, M>(BULK))
fdm2_kernel(const __grid_constant__ Fdm2Params<D, M> p) {
  extern __shared__ __align__(16) double sm[];
  fdm_group<D, M, PATCH, fdm2_groups<D, M>(), BULK>(p, p.list, p.packed, p.start, p.count,
                                                    blockIdx.x, sm, false);
}

// fdm6: persistent variant of fdm2 with staggered starts.  All CTAs of a
// launch have the same work, so in fdm2 every wave gathers, contracts and
// scatters in lock-step and the memory and DFMA phases of co-resident CTAs do
// not overlap.  Here the k-th CTA slot of each SM starts k * stagger_ns late
// and then walks its groups back to back, keeping the phases interleaved.
template <int D, int M, bool PATCH>
__global__ void __launch_bounds__(fdm2_groups<D, M>() * Lay<D, M>::F)
fdm6_kernel(const __grid_constant__ Fdm2Params<D, M> p, int64_t ngroups, int stagger_ns,
            int nsm) {
  extern __shared__ __align__(16) double sm[];
  if (stagger_ns > 0) {
    const int slot = (int)(blockIdx.x / nsm);
    for (int i = 0; i < slot; ++i) __nanosleep(stagger_ns);
  }
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    fdm_group<D, M, PATCH, fdm2_groups<D, M>()>(p, p.list, p.packed, p.start, p.count, grp, sm,
                                                false);
    __syncthreads();
  }
}



// ---------------------------------------------------------------------------
// fdm5: persistent, software-pipelined solves.  Each CTA walks its groups of
// G subdomains; cp.async brings the r rows of the next group into the second
// (padded) tensor buffer and the x rows of the current group into an
// unpadded buffer while the current group is contracted, so neither the
// gather of r nor the load half of the x update is exposed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(double* sdst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

template <int D, int M, bool PATCH>
struct Fdm5Shape {
  using R = Rows<D, M, PATCH>;
  static constexpr int N = R::N;
  static constexpr int NEc = (D == 3) ? N * N * N : N * N;
  static constexpr int G = fdm2_groups<D, M>();
  static constexpr int NT = G * Lay<D, M>::F;
  static constexpr int SZ = Lay<D, M>::SZ;
  static constexpr int XSZ = R::SLOTS * NEc;
  static constexpr int SMEM = 2 * G * SZ + G * XSZ;  // doubles
};

template <int D, int M, bool PATCH>
__global__ void __launch_bounds__(Fdm5Shape<D, M, PATCH>::NT)
fdm5_kernel(const __grid_constant__ Fdm2Params<D, M> p, int64_t ngroups) {
  using L = Lay<D, M>;
  using R = Rows<D, M, PATCH>;
  using S = Fdm5Shape<D, M, PATCH>;
  constexpr int N = S::N, G = S::G, F = L::F, NT = S::NT;
  extern __shared__ __align__(16) double sm[];
  double* Xs = sm + 2 * G * S::SZ;
  __shared__ int s_info[2][G][8];            // digit[3], cls, active
  __shared__ int64_t s_cell[2][G][R::SLOTS];  // dof offset of each cell
  const int tid = threadIdx.x;
  const int g = tid / F, f = tid - (tid / F) * F;

  auto info = [&](int64_t grp, int st) {
    if (tid < G) {
      const int64_t idx = grp * G + tid;
      int* inf = s_info[st][tid];
      inf[7] = idx < p.count;
      int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
      if (inf[7]) {
        const int id = p.list ? p.list[idx] : (int)(p.start + idx);
        subdomain_info<D, PATCH>(p.geo, id, p.packed != 0, digit, base);
      }
      int cls = 0;
#pragma unroll
      for (int t = D - 1; t >= 0; --t) cls = cls * 4 + digit[t];
#pragma unroll
      for (int t = 0; t < 3; ++t) inf[t] = digit[t];
      inf[6] = cls;
#pragma unroll
      for (int s = 0; s < R::SLOTS; ++s) {
        int c[3] = {base[0] + (s & 1), base[1] + ((s >> 1) & 1), base[2] + ((s >> 2) & 1)};
        if (!PATCH) c[0] = base[0], c[1] = base[1], c[2] = base[2];
        s_cell[st][tid][s] = (int64_t)cell_local<D>(p.geo, c) * S::NEc;
      }
    }
  };
  auto issue_r = [&](int st) {
    double* base = sm + st * G * S::SZ;
    for (int row = tid; row < G * R::RPS; row += NT) {
      const int gg = row / R::RPS;
      if (!s_info[st][gg][7]) continue;
      int slot, goff, soff;
      R::map(row - gg * R::RPS, slot, goff, soff);
      const double* src = p.r + s_cell[st][gg][slot] + goff;
      double* dst = base + gg * S::SZ + soff;
#pragma unroll
      for (int i = 0; i < N; ++i) cp_async8(dst + i, src + i);
    }
    cp_async_commit();
  };
  auto issue_x = [&](int st) {
    for (int row = tid; row < G * R::RPS; row += NT) {
      const int gg = row / R::RPS;
      if (!s_info[st][gg][7]) continue;
      const int rr = row - gg * R::RPS;
      const int slot = rr / R::RPC, w = rr - slot * R::RPC;
      const double* src = p.x + s_cell[st][gg][slot] + w * N;
      double* dst = Xs + gg * S::XSZ + slot * S::NEc + w * N;
      if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N; i += 2) cp_async16(dst + i, src + i);
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) cp_async8(dst + i, src + i);
      }
    }
    cp_async_commit();
  };

  int64_t grp = blockIdx.x;
  if (grp >= ngroups) return;
  info(grp, 0);
  __syncthreads();
  issue_r(0);
  for (int st = 0; grp < ngroups; grp += gridDim.x, st ^= 1) {
    issue_x(st);
    const int64_t nxt = grp + gridDim.x;
    const bool more = nxt < ngroups;
    if (more) {
      info(nxt, st ^ 1);
      __syncthreads();
      issue_r(st ^ 1);
      cp_async_wait<2>();  // r of this group landed (x of it and r of the next may fly)
    } else {
      cp_async_wait<1>();
    }
    __syncthreads();
    const int* dg = s_info[st][g];
    const bool active = dg[7];
    double* buf = sm + (st * G + g) * S::SZ;
#pragma unroll
    for (int t = 0; t < D - 1; ++t) {
      if (active) fdm_fiber<M, true>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
      __syncthreads();
    }
    if (active) {
      constexpr int t = D - 1;
      const int sb = L::sbase(t, f), ss = L::sstride(t);
      const double* inv = p.invsum + (int64_t)dg[6] * L::NE + L::gbase(t, f);
      double v[M], o[M];
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = buf[sb + k * ss];
      fdm_matvec<M, true>(p.mats, p.eo, dg[t], v, o);
#pragma unroll
      for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * L::gstride(t));
      fdm_matvec<M, false>(p.mats, p.eo, dg[t], o, v);
#pragma unroll
      for (int k = 0; k < M; ++k) buf[sb + k * ss] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < D - 1; ++s) {
      const int t = D - 2 - s;
      if (active) fdm_fiber<M, false>(p.mats, p.eo, dg[t], buf, L::sbase(t, f), L::sstride(t));
      __syncthreads();
    }
    if (more) cp_async_wait<1>();  // x of this group landed
    else cp_async_wait<0>();
    __syncthreads();
    double* rb = sm + st * G * S::SZ;
    for (int row = tid; row < G * R::RPS; row += NT) {
      const int gg = row / R::RPS;
      if (!s_info[st][gg][7]) continue;
      int slot, goff, soff;
      R::map(row - gg * R::RPS, slot, goff, soff);
      const double* y = rb + gg * S::SZ + soff;
      const double* xs = Xs + gg * S::XSZ + slot * S::NEc + goff;
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = xupd(xs[i], p.omega, y[i]);
      row_store<N>(p.x + s_cell[st][gg][slot] + goff, v);
    }
    __syncthreads();  // X and this stage's buffers are refilled next
  }
}

// Additive patch step over 2^d-patch clusters (vertices {2a+1, 2a+2}^d): one
// group of threads owns a cluster and solves its patches one after another,
// so the cluster's 3^d cells of r and x stay in L1/L2 across the 2^d solves
// (~3^d/8 cell loads per patch instead of 2^d).  Clusters of one launch share
// the parity of a (2^d launches per step): they are 2 cells apart, so their
// writes are disjoint and no atomics are needed.
template <int D, int M>
__global__ void __launch_bounds__(fdm2_groups<D, M>() * Lay<D, M>::F)
cluster_kernel(const __grid_constant__ Fdm2Params<D, M> p) {
  extern __shared__ __align__(16) double sm[];
#pragma unroll 1
  for (int delta = 0; delta < (1 << D); ++delta) {
    fdm_group<D, M, true, fdm2_groups<D, M>()>(p, p.list, 1, 0, p.count, blockIdx.x, sm, false,
                                               delta);
    __syncthreads();  // the next patch of each cluster overlaps this one
  }
}

template <int D, int M>
__host__ __device__ constexpr int fdm2_smem_doubles() {
  return fdm2_groups<D, M>() * fdm_gstride<D, M, fdm2_groups<D, M>()>();
}

}  // namespace dgb
