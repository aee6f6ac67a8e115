// fdm7.cuh - bulk vertex-patch solve with two fibers per thread.
//
// Same algorithm, data movement and arithmetic as fdm2_kernel<3, M, patch,
// bulk> (fdm2.cuh): TMA bulk copies of the 8 cells of R_j r into the dense
// staging, 2d-1 contraction passes in place, omega * y written densely and
// reduce-added into x by the TMA engine.  The difference is the thread map:
// a thread owns fibers h and h + M^2/2 of its patch in every pass, so each
// LDCU.128 of the (patch-uniform) 1D matrix feeds four DFMAs instead of two
// and the index arithmetic is shared.  ncu of fdm2 at cfg 5 (profiles/r02):
// LDCU is 19% and integer / control another ~15% of the issued instructions
// next to 45% fp64.  CTA = G patches x M^2/2 threads.
//
// Measured (r02, cfg 5, bitwise-equal results): 2.43 ms with a 96-register
// cap (two CTAs of 288 threads per SM: the register file is per scheduler, 5
// warps x 32 x 96 is what fits; ~600 B of spills) and 4.24 ms at 110-118
// registers (one CTA per SM) against 1.79 ms for fdm2 at 36 warps per SM:
// the solve's throughput follows the number of resident warps, not the
// per-thread instruction count (ncu: profiles/r02/ncu_cfg5_fdm7_two_fibers_
// variant_summary.txt, 8 warps per SM, issue 28%, fp64 pipe 25%).  Kept
// opt-in (DGB_FDM7=1 / 2, DGB_EXPERIMENTAL builds).
#pragma once
#include "fdm2.cuh"

namespace dgb {

template <int M>
struct Fdm7Shape {
  static constexpr int G = 4;                 // patches per CTA
  static constexpr int TPP = M * M / 2;       // threads per patch
  static constexpr int NT = G * TPP;
  static constexpr int GSZ = fdm_gstride<3, M, G>();
  static constexpr int SMEM = G * GSZ;        // doubles
};

// two products with the same matrix: the constant loads are shared
template <int M, bool FWD>
__device__ __forceinline__ void fdm_matvec2(const FdmMats<M>& m, int eo, int digit,
                                            const double (&v0)[M], double (&o0)[M],
                                            const double (&v1)[M], double (&o1)[M]) {
  if (eo && digit == 0) {
    if (FWD) {
      matvec_eo_fwd<M>(m.eo[0], m.eo[1], v0, o0);
      matvec_eo_fwd<M>(m.eo[0], m.eo[1], v1, o1);
    } else {
      matvec_eo_bwd<M>(m.eo[2], m.eo[3], v0, o0);
      matvec_eo_bwd<M>(m.eo[2], m.eo[3], v1, o1);
    }
    return;
  }
  // boundary digits: the per-fiber products of fdm2 (a merged switch over
  // both products compiles to register-indexed constant loads, LDC per DFMA)
  matvec_digit<M>(FWD ? m.fwd : m.bwd, digit, v0, o0);
  matvec_digit<M>(FWD ? m.fwd : m.bwd, digit, v1, o1);
}

// MAXR: register cap (112 = two CTAs of 288 threads per SM)
template <int M, int MAXR>
__global__ void __launch_bounds__(Fdm7Shape<M>::NT) __maxnreg__(MAXR)
fdm7_kernel(const __grid_constant__ Fdm2Params<3, M> p) {
  constexpr int D = 3;
  using L = Lay<D, M>;
  using R = Rows<D, M, true>;
  using S = Fdm7Shape<M>;
  constexpr int N = M / 2, NEc = N * N * N;
  constexpr int G = S::G, TPP = S::TPP, NT = S::NT, GSZ = S::GSZ;
  static_assert(N % 2 == 0 && N % 8 != 0, "dense rows read with plain 16-byte accesses");
  static_assert(dense_off<NEc>(R::SLOTS - 1) + NEc <= GSZ, "dense staging fits");
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_info[G][8];
  __shared__ int64_t s_cell[G][R::SLOTS];
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  const int64_t grp = blockIdx.x;
  if (tid < 32) {
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      const int64_t left = p.count - grp * G;
      const int nact = left < G ? (int)left : G;
      mbar_expect_tx(&s_bar, (unsigned)(nact * R::SLOTS * NEc * 8));
    }
    __syncwarp();
    for (int l = tid; l < G * R::SLOTS; l += 32) {
      const int gg = l / R::SLOTS, sl = l - gg * R::SLOTS;
      const int64_t idx = grp * G + gg;
      const bool act = idx < p.count;
      int digit[3] = {0, 0, 0}, base[3] = {0, 0, 0};
      if (act) subdomain_info<D, true>(p.geo, p.list ? p.list[idx] : (int)(p.start + idx),
                                       p.packed != 0, digit, base);
      if (sl == 0) {
        int* inf = s_info[gg];
        inf[0] = digit[0], inf[1] = digit[1], inf[2] = digit[2];
        inf[6] = (digit[2] * 4 + digit[1]) * 4 + digit[0];
        inf[7] = act;
      }
      int c[3] = {base[0] + (sl & 1), base[1] + ((sl >> 1) & 1), base[2] + ((sl >> 2) & 1)};
      const int64_t off = act ? (int64_t)cell_local<D>(p.geo, c) * NEc : 0;
      s_cell[gg][sl] = off;
      if (act) bulk_load(sm + gg * GSZ + dense_off<NEc>(sl), p.r + off, NEc * 8, &s_bar);
    }
  }
  __syncthreads();
  const int g = tid / TPP, h = tid - g * TPP;
  const int f0 = h, f1 = h + TPP;
  const bool active = s_info[g][7];
  const int* dg = s_info[g];
  double* buf = sm + g * GSZ;
  double va[M], oa[M], vb[M], ob[M];
  // ---- direction 0 forward, straight from the dense staging
  mbar_wait(&s_bar, 0);
  if (active) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      int slot0, goff;
      fiber_rows<D, M, true>(q ? f1 : f0, slot0, goff);
      double (&v)[M] = q ? vb : va;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const double* src = buf + dense_off<NEc>(slot0 + hh) + goff;
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          const double2 t = *reinterpret_cast<const double2*>(src + i);
          v[hh * N + i] = t.x;
          v[hh * N + i + 1] = t.y;
        }
      }
    }
    fdm_matvec2<M, true>(p.mats, p.eo, dg[0], va, oa, vb, ob);
  }
  __syncthreads();  // all dense rows read before the padded tensor overwrites them
  if (active) {
    const int sa = L::sbase(0, f0), sb = L::sbase(0, f1);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      buf[sa + k] = oa[k];
      buf[sb + k] = ob[k];
    }
  }
  __syncthreads();
  // ---- direction 1 forward
  if (active) {
    const int sa = L::sbase(1, f0), sb = L::sbase(1, f1), ss = L::sstride(1);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      va[k] = buf[sa + k * ss];
      vb[k] = buf[sb + k * ss];
    }
    fdm_matvec2<M, true>(p.mats, p.eo, dg[1], va, oa, vb, ob);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      buf[sa + k * ss] = oa[k];
      buf[sb + k * ss] = ob[k];
    }
  }
  __syncthreads();
  // ---- direction 2: forward, 1/Lambda, backward; the G patches interleaved
  {
    const int gi = tid % G;                    // NT % G == 0: both fibers in patch gi
    const int fa = tid / G, fb = (tid + NT) / G;
    if (s_info[gi][7]) {
      const int* dgi = s_info[gi];
      double* bufi = sm + gi * GSZ;
      const int sa = L::sbase(2, fa), sb = L::sbase(2, fb), ss = L::sstride(2);
      const double* inv = p.invsum + (int64_t)dgi[6] * L::NE;
      const int ga = L::gbase(2, fa), gb = L::gbase(2, fb);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        va[k] = bufi[sa + k * ss];
        vb[k] = bufi[sb + k * ss];
      }
      fdm_matvec2<M, true>(p.mats, p.eo, dgi[2], va, oa, vb, ob);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        oa[k] *= __ldg(inv + ga + k * L::gstride(2));
        ob[k] *= __ldg(inv + gb + k * L::gstride(2));
      }
      fdm_matvec2<M, false>(p.mats, p.eo, dgi[2], oa, va, ob, vb);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        bufi[sa + k * ss] = va[k];
        bufi[sb + k * ss] = vb[k];
      }
    }
  }
  __syncthreads();
  // ---- direction 1 backward
  if (active) {
    const int sa = L::sbase(1, f0), sb = L::sbase(1, f1), ss = L::sstride(1);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      va[k] = buf[sa + k * ss];
      vb[k] = buf[sb + k * ss];
    }
    fdm_matvec2<M, false>(p.mats, p.eo, dg[1], va, oa, vb, ob);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      buf[sa + k * ss] = oa[k];
      buf[sb + k * ss] = ob[k];
    }
  }
  __syncthreads();
  // ---- direction 0 backward; omega * y densely over the tensor, bulk reduce-add
  if (active) {
    const int sa = L::sbase(0, f0), sb = L::sbase(0, f1);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      va[k] = buf[sa + k];
      vb[k] = buf[sb + k];
    }
    fdm_matvec2<M, false>(p.mats, p.eo, dg[0], va, oa, vb, ob);
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      int slot0, goff;
      fiber_rows<D, M, true>(q ? f1 : f0, slot0, goff);
      const double (&o)[M] = q ? ob : oa;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        double* dst = buf + dense_off<NEc>(slot0 + hh) + goff;
#pragma unroll
        for (int i = 0; i < N; i += 2)
          *reinterpret_cast<double2*>(dst + i) = make_double2(
              __dmul_rn(p.omega, o[hh * N + i]), __dmul_rn(p.omega, o[hh * N + i + 1]));
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
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
}

}  // namespace dgb
