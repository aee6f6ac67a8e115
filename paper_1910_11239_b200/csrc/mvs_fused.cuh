// mvs_fused.cuh - one colour of the multiplicative vertex-patch sweep in one
// launch: restricted residual and patch solve fused per patch.
//
// LevelSmoother.smooth_multiplicative (smoothers.py:157-166): for each colour,
// r = b - A x, then x += omega R_j^T A_j^-1 R_j r for the colour's patches.
// Patches of one structured colour share neither a cell nor a face
// (mesh.py:360-375), so everything a patch's residual reads -- its 8 cells
// and their face neighbours -- is written by no other patch of the launch:
// a CTA can form R_j r itself, solve, and update x in place.  Against the
// two-launch form (res3 on the colour's cells, then fdm2 on its patches) r
// never goes to memory (2 x 8 B per patch dof less DRAM / L2 traffic per
// colour, x of the patch read once more from L1/L2 instead of DRAM), a sweep
// is 16 launches instead of 32, and the two kernels' tail waves merge.
//
// CTA = one patch, M^2 = 4 n^2 threads.  The residual runs the three passes
// of res3 (same device functions, bitwise the same r) on 4 cells at a time
// (slots 0-3 = lower half of the patch tensor, then slots 4-7), each thread
// a fiber of one cell; r lands in the padded (2n)^3 patch tensor in shared
// memory, whose upper half aliases the residual's scratch.  The solve is
// fdm2's sequence (2d-1 in-place passes, the last one writing
// x += omega y straight to the cell rows), one fiber per thread.
//
// Measured (r02, cfg 3: 3D Q7, 32^3 cells, 16 colours; results bitwise equal
// to the two-launch sweep): 2.272 ms per sweep with three CTAs per SM (76
// registers, 72.7 KB of shared memory), 2.405 ms with two, against 2.046 ms
// for res3 + fdm2: the CTA walks residual round 0, round 1 and the solve one
// after the other behind ten barriers, and the saved traffic (the sweep is
// not DRAM-bound: 42% of HBM in the residual) does not pay for that.  Opt-in
// (DGB_MVS_FUSED=1) in DGB_EXPERIMENTAL builds.
#pragma once
#include "res3.cuh"

namespace dgb {

template <int N>
struct MvsShape {
  static constexpr int M = 2 * N;
  using LM = Lay<3, M>;
  using S3 = Res3Shape<N>;
  static constexpr int NT = M * M;                       // = 4 cells x N^2 fibers
  static constexpr int HALF = LM::P * M * N;             // planes j2 < N of the patch tensor
  static constexpr int SCR = 4 * S3::CS;                 // residual scratch of 4 cells
  static constexpr int SMEM = HALF + (SCR > HALF ? SCR : HALF);  // doubles
};

template <int N>
struct MvsParams {
  Res2Params<3, N> res;     // x, b, geo, residual tables (list / r unused)
  FdmMats<2 * N> fm;        // patch eigenvectors per digit
  double* x;                // updated in place
  const int32_t* patches;   // packed vertex coordinates of the colour
  int64_t count;
  const double* invsum;
  double omega;
  int eo;
};

template <int N, int MINB>
__global__ void __launch_bounds__(MvsShape<N>::NT, MINB)
mvs_fused_kernel(const __grid_constant__ MvsParams<N> P) {
  using SH = MvsShape<N>;
  using S3 = Res3Shape<N>;
  using L = Lay<3, N>;
  using LM = typename SH::LM;
  constexpr int M = SH::M, F = N * N, NE = L::NE;
  extern __shared__ __align__(16) double sm[];
  double* T = sm;                    // patch tensor; planes >= N alias the scratch
  double* scr = sm + SH::HALF;
  __shared__ int s_dig[3], s_base[3];
  const int tid = threadIdx.x;
  const Res2Params<3, N>& p = P.res;
  if (tid == 0) {
    int digit[3], base[3];
    subdomain_info<3, true>(p.geo, P.patches[blockIdx.x], true, digit, base);
#pragma unroll
    for (int t = 0; t < 3; ++t) s_dig[t] = digit[t], s_base[t] = base[t];
  }
  __syncthreads();
  const int g = tid / F, f = tid - g * F;   // cell of the round, fiber
  const int fa = f % N, fb = f / N;
  double* A = scr + g * S3::CS;
  double* B = A + L::SZ;
  double* F1 = B + L::SZ;
  double* F2 = F1 + 4 * S3::FP;
  // r of cell `slot` at (i0, i1, i2) = (fa, fb, k) is patch entry
  // (s0 n + fa, s1 n + fb, s2 n + k)
  auto cell_of = [&](int slot, int (&c)[3], int (&dig)[3]) -> int64_t {
    c[0] = s_base[0] + (slot & 1);
    c[1] = s_base[1] + ((slot >> 1) & 1);
    c[2] = s_base[2] + (slot >> 2);
#pragma unroll
    for (int t = 0; t < 3; ++t) dig[t] = (c[t] == 0 ? 1 : 0) | (c[t] == p.geo.nc[t] - 1 ? 2 : 0);
    return (int64_t)cell_local<3>(p.geo, c) * NE;
  };
  {
    // round 0: slots 0-3, the lower half of the patch tensor (not aliased):
    // the last pass writes r straight into it
    int c[3], dig[3];
    const int64_t cb = cell_of(g, c, dig);
    res3_pass0<N>(p, true, f, fa, fb, c, dig, cb, A, B, F1, F2);
    __syncthreads();
    double* dst = T + ((g & 1) * N + fa) + LM::P * (((g >> 1) & 1) * N + fb);
    res3_tail_to<N>(p, true, f, fa, fb, dig, cb, A, B, F1, F2,
                    [&](int k, double v) { dst[LM::P * M * k] = v; });
    __syncthreads();  // the scratch is rewritten by round 1
  }
  {
    // round 1: slots 4-7; their half of the tensor overlays the scratch, so r
    // waits in registers until every thread is done reading it
    int c[3], dig[3];
    const int64_t cb = cell_of(4 + g, c, dig);
    res3_pass0<N>(p, true, f, fa, fb, c, dig, cb, A, B, F1, F2);
    __syncthreads();
    double rr[N];
    res3_tail_to<N>(p, true, f, fa, fb, dig, cb, A, B, F1, F2,
                    [&](int k, double v) { rr[k] = v; });
    __syncthreads();
    double* dst = T + ((g & 1) * N + fa) + LM::P * (((g >> 1) & 1) * N + fb) + LM::P * M * N;
#pragma unroll
    for (int k = 0; k < N; ++k) dst[LM::P * M * k] = rr[k];
    __syncthreads();
  }
  // ---- patch solve on T (fdm2's pass sequence), one fiber per thread
  const int cls = (s_dig[2] * 4 + s_dig[1]) * 4 + s_dig[0];
  fdm_fiber<M, true>(P.fm, P.eo, s_dig[0], T, LM::sbase(0, tid), LM::sstride(0));
  __syncthreads();
  fdm_fiber<M, true>(P.fm, P.eo, s_dig[1], T, LM::sbase(1, tid), LM::sstride(1));
  __syncthreads();
  {
    const int sb = LM::sbase(2, tid), ss = LM::sstride(2);
    const double* inv = P.invsum + (int64_t)cls * LM::NE + LM::gbase(2, tid);
    double v[M], o[M];
#pragma unroll
    for (int k = 0; k < M; ++k) v[k] = T[sb + k * ss];
    fdm_matvec<M, true>(P.fm, P.eo, s_dig[2], v, o);
#pragma unroll
    for (int k = 0; k < M; ++k) o[k] *= __ldg(inv + k * LM::gstride(2));
    fdm_matvec<M, false>(P.fm, P.eo, s_dig[2], o, v);
#pragma unroll
    for (int k = 0; k < M; ++k) T[sb + k * ss] = v[k];
  }
  __syncthreads();
  fdm_fiber<M, false>(P.fm, P.eo, s_dig[1], T, LM::sbase(1, tid), LM::sstride(1));
  __syncthreads();
  {
    // last backward contraction (direction 0) and x += omega R_j^T y, row by row
    double v[M], o[M];
    const int sb = LM::sbase(0, tid);
#pragma unroll
    for (int k = 0; k < M; ++k) v[k] = T[sb + k];
    fdm_matvec<M, false>(P.fm, P.eo, s_dig[0], v, o);
    int slot0, goff;
    fiber_rows<3, M, true>(tid, slot0, goff);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int slot = slot0 + hh;
      int c[3] = {s_base[0] + (slot & 1), s_base[1] + ((slot >> 1) & 1), s_base[2] + (slot >> 2)};
      reg_update<N, M>(P.x + (int64_t)cell_local<3>(p.geo, c) * NE + goff, o, hh, P.omega, 0, false);
    }
  }
}

}  // namespace dgb
