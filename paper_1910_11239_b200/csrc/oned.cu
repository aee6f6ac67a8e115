// oned.cu - one-dimensional levels (mesh.py:144; fastdiag.py:245,284).
//
// The reference's operator, cell solvers and vertex-patch solvers are
// dimension independent; in 1D a cell holds n <= 16 and a patch 2n <= 32
// unknowns, the operator is the block-tridiagonal A_g itself
// (A_diag(digit) on the diagonal, the rank-2 coupling a_pm off it,
// polybasis.py:247-284) and a local solve is Z diag(1/lambda) Z^T.  These
// levels are tiny, so one thread owns one cell or one patch and reads the
// level's tables from global memory; the host dispatchers
// (dispatch_residual / dispatch_cell_fdm / dispatch_patch_fdm) route d = 1
// here, so every entry point of the C ABI works unchanged.
#include "launch.h"
#include "fdm2.cuh"

namespace dgb {

struct OneDParams {
  const double* x;
  const double* b;  // residual: nullptr -> v = A x;  solves: unused
  double* r;        // residual output, or the solves' right-hand side
  double* xo;       // solves: x += omega A_j^-1 R_j r
  const int32_t* list;
  int64_t start, count;
  int packed, atomic, n;
  int nc, zb;       // global cells, first stored cell
  double alpha, beta, betap, omega;
  const double *adiag, *bg;    // [digit][i*n+k], [2][n]
  const double *z, *zt, *inv;  // [digit][k*m+i], [digit][k*m+i], [digit][m]
};

constexpr int kOneMax = 32;

__global__ void oned_residual_kernel(const OneDParams p) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= p.count) return;
  const int n = p.n;
  // packed entries are global cell coordinates, plain ones local ids
  const int c = p.list ? (p.packed ? p.list[idx] : p.list[idx] + p.zb) : (int)(p.start + idx) + p.zb;
  const int digit = (c == 0 ? 1 : 0) | (c == p.nc - 1 ? 2 : 0);
  const double* xc = p.x + (int64_t)(c - p.zb) * n;
  const double* A = p.adiag + digit * n * n;
  const double *bg0 = p.bg, *bg1 = p.bg + n;
  double o[16];
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = fma(A[i * n + k], xc[k], s);
    o[i] = s;
  }
  if (!(digit & 2)) {  // a_pm x_R
    const double* xr = xc + n;
    double g = 0.0;
    for (int k = 0; k < n; ++k) g = fma(bg0[k], xr[k], g);
    const double r_all = p.betap * xr[0], r_hi = p.alpha * xr[0] + p.beta * g;
    for (int i = 0; i < n; ++i) o[i] = fma(bg1[i], r_all, o[i]);
    o[n - 1] += r_hi;
  }
  if (!(digit & 1)) {  // a_pm^T x_L
    const double* xl = xc - n;
    double g = 0.0;
    for (int k = 0; k < n; ++k) g = fma(bg1[k], xl[k], g);
    const double l_all = p.beta * xl[n - 1], l_lo = p.alpha * xl[n - 1] + p.betap * g;
    for (int i = 0; i < n; ++i) o[i] = fma(bg0[i], l_all, o[i]);
    o[0] += l_lo;
  }
  double* rc = p.r + (int64_t)(c - p.zb) * n;
  const double* bc = p.b ? p.b + (int64_t)(c - p.zb) * n : nullptr;
  for (int i = 0; i < n; ++i) rc[i] = bc ? bc[i] - o[i] : o[i];
}

// cells (m = n) and vertex patches (m = 2n: cells v-1 and v are contiguous)
template <bool PATCH>
__global__ void oned_fdm_kernel(const OneDParams p) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= p.count) return;
  const int n = p.n, m = PATCH ? 2 * n : n;
  int c, digit;
  if (PATCH) {
    // packed entries are vertex coordinates, plain ones global patch ids
    const int e = p.list ? p.list[idx] : (int)(p.start + idx);
    const int v = p.packed ? e : e + 1;
    c = v - 1;
    digit = (v == 1 ? 1 : 0) | (v == p.nc - 1 ? 2 : 0);
  } else {
    c = p.list ? (p.packed ? p.list[idx] : p.list[idx] + p.zb) : (int)(p.start + idx) + p.zb;
    digit = (c == 0 ? 1 : 0) | (c == p.nc - 1 ? 2 : 0);
  }
  const double* rv = p.r + (int64_t)(c - p.zb) * n;
  double* xv = p.xo + (int64_t)(c - p.zb) * n;
  const double* Z = p.z + digit * m * m;
  const double* Zt = p.zt + digit * m * m;
  const double* inv = p.inv + digit * m;
  double y[kOneMax];
  for (int i = 0; i < m; ++i) {  // y = diag(1/lambda) Z^T r
    double s = 0.0;
    for (int k = 0; k < m; ++k) s = fma(Z[k * m + i], rv[k], s);
    y[i] = s * inv[i];
  }
  for (int i = 0; i < m; ++i) {  // x += omega Z y
    double s = 0.0;
    for (int k = 0; k < m; ++k) s = fma(Zt[k * m + i], y[k], s);
    if (p.atomic) atomicAdd(xv + i, p.omega * s);
    else xv[i] = xupd(xv[i], p.omega, s);
  }
}

static OneDParams oned_common(const Geo& geo, int n) {
  OneDParams p{};
  p.n = n;
  p.nc = geo.nc[0];
  p.zb = geo.zb;
  return p;
}

int oned_residual(int n, const ResArgs& q, const OneDTables& t, cudaStream_t st) {
  if (q.count <= 0) return DG_OK;
  OneDParams p = oned_common(q.geo, n);
  p.x = q.x;
  p.b = q.b;
  p.r = q.r;
  p.list = q.list;
  p.start = q.start;
  p.count = q.count;
  p.packed = q.packed;
  p.alpha = q.alpha;
  p.beta = q.beta;
  p.betap = q.betap;
  p.adiag = t.adiag;
  p.bg = t.bg;
  oned_residual_kernel<<<(unsigned)((q.count + 127) / 128), 128, 0, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int oned_fdm(int n, bool patch, const FdmArgs& q, cudaStream_t st) {
  if (q.count <= 0) return DG_OK;
  if (!q.zd || !q.ztd || !q.invsum) return fail(DG_EINVAL, "1D solve: device tables missing");
  OneDParams p = oned_common(q.geo, n);
  p.r = const_cast<double*>(q.r);
  p.xo = q.x;
  p.list = q.list;
  p.start = q.start;
  p.count = q.count;
  p.packed = q.packed;
  p.atomic = q.atomic;
  p.omega = q.omega;
  p.z = q.zd;
  p.zt = q.ztd;
  p.inv = q.invsum;
  const unsigned grid = (unsigned)((q.count + 127) / 128);
  if (patch) oned_fdm_kernel<true><<<grid, 128, 0, st>>>(p);
  else oned_fdm_kernel<false><<<grid, 128, 0, st>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

}  // namespace dgb
