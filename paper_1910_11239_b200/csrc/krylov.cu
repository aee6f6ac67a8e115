// krylov.cu - fused vector kernels of the device-resident preconditioned CG
// (reference: dgmg.krylov.pcg, krylov.py:69-123).
//
//   dg_cg_update: x += a p; r -= a Ap; |r|^2        (krylov.py:103-107)
//   dg_xpby:      p = z + beta p                    (krylov.py:119-120)
//   dg_dot:       a . b                             (krylov.py:92, 101, 114)
//
// HBM-bound streaming kernels: 16-byte loads, a fixed grid of 4 CTAs per SM,
// fp64 partial sums per CTA reduced by a second one-CTA launch in a fixed
// order, so every dot product is deterministic run to run.
#include "launch.h"

namespace dgb {

constexpr int KT = 256;     // threads per CTA
constexpr int KMAXG = 1024; // partial-sum slots

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[KT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  v = 0.0;
  if (w == 0) {
    v = lane < KT / 32 ? ws[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

__global__ void __launch_bounds__(KT) dot_kernel(const double* __restrict__ a,
                                                 const double* __restrict__ b, int64_t n,
                                                 int vec, double* __restrict__ part) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * KT;
  if (vec) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n / 2; i += stride) {
      const double2 u = a2[i], v = b2[i];
      s = fma(u.x, v.x, s);
      s = fma(u.y, v.y, s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s = fma(a[n - 1], b[n - 1], s);
  } else {
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += stride)
      s = fma(a[i], b[i], s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(KT) cg_update_kernel(double* __restrict__ x,
                                                       double* __restrict__ r,
                                                       const double* __restrict__ p,
                                                       const double* __restrict__ ap, double a,
                                                       int64_t n, int vec,
                                                       double* __restrict__ part) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * KT;
  if (vec) {
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(ap);
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n / 2; i += stride) {
      double2 xv = x2[i], rv = r2[i];
      const double2 pv = p2[i], qv = q2[i];
      xv.x = fma(a, pv.x, xv.x);
      xv.y = fma(a, pv.y, xv.y);
      rv.x = fma(-a, qv.x, rv.x);
      rv.y = fma(-a, qv.y, rv.y);
      x2[i] = xv;
      r2[i] = rv;
      s = fma(rv.x, rv.x, s);
      s = fma(rv.y, rv.y, s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
      const int64_t i = n - 1;
      x[i] = fma(a, p[i], x[i]);
      r[i] = fma(-a, ap[i], r[i]);
      s = fma(r[i], r[i], s);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += stride) {
      x[i] = fma(a, p[i], x[i]);
      const double rv = fma(-a, ap[i], r[i]);
      r[i] = rv;
      s = fma(rv, rv, s);
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(KT) finish_kernel(const double* __restrict__ part, int np,
                                                    double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += KT) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(KT) xpby_kernel(const double* __restrict__ z, double beta,
                                                  double* __restrict__ p, int64_t n, int vec) {
  const int64_t stride = (int64_t)gridDim.x * KT;
  if (vec) {
    const double2* z2 = reinterpret_cast<const double2*>(z);
    double2* p2 = reinterpret_cast<double2*>(p);
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n / 2; i += stride) {
      double2 pv = p2[i];
      const double2 zv = z2[i];
      pv.x = fma(beta, pv.x, zv.x);
      pv.y = fma(beta, pv.y, zv.y);
      p2[i] = pv;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) p[n - 1] = fma(beta, p[n - 1], z[n - 1]);
  } else {
    for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += stride)
      p[i] = fma(beta, p[i], z[i]);
  }
}

static int grid_for(int64_t n) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  const int64_t want = (n / 2 + KT - 1) / KT;
  int64_t g = std::min<int64_t>(4 * (int64_t)sms, want);
  g = std::min<int64_t>(g, KMAXG);
  return (int)std::max<int64_t>(1, g);
}

static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace dgb

extern "C" {

int dg_dot(const double* a, const double* b, int64_t n, double* part, double* out,
           void* stream) {
  using namespace dgb;
  if (!a || !b || !part || !out || n < 0) return fail(DG_EINVAL, "dg_dot: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n);
  dot_kernel<<<g, KT, 0, st>>>(a, b, n, al16(a) && al16(b), part);
  finish_kernel<<<1, KT, 0, st>>>(part, g, out);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dg_cg_update(double* x, double* r, const double* p, const double* ap, double alpha,
                 int64_t n, double* part, double* out, void* stream) {
  using namespace dgb;
  if (!x || !r || !p || !ap || !part || !out || n < 0)
    return fail(DG_EINVAL, "dg_cg_update: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n);
  const int vec = al16(x) && al16(r) && al16(p) && al16(ap);
  cg_update_kernel<<<g, KT, 0, st>>>(x, r, p, ap, alpha, n, vec, part);
  finish_kernel<<<1, KT, 0, st>>>(part, g, out);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dg_xpby(const double* z, double beta, double* p, int64_t n, void* stream) {
  using namespace dgb;
  if (!z || !p || n < 0) return fail(DG_EINVAL, "dg_xpby: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  xpby_kernel<<<grid_for(n), KT, 0, st>>>(z, beta, p, n, al16(z) && al16(p));
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

}  // extern "C"
