// coarse.cu - setup-side tensor kernels: the exact coarse solve on Cartesian
// levels and the sum-factorised load-vector contractions.
//
// Coarse solve (CoarseSolver "direct", multigrid.py:148-195): on a uniform
// Cartesian level the SIPG matrix is the Kronecker sum
//   A = sum_t M_g (x) .. (x) A_g^(t) (x) .. (x) M_g
// of GLOBAL 1D matrices (A_g block tridiagonal over the n_c,t cells of
// direction t), so with the generalised eigenpairs
// A_g^(t) Z_t = M_g Z_t diag(lambda_t), Z_t^T M_g Z_t = I of each direction
//   A^-1 = (Z_d (x) .. (x) Z_1) diag(1 / sum_t lambda_t) (Z_d (x) .. (x) Z_1)^T
// exactly: a direct solve in O(N sum_t N_t) work that replaces the
// reference's dense Cholesky / sparse LU (scipy) on the device.  The vector
// is permuted from the canonical cell-major layout to the direction-major
// global tensor (dg_canonical_tensor), contracted mode by mode
// (dg_mode_contract), scaled (dg_kron_scale) and brought back.
//
// Load vector (compute_rhs, dgop.py:800-871): the same mode contraction with
// the n x n_q basis-value matrix maps weighted quadrature values to nodal
// coefficients (`_tensor.backward_all`, _tensor.py:81-97).
#include "launch.h"

namespace dgb {

// out[o, i, r] = sum_k S(i, k) in[o, k, r];  S(i, k) = S[i*ld_i + k*ld_k]
__global__ void mode_contract_kernel(const double* __restrict__ in, double* __restrict__ out,
                                     const double* __restrict__ S, int64_t outer, int K, int I,
                                     int64_t inner, int ld_i, int ld_k) {
  const int64_t total = outer * I * inner;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % inner;
    const int64_t oi = e / inner;
    const int i = (int)(oi % I);
    const int64_t o = oi / I;
    const double* src = in + (o * K) * inner + r;
    const double* row = S + (int64_t)i * ld_i;
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(__ldg(row + (int64_t)k * ld_k), __ldg(src + k * inner), s);
    out[e] = s;
  }
}

struct CanonParams {
  const double* in;
  double* out;
  int d, n;
  int nc[3];
  int to_tensor;  // 1: canonical -> tensor, 0: tensor -> canonical
};

// tensor index e = j_0 + N_0 (j_1 + N_1 j_2), j_t = c_t n + i_t, N_t = nc_t n;
// canonical dof = cell n^d + i_0 + n i_1 + n^2 i_2, cell = c_0 + nc_0 (c_1 + nc_1 c_2)
__global__ void canonical_tensor_kernel(const CanonParams p) {
  int64_t N[3] = {1, 1, 1};
  int64_t total = 1, nd = 1;
  for (int t = 0; t < p.d; ++t) {
    N[t] = (int64_t)p.nc[t] * p.n;
    total *= N[t];
    nd *= p.n;
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, cell = 0, cm = 1, off = 0, om = 1;
    for (int t = 0; t < p.d; ++t) {
      const int64_t j = rem % N[t];
      rem /= N[t];
      cell += (j / p.n) * cm;
      cm *= p.nc[t];
      off += (j % p.n) * om;
      om *= p.n;
    }
    const int64_t g = cell * nd + off;
    if (p.to_tensor) p.out[e] = p.in[g];
    else p.out[g] = p.in[e];
  }
}

// T[j] *= 1 / (lam_0[j_0] + lam_1[j_1] + lam_2[j_2])
__global__ void kron_scale_kernel(double* T, const double* l0, const double* l1,
                                  const double* l2, int N0, int N1, int N2) {
  const int64_t total = (int64_t)N0 * N1 * N2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j0 = (int)(e % N0);
    const int64_t q = e / N0;
    const int j1 = (int)(q % N1), j2 = (int)(q / N1);
    double s = l0[j0];
    if (l1) s += l1[j1];
    if (l2) s += l2[j2];
    T[e] = T[e] / s;
  }
}

static unsigned grid_for(int64_t total) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
}

}  // namespace dgb

using namespace dgb;

extern "C" {

int dg_mode_contract(const double* in, double* out, const double* S, int64_t outer, int K,
                     int I, int64_t inner, int transposed, void* stream) {
  if (!in || !out || !S) return fail(DG_EINVAL, "null argument");
  if (in == out) return fail(DG_EINVAL, "mode contraction: output must not alias input");
  if (outer < 0 || inner < 1 || K < 1 || I < 1) return fail(DG_EINVAL, "bad contraction shape");
  const int64_t total = outer * I * inner;
  if (total == 0) return DG_OK;
  // S is I x K row-major, or K x I row-major when transposed
  const int ld_i = transposed ? 1 : K, ld_k = transposed ? I : 1;
  mode_contract_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(in, out, S, outer, K, I,
                                                                         inner, ld_i, ld_k);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dg_canonical_tensor(int dim, int degree, const int* ncells, const double* in, double* out,
                        int to_tensor, void* stream) {
  if (!ncells || !in || !out) return fail(DG_EINVAL, "null argument");
  if (in == out) return fail(DG_EINVAL, "layout change: output must not alias input");
  if (dim < 1 || dim > 3 || degree < 1) return fail(DG_EINVAL, "bad level shape");
  CanonParams p{};
  p.in = in;
  p.out = out;
  p.d = dim;
  p.n = degree + 1;
  int64_t total = 1;
  for (int t = 0; t < 3; ++t) {
    p.nc[t] = t < dim ? ncells[t] : 1;
    if (p.nc[t] < 1) return fail(DG_EINVAL, "ncells must be >= 1");
    if (t < dim) total *= (int64_t)p.nc[t] * p.n;
  }
  p.to_tensor = to_tensor;
  canonical_tensor_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int dg_kron_scale(double* tensor, const double* lam0, const double* lam1, const double* lam2,
                  int n0, int n1, int n2, void* stream) {
  if (!tensor || !lam0) return fail(DG_EINVAL, "null argument");
  if (n0 < 1 || n1 < 1 || n2 < 1) return fail(DG_EINVAL, "bad tensor shape");
  kron_scale_kernel<<<grid_for((int64_t)n0 * n1 * n2), 256, 0, (cudaStream_t)stream>>>(
      tensor, lam0, lam1, lam2, n0, n1, n2);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

}  // extern "C"
