// Scatter-update microbenchmark on B200: x[i] += w*y[i] over a large vector,
// done as (a) load-add-store, (b) red.global.add.f64 (fire-and-forget),
// (c) cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 from smem
// in 1728-byte chunks (one Q5 cell).  Reports effective GB/s of x updated.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while(0)

__global__ void rmw(double* x, const double* y, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long)gridDim.x * blockDim.x) x[i] += 0.5 * y[i];
}
__global__ void red(double* x, const double* y, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long)gridDim.x * blockDim.x) {
    double v = 0.5 * y[i];
    asm volatile("red.global.add.f64 [%0], %1;" :: "l"(x + i), "d"(v) : "memory");
  }
}
// each CTA: chunks of 216 doubles; stage w*y in smem then bulk-reduce into x
__global__ void bulkred(double* x, const double* y, long nchunks) {
  __shared__ __align__(128) double buf[2][216];
  int s = 0;
  for (long c = blockIdx.x; c < nchunks; c += gridDim.x, s ^= 1) {
    // make sure the bulk op that last read buf[s] has finished reading smem
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < 216; i += blockDim.x) buf[s][i] = 0.5 * y[c * 216 + i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(buf[s]);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                   :: "l"(x + c * 216), "r"(sa), "r"(216 * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const long n = 216L * 262144;  // 56.6M doubles (cfg5 vector)
  double *x, *y;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8));
  CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(y, 0, n * 8));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    rmw<<<148 * 8, 256>>>(x, y, n); cudaEventRecord(a); rmw<<<148 * 8, 256>>>(x, y, n); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"rmw\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, n * 8 / ms / 1e6);
    red<<<148 * 8, 256>>>(x, y, n); cudaEventRecord(a); red<<<148 * 8, 256>>>(x, y, n); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"red.add.f64\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, n * 8 / ms / 1e6);
    bulkred<<<148 * 16, 128>>>(x, y, n / 216); cudaEventRecord(a); bulkred<<<148 * 16, 128>>>(x, y, n / 216); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"cp.reduce.async.bulk.add.f64\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, n * 8 / ms / 1e6);
  }
  CK(cudaGetLastError());
  // L2-resident variant: 8 MB region updated repeatedly (what a locality-friendly schedule sees)
  const long m = 1L << 20;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); for (int k = 0; k < 20; ++k) rmw<<<148 * 8, 256>>>(x, y, m); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"rmw_l2\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, 20 * m * 8 / ms / 1e6);
    cudaEventRecord(a); for (int k = 0; k < 20; ++k) red<<<148 * 8, 256>>>(x, y, m); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"red_l2\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, 20 * m * 8 / ms / 1e6);
    cudaEventRecord(a); for (int k = 0; k < 20; ++k) bulkred<<<148 * 16, 128>>>(x, y, m / 216); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("{\"kind\": \"bulkred_l2\", \"ms\": %.3f, \"x_GBps\": %.1f}\n", ms, 20 * (m / 216) * 216 * 8 / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
