// launch.h - host-side launch arguments and the per-kernel-family dispatch
// entry points (each kernel family is its own compilation unit).
#pragma once
#include "../../include/dgmg_b200.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace dgb {

int fail(int code, const std::string& msg);

#define DG_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return fail(DG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// device tables of a one-dimensional level (oned.cu)
struct OneDTables {
  const double* adiag = nullptr;  // [digit][i*n+k]
  const double* bg = nullptr;     // [2][n]
};

// host-side launch arguments (the kernels' parameter structs are built from these)
struct ResArgs {
  const double* x = nullptr;
  const double* b = nullptr;
  double* r = nullptr;
  const int32_t* list = nullptr;
  int64_t start = 0;
  int64_t count = 0;
  int packed = 0;
  int block_list = 0;  // list = vertex-patch cells, 2x2x2 blocks of 8 in slot order
  double alpha = 0, beta = 0, betap = 0;
  OneDTables oned;     // d = 1 only
  Geo geo;
};

struct FdmArgs {
  const double* r = nullptr;
  double* x = nullptr;
  const int32_t* list = nullptr;
  int64_t start = 0;
  int64_t count = 0;
  int packed = 0;
  int atomic = 0;
  int cluster = 0;  // list holds cluster base vertices (cluster_kernel)
  int pv_lo = 0, pv_hi = 0;
  const double* invsum = nullptr;
  const double* zd = nullptr;   // device Z per digit (row-major m x m), tensor-core path
  const double* ztd = nullptr;  // device Z^T per digit
  const double* eod = nullptr;  // device even/odd halves of the interior digit (4 tables)
  int* counter = nullptr;       // device work counter of the persistent solve (fdm2p.cuh)
  double* big_scratch = nullptr;  // per-CTA tensors of the generic kernel (fdmg.cuh), or null
  int big_slots = 0;              // tensors big_scratch holds
  double omega = 0;
  Geo geo;
};

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

// FNV-1a hash of every DGB_* environment entry: part of the CUDA-graph cache
// key, so a run-time switch flipped after a capture takes effect
uint64_t switch_signature();

template <typename K>
inline int resident_ctas(K k, int threads, size_t smem, int* out) {
  int per_sm = 0, dev = 0, sms = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem));
  DG_CUDA(cudaGetDevice(&dev));
  DG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *out = std::max(1, per_sm) * sms;
  return DG_OK;
}

struct HostRes {
  const double* mass;   // n*n
  const double* adiag;  // 4*n*n
  const double* bg;     // 2*n
  const double* eo;     // 4*(n/2)^2 or nullptr
};

struct FlowTask;

struct FlowDev {
  FlowTask* tasks = nullptr;
  int32_t* succ = nullptr;
  int32_t* plist = nullptr;
  int* state = nullptr;       // live scheduler state
  int* state_init = nullptr;  // its initial image (copied in before each step)
  int ntasks = 0;
  int64_t units = 0;
};

#define DG_N_CASES(X, D) \
  X(D, 2) X(D, 3) X(D, 4) X(D, 5) X(D, 6) X(D, 7) X(D, 8) X(D, 9) X(D, 10) \
  X(D, 11) X(D, 12) X(D, 13) X(D, 14) X(D, 15) X(D, 16)

int dispatch_residual(int d, int n, const ResArgs& p, const HostRes& h, cudaStream_t st);
int dispatch_cell_fdm(int d, int n, const FdmArgs& p, const double* hz, const double* hzt,
                      const double* heo, cudaStream_t st);
int dispatch_patch_fdm(int d, int n, const FdmArgs& p, const double* hz, const double* hzt,
                       const double* heo, cudaStream_t st);
size_t patch_fdm_scratch_bytes(int d, int n);
bool mvs_fused_supported(int d, int n);
int dispatch_mvs_fused(int d, int n, const ResArgs& ra, const FdmArgs& fa, const HostRes& h,
                       const double* hz, const double* hzt, const double* heo, cudaStream_t st);
int oned_residual(int n, const ResArgs& p, const OneDTables& t, cudaStream_t st);
int oned_fdm(int n, bool patch, const FdmArgs& p, cudaStream_t st);
bool flow_shape(int d, int n, int* gp, int* gr);
int dispatch_flow(int d, int n, const ResArgs& ra, const FdmArgs& fa, const HostRes& h,
                  const double* hz, const double* hzt, const double* heo, const FlowDev& fd,
                  cudaStream_t st);

}  // namespace dgb
