// Shared device-side definitions for the dicb200 kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "dicb200.h"

namespace dicb200 {

// Regular POI lattice: grid_subsets (image.cpp:140-158) keeps a centre iff
// subset_fits, which is separable in x and y, so the kept centres form the
// Cartesian product xs x ys. Subset index k = iy * nx + ix (y-outer, x-inner).
struct Lattice {
  int x0, y0, step, nx, ny;
  __host__ __device__ int cx(int ix) const { return x0 + ix * step; }
  __host__ __device__ int cy(int iy) const { return y0 + iy * step; }
};

struct ImageView {
  const void* data;
  int width, height, pitch;  // pitch in elements
};

// One BFS candidate partial: argmax under the reference order
// (c desc, dy asc, dx asc) (integer_search.cpp:43-48) plus the evaluation
// count (non-degenerate, in-window candidates).
struct BestPartial {
  double c;
  int dx, dy;
  int count;
  int found;
};

// improves(c, dx, dy, best...) of integer_search.cpp:43-48.
__host__ __device__ inline bool improves(double c, int dx, int dy, double bc, int bdx, int bdy) {
  if (c > bc) return true;
  if (c < bc) return false;
  if (dy != bdy) return dy < bdy;
  return dx < bdx;
}

__device__ inline void merge_best(BestPartial& a, const BestPartial& b) {
  if (b.found && (!a.found || improves(b.c, b.dx, b.dy, a.c, a.dx, a.dy))) {
    a.c = b.c;
    a.dx = b.dx;
    a.dy = b.dy;
    a.found = 1;
  }
  a.count += b.count;
}

// ZNCC from exact integer moments. With n = (2M+1)^2:
//   num = n*Sfg - Sf*Sg, vf = n*Sff - Sf^2, vg = n*Sgg - Sg^2 (all exact int64),
//   zncc = num / (sqrt(vf) * sqrt(vg)),
// algebraically identical to correlation.cpp:41-72 (cross/(||f-fbar|| ||g-gbar||));
// vg == 0 <=> the reference's "degenerate target subset" (constant window).
__device__ inline double zncc_from_moments(int64_t n, int64_t sfg, int64_t sf, int64_t sg, int64_t sgg,
                                           double sqrt_vf) {
  const int64_t num = n * sfg - sf * sg;
  const int64_t vg = n * sgg - sg * sg;
  return (double)num / (sqrt_vf * sqrt((double)vg));
}

// Launch accounting (bench.py "gpu_launches").
void count_launch(int n = 1);

// Stage timing scope (dicb200_profile_*): CUDA events around the enqueued work.
struct StageTimer {
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  StageTimer(int s, cudaStream_t stream);
  ~StageTimer();
};

}  // namespace dicb200

#define DICB200_CUDA_TRY(expr)                                              \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::dicb200::cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)

namespace dicb200 {
dicb200_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);
void set_error(const char* msg);
// DICB200_HOST_TRACE=1: reports host-side gaps > 5 ms between consecutive
// marks on this thread (enqueue stalls that would starve the GPU)
void host_trace(const char* what, long i = 0);
// cudaFuncAttributeMaxDynamicSharedMemorySize is per-kernel (and per-device) state: concurrent host
// callers that set it to what THEIR launch needs race - the one that set the larger value can find
// it lowered before it launches (cudaErrorInvalidValue; seen with four threads in
// dicb200_analyze_pair). The limit therefore only ever grows.
cudaError_t set_dyn_smem(const void* kernel, size_t bytes);
template <typename K>
inline cudaError_t set_dyn_smem(K kernel, size_t bytes) {
  return set_dyn_smem(reinterpret_cast<const void*>(kernel), bytes);
}

}  // namespace dicb200
