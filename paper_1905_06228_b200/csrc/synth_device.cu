// Device renderer for the synthetic BASELINE frames: one
// thread per pixel running the SAME per-pixel code as the host renderer
// (synth_math.h: explicit IEEE roundings, portable exp/sin/cos), over the same
// blob list and binning (synth.c) — frames are bit-identical to
// dicb200_synth_render's by construction (tests/test_gpu_synth.py checks every
// BASELINE frame kind). Used by bench.py so 65-frame 2048^2 sequences are
// generated in milliseconds instead of seconds of host cores.
#include <cmath>

#include "common.cuh"
#include "synth_internal.h"
#include "synth_math.h"

namespace dicb200 {
namespace {

__global__ void render_kernel(dicb200_synth_spec sp, const blob_t* blobs, const int* cell_start, const int* items,
                              int gx, int gy, int reach_cells, void* out, int pitch) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= sp.width) return;
  const double q = sx_pixel(&sp, blobs, cell_start, items, gx, gy, reach_cells, x, y);
  if (sp.dtype == DICB200_U8)
    reinterpret_cast<uint8_t*>(out)[(size_t)y * pitch + x] = (uint8_t)q;
  else
    reinterpret_cast<uint16_t*>(out)[(size_t)y * pitch + x] = (uint16_t)q;
}

}  // namespace
}  // namespace dicb200

extern "C" int dicb200_synth_render_device(const dicb200_synth_spec* sp, void* out_dev, int32_t pitch, void* stream) {
  using namespace dicb200;
  if (sp->width < 1 || sp->height < 1 || sp->blob_count < 0 || pitch < sp->width) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  synth_blobs_t B;
  dicb200_synth_blobs(sp, &B);
  const int ncell = B.gx * B.gy;
  blob_t* dblobs = nullptr;
  int *dstart = nullptr, *ditems = nullptr;
  int rc = 0;
  if (cudaMalloc(&dblobs, sizeof(blob_t) * (B.n > 0 ? B.n : 1)) != cudaSuccess ||
      cudaMalloc(&dstart, sizeof(int) * (ncell + 1)) != cudaSuccess ||
      cudaMalloc(&ditems, sizeof(int) * (B.n > 0 ? B.n : 1)) != cudaSuccess) {
    rc = 2;
  } else {
    cudaMemcpyAsync(dblobs, B.blobs, sizeof(blob_t) * B.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dstart, B.cell_start, sizeof(int) * (ncell + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(ditems, B.items, sizeof(int) * B.n, cudaMemcpyHostToDevice, st);
    dim3 grid((sp->width + 127) / 128, sp->height);
    render_kernel<<<grid, 128, 0, st>>>(*sp, dblobs, dstart, ditems, B.gx, B.gy, B.reach_cells, out_dev, pitch);
    if (cudaGetLastError() != cudaSuccess) rc = 3;
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = 3;
  }
  cudaFree(dblobs);
  cudaFree(dstart);
  cudaFree(ditems);
  dicb200_synth_blobs_free(&B);
  return rc;
}
