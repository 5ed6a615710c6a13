// Device renderer for the synthetic BASELINE frames:
// same blob list, binning, preimage map and 5-sigma cut-off as the host
// renderer (synth.c); one thread per pixel. Used by bench.py so 65-frame
// 2048^2 sequences are generated in milliseconds instead of minutes on host
// cores. (Host and device exp() may differ in the last ulp, so a rare pixel
// can round differently; parity tests always feed the SAME frame to both the
// oracle and the device path.)
#include <cmath>

#include "common.cuh"
#include "synth_internal.h"

namespace dicb200 {
namespace {

__device__ void displacement(const dicb200_synth_spec& sp, double yx, double yy, double* dx, double* dy) {
  const double* a = sp.a;
  if (sp.field == DICB200_FIELD_AFFINE) {
    const double rx = yx - a[6], ry = yy - a[7];
    *dx = a[0] + a[1] * rx + a[2] * ry;
    *dy = a[3] + a[4] * rx + a[5] * ry;
  } else if (sp.field == DICB200_FIELD_SINUSOID) {
    *dx = a[0] * sin(2.0 * M_PI * yy / a[1]);
    *dy = a[2] * cos(2.0 * M_PI * yx / a[3]);
  } else {
    *dx = 0.0;
    *dy = 0.0;
  }
}

__device__ void preimage(const dicb200_synth_spec& sp, double x, double y, double* px, double* py) {
  const double* a = sp.a;
  if (sp.field == DICB200_FIELD_AFFINE) {
    const double m00 = 1.0 + a[1], m01 = a[2], m10 = a[4], m11 = 1.0 + a[5];
    const double det = m00 * m11 - m01 * m10;
    const double bx = x - a[6] - a[0], by = y - a[7] - a[3];
    *px = a[6] + (m11 * bx - m01 * by) / det;
    *py = a[7] + (-m10 * bx + m00 * by) / det;
  } else if (sp.field == DICB200_FIELD_SINUSOID) {
    double yx = x, yy = y;
    for (int it = 0; it < 60; ++it) {
      double dx, dy;
      displacement(sp, yx, yy, &dx, &dy);
      const double nx = x - dx, ny = y - dy;
      const double ch = fabs(nx - yx) + fabs(ny - yy);
      yx = nx;
      yy = ny;
      if (ch < 1e-13) break;
    }
    *px = yx;
    *py = yy;
  } else {
    *px = x;
    *py = y;
  }
}

__global__ void render_kernel(dicb200_synth_spec sp, const blob_t* blobs, const int* cell_start, const int* items,
                              int gx, int gy, int reach_cells, void* out, int pitch) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= sp.width) return;
  double qx, qy;
  preimage(sp, x, y, &qx, &qy);
  double v = sp.background;
  const int cx = (int)floor(qx / CELL), cy = (int)floor(qy / CELL);
  for (int by = cy - reach_cells; by <= cy + reach_cells; ++by) {
    if (by < 0 || by >= gy) continue;
    for (int bx = cx - reach_cells; bx <= cx + reach_cells; ++bx) {
      if (bx < 0 || bx >= gx) continue;
      const int c = by * gx + bx;
      for (int i = cell_start[c]; i < cell_start[c + 1]; ++i) {
        const blob_t b = blobs[items[i]];
        const double ddx = qx - b.cx, ddy = qy - b.cy;
        const double r2 = ddx * ddx + ddy * ddy;
        if (r2 <= b.reach2) v += b.peak * exp(-r2 * b.inv2s2);
      }
    }
  }
  const double maxv = (double)sp.max_value;
  if (v < 0.0) v = 0.0;
  if (v > maxv) v = maxv;
  const double q = floor(v + 0.5);
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
