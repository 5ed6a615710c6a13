// K1-FP — integer search on fractional (floating-point) gray levels: the
// reference's own zncc / subset_stats / bfs_search (correlation.cpp:9-72,
// integer_search.cpp:52-79) restated for the device in its exact evaluation
// order, so the correlation values are the reference's bit for bit.
//
// The BASELINE configurations are integer images (the exact-integer kernels,
// bfs.cu / bfs_tc.cu / bfs_bs.cu); fractional gray levels — the reference's
// synth_speckle / synth_warped_pair frames its unit tests use
// (synth.cpp:51-87) — come here instead of being quantized. Images are fp64
// on the device (f32 inputs are widened exactly).
//
// CTA per POI. Its reference subset is centred once (the mean from one
// sequential sum, the norm from one sequential sum of squares: thread 0, the
// reference's loop order) and its candidate window staged in shared memory
// (global reads when it does not fit: whole-image domain). One THREAD per
// candidate then runs zncc exactly as the reference does — sequential
// row-major sum, mean = sum / n, sequential cross and sum of squares of the
// centred values, IEEE _rn operations (no FMA contraction, like the
// reference build's -ffp-contract=off) — so every value, every degenerate
// skip ("norm <= 0") and every argmax decision (improves(), integer_search.cpp:
// 43-48) is the reference's. Surface mode writes each candidate's value (NaN =
// no result) for the swarm walk (pso.cu).
#include "bfs_fp.cuh"

namespace dicb200 {

namespace {

constexpr int kFpThreads = 256;

__device__ __forceinline__ double tgt_at(const double* win, int wpitch, const ImageView& t, int wx0, int wy0, int x,
                                         int y) {
  if (win) return win[(y - wy0) * wpitch + (x - wx0)];
  return static_cast<const double*>(t.data)[(size_t)y * t.pitch + x];
}

__global__ void __launch_bounds__(kFpThreads) bfs_fp_kernel(FpParams p) {
  extern __shared__ __align__(16) double fp_smem[];
  __shared__ double s_norm;
  __shared__ double red_c[kFpThreads / 32];
  __shared__ int red_d[kFpThreads / 32][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t k = blockIdx.x;
  const int ix = (int)(k % p.lat.nx), iy = p.row_begin + (int)(k / p.lat.nx);
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, side = 2 * M + 1, n = side * side;
  const int W = p.tgt.width, H = p.tgt.height;
  // candidate domain: feasible_window (integer_search.cpp:11-21) or whole_image_window (:23-33)
  int lo_dx, hi_dx, lo_dy, hi_dy;
  if (p.whole) {
    lo_dx = M - cx, hi_dx = W - 1 - M - cx, lo_dy = M - cy, hi_dy = H - 1 - M - cy;
  } else {
    lo_dx = max(-p.R, M - cx), hi_dx = min(p.R, W - 1 - M - cx);
    lo_dy = max(-p.R, M - cy), hi_dy = min(p.R, H - 1 - M - cy);
  }
  double* cen = fp_smem;  // centred reference subset [n]
  double* win = p.stage_window ? fp_smem + ((n + 1) & ~1) : nullptr;
  const int wx0 = cx + lo_dx - M, wy0 = cy + lo_dy - M;
  const int ww = hi_dx - lo_dx + side, wh = hi_dy - lo_dy + side;
  // ---- subset_stats (correlation.cpp:9-39)
  const double* ref = static_cast<const double*>(p.ref.data);
  if (tid == 0) {
    double sum = 0.0;
    for (int dy = -M; dy <= M; ++dy) {
      const double* row = ref + (size_t)(cy + dy) * p.ref.pitch + (cx - M);
      for (int i = 0; i < side; ++i) sum = __dadd_rn(sum, row[i]);
    }
    red_c[0] = __ddiv_rn(sum, (double)n);
  }
  __syncthreads();
  const double mean_f = red_c[0];
  for (int t = tid; t < n; t += kFpThreads) {
    const int r = t / side, c = t - r * side;
    cen[t] = __dsub_rn(ref[(size_t)(cy - M + r) * p.ref.pitch + (cx - M + c)], mean_f);
  }
  if (win && lo_dx <= hi_dx && lo_dy <= hi_dy)
    for (int t = tid; t < ww * wh; t += kFpThreads) {
      const int r = t / ww, c = t - r * ww;
      win[t] = static_cast<const double*>(p.tgt.data)[(size_t)(wy0 + r) * p.tgt.pitch + (wx0 + c)];
    }
  __syncthreads();
  if (tid == 0) {
    double sumsq = 0.0;
    for (int t = 0; t < n; ++t) sumsq = __dadd_rn(sumsq, __dmul_rn(cen[t], cen[t]));
    s_norm = __dsqrt_rn(sumsq);
  }
  __syncthreads();
  const double norm_f = s_norm;
  // ---- bfs_search: thread per candidate, row-major candidate index
  BestPartial b;
  b.c = -2.0;
  b.dx = b.dy = 0;
  b.count = 0;
  b.found = 0;
  const int fw = hi_dx - lo_dx + 1, fh = hi_dy - lo_dy + 1;
  const int EW = 2 * p.R + 1;
  if (fw > 0 && fh > 0) {
    for (int cidx = tid; cidx < fw * fh; cidx += kFpThreads) {
      const int ry = cidx / fw, dx = lo_dx + (cidx - ry * fw), dy = lo_dy + ry;
      const int x0 = cx + dx - M, y0 = cy + dy - M;
      double z = __longlong_as_double(0x7ff8000000000000ll);  // no result
      if (norm_f > 0.0) {  // "degenerate subset" (correlation.cpp:43): every candidate throws
        double sum = 0.0;
        for (int oy = 0; oy < side; ++oy)
          for (int i = 0; i < side; ++i) sum = __dadd_rn(sum, tgt_at(win, ww, p.tgt, wx0, wy0, x0 + i, y0 + oy));
        const double mean = __ddiv_rn(sum, (double)n);
        double cross = 0.0, sumsq = 0.0;
        int kk = 0;
        for (int oy = 0; oy < side; ++oy)
          for (int i = 0; i < side; ++i, ++kk) {
            const double g = __dsub_rn(tgt_at(win, ww, p.tgt, wx0, wy0, x0 + i, y0 + oy), mean);
            cross = __dadd_rn(cross, __dmul_rn(cen[kk], g));
            sumsq = __dadd_rn(sumsq, __dmul_rn(g, g));
          }
        const double nrm = __dsqrt_rn(sumsq);
        if (nrm > 0.0) {  // "degenerate target subset" (correlation.cpp:70): skipped, not counted
          z = __ddiv_rn(cross, __dmul_rn(norm_f, nrm));
          ++b.count;
          if (!b.found || improves(z, dx, dy, b.c, b.dx, b.dy)) {
            b.found = 1;
            b.c = z;
            b.dx = dx;
            b.dy = dy;
          }
        }
      }
      if (p.surface) p.surface[k * (size_t)EW * EW + (size_t)(dy + p.R) * EW + (dx + p.R)] = z;
    }
  }
  if (p.surface) {  // positions outside the feasible window: no result
    for (int t = tid; t < EW * EW; t += kFpThreads) {
      const int dy = t / EW - p.R, dx = t % EW - p.R;
      if (dx < lo_dx || dx > hi_dx || dy < lo_dy || dy > hi_dy)
        p.surface[k * (size_t)EW * EW + t] = __longlong_as_double(0x7ff8000000000000ll);
    }
    return;  // the swarm walk writes the record
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    BestPartial q;
    q.c = __shfl_xor_sync(0xffffffffu, b.c, o);
    q.dx = __shfl_xor_sync(0xffffffffu, b.dx, o);
    q.dy = __shfl_xor_sync(0xffffffffu, b.dy, o);
    q.count = __shfl_xor_sync(0xffffffffu, b.count, o);
    q.found = __shfl_xor_sync(0xffffffffu, b.found, o);
    merge_best(b, q);
  }
  if (lane == 0) {
    red_c[warp] = b.c;
    red_d[warp][0] = b.dx;
    red_d[warp][1] = b.dy;
    red_d[warp][2] = b.count;
    red_d[warp][3] = b.found;
  }
  __syncthreads();
  if (tid == 0) {
    BestPartial t;
    t.c = -2.0;
    t.dx = t.dy = 0;
    t.count = 0;
    t.found = 0;
    for (int w2 = 0; w2 < kFpThreads / 32; ++w2) {
      BestPartial q;
      q.c = red_c[w2];
      q.dx = red_d[w2][0];
      q.dy = red_d[w2][1];
      q.count = red_d[w2][2];
      q.found = red_d[w2][3];
      merge_best(t, q);
    }
    write_integer_record(p.rec[k], cx, cy, t, p.subpixel_none);
  }
}

__global__ void widen_f32_kernel(const float* src, int pitch, double* dst, int w, int h) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x < w) dst[(size_t)y * w + x] = (double)src[(size_t)y * pitch + x];
}

template <typename Pix>
__global__ void widen_int_kernel(const Pix* src, int pitch, double* dst, int w, int h) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x < w) dst[(size_t)y * w + x] = (double)src[(size_t)y * pitch + x];
}

}  // namespace

cudaError_t bfs_fp_launch(FpParams p, int rows, cudaStream_t st) {
  const int side = 2 * p.M + 1, n = side * side;
  const int EW = p.whole ? 0 : 2 * p.R + 1;
  size_t smem = (size_t)((n + 1) & ~1) * 8;
  const size_t wbytes = p.whole ? 0 : (size_t)(EW + side - 1) * (EW + side - 1) * 8;
  p.stage_window = !p.whole && smem + wbytes <= 160 * 1024;
  if (p.stage_window) smem += wbytes;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_dyn_smem(bfs_fp_kernel, smem);
  if (e != cudaSuccess) return e;
  const size_t npoi = (size_t)rows * p.lat.nx;
  if (npoi == 0) return cudaSuccess;
  bfs_fp_kernel<<<(unsigned)npoi, kFpThreads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t widen_f32_to_f64(const float* src, int pitch, double* dst, int w, int h, cudaStream_t st) {
  widen_f32_kernel<<<dim3((w + 255) / 256, h), 256, 0, st>>>(src, pitch, dst, w, h);
  count_launch();
  return cudaGetLastError();
}

cudaError_t widen_int_to_f64(const void* src, int elem_size, int pitch, double* dst, int w, int h, cudaStream_t st) {
  const dim3 grid((w + 255) / 256, h);
  if (elem_size == 1)
    widen_int_kernel<uint8_t><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(src), pitch, dst, w, h);
  else
    widen_int_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(src), pitch, dst, w, h);
  count_launch();
  return cudaGetLastError();
}

}  // namespace dicb200
