// K3/K4 — sub-pixel refinement: IC-GN (icgn_precompute + refine_icgn,
// subpixel.cpp:191-222, 301-359) and Newton-Raphson (refine_nr,
// subpixel.cpp:224-299), first-order warp, bilinear interpolation
// (interp_bilinear / grad_bilinear, subpixel.cpp:59-128).
//
// One WARP per POI; a CTA (8 warps) takes a strip of 8 neighbouring POIs of
// one grid row, which share one staged fp32 reference region (subsets + 1 px
// gradient border) and one staged fp32 target region (union of the 8
// neighbourhoods of the integer estimates + pad_for(method)). After staging there are no
// block barriers: every reduction is a warp shuffle and the 6x6 algebra runs
// lane-parallel in fp64 on the same warp. Samples whose warped subset leaves
// the staged region (or needs domain checks near the image border) take the
// checked slow path with global loads, so any drift is handled exactly.
//
// Each iteration is ONE pass over the pixels: warp + gather + bilinear
// (+ gradient for NR) in fp32 on subset-local coordinates, per-lane fp32
// partials, fp64 warp reductions. The reference forms e_k (:331) / coeff_k
// (:258) after gbar and ng are known; the update sums are expanded exactly,
//   sum e_k sd_k = sum f_k sd_k - (nf/ng) [ sum g'_k sd_k - (gbar - fbar) sum sd_k ],
// g' = g - fbar, with the reference-side sums (sum f sd, sum sd, Hessian
// moments) precomputed in ONE pass: fp32 per-lane partials (<= 53 terms),
// fp64 across lanes; subset_stats sums (sum f, sum f^2) exact in fp64.
// 6x6 solves: warp-parallel Cholesky H^-1 (H is SPD: J^T J); IC-GN keeps H^-1
// in registers for all iterations. "Degenerate target" (ng == 0 in the
// reference) is detected exactly as "all samples equal" (min == max).
// Convergence test, guard band M+2, domain checks, |det| < 1e-8, non-finite
// steps and the final re-sample + ZNCC follow subpixel.cpp; failure semantics
// follow pipeline.cpp:82-133 (status set, converged = 0, integer fields kept).
#include <cstdlib>

#include "common.cuh"
#include "linalg.cuh"
#include <type_traits>

#include "refine.cuh"
#include "tma.cuh"

namespace dicb200 {

namespace {

constexpr int kWarps = 8;        // POIs per CTA
constexpr int kNT = 32 * kWarps;
// staged target margin around each neighbourhood (px): NR's iterates wander
// further (C3: drifting, non-converging POIs) than IC-GN's
__host__ __device__ constexpr int pad_for(int method) { return method == 0 ? 32 : 4; }
constexpr int kSpread = 12;      // max spread of integer estimates folded into one region

template <typename Pix>
__device__ __forceinline__ float gpx(const ImageView& im, int x, int y) {
  return (float)__ldg(reinterpret_cast<const Pix*>(im.data) + (size_t)y * im.pitch + x);
}

// Region rows [0, H) x [0, P) of `im` at (X0, Y0) -> dst (fp32, pitch P), zero
// outside the image; warp w takes rows w, w + kWarps, ...
template <typename Pix>
__device__ __forceinline__ void stage_rows(const ImageView& im, int X0, int Y0, int P, int H, float* dst, int warp,
                                           int lane) {
  const Pix* base = reinterpret_cast<const Pix*>(im.data);
  for (int y = warp; y < H; y += kWarps) {
    const int gy = Y0 + y;
    const bool yin = gy >= 0 && gy < im.height;
    const Pix* src = base + (size_t)(yin ? gy : 0) * im.pitch;
    float* d = dst + y * P;
    for (int c0 = 0; c0 < P; c0 += 128) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = c0 + u * 32 + lane, gx = X0 + x;
        v[u] = (x < P && yin && gx >= 0 && gx < im.width) ? (float)__ldg(src + gx) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u * 32 + lane < P) d[c0 + u * 32 + lane] = v[u];
    }
  }
}

struct Win {
  const float* w;  // S x S fp32 copy of the target around (bx, by), row pitch P
  int S, P, ox, oy;  // ox, oy: global coords of w[0]
};

template <typename Pix>
__device__ __forceinline__ float tap(const Win& wn, const ImageView& im, int x, int y) {
  const int lx = x - wn.ox, ly = y - wn.oy;
  if ((unsigned)lx < (unsigned)wn.S && (unsigned)ly < (unsigned)wn.S) return wn.w[ly * wn.P + lx];
  return gpx<Pix>(im, x, y);
}

// interp_bilinear (subpixel.cpp:59-102) at global (bx + xl, by + yl).
template <typename Pix>
__device__ __forceinline__ bool bilinear(const Win& wn, const ImageView& im, int bx, int by, float xl, float yl,
                                         float& g) {
  if (!(xl >= (float)(-bx) && xl <= (float)(im.width - 1 - bx) && yl >= (float)(-by) &&
        yl <= (float)(im.height - 1 - by)))
    return false;
  int x0 = bx + (int)floorf(xl), y0 = by + (int)floorf(yl);
  if (x0 > im.width - 2) x0 = im.width - 2;
  if (y0 > im.height - 2) y0 = im.height - 2;
  const float fx = xl - (float)(x0 - bx), fy = yl - (float)(y0 - by);
  // slow path: the four corners straight from global memory (L1), loads issued
  // together (no window test per tap)
  (void)wn;
  const int x1 = min(x0 + 1, im.width - 1), y1 = min(y0 + 1, im.height - 1);
  const float f00 = gpx<Pix>(im, x0, y0), f10 = gpx<Pix>(im, x1, y0);
  const float f01 = gpx<Pix>(im, x0, y1), f11 = gpx<Pix>(im, x1, y1);
  const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f00 + f11) - f10 - f01;
  const float v = fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
  const float lo = fminf(fminf(f00, f10), fminf(f01, f11));
  const float hi = fmaxf(fmaxf(f00, f10), fmaxf(f01, f11));
  g = fminf(fmaxf(v, lo), hi);
  return true;
}

// grad_bilinear (subpixel.cpp:104-128): node central differences, bilinearly
// weighted, zero weights skipped (keeps the taps inside the image).
template <typename Pix>
__device__ __forceinline__ bool grad_bilinear(const Win& wn, const ImageView& im, int bx, int by, float xl,
                                              float yl, float& gx, float& gy) {
  if (!(xl >= (float)(1 - bx) && xl <= (float)(im.width - 2 - bx) && yl >= (float)(1 - by) &&
        yl <= (float)(im.height - 2 - by)))
    return false;
  const float flx = floorf(xl), fly = floorf(yl);
  const int x0 = bx + (int)flx, y0 = by + (int)fly;
  const float fx = xl - flx, fy = yl - fly;
  const float wx[2] = {1.0f - fx, fx}, wy[2] = {1.0f - fy, fy};
  // the 12 taps of the four nodes' central differences, loaded together from
  // global memory (coordinates clamped: a clamped tap only ever meets a zero
  // weight, and fmaf(0, d, a) == a, so the sums equal the reference's
  // zero-weight skipping exactly)
  (void)wn;
  const int W1 = im.width - 1, H1 = im.height - 1;
  const int xm = max(x0 - 1, 0), xa = min(x0 + 1, W1), xb = min(x0 + 2, W1);
  const int ym = max(y0 - 1, 0), ya = min(y0 + 1, H1), yb = min(y0 + 2, H1);
  const float t_m0 = gpx<Pix>(im, xm, y0), t_a0 = gpx<Pix>(im, xa, y0), t_b0 = gpx<Pix>(im, xb, y0);
  const float t_0m = gpx<Pix>(im, x0, ym), t_0a = gpx<Pix>(im, x0, ya), t_0b = gpx<Pix>(im, x0, yb);
  const float t_am = gpx<Pix>(im, xa, ym), t_aa = gpx<Pix>(im, xa, ya), t_ab = gpx<Pix>(im, xa, yb);
  const float t_ma = gpx<Pix>(im, xm, ya), t_ba = gpx<Pix>(im, xb, ya), t_00 = gpx<Pix>(im, x0, y0);
  // node (x0 + a, y0 + b): d/dx = t(x+1) - t(x-1), d/dy = t(y+1) - t(y-1)
  const float ddx[2][2] = {{t_a0 - t_m0, t_b0 - t_00}, {t_aa - t_ma, t_ba - t_0a}};
  const float ddy[2][2] = {{t_0a - t_0m, t_aa - t_am}, {t_0b - t_00, t_ab - t_a0}};
  float ax = 0.f, ay = 0.f;
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const float w = wx[a] * wy[b] * 0.5f;
      ax = fmaf(w, ddx[b][a], ax);
      ay = fmaf(w, ddy[b][a], ay);
    }
  gx = ax;
  gy = ay;
  return true;
}

// ---- bicubic variant (dicb200_run_config.interp = DICB200_INTERP_BICUBIC) ----
// Keys cubic convolution (a = -0.5) and its derivative; the CPU restatement is
// oracle/dic_oracle.c (bicubic_eval), same tap order and row-first summation.
__device__ __forceinline__ void keys_weights(float f, float (&w)[4], float (&d)[4]) {
  w[0] = ((-0.5f * f + 1.0f) * f - 0.5f) * f;
  w[1] = (1.5f * f - 2.5f) * f * f + 1.0f;
  w[2] = ((-1.5f * f + 2.0f) * f + 0.5f) * f;
  w[3] = (0.5f * f - 0.5f) * f * f;
  d[0] = (-1.5f * f + 2.0f) * f - 0.5f;
  d[1] = (4.5f * f - 5.0f) * f;
  d[2] = (-4.5f * f + 4.0f) * f + 0.5f;
  d[3] = (1.5f * f - 1.0f) * f;
}

// 4 x 4 taps at rows/columns (0..3) of `tap(i, j)`, weights in x / y.
template <bool GRADS, typename TapF>
__device__ __forceinline__ float bicubic_sum(const TapF& tap, float fx, float fy, float& gx, float& gy) {
  float wx[4], dwx[4], wy[4], dwy[4];
  keys_weights(fx, wx, dwx);
  keys_weights(fy, wy, dwy);
  float v = 0.f, vx = 0.f, vy = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float r = 0.f, rd = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float t = tap(i, j);
      r = fmaf(wx[i], t, r);
      if (GRADS) rd = fmaf(dwx[i], t, rd);
    }
    v = fmaf(wy[j], r, v);
    if (GRADS) {
      vx = fmaf(wy[j], rd, vx);
      vy = fmaf(dwy[j], r, vy);
    }
  }
  if (GRADS) {
    gx = vx;
    gy = vy;
  }
  return v;
}

// Checked path: global taps, domain checks and replicated borders as the oracle.
template <typename Pix, bool GRADS>
__device__ __forceinline__ bool bicubic_global(const ImageView& im, int bx, int by, float xl, float yl, float& g,
                                               float& gx, float& gy) {
  if (!(xl >= (float)(-bx) && xl <= (float)(im.width - 1 - bx) && yl >= (float)(-by) &&
        yl <= (float)(im.height - 1 - by)))
    return false;
  if (GRADS && !(xl >= (float)(1 - bx) && xl <= (float)(im.width - 2 - bx) && yl >= (float)(1 - by) &&
                 yl <= (float)(im.height - 2 - by)))
    return false;
  int x0 = bx + (int)floorf(xl), y0 = by + (int)floorf(yl);
  if (x0 > im.width - 2) x0 = im.width - 2;
  if (y0 > im.height - 2) y0 = im.height - 2;
  const float fx = xl - (float)(x0 - bx), fy = yl - (float)(y0 - by);
  auto tap = [&](int i, int j) {
    const int x = min(max(x0 - 1 + i, 0), im.width - 1), y = min(max(y0 - 1 + j, 0), im.height - 1);
    return gpx<Pix>(im, x, y);
  };
  g = bicubic_sum<GRADS>(tap, fx, fy, gx, gy);
  return true;
}

__device__ __forceinline__ double warp_sum1(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-thread partials -> per-warp sums in rb[warp][base + i] (one value live at a time).
// Transposed warp reduction by recursive halving: N (power of two <= 32)
// per-lane partials in, lane l gets the warp total of value (l >> (5 - log2 N)).
// (N-1) x (4 SEL + 2 SHFL + DADD) instead of N x 5 x (2 SHFL + DADD).
template <int N>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[N]) {
  const int lane = threadIdx.x & 31;
  constexpr int L = N == 1 ? 0 : N == 2 ? 1 : N == 4 ? 2 : N == 8 ? 3 : N == 16 ? 4 : 5;
  static_assert((1 << L) == N, "N must be a power of two <= 32");
#pragma unroll
  for (int st = 0; st < L; ++st) {
    const int m = 16 >> st;
    const int half = N >> (st + 1);
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      const double send = upper ? v[j] : v[j + half];
      const double keep = upper ? v[j + half] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  double r = v[0];
#pragma unroll
  for (int m = 16 >> L; m; m >>= 1) r += __shfl_xor_sync(0xffffffffu, r, m);
  return r;
}

// Broadcast value j (held by lanes j << (5 - L)) of a transposed reduction.
template <int N>
__device__ __forceinline__ double tget(double r, int j) {
  constexpr int L = N == 1 ? 0 : N == 2 ? 1 : N == 4 ? 2 : N == 8 ? 3 : N == 16 ? 4 : 5;
  return __shfl_sync(0xffffffffu, r, j << (5 - L));
}

__device__ __forceinline__ double warp_det(const double* p) {
  return __dsub_rn(__dmul_rn(1.0 + p[1], 1.0 + p[5]), __dmul_rn(p[2], p[4]));
}

// compose_with_inverse (subpixel.cpp:53-57, affine_inverse :26-38). p layout: u,ux,uy,v,vx,vy.
__device__ int compose_with_inverse(double* p, const double* inc) {
  if (inc[0] == 0 && inc[3] == 0 && inc[1] == 0 && inc[2] == 0 && inc[4] == 0 && inc[5] == 0) return 0;
  const double a00 = 1.0 + inc[1], a01 = inc[2];
  const double a10 = inc[4], a11 = 1.0 + inc[5];
  const double det = __dsub_rn(__dmul_rn(a00, a11), __dmul_rn(a01, a10));
  if (fabs(det) < 1e-8) return DICB200_POI_INCREMENT_NOT_INVERTIBLE;
  const double rdet = 1.0 / det;  // one division (the reference divides each cofactor)
  const double i00 = a11 * rdet, i01 = -a01 * rdet;
  const double i10 = -a10 * rdet, i11 = a00 * rdet;
  const double inv[9] = {i00, i01, -__dadd_rn(__dmul_rn(i00, inc[0]), __dmul_rn(i01, inc[3])),
                         i10, i11, -__dadd_rn(__dmul_rn(i10, inc[0]), __dmul_rn(i11, inc[3])),
                         0.0, 0.0, 1.0};
  const double w[9] = {1.0 + p[1], p[2], p[0], p[4], 1.0 + p[5], p[3], 0.0, 0.0, 1.0};
  double c[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = __dmul_rn(w[i * 3 + 0], inv[0 * 3 + j]);
      s = __dadd_rn(s, __dmul_rn(w[i * 3 + 1], inv[1 * 3 + j]));
      s = __dadd_rn(s, __dmul_rn(w[i * 3 + 2], inv[2 * 3 + j]));
      c[i * 3 + j] = s;
    }
  p[1] = c[0] - 1.0;
  p[2] = c[1];
  p[0] = c[2];
  p[4] = c[3];
  p[5] = c[4] - 1.0;
  p[3] = c[5];
  return 0;
}

// 18 moment sums mo[k*6+w] (k: 0 aa, 1 ab, 2 bb; w: 1,dx,dy,dx^2,dxdy,dy^2) -> symmetric
// H = sum sd sd^T, sd = [a, a dx, a dy, b, b dx, b dy] (subpixel.cpp:210-212, :261-263).
__device__ void assemble_hessian(const double* mo, double scale, double* H) {
  const int map[6][6][2] = {
      {{0, 0}, {0, 1}, {0, 2}, {1, 0}, {1, 1}, {1, 2}}, {{0, 1}, {0, 3}, {0, 4}, {1, 1}, {1, 3}, {1, 4}},
      {{0, 2}, {0, 4}, {0, 5}, {1, 2}, {1, 4}, {1, 5}}, {{1, 0}, {1, 1}, {1, 2}, {2, 0}, {2, 1}, {2, 2}},
      {{1, 1}, {1, 3}, {1, 4}, {2, 1}, {2, 3}, {2, 4}}, {{1, 2}, {1, 4}, {1, 5}, {2, 2}, {2, 4}, {2, 5}},
  };
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) H[i * 6 + j] = mo[map[i][j][0] * 6 + map[i][j][1]] * scale;
}

// Warp-parallel Cholesky of the SPD 6x6 H (lane i < 6 holds row i in h[]),
// then lane c < 6 solves H x = e_c: returns row c of H^-1 in hinv[] (H^-1 is
// symmetric). pd = all pivots > 0. Runs on all 32 lanes of one warp.
__device__ void warp_cholesky_inverse(double (&h)[6], double (&hinv)[6], bool& pd) {
  const int lane = threadIdx.x & 31;
  double L[6][6], rdiag[6];  // rdiag: 1 / L[j][j], one division per pivot
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    // pivot on lane j: d = h[j][j] - sum_k<j L[j][k]^2 (lane j's h[k<j] already hold L[j][k])
    double d = h[j];
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) d -= h[k2] * h[k2];
    d = __shfl_sync(0xffffffffu, d, j);
    ok = ok && d > 0.0;
    const double dd = d > 0.0 ? d : 1.0, rj = rsqrt(dd), ljj = dd * rj;  // sqrt and its reciprocal, one MUFU
    // broadcast row j of L (k < j) and finish column j on lanes i > j
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) L[j][k2] = __shfl_sync(0xffffffffu, h[k2], j);
    L[j][j] = ljj;
    rdiag[j] = rj;
    double v = h[j];
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) v -= h[k2] * L[j][k2];
    if (lane > j) h[j] = v * rdiag[j];
    if (lane == j) h[j] = ljj;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int k2 = 0; k2 < i; ++k2) L[i][k2] = __shfl_sync(0xffffffffu, h[k2], i);
  // forward / back substitution for e_lane
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k2 = 0; k2 < i; ++k2) v -= L[i][k2] * y[k2];
    y[i] = v * rdiag[i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k2 = i + 1; k2 < 6; ++k2) v -= L[k2][i] * hinv[k2];
    hinv[i] = v * rdiag[i];
  }
  pd = ok;
}


struct StripGeom {
  int rX0, rY0, rP, rH;   // reference region: global origin, pitch (floats), rows
  int tX0, tY0, tP, tH;   // target region
};

template <typename Pix>
__device__ __forceinline__ bool sample_slow(const Win& wn, const ImageView& im, int bx, int by, float xl, float yl,
                                            bool grads, float& g, float& gx, float& gy) {
  bool ok = bilinear<Pix>(wn, im, bx, by, xl, yl, g);
  if (grads) ok = ok && grad_bilinear<Pix>(wn, im, bx, by, xl, yl, gx, gy);
  return ok;
}

// Lane-parallel step from H^-1 rows (lane i < 6 holds row i) and the rhs;
// returns the 6-vector on every lane.
__device__ __forceinline__ void hinv_step(const double (&hinv)[6], const double (&rhs)[6], double (&step)[6],
                                          bool& finite) {
  double si = 0.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) si = fma(hinv[j], -rhs[j], si);
  finite = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    step[j] = __shfl_sync(0xffffffffu, si, j);
    finite = finite && isfinite(step[j]);
  }
}


// Strided pixel walk of one warp over a (2M+1)^2 subset: lane handles pixels
// k = lane + 32 i (consecutive lanes -> consecutive pixels: conflict-free smem).
struct Walk {
  int npl, last_valid;     // trips; whether the last trip is a real pixel for this lane
  float dxf, dyf;          // subset-local coordinates of the current pixel
  float r32f, q32f, sidef, Mf;
  int roff, roff_step, roff_wrap;  // reference-region offset (rr * rP + cc)
  __device__ __forceinline__ void init(int M, int lane, int rP) {
    const int side = 2 * M + 1, n = side * side;
    npl = (n + 31) / 32;
    last_valid = lane + 32 * (npl - 1) < n;
    const int rr = lane / side, cc = lane - rr * side;
    const int q = 32 / side, r = 32 - q * side;
    dxf = (float)(cc - M);
    dyf = (float)(rr - M);
    r32f = (float)r;
    q32f = (float)q;
    sidef = (float)side;
    Mf = (float)M;
    roff = rr * rP + cc;
    roff_step = q * rP + r;
    roff_wrap = rP - side;
  }
  __device__ __forceinline__ void advance() {
    dxf += r32f;
    dyf += q32f;
    roff += roff_step;
    if (dxf > Mf) {
      dxf -= sidef;
      dyf += 1.0f;
      roff += roff_wrap;
    }
  }
};

struct WarpConst {
  double scf, nf;
  double A[6], S[6];
};

struct PassCtx {
  const float* T;   // target region
  const float* Rs;  // reference pixel (0,0) of the subset in the reference region
  const float2* Gs;  // IC-GN: (2 df/dx, 2 df/dy) of that pixel (gradient region)
  int tP, rP;
  float offx, offy;  // subset-local -> target-region coordinates
  int ioffx, ioffy;  // the same offsets as integers (exact floor/frac in local coordinates)
  float fbar;
  float ul, vl, ux, uy, vx, vy;
  Win wn;
  int bx, by;
};

enum { kIcgn = 0, kNr = 1, kFinal = 2 };

// One pass over the subset pixels for the current warp parameters.
// kIcgn : acc = {sum g', sum g'^2, -, sum g' 2gx {1,dx,dy}, sum g' 2gy {1,dx,dy}}
// kNr   : acc = {sum g', sum g'^2, sum cf g', sum cf J[6], sum g' J[6], sum J[6], moments[18]}
// kFinal: acc = {sum g', sum g'^2, sum cf g'}

// ---- packed FP32x2 (FFMA2 / FADD2 / FMUL2, sm_100a) ----
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk2(float a, float b) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(f2x v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// First IC-GN pass: the warp is the integer displacement with zero gradients,
// so every sample sits exactly on a target node and the bilinear value is the
// node itself (fma(a, 0, f00) == f00): one load per pixel, bit-identical sums
// to icgn_pass_fast2 at these parameters.
__device__ __forceinline__ void icgn_pass_node(const PassCtx& c, const Walk& w0, float* acc, float& gmin,
                                               float& gmax) {
  float s0 = 0.f, s1 = 0.f;
  f2x a36 = pk2(0.f, 0.f), a47 = a36, a58 = a36;
  gmin = 3.0e38f;
  gmax = -3.0e38f;
  const f2x step = pk2(w0.r32f, w0.q32f), wrap = pk2(-w0.sidef, 1.0f);
  f2x dxy = pk2(w0.dxf, w0.dyf);
  int roff = w0.roff;
  const int side = (int)w0.sidef, q = (int)w0.q32f, r = (int)w0.r32f;
  const int tstep = q * c.tP + r, twrap = c.tP - side;
  const float* Tb = c.T + c.ioffy * c.tP + c.ioffx;
  int toff = (int)w0.dyf * c.tP + (int)w0.dxf;
  const int cnt = w0.npl - (w0.last_valid ? 0 : 1);
#pragma unroll 2
  for (int i = 0; i < cnt; ++i) {
    float dx, dy;
    up2(dxy, dx, dy);
    const float gv = Tb[toff];
    gmin = fminf(gmin, gv);
    gmax = fmaxf(gmax, gv);
    const float2 gg = c.Gs[roff];
    const float gp = gv - c.fbar;
    s0 += gp;
    s1 = fmaf(gp, gp, s1);
    const f2x txy = mul2(pk2(gg.x, gg.y), pk2(gp, gp));
    a36 = add2(a36, txy);
    a47 = fma2(txy, pk2(dx, dx), a47);
    a58 = fma2(txy, pk2(dy, dy), a58);
    dxy = add2(dxy, step);
    roff += w0.roff_step;
    toff += tstep;
    float ndx, ndy;
    up2(dxy, ndx, ndy);
    if (ndx > w0.Mf) {
      dxy = add2(dxy, wrap);
      roff += w0.roff_wrap;
      toff += twrap;
    }
  }
  acc[0] = s0;
  acc[1] = s1;
  acc[2] = 0.f;
  up2(a36, acc[3], acc[6]);
  up2(a47, acc[4], acc[7]);
  up2(a58, acc[5], acc[8]);
}

// Fast IC-GN pass with packed x/y arithmetic: same sums as pixel_pass<true, kIcgn>.
__device__ __forceinline__ void icgn_pass_fast2(const PassCtx& c, const Walk& w0, float* acc, float& gmin,
                                                float& gmax) {
  float s0 = 0.f, s1 = 0.f;
  f2x a36 = pk2(0.f, 0.f), a47 = a36, a58 = a36;
  gmin = 3.0e38f;
  gmax = -3.0e38f;
  const f2x uvl = pk2(c.ul, c.vl);
  const f2x uxvx = pk2(c.ux, c.vx), uyvy = pk2(c.uy, c.vy);
  const f2x step = pk2(w0.r32f, w0.q32f), wrap = pk2(-w0.sidef, 1.0f);
  f2x dxy = pk2(w0.dxf, w0.dyf);
  int roff = w0.roff;
  const int cnt = w0.npl - (w0.last_valid ? 0 : 1);
  const float* Tb = c.T + c.ioffy * c.tP + c.ioffx;  // target-region origin in subset-local coordinates
#pragma unroll 4
  for (int i = 0; i < cnt; ++i) {
    float dx, dy;
    up2(dxy, dx, dy);
    f2x xy = add2(dxy, uvl);
    xy = fma2(uxvx, pk2(dx, dx), xy);
    xy = fma2(uyvy, pk2(dy, dy), xy);
    float xl, yl;
    up2(xy, xl, yl);
    const float flx = floorf(xl), fly = floorf(yl);  // subset-local: exact frac
    const float fx = xl - flx, fy = yl - fly;
    const float* t = Tb + (int)fly * c.tP + (int)flx;
    const float f00 = t[0], f10 = t[1], f01 = t[c.tP], f11 = t[c.tP + 1];
    const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f11 - f10) - a01;
    const float gv = fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
    gmin = fminf(gmin, gv);
    gmax = fmaxf(gmax, gv);
    const float2 gg = c.Gs[roff];
    const float gp = gv - c.fbar;
    s0 += gp;
    s1 = fmaf(gp, gp, s1);
    const f2x txy = mul2(pk2(gg.x, gg.y), pk2(gp, gp));
    a36 = add2(a36, txy);
    a47 = fma2(txy, pk2(dx, dx), a47);
    a58 = fma2(txy, pk2(dy, dy), a58);
    // advance the strided walk
    dxy = add2(dxy, step);
    roff += w0.roff_step;
    float ndx, ndy;
    up2(dxy, ndx, ndy);
    if (ndx > w0.Mf) {
      dxy = add2(dxy, wrap);
      roff += w0.roff_wrap;
    }
  }
  acc[0] = s0;
  acc[1] = s1;
  acc[2] = 0.f;
  up2(a36, acc[3], acc[6]);
  up2(a47, acc[4], acc[7]);
  up2(a58, acc[5], acc[8]);
}

// Final ZNCC pass with the packed walk of icgn_pass_fast2: the same values as
// pixel_pass<true, kFinal> (IEEE fma per lane, pixel_pass's bilinear rounding
// order): acc = {sum g', sum g'^2, sum (f - fbar) g'}.
__device__ __forceinline__ void final_pass_fast2(const PassCtx& c, const Walk& w0, float* acc, float& gmin,
                                                 float& gmax) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  gmin = 3.0e38f;
  gmax = -3.0e38f;
  const f2x uvl = pk2(c.ul, c.vl);
  const f2x uxvx = pk2(c.ux, c.vx), uyvy = pk2(c.uy, c.vy);
  const f2x step = pk2(w0.r32f, w0.q32f), wrap = pk2(-w0.sidef, 1.0f);
  f2x dxy = pk2(w0.dxf, w0.dyf);
  int roff = w0.roff;
  const int cnt = w0.npl - (w0.last_valid ? 0 : 1);
  const float* Tb = c.T + c.ioffy * c.tP + c.ioffx;
#pragma unroll 2
  for (int i = 0; i < cnt; ++i) {
    float dx, dy;
    up2(dxy, dx, dy);
    f2x xy = add2(dxy, uvl);
    xy = fma2(uxvx, pk2(dx, dx), xy);
    xy = fma2(uyvy, pk2(dy, dy), xy);
    float xl, yl;
    up2(xy, xl, yl);
    const float flx = floorf(xl), fly = floorf(yl);
    const float fx = xl - flx, fy = yl - fly;
    const float* t = Tb + (int)fly * c.tP + (int)flx;
    const float f00 = t[0], f10 = t[1], f01 = t[c.tP], f11 = t[c.tP + 1];
    const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f00 + f11) - f10 - f01;
    const float gv = fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
    gmin = fminf(gmin, gv);
    gmax = fmaxf(gmax, gv);
    const float gp = gv - c.fbar;
    s0 += gp;
    s1 = fmaf(gp, gp, s1);
    s2 = fmaf(c.Rs[roff] - c.fbar, gp, s2);
    dxy = add2(dxy, step);
    roff += w0.roff_step;
    float ndx, ndy;
    up2(dxy, ndx, ndy);
    if (ndx > w0.Mf) {
      dxy = add2(dxy, wrap);
      roff += w0.roff_wrap;
    }
  }
  acc[0] = s0;
  acc[1] = s1;
  acc[2] = s2;
}

// ---- fixed-geometry IC-GN passes (subset side and strip geometry known at
// compile time: C4 / C5) ----
// The subset is walked in two parts with a FIXED column per lane, so the
// per-pixel walk is one row step and the dx-weighted sums factor out of the
// pixel loop (sum txy dx = dx sum txy per lane):
//   part A: NA blocks of 32 columns, lane = column, one subset row per trip;
//   part B: the BW = side mod 32 remaining columns, RPT = 32 / BW rows per
//           trip (lanes >= RPT * BW and rows past the subset carry weight 0).
// The target region is staged as VERTICAL PAIRS T2[y][x] = (T[y][x], T[y+1][x]),
// so a bilinear sample is two 8-byte loads (left / right column pairs) and one
// packed lerp. floor / fraction / tap address come from the float bits of
// (xy - 0.5) + 1.5 * 2^23 (round to nearest integer = floor(xy), or xy - 1 at an
// exact integer, where the fraction is then 1 and the lerp gives the same node
// value): no conversion instructions.
template <int M>
struct FixedMap {
  static constexpr int SIDE = 2 * M + 1;
  static constexpr int NA = SIDE / 32;
  static constexpr int BW = SIDE % 32;
  static constexpr int RPT = BW ? 32 / BW : 1;
  static constexpr int NB = BW ? (SIDE + RPT - 1) / RPT : 0;
};

struct FixedCtx {
  uint32_t t2;   // shared address: T2 pair of subset-local (0, 0) minus the magic bias (see fixed_tap)
  uint32_t tn;   // shared address: T2 pair of subset-local (-M, -M) at the integer estimate (node pass)
  uint32_t g2;   // shared address: G2 (2 grad f) at subset pixel (-M, -M)
  uint32_t r;    // shared address: R (f) at subset pixel (-M, -M)
  float fbar;
  f2x o;         // (ul, vl) + kFixedK: warped origin, shifted to positive coordinates
  f2x A, B;      // (1 + ux, vx), (uy, 1 + vy)
};

constexpr int kFixedK = 32;            // fixed passes sample at subset-local + kFixedK (> 0)
constexpr uint32_t kMagicBits = 0x4B000000u;  // bit pattern of 2^23

__device__ __forceinline__ uint32_t fbits(float v) { return __float_as_uint(v); }
// Shared-memory loads by address. `volatile`: a plain asm counts as a pure
// function of its inputs, so the compiler may hoist it above the branch that
// makes the address valid (it did: the node pass's loads moved out of the
// iteration loop and faulted for a POI whose integer estimate lies outside the
// strip's staged target window — the POI itself runs the checked path).
__device__ __forceinline__ float lds1(uint32_t a) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ f2x lds2x(uint32_t a) {
  f2x r;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(a));
  return r;
}

// Bilinear sample at xk = subset-local position + kFixedK (packed x/y, >= 1 on
// the fast path). xk + (2^23 - 0.5) lands in [2^23, 2^24), whose integers are
// exactly the representable values: the sum rounds to 2^23 + round(xk - 0.5) =
// 2^23 + floor(xk) (or floor(xk) - 1 at an exact integer, where the fraction
// is then 1 and the lerp returns the same node value), and its bit pattern is
// 0x4B000000 + that floor.
template <int TP>
__device__ __forceinline__ float fixed_tap(const FixedCtx& c, f2x xk) {
  const f2x v = add2(xk, pk2(8388607.5f, 8388607.5f));
  const f2x fr = fma2(add2(v, pk2(-8388608.0f, -8388608.0f)), pk2(-1.0f, -1.0f), xk);  // xk - floor: exact
  float vx, vy, fx, fy;
  up2(v, vx, vy);
  up2(fr, fx, fy);
  // c.t2 carries -(0x4B000000 (TP + 1)) * 8 (mod 2^32)
  uint32_t a;
  if ((TP & (TP - 1)) == 0) {
    // shifts and a three-input add, kept on the ALU pipe (funnel shifts: ptxas
    // turns shl + add into IMAD, and the fixed passes are bound by the FMA pipe,
    // where packed FP32x2 instructions take two issue cycles each)
    constexpr int LG = TP == 128 ? 10 : TP == 64 ? 9 : TP == 32 ? 8 : 0;
    uint32_t sy, sx;
    asm("shf.l.clamp.b32 %0, 0, %1, %2;" : "=r"(sy) : "r"(fbits(vy)), "n"(LG));  // high word of {v : 0} << LG
    asm("shf.l.clamp.b32 %0, 0, %1, 3;" : "=r"(sx) : "r"(fbits(vx)));
    a = sy + sx + c.t2;
  } else {
    a = fbits(vy) * (uint32_t)(TP * 8) + (fbits(vx) * 8u + c.t2);
  }
  const f2x p0 = lds2x(a), p1 = lds2x(a + 8u);  // (f00, f01), (f10, f11)
  const f2x d = fma2(p0, pk2(-1.0f, -1.0f), p1);
  const f2x cc = fma2(d, pk2(fx, fx), p0);  // (top, bottom) at fx
  float top, bot;
  up2(cc, top, bot);
  return fmaf(fy, bot - top, top);
}

// KIND 0: node pass (integer start), 1: IC-GN pass, 2: final ZNCC pass.
// acc: {sum g', sum g'^2, sum f g' (final), sum g' 2gx {1,dx,dy}, sum g' 2gy {1,dx,dy}}
template <int M, int TP, int RP, int KIND>
__device__ __forceinline__ void fixed_pass(const FixedCtx& c, float* acc) {
  using F = FixedMap<M>;
  const int lane = threadIdx.x & 31;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  f2x a36 = pk2(0.f, 0.f), a58 = a36, a47 = a36;
  // ---- part A: lane = column, one row per trip ----
#pragma unroll
  for (int blk = 0; blk < F::NA; ++blk) {
    const int col = 32 * blk + lane;
    const float dxf = (float)(col - M);
    const f2x base = fma2(c.A, pk2(dxf, dxf), c.o);
    const uint32_t gcol = c.g2 + (uint32_t)col * 8u, rcol = c.r + (uint32_t)col * 4u;
    const uint32_t ncol = c.tn + (uint32_t)col * 8u;
    f2x bsum = pk2(0.f, 0.f);
    f2x dy2 = pk2((float)-M, (float)-M);  // (dy, dy), stepped as a pair: one packed add per row
#pragma unroll 4
    for (int t = 0; t < F::SIDE; ++t, dy2 = add2(dy2, pk2(1.0f, 1.0f))) {
      float g;
      if (KIND == 0)
        g = lds1(ncol + (uint32_t)(t * TP * 8));
      else
        g = fixed_tap<TP>(c, fma2(c.B, dy2, base));
      const float gp = g - c.fbar;
      s0 += gp;
      s1 = fmaf(gp, gp, s1);
      if (KIND == 2) {
        s2 = fmaf(lds1(rcol + (uint32_t)(t * RP * 4)) - c.fbar, gp, s2);
      } else {
        const f2x txy = mul2(lds2x(gcol + (uint32_t)(t * RP * 8)), pk2(gp, gp));
        bsum = add2(bsum, txy);
        a58 = fma2(txy, dy2, a58);
      }
    }
    if (KIND != 2) {
      a36 = add2(a36, bsum);
      a47 = fma2(bsum, pk2(dxf, dxf), a47);
    }
  }
  // ---- part B: the remaining BW columns, RPT rows per trip ----
  if (F::BW) {
    const int lc = lane % F::BW, lr = lane / F::BW;
    const bool lane_ok = lane < F::RPT * F::BW;
    const int col = 32 * F::NA + lc;
    const float dxf = (float)(col - M);
    const f2x base = fma2(c.A, pk2(dxf, dxf), c.o);
    const uint32_t gcol = c.g2 + (uint32_t)(col + lr * RP) * 8u, rcol = c.r + (uint32_t)(col + lr * RP) * 4u;
    const uint32_t ncol = c.tn + (uint32_t)(col + lr * TP) * 8u;
    f2x bsum = pk2(0.f, 0.f);
    // trips 0 .. NB-2: every lane's row is inside the subset (also the idle
    // lanes', whose weight is 0), so weight, row offsets and dy need no selects
    {
      const float w = lane_ok ? 1.0f : 0.0f, nfw = -c.fbar * w;
      f2x dy2 = pk2((float)(lr - M), (float)(lr - M));
#pragma unroll 2
      for (int t = 0; t < F::NB - 1; ++t, dy2 = add2(dy2, pk2((float)F::RPT, (float)F::RPT))) {
        float g;
        if (KIND == 0)
          g = lds1(ncol + (uint32_t)(t * F::RPT * TP * 8));
        else
          g = fixed_tap<TP>(c, fma2(c.B, dy2, base));
        const float gp = fmaf(g, w, nfw);
        s0 += gp;
        s1 = fmaf(gp, gp, s1);
        if (KIND == 2) {
          s2 = fmaf(lds1(rcol + (uint32_t)(t * F::RPT * RP * 4)) - c.fbar, gp, s2);
        } else {
          const f2x txy = mul2(lds2x(gcol + (uint32_t)(t * F::RPT * RP * 8)), pk2(gp, gp));
          bsum = add2(bsum, txy);
          a58 = fma2(txy, dy2, a58);
        }
      }
    }
    for (int t = F::NB - 1; t < F::NB; ++t) {  // last trip: rows past the subset carry weight 0
      const int row = t * F::RPT + lr;
      const bool ok = lane_ok && row < F::SIDE;
      const int rr = ok ? row : 0;  // weight 0: any valid pixel, contribution dropped
      const float w = ok ? 1.0f : 0.0f;
      const float dyf = (float)(rr - M);
      const f2x dy2 = pk2(dyf, dyf);
      const int roff = (ok ? t * F::RPT : -lr);
      float g;
      if (KIND == 0)
        g = lds1(ncol + (uint32_t)(roff * TP * 8));
      else
        g = fixed_tap<TP>(c, fma2(c.B, dy2, base));
      const float gp = fmaf(g, w, -c.fbar * w);
      s0 += gp;
      s1 = fmaf(gp, gp, s1);
      if (KIND == 2) {
        s2 = fmaf(lds1(rcol + (uint32_t)(roff * RP * 4)) - c.fbar, gp, s2);
      } else {
        const f2x txy = mul2(lds2x(gcol + (uint32_t)(roff * RP * 8)), pk2(gp, gp));
        bsum = add2(bsum, txy);
        a58 = fma2(txy, dy2, a58);
      }
    }
    if (KIND != 2) {
      a36 = add2(a36, bsum);
      a47 = fma2(bsum, pk2(dxf, dxf), a47);
    }
  }
  acc[0] = s0;
  acc[1] = s1;
  acc[2] = s2;
  up2(a36, acc[3], acc[6]);
  up2(a47, acc[4], acc[7]);
  up2(a58, acc[5], acc[8]);
}

// NODE: the integer start (u, v integral, zero gradients) — every sample and
// its bilinear gradient sit on a node: value t[0], gradient half the central
// differences, exactly what the weighted forms give with weights (1, 0, 0, 0).
template <bool FAST, int KIND, typename Pix, bool NODE = false, int INTERP = 0>
__device__ __forceinline__ void pixel_pass(const PassCtx& c, const ImageView& tgt, const Walk& w0,
                                           float* acc, int& bad, float& gmin, float& gmax) {
  constexpr int NV = KIND == kNr ? 39 : 9;
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.f;
  gmin = 3.0e38f;
  gmax = -3.0e38f;
  bad = 0;
  Walk w = w0;
  const int cnt = w.npl - (w.last_valid ? 0 : 1);
  const float* Tb = c.T + c.ioffy * c.tP + c.ioffx;  // target-region origin in subset-local coordinates
#pragma unroll 2
  for (int i = 0; i < cnt; ++i) {
    const float dx = w.dxf, dy = w.dyf;
    const float xl = fmaf(c.uy, dy, fmaf(c.ux, dx, dx + c.ul));
    const float yl = fmaf(c.vy, dy, fmaf(c.vx, dx, dy + c.vl));
    float gv, gx = 0.f, gy = 0.f;
    if (FAST && NODE) {
      const float* t = Tb + (int)dy * c.tP + (int)dx;
      gv = t[0];
      if (KIND == kNr) {
        gx = 0.5f * (t[1] - t[-1]);
        gy = 0.5f * (t[c.tP] - t[-c.tP]);
      }
    } else if (FAST && INTERP == DICB200_INTERP_BICUBIC) {
      const float flx = floorf(xl), fly = floorf(yl);
      const float* t = Tb + ((int)fly - 1) * c.tP + (int)flx - 1;
      const int tP = c.tP;
      gv = bicubic_sum<KIND == kNr>([&](int i, int j) { return t[j * tP + i]; }, xl - flx, yl - fly, gx, gy);
    } else if (FAST) {
      const float flx = floorf(xl), fly = floorf(yl);  // subset-local: exact frac
      const float fx = xl - flx, fy = yl - fly;
      const float* t = Tb + (int)fly * c.tP + (int)flx;
      const float f00 = t[0], f10 = t[1], f01 = t[c.tP], f11 = t[c.tP + 1];
      const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f00 + f11) - f10 - f01;
      gv = fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
      if (KIND == kNr) {
        const int P2 = 2 * c.tP;
        const float dx00 = f10 - t[-1], dx10 = t[2] - f00, dx01 = f11 - t[c.tP - 1], dx11 = t[c.tP + 2] - f01;
        const float dy00 = f01 - t[-c.tP], dy10 = f11 - t[1 - c.tP], dy01 = t[P2] - f00, dy11 = t[P2 + 1] - f10;
        const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
        gx = 0.5f * (w00 * dx00 + w10 * dx10 + w01 * dx01 + w11 * dx11);
        gy = 0.5f * (w00 * dy00 + w10 * dy10 + w01 * dy01 + w11 * dy11);
      }
    } else if (INTERP == DICB200_INTERP_BICUBIC) {
      gv = 0.f;
      bad |= !bicubic_global<Pix, KIND == kNr>(tgt, c.bx, c.by, xl, yl, gv, gx, gy);
    } else {
      gv = 0.f;
      bool ok = bilinear<Pix>(c.wn, tgt, c.bx, c.by, xl, yl, gv);
      if (KIND == kNr) ok = ok && grad_bilinear<Pix>(c.wn, tgt, c.bx, c.by, xl, yl, gx, gy);
      bad |= !ok;
    }
    gmin = fminf(gmin, gv);
    gmax = fmaxf(gmax, gv);
    const float* q = c.Rs + w.roff;
    const float gp = gv - c.fbar;
    acc[0] += gp;
    acc[1] = fmaf(gp, gp, acc[1]);
    if (KIND != kIcgn) acc[2] = fmaf(q[0] - c.fbar, gp, acc[2]);
    if (KIND == kIcgn) {
      const float2 gg = c.Gs[w.roff];  // 2 grad f, staged once per strip
      const float tx = gp * gg.x, ty = gp * gg.y;
      acc[3] += tx;
      acc[4] = fmaf(tx, dx, acc[4]);
      acc[5] = fmaf(tx, dy, acc[5]);
      acc[6] += ty;
      acc[7] = fmaf(ty, dx, acc[7]);
      acc[8] = fmaf(ty, dy, acc[8]);
    } else if (KIND == kNr) {
      const float cfv = q[0] - c.fbar;
      const float J[6] = {gx, gx * dx, gx * dy, gy, gy * dx, gy * dy};
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        acc[3 + j] = fmaf(cfv, J[j], acc[3 + j]);
        acc[9 + j] = fmaf(gp, J[j], acc[9 + j]);
        acc[15 + j] += J[j];
      }
      const float wv[6] = {1.f, dx, dy, dx * dx, dx * dy, dy * dy};
      const float aa = gx * gx, ab = gx * gy, bb = gy * gy;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        acc[21 + j] = fmaf(aa, wv[j], acc[21 + j]);
        acc[27 + j] = fmaf(ab, wv[j], acc[27 + j]);
        acc[33 + j] = fmaf(bb, wv[j], acc[33 + j]);
      }
    }
    w.advance();
  }
}

// Row `lane` (< 6) of H = scale * assemble(mo); other lanes get row 0.
__device__ __forceinline__ void hessian_row(const double* mo, double scale, int lane, double (&h)[6]) {
  const int map[6][6][2] = {
      {{0, 0}, {0, 1}, {0, 2}, {1, 0}, {1, 1}, {1, 2}}, {{0, 1}, {0, 3}, {0, 4}, {1, 1}, {1, 3}, {1, 4}},
      {{0, 2}, {0, 4}, {0, 5}, {1, 2}, {1, 4}, {1, 5}}, {{1, 0}, {1, 1}, {1, 2}, {2, 0}, {2, 1}, {2, 2}},
      {{1, 1}, {1, 3}, {1, 4}, {2, 1}, {2, 3}, {2, 4}}, {{1, 2}, {1, 4}, {1, 5}, {2, 2}, {2, 4}, {2, 5}},
  };
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double v = mo[map[0][j][0] * 6 + map[0][j][1]];
#pragma unroll
    for (int r = 1; r < 6; ++r)
      if (r == lane) v = mo[map[r][j][0] * 6 + map[r][j][1]];
    h[j] = v * scale;
  }
}

// Fixed-geometry variant (FM > 0, IC-GN only): subset half-width FM and
// lattice step FSTEP known at compile time, strip regions of static shape
// (target staged as vertical pairs, around the median integer estimate +-
// kFixedSpread), fixed_pass for every staged-region pass.
constexpr int kFixedPad = 3, kFixedSpread = 3;
template <int FM, int FSTEP>
struct FixedGeom {
  static constexpr int SIDE = 2 * FM + 1, SPAN = FSTEP * (kWarps - 1);
  // reference pitch: the SPAN + SIDE + 2 region columns plus up to 3 columns of
  // slack, a multiple of 4 (the pre-converted TMA boxes start 16-byte aligned)
  static constexpr int RP = (SPAN + SIDE + 2 + 3 + 3) & ~3, RH = SIDE + 2;
  // target pitch: the region plus one column of slack (even box start for the
  // pre-converted pairs), padded to a power of two when that costs < 8 columns
  // of pairs (the tap address is then two shifts on the ALU pipe instead of
  // IMADs), else to an even width (16-byte box rows)
  static constexpr int TP0 = SPAN + SIDE + 2 * kFixedPad + 2 * kFixedSpread + 1;
  static constexpr int TP = (TP0 <= 128 && TP0 > 80) ? 128 : (TP0 <= 64 && TP0 > 56) ? 64 : (TP0 + 1) & ~1;
  static constexpr int TH = SIDE + 2 * kFixedPad + 2 * kFixedSpread;  // float rows; TH - 1 pair rows
  // floats; 128-byte aligned (TMA destinations of the pre-converted staging)
  static constexpr size_t G2_OFF = (((size_t)RH * RP + 31) & ~(size_t)31);
  static constexpr size_t T2_OFF = ((G2_OFF + 2 * (size_t)RH * RP) + 31) & ~(size_t)31;
  static constexpr size_t SMEM = 4 * (T2_OFF + 2 * (size_t)(TH - 1) * TP);
  // TMA boxes of the raw u8/u16 regions (inner extent a multiple of 16 bytes),
  // landed inside the gradient area, which is only written after they are converted
  template <int ES>
  struct Raw {
    // box starts are aligned down to 16 bytes (measured: an unaligned inner
    // start coordinate faults, tools/microbench/tma_check.cu), so the boxes are
    // up to 16 bytes wider than the regions
    static constexpr int AE = 16 / ES;
    static constexpr int RBW = ((RP + AE - 1 + AE - 1) / AE) * AE, TBW = ((TP + AE - 1 + AE - 1) / AE) * AE;
    static constexpr size_t T_BYTES = (size_t)TH * TBW * ES, R_BYTES = (size_t)RH * RBW * ES;
    static constexpr uint32_t BYTES = (uint32_t)(T_BYTES + R_BYTES);
    // TMA destinations are 128-byte aligned (raw_dst); worst-case padding included
    static_assert(SIDE <= 3 || 4 * G2_OFF + 127 + ((T_BYTES + 127) & ~(size_t)127) + R_BYTES <= 4 * T2_OFF,
                  "raw TMA boxes must fit in the gradient area");
  };
};

// 128-byte aligned TMA destinations of the raw target / reference boxes inside
// the gradient area starting at `area`.
template <typename RAW>
__device__ __forceinline__ void raw_dst(float* area, unsigned char** t, unsigned char** r) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(area);
  const uint32_t pt = (128u - (a & 127u)) & 127u;
  unsigned char* b = reinterpret_cast<unsigned char*>(area);
  *t = b + pt;
  *r = b + pt + ((RAW::T_BYTES + 127) & ~(size_t)127);
}

// Rows [0, H-1) of vertical pairs (T[y][x], T[y+1][x]) of `im` at (X0, Y0), zero outside.
template <typename Pix>
__device__ __forceinline__ void stage_pairs(const ImageView& im, int X0, int Y0, int P, int H, float2* dst, int warp,
                                            int lane) {
  const Pix* base = reinterpret_cast<const Pix*>(im.data);
  for (int y = warp; y < H - 1; y += kWarps) {
    const int gy = Y0 + y;
    const bool y0in = gy >= 0 && gy < im.height, y1in = gy + 1 >= 0 && gy + 1 < im.height;
    const Pix* r0 = base + (size_t)(y0in ? gy : 0) * im.pitch;
    const Pix* r1 = base + (size_t)(y1in ? gy + 1 : 0) * im.pitch;
    float2* d = dst + y * P;
    for (int x = lane; x < P; x += 32) {
      const int gx = X0 + x;
      const bool xin = gx >= 0 && gx < im.width;
      d[x] = make_float2(xin && y0in ? (float)__ldg(r0 + gx) : 0.f, xin && y1in ? (float)__ldg(r1 + gx) : 0.f);
    }
  }
}

template <typename Pix, int METHOD, int FM = 0, int FSTEP = 0, int INTERP = 0>
__global__ void __launch_bounds__(kNT, 2) refine_strip_kernel(RefineParams p, const __grid_constant__ TmaPair tm) {
  constexpr bool FIXED = FM > 0;
  using FG = FixedGeom<FIXED ? FM : 1, FIXED ? FSTEP : 1>;
  using RAW = typename FG::template Raw<(int)sizeof(Pix)>;
  extern __shared__ __align__(128) float smem_f[];
  __shared__ uint64_t s_bar;  // TMA staging completion
  __shared__ int s_idx[kWarps], s_idy[kWarps], s_ok[kWarps];
  __shared__ WarpConst s_const[kWarps];
  __shared__ StripGeom G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = p.M, side = 2 * M + 1, n = side * side;
  // strip of this CTA: launch order from p.order (NR: likely long walks first), else the grid
  const int strip = p.order ? p.order[blockIdx.y * gridDim.x + blockIdx.x] : (int)(blockIdx.y * gridDim.x + blockIdx.x);
  const int iy = p.row_begin + strip / (int)gridDim.x;
  const int ix0 = (strip % (int)gridDim.x) * p.spc;
  const int ts = min(p.spc, p.lat.nx - ix0);
  const int cy = p.lat.cy(iy);
  const size_t rec0 = (size_t)(iy - p.row_begin) * p.lat.nx + ix0;

  // ---- strip geometry from the integer estimates ----
  if (!FIXED && tid < kWarps) {
    int ok = 0, dx = 0, dy = 0;
    if (tid < ts) {
      const dicb200_poi_record& r = p.rec[rec0 + tid];
      ok = r.status == DICB200_POI_OK;
      dx = r.integer_dx;
      dy = r.integer_dy;
    }
    s_ok[tid] = ok;
    s_idx[tid] = dx;
    s_idy[tid] = dy;
  }
  if (FIXED) {
    // static region around the median integer estimate, computed by warp 0
    // (lanes = the strip's POIs; ranks by shuffles), then lane 0 issues the TMA
    // copies of both raw regions before the block syncs
    if (warp == 0) {
      int ok = 0, dx = 0, dy = 0;
      if (lane < ts) {
        const dicb200_poi_record& r = p.rec[rec0 + lane];
        ok = r.status == DICB200_POI_OK;
        dx = r.integer_dx;
        dy = r.integer_dy;
      }
      if (lane < kWarps) {
        s_ok[lane] = ok;
        s_idx[lane] = dx;
        s_idy[lane] = dy;
      }
      const unsigned valid = __ballot_sync(0xffffffffu, ok);
      const int nv = __popc(valid);
      int rx = 0, ry = 0;  // rank of this lane's estimate among the valid ones (ties by lane)
#pragma unroll
      for (int j = 0; j < kWarps; ++j) {
        const int ox = __shfl_sync(0xffffffffu, dx, j), oy = __shfl_sync(0xffffffffu, dy, j);
        const bool vj = (valid >> j) & 1u;
        rx += vj && (ox < dx || (ox == dx && j < lane));
        ry += vj && (oy < dy || (oy == dy && j < lane));
      }
      const unsigned mx = __ballot_sync(0xffffffffu, ok && rx == nv / 2);
      const unsigned my = __ballot_sync(0xffffffffu, ok && ry == nv / 2);
      const int dxc = nv ? __shfl_sync(0xffffffffu, dx, __ffs(mx) - 1) : 0;
      const int dyc = nv ? __shfl_sync(0xffffffffu, dy, __ffs(my) - 1) : 0;
      if (lane == 0) {
        const int cx0 = p.lat.cx(ix0);
        G.rX0 = cx0 - M - 1;
        G.rY0 = cy - M - 1;
        G.rP = FG::RP;
        G.rH = FG::RH;
        G.tX0 = cx0 + dxc - kFixedSpread - M - kFixedPad;
        G.tY0 = cy + dyc - kFixedSpread - M - kFixedPad;
        G.tP = FG::TP;
        G.tH = FG::TH;
        if (p.use_tma == 2) {
          // pre-converted images (fp32 reference, its 2 grad, target vertical
          // pairs): the regions land in their final layout; the origins move to
          // the aligned box starts (the pitches carry the slack)
          G.rX0 &= ~3;
          G.tX0 &= ~1;
          tma_mbar_init(&s_bar, 1);
          tma_mbar_expect_tx(&s_bar, (uint32_t)(4 * FG::RP * FG::RH + 8 * FG::RP * FG::RH + 8 * FG::TP * (FG::TH - 1)));
          tma_load_2d(smem_f + FG::T2_OFF, &tm.tgt, G.tX0, G.tY0, &s_bar);
          tma_load_2d(smem_f, &tm.ref, G.rX0, G.rY0, &s_bar);
          tma_load_2d(smem_f + FG::G2_OFF, &tm.aux, G.rX0, G.rY0, &s_bar);
        } else if (p.use_tma) {
          tma_mbar_init(&s_bar, 1);
          unsigned char *rt, *rr;
          raw_dst<RAW>(smem_f + FG::G2_OFF, &rt, &rr);
          tma_mbar_expect_tx(&s_bar, RAW::BYTES);
          tma_load_2d(rt, &tm.tgt, G.tX0 & ~(RAW::AE - 1), G.tY0, &s_bar);
          tma_load_2d(rr, &tm.ref, G.rX0 & ~(RAW::AE - 1), G.rY0, &s_bar);
        }
      }
    }
  }
  __syncthreads();
  if (!FIXED && tid == 0) {
    int first = -1;
    for (int s = 0; s < ts; ++s)
      if (s_ok[s]) {
        first = s;
        break;
      }
    int dxlo = 0, dxhi = 0, dylo = 0, dyhi = 0;
    if (first >= 0) {
      dxlo = dxhi = s_idx[first];
      dylo = dyhi = s_idy[first];
      for (int s = 0; s < ts; ++s)
        if (s_ok[s]) {
          dxlo = min(dxlo, s_idx[s]);
          dxhi = max(dxhi, s_idx[s]);
          dylo = min(dylo, s_idy[s]);
          dyhi = max(dyhi, s_idy[s]);
        }
      // bound the region: outliers beyond kSpread fall back to the slow path
      dxlo = max(dxlo, s_idx[first] - kSpread);
      dxhi = min(dxhi, s_idx[first] + kSpread);
      dylo = max(dylo, s_idy[first] - kSpread);
      dyhi = min(dyhi, s_idy[first] + kSpread);
    }
    const int cx0 = p.lat.cx(ix0), cx1 = p.lat.cx(ix0 + ts - 1);
    G.rX0 = cx0 - M - 1;
    G.rY0 = cy - M - 1;
    G.rP = (cx1 - cx0) + side + 2;
    G.rH = side + 2;
    constexpr int kPad = FIXED ? kFixedPad : pad_for(METHOD);
    G.tX0 = cx0 + dxlo - M - kPad;
    G.tY0 = cy + dylo - M - kPad;
    G.tP = (cx1 - cx0) + (dxhi - dxlo) + side + 2 * kPad;
    G.tH = (dyhi - dylo) + side + 2 * kPad;
  }
  if (!FIXED) __syncthreads();
  const StripGeom g = G;
  float* R = smem_f;                    // reference region [rH][rP]
  float* T = smem_f + g.rH * g.rP;      // target region [tH][tP]
  // IC-GN: gradient region (2 grad f) [rH][rP] as float2, 8-byte aligned
  float2* G2 = reinterpret_cast<float2*>(smem_f + ((g.rH * g.rP + g.tH * g.tP + 1) & ~1));
  float2* T2 = nullptr;  // fixed geometry: target as vertical pairs [tH - 1][tP]
  if (FIXED) {
    G2 = reinterpret_cast<float2*>(smem_f + FG::G2_OFF);
    T2 = reinterpret_cast<float2*>(smem_f + FG::T2_OFF);
    T = nullptr;
  }
  // ---- stage both regions (fp32), zero outside the images: one warp per
  // region row, 4 independent loads per lane in flight, no index division ----
  if (FIXED && p.use_tma == 2) {
    tma_mbar_wait(&s_bar, 0);  // R, G2 and T2 in place: no conversion, no barrier
  } else if (FIXED && p.use_tma) {
    // raw u8/u16 boxes (TMA, zero outside the image) -> fp32 reference rows and
    // target vertical pairs, shared memory to shared memory
    tma_mbar_wait(&s_bar, 0);
    unsigned char *rtb, *rrb;
    raw_dst<RAW>(smem_f + FG::G2_OFF, &rtb, &rrb);
    const Pix* rr = reinterpret_cast<const Pix*>(rrb);
    const Pix* rt = reinterpret_cast<const Pix*>(rtb);
    const int oxr = g.rX0 & (RAW::AE - 1), oxt = g.tX0 & (RAW::AE - 1);
    for (int y = warp; y < FG::RH; y += kWarps) {
      const Pix* src = rr + y * RAW::RBW + oxr;
#pragma unroll
      for (int x = lane; x < FG::RP; x += 32) R[y * FG::RP + x] = (float)src[x];
    }
    for (int y = warp; y < FG::TH - 1; y += kWarps) {
      const Pix* s0 = rt + y * RAW::TBW + oxt;
#pragma unroll
      for (int x = lane; x < FG::TP; x += 32)
        T2[y * FG::TP + x] = make_float2((float)s0[x], (float)s0[x + RAW::TBW]);
    }
  } else {
    stage_rows<Pix>(p.ref, g.rX0, g.rY0, g.rP, g.rH, R, warp, lane);
    if (FIXED)
      stage_pairs<Pix>(p.tgt, g.tX0, g.tY0, g.tP, g.tH, T2, warp, lane);
    else
      stage_rows<Pix>(p.tgt, g.tX0, g.tY0, g.tP, g.tH, T, warp, lane);
  }
  const bool preconv = FIXED && p.use_tma == 2;  // the gradients came with the pre-converted images
  if (!preconv) __syncthreads();
  if (preconv) {
  } else if (FIXED) {  // static region shape: four independent columns per lane in flight
    for (int y = warp; y < FG::RH; y += kWarps) {
      const bool yin = y >= 1 && y < FG::RH - 1;
      const float* r0 = R + y * FG::RP;
#pragma unroll
      for (int x0 = 0; x0 < FG::RP; x0 += 128) {
        float2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int x = x0 + 32 * u + lane;
          v[u] = make_float2(0.f, 0.f);
          if (yin && x >= 1 && x < FG::RP - 1)
            v[u] = make_float2(r0[x + 1] - r0[x - 1], r0[x + FG::RP] - r0[x - FG::RP]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (x0 + 32 * u + lane < FG::RP) G2[y * FG::RP + x0 + 32 * u + lane] = v[u];
      }
    }
    __syncthreads();
  } else if (METHOD == 1) {  // central differences of the reference (icgn_precompute, subpixel.cpp:207-208), x2
    for (int y = warp; y < g.rH; y += kWarps) {
      const bool yin = y >= 1 && y < g.rH - 1;
      for (int x = lane; x < g.rP; x += 32) {
        const int i = y * g.rP + x;
        float2 v = make_float2(0.f, 0.f);
        if (yin && x >= 1 && x < g.rP - 1) v = make_float2(R[i + 1] - R[i - 1], R[i + g.rP] - R[i - g.rP]);
        G2[i] = v;
      }
    }
    __syncthreads();
  }
  // ==== from here on every warp is independent (no block barriers) ====
  if (warp >= ts || !s_ok[warp]) return;
  dicb200_poi_record* rec = p.rec + rec0 + warp;
  const int cx = p.lat.cx(ix0 + warp);
  const int idx = s_idx[warp], idy = s_idy[warp];
  const int bx = cx + idx, by = cy + idy;

  auto fail = [&](int code) {
    if (lane == 0) {
      rec->status = code;
      rec->converged = 0;
    }
  };
  if (METHOD == 1 && (cx - M - 1 < 0 || cx + M + 1 > p.ref.width - 1 || cy - M - 1 < 0 ||
                      cy + M + 1 > p.ref.height - 1)) {
    fail(DICB200_POI_BORDER_GRADIENTS);  // subpixel.cpp:193-195
    return;
  }
  Walk wk;
  wk.init(M, lane, g.rP);
  const float* Rs = R + g.rP + (cx - M - g.rX0);  // reference pixel (0,0) of this subset
  const float2* Gs = G2 + g.rP + (cx - M - g.rX0);

  double* crec = (METHOD == 1 && p.cache)
                     ? p.cache + ((size_t)iy * p.lat.nx + ix0 + warp) * kIcgnCacheStride
                     : nullptr;
  auto store_fail = [&](int code) {
    if (crec && lane == 0) crec[0] = 1.0 + code;
  };
  WarpConst& C = s_const[warp];
  double fbar, nf;
  double hinv[6] = {0, 0, 0, 0, 0, 0};
  const double tag = crec ? crec[0] : 0.0;
  if (tag != 0.0) {  // reference-side constants of this POI from an earlier pair
    if (tag != 1.0) {
      fail((int)tag - 1);
      return;
    }
    fbar = crec[1];
    nf = crec[2];
    if (lane == 0) C.scf = crec[3];
    if (lane < 12) (lane < 6 ? C.A[lane] : C.S[lane - 6]) = crec[4 + lane];
    if (lane < 6)
#pragma unroll
      for (int j = 0; j < 6; ++j) hinv[j] = crec[16 + 6 * lane + j];
    if (lane == 0) C.nf = nf;
  } else {
  // ---- one precompute pass: exact subset_stats sums (fp64) and, for IC-GN,
  // the reference-side update constants in fp32 per lane (<= npl terms):
  // sum f*sd, sum sd, and the Hessian moments of sd = (2 grad) x {1,dx,dy}.
  // A = sum (f - fbar) sd = sum f sd - fbar sum sd needs no second pass.
  {
    double sf = 0.0, sff = 0.0;
    float a[30];
#pragma unroll
    for (int j = 0; j < 30; ++j) a[j] = 0.f;
    Walk w = wk;
    for (int i = 0; i < w.npl; ++i) {
      if (i < w.npl - 1 || w.last_valid) {
        const float* q = Rs + w.roff;
        const float f = q[0];
        sf += (double)f;
        sff = fma((double)f, (double)f, sff);
        if (METHOD == 1) {
          const float2 gg = Gs[w.roff];
          const float ga = gg.x, gb = gg.y;  // 2 * gradient (exact)
          const float dx = w.dxf, dy = w.dyf;
          const float w6[6] = {1.f, dx, dy, dx * dx, dx * dy, dy * dy};
          const float aa = ga * ga, ab = ga * gb, bb = gb * gb;
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            a[j] = fmaf(aa, w6[j], a[j]);
            a[6 + j] = fmaf(ab, w6[j], a[6 + j]);
            a[12 + j] = fmaf(bb, w6[j], a[12 + j]);
          }
          const float fga = f * ga, fgb = f * gb;
          a[18] += fga;
          a[19] = fmaf(fga, dx, a[19]);
          a[20] = fmaf(fga, dy, a[20]);
          a[21] += fgb;
          a[22] = fmaf(fgb, dx, a[22]);
          a[23] = fmaf(fgb, dy, a[23]);
          a[24] += ga;
          a[25] = fmaf(ga, dx, a[25]);
          a[26] = fmaf(ga, dy, a[26]);
          a[27] += gb;
          a[28] = fmaf(gb, dx, a[28]);
          a[29] = fmaf(gb, dy, a[29]);
        }
      }
      w.advance();
    }
    sf = warp_sum1(sf);
    sff = warp_sum1(sff);
    double vfn;  // sum of squared centred values (subset_stats' norm^2, correlation.cpp:27-36)
    if (std::is_floating_point<Pix>::value) {
      // fractional levels: the sums are not exact, so the norm takes the
      // reference's second pass over the centred values
      const double mean = sf / (double)n;
      double s2 = 0.0;
      Walk w2 = wk;
      for (int i = 0; i < w2.npl; ++i) {
        if (i < w2.npl - 1 || w2.last_valid) {
          const double c = (double)Rs[w2.roff] - mean;
          s2 = fma(c, c, s2);
        }
        w2.advance();
      }
      vfn = warp_sum1(s2);
    } else {  // integer levels: n sum f^2 - (sum f)^2 is exact
      vfn = (double)((int64_t)n * (int64_t)sff - (int64_t)sf * (int64_t)sf) / (double)n;
    }
    if (!(vfn > 0.0)) {  // constant subset (exact test for integer levels)
      fail(METHOD == 1 ? DICB200_POI_DEGENERATE_TEXTURE : DICB200_POI_DEGENERATE_SUBSET);
      store_fail(DICB200_POI_DEGENERATE_TEXTURE);
      return;
    }
    fbar = sf / (double)n;  // correlation.cpp:25: exact sum / n
    nf = sqrt(vfn);
    if (lane == 0) {
      C.scf = sf - (double)n * fbar;  // sum of centred values
      C.nf = nf;
    }
    if (METHOD == 1) {
      double v32[32];
#pragma unroll
      for (int j = 0; j < 30; ++j) v32[j] = a[j];
      v32[30] = v32[31] = 0.0;
      const double r = warp_transpose_sum<32>(v32);  // lane l holds total l
      // lanes 18..23: sum f sd (x2), 24..29: sum sd (x2)
      if (lane >= 24 && lane < 30) C.S[lane - 24] = 0.5 * r;
      __syncwarp();
      if (lane >= 18 && lane < 24) C.A[lane - 18] = 0.5 * r - fbar * C.S[lane - 18];
      double mo[18];
#pragma unroll
      for (int j = 0; j < 18; ++j) mo[j] = __shfl_sync(0xffffffffu, r, j);
      double h[6];
      hessian_row(mo, 0.25, lane, h);
      double hf2 = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) hf2 += h[j] * h[j];
      bool pd;
      warp_cholesky_inverse(h, hinv, pd);
      double if2 = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) if2 += lane < 6 ? hinv[j] * hinv[j] : 0.0;
      hf2 = warp_sum1(lane < 6 ? hf2 : 0.0);
      if2 = warp_sum1(if2);
      // cond(H) <= ||H||_F ||H^-1||_F; exact eigenvalues only when inconclusive (subpixel.cpp:215-219)
      int accept = pd && sqrt(hf2) * sqrt(if2) < 1e12;
      if (!accept && pd) {
        if (lane == 0) {
          double H[36];
          assemble_hessian(mo, 0.25, H);
          double lo, hi;
          jacobi6_minmax(H, &lo, &hi);
          accept = lo > 0.0 && hi / lo < 1e12;
        }
        accept = __shfl_sync(0xffffffffu, accept, 0);
      }
      if (!accept) {
        fail(DICB200_POI_DEGENERATE_TEXTURE);
        store_fail(DICB200_POI_DEGENERATE_TEXTURE);
        return;
      }
      if (crec) {  // keep this POI's constants for the next pair on the same reference
        __syncwarp();
        if (lane == 0) {
          crec[1] = fbar;
          crec[2] = nf;
          crec[3] = C.scf;
        }
        if (lane < 12) crec[4 + lane] = lane < 6 ? C.A[lane] : C.S[lane - 6];
        if (lane < 6)
#pragma unroll
          for (int j = 0; j < 6; ++j) crec[16 + 6 * lane + j] = hinv[j];
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          crec[0] = 1.0;
        }
      }
    }
  }
  }  // precompute
  const float fbarf = (float)fbar;
  __syncwarp();

  // ---- iterations (all lanes hold the same warp parameters) ----
  double P[6] = {(double)idx, 0.0, 0.0, (double)idy, 0.0, 0.0};  // u, ux, uy, v, vx, vy
  int iterations = 0, converged = 0, done = 0;
  const double n_d = (double)n, inv_n = 1.0 / n_d;
  const double lim = (double)(M + 2);
  PassCtx pc;
  pc.T = T;
  pc.Rs = Rs;
  pc.Gs = Gs;
  pc.tP = g.tP;
  pc.rP = g.rP;
  pc.offx = (float)(bx - g.tX0);
  pc.offy = (float)(by - g.tY0);
  pc.ioffx = bx - g.tX0;
  pc.ioffy = by - g.tY0;
  pc.fbar = fbarf;
  pc.wn.w = T;
  pc.wn.S = min(g.tP, g.tH);
  pc.wn.P = g.tP;
  pc.wn.ox = g.tX0;
  pc.wn.oy = g.tY0;
  pc.bx = bx;
  pc.by = by;
  FixedCtx fc;
  if (FIXED) {
    const uint32_t t2b = smem_addr(T2);
    fc.t2 = t2b + (uint32_t)(((pc.ioffy - kFixedK) * FG::TP + (pc.ioffx - kFixedK)) * 8) -
            kMagicBits * (uint32_t)((FG::TP + 1) * 8);
    // the node pass's window [ioff - M, ioff + M]^2 lies inside the staged pairs
    // whenever the first iteration is `fast`; otherwise (an integer estimate far
    // from the strip's median) the address is parked on the region's origin
    const bool tn_in = pc.ioffx - M >= 0 && pc.ioffx + M < FG::TP && pc.ioffy - M >= 0 && pc.ioffy + M <= FG::TH - 2;
    fc.tn = t2b + (tn_in ? (uint32_t)(((pc.ioffy - M) * FG::TP + (pc.ioffx - M)) * 8) : 0u);
    fc.g2 = smem_addr(Gs);
    fc.r = smem_addr(Rs);
    fc.fbar = fbarf;
  }
  double zncc = 0.0;
  int status = DICB200_POI_OK;
  bool force_slow = false;  // fixed passes: exact min == max recheck on the checked path
  for (int iter = 1;; ++iter) {
    const bool final_pass = iter > p.max_iter || done;
    {  // check_guard (subpixel.cpp:134-141)
      const double ccx = cx + P[0], ccy = cy + P[3];
      if (!(ccx >= lim && ccx <= p.tgt.width - 1 - lim && ccy >= lim && ccy <= p.tgt.height - 1 - lim)) {
        status = DICB200_POI_DRIFTED;
        break;
      }
    }
    pc.ul = (float)(P[0] - idx);
    pc.vl = (float)(P[3] - idy);
    pc.ux = (float)P[1];
    pc.uy = (float)P[2];
    pc.vx = (float)P[4];
    pc.vy = (float)P[5];
    const bool grads = METHOD == 0 && !final_pass;
    bool fast;
    {
      const float Mf = (float)M;
      const float ex = fabsf(Mf + Mf * pc.ux) + fabsf(Mf * pc.uy), ey = fabsf(Mf * pc.vx) + fabsf(Mf + Mf * pc.vy);
      const float lo_x = pc.ul - ex, hi_x = pc.ul + ex, lo_y = pc.vl - ey, hi_y = pc.vl + ey;
      // taps beyond the sample's cell: bilinear +-1 (NR central differences +-2); bicubic -1 / +2
      const float mg = (grads || INTERP == DICB200_INTERP_BICUBIC) ? 2.0f : 1.0f;
      fast = pc.offx + lo_x - mg >= 0.0f && pc.offx + hi_x + mg + 1.0f <= (float)(g.tP - 1) &&
             pc.offy + lo_y - mg >= 0.0f && pc.offy + hi_y + mg + 1.0f <= (float)(g.tH - 1) &&
             (float)bx + lo_x - mg >= 0.0f && (float)bx + hi_x + mg <= (float)(p.tgt.width - 1) &&
             (float)by + lo_y - mg >= 0.0f && (float)by + hi_y + mg <= (float)(p.tgt.height - 1);
    }
    constexpr int NV = METHOD == 1 ? 9 : 39;
    float acc[NV];
    int bad = 0;
    float gmin, gmax;
    // fixed passes also need the shifted sample coordinates >= 1 (fixed_tap)
    const bool fixed_fast = FIXED && fast && !force_slow &&
                            pc.ul - fabsf((float)M + (float)M * pc.ux) - fabsf((float)M * pc.uy) + (float)kFixedK >= 1.0f &&
                            pc.vl - fabsf((float)M * pc.vx) - fabsf((float)M + (float)M * pc.vy) + (float)kFixedK >= 1.0f;
    if (fixed_fast) {
      fc.o = pk2(pc.ul + (float)kFixedK, pc.vl + (float)kFixedK);
      fc.A = pk2(1.0f + pc.ux, pc.vx);
      fc.B = pk2(pc.uy, 1.0f + pc.vy);
      if (final_pass)
        fixed_pass<FIXED ? FM : 1, FG::TP, FG::RP, 2>(fc, acc);
      else if (iter == 1)
        fixed_pass<FIXED ? FM : 1, FG::TP, FG::RP, 0>(fc, acc);
      else
        fixed_pass<FIXED ? FM : 1, FG::TP, FG::RP, 1>(fc, acc);
      gmin = 0.f;  // no min / max in the fixed passes: see the ng2 test below
      gmax = 1.f;
    } else if (FIXED) {  // checked path (global memory) only
      if (final_pass)
        pixel_pass<false, kFinal, Pix>(pc, p.tgt, wk, acc, bad, gmin, gmax);
      else
        pixel_pass<false, kIcgn, Pix>(pc, p.tgt, wk, acc, bad, gmin, gmax);
    } else if (final_pass) {
      if (fast && METHOD == 1 && INTERP == DICB200_INTERP_BILINEAR)
        final_pass_fast2(pc, wk, acc, gmin, gmax);
      else if (fast)
        pixel_pass<true, kFinal, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
      else
        pixel_pass<false, kFinal, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
    } else if (METHOD == 1) {
      // the integer start samples on the nodes: value = node for either interpolant
      if (fast && iter == 1)
        icgn_pass_node(pc, wk, acc, gmin, gmax);
      else if (fast && INTERP == DICB200_INTERP_BILINEAR)
        icgn_pass_fast2(pc, wk, acc, gmin, gmax);
      else if (fast)
        pixel_pass<true, kIcgn, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
      else
        pixel_pass<false, kIcgn, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
    } else {
      // nodes: bicubic's analytic gradient there is the central difference too
      if (fast && iter == 1)
        pixel_pass<true, kNr, Pix, true>(pc, p.tgt, wk, acc, bad, gmin, gmax);
      else if (fast)
        pixel_pass<true, kNr, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
      else
        pixel_pass<false, kNr, Pix, false, INTERP>(pc, p.tgt, wk, acc, bad, gmin, gmax);
    }
    // ---- warp reductions ----
    if (!fixed_fast) {  // the fixed passes track no min / max (see the ng2 test below)
      bad = __any_sync(0xffffffffu, bad);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        gmin = fminf(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
        gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      }
    }
    double t0, t1, t2 = 0.0, G6[6] = {0, 0, 0, 0, 0, 0};
    if (METHOD == 1 && !final_pass) {
      double v8[8] = {acc[0], acc[1], acc[3], acc[4], acc[5], acc[6], acc[7], acc[8]};
      const double r = warp_transpose_sum<8>(v8);
      t0 = tget<8>(r, 0);
      t1 = tget<8>(r, 1);
#pragma unroll
      for (int j = 0; j < 6; ++j) G6[j] = tget<8>(r, 2 + j);
    } else {
      double v4[4] = {acc[0], acc[1], acc[2], 0.0};
      const double r = warp_transpose_sum<4>(v4);
      t0 = tget<4>(r, 0);
      t1 = tget<4>(r, 1);
      t2 = tget<4>(r, 2);
    }
    const double delta = t0 * inv_n;                         // gbar - fbar
    const double ng2 = fmax(t1 - n_d * delta * delta, 0.0);  // sum (g - gbar)^2
    const double rng = rsqrt(ng2);                           // one MUFU + refinement, no divisions
    const double ng = ng2 * rng;
    if (fixed_fast && !(ng2 > 1e-4 * t1)) {
      // (nearly) constant warped target: decide "degenerate target" exactly
      // (min == max over the samples) on the checked path
      force_slow = true;
      --iter;
      continue;
    }
    force_slow = false;
    if (bad) {
      status = DICB200_POI_DRIFTED;
      break;
    }
    if (!(gmax > gmin) || !(ng > 0.0)) {
      status = DICB200_POI_DEGENERATE_TARGET;
      break;
    }
    if (final_pass) {
      zncc = (t2 - delta * C.scf) / (C.nf * ng);  // cross / (nf ng)
      break;
    }
    double step[6];
    bool finite;
    if (METHOD == 1) {
      // rhs = sum e_k sd_k (subpixel.cpp:328-333), expanded; step = H^-1 (-rhs)
      const double ratio = C.nf * rng;
      double rhs[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) rhs[j] = C.A[j] - ratio * (0.5 * G6[j] - delta * C.S[j]);
      hinv_step(hinv, rhs, step, finite);
      if (!finite) {
        status = DICB200_POI_DEGENERATE_TEXTURE;
        break;
      }
      const int st = compose_with_inverse(P, step);
      if (st != DICB200_POI_OK) {
        status = st;
        break;
      }
    } else {
      // NR (subpixel.cpp:247-279): gradient = -2/(nf ng) sum coeff J, H = 2/ng^2 sum J J^T,
      // additive update
      const double kap = (t2 - delta * C.scf) / ng2;  // cross / ng^2
      const double scale = -2.0 / (C.nf * ng);
      double v32[32], v4[4];
#pragma unroll
      for (int j = 0; j < 32; ++j) v32[j] = acc[3 + j];
#pragma unroll
      for (int j = 0; j < 4; ++j) v4[j] = acc[35 + j];
      const double ra = warp_transpose_sum<32>(v32), rb2 = warp_transpose_sum<4>(v4);
      double grad[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const double cj = tget<32>(ra, j), gj = tget<32>(ra, 6 + j), sj = tget<32>(ra, 12 + j);
        grad[j] = scale * (cj - kap * (gj - delta * sj));
      }
      double mo[18];
#pragma unroll
      for (int j = 0; j < 14; ++j) mo[j] = tget<32>(ra, 18 + j);
#pragma unroll
      for (int j = 0; j < 4; ++j) mo[14 + j] = tget<4>(rb2, j);
      double h[6], hi6[6];
      hessian_row(mo, 2.0 / ng2, lane, h);
      bool pd;
      warp_cholesky_inverse(h, hi6, pd);
      hinv_step(hi6, grad, step, finite);  // step = H^-1 (-gradient)
      if (!pd || !finite) {
        status = DICB200_POI_DEGENERATE_SUBSET;
        break;
      }
#pragma unroll
      for (int j = 0; j < 6; ++j) P[j] += step[j];
    }
    if (fabs(warp_det(P)) < 1e-8) {
      status = DICB200_POI_WARP_NOT_INVERTIBLE;
      break;
    }
    iterations = iter;
    if (fmax(fabs(step[0]), fabs(step[3])) < p.tol) {
      converged = 1;
      done = 1;
    }
  }
  if (lane == 0) {
    if (status == DICB200_POI_OK) {
      rec->u = P[0];
      rec->v = P[3];
      rec->zncc = zncc;
      rec->iterations = iterations;
      rec->converged = converged;
    } else {
      rec->status = status;
      rec->converged = 0;
    }
  }
}

}  // namespace

static size_t strip_smem(int M, int step, int spc, int method) {
  const int side = 2 * M + 1;
  const int span = step * (spc - 1);
  const size_t ref = (size_t)(side + 2) * (span + side + 2);
  const int kPad = pad_for(method);
  const size_t tgt = (size_t)(side + 2 * kPad + 2 * kSpread) * (span + 2 * kSpread + side + 2 * kPad);
  return (size_t)4 * (((ref + tgt + 1) & ~(size_t)1) + (method == 1 ? 2 * ref : 0));
}

bool refine_plan(int M, int* ppt_out, int* nt_out) {
  *ppt_out = ((2 * M + 1) * (2 * M + 1) + 31) / 32;
  *nt_out = kNT;
  return M >= 1 && strip_smem(M, 1, 1, 1) <= 100 * 1024;
}

void icgn_cache_free(IcgnRefCache& c, cudaStream_t st, bool async) {
  for (void* b : {(void*)c.data, c.rimg, c.gimg, c.timg})
    if (b) async ? cudaFreeAsync(b, st) : cudaFree(b);
  c = IcgnRefCache{};
}

// ---- pre-converted staging images of the fixed-geometry IC-GN kernels ----
// The strips' TMA boxes then land in their final layout (no shared-memory
// conversion pass, no gradient pass, no block barriers): the reference as fp32
// and its central differences (2 grad f, zero outside the image — exactly the
// values the strip staging computed from its zero-filled region), and the
// target as vertical pairs (T[y][x], T[y+1][x]). Dense rows of `wp` elements.
template <typename Pix>
__device__ __forceinline__ float img_at(const ImageView& im, int x, int y) {
  return (x >= 0 && x < im.width && y >= 0 && y < im.height) ? gpx<Pix>(im, x, y) : 0.f;
}

template <typename Pix>
__global__ void __launch_bounds__(256) ref_images_kernel(ImageView im, int wp, float* R, float2* G) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= wp) return;
  const size_t o = (size_t)y * wp + x;
  R[o] = img_at<Pix>(im, x, y);
  G[o] = make_float2(img_at<Pix>(im, x + 1, y) - img_at<Pix>(im, x - 1, y),
                     img_at<Pix>(im, x, y + 1) - img_at<Pix>(im, x, y - 1));
}

// four pairs per thread (wp is a multiple of 4): 16-byte stores
template <typename Pix>
__global__ void __launch_bounds__(256) pair_image_kernel(ImageView im, int wp, float2* T2) {
  const int x = 4 * (blockIdx.x * blockDim.x + threadIdx.x), y = blockIdx.y;
  if (x >= wp) return;
  float a[4], b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[j] = img_at<Pix>(im, x + j, y);
    b[j] = img_at<Pix>(im, x + j, y + 1);
  }
  float4* d = reinterpret_cast<float4*>(T2 + (size_t)y * wp + x);
  d[0] = make_float4(a[0], b[0], a[1], b[1]);
  d[1] = make_float4(a[2], b[2], a[3], b[3]);
}

// NR launch order (bit-identical results: only the order in which strips start
// changes). A POI whose integer estimate correlates poorly is the one whose
// Newton walk runs long (C3: ~2 % of the POIs take 14-50 iterations against ~4
// for the rest, and a CTA lasts as long as its slowest warp), so strips are
// started in four buckets of their worst integer ZNCC, worst first: the long
// walks overlap the bulk instead of trailing it. One CTA: counts, offsets,
// scatter (order within a bucket is arbitrary).
__global__ void __launch_bounds__(1024) strip_order_kernel(const dicb200_poi_record* rec, int nx, int rows, int spc,
                                                           int* order) {
  __shared__ int cnt[4], off[4];
  const int nsx = (nx + spc - 1) / spc, ns = nsx * rows;
  auto bucket = [&](int st) {
    const int iy = st / nsx, ix0 = (st % nsx) * spc;
    float worst = 1.0f;
    for (int j = 0; j < spc && ix0 + j < nx; ++j) {
      const dicb200_poi_record& r = rec[(size_t)iy * nx + ix0 + j];
      if (r.status == DICB200_POI_OK && r.zncc == r.zncc) worst = fminf(worst, (float)r.zncc);
    }
    return worst < 0.5f ? 0 : worst < 0.8f ? 1 : worst < 0.95f ? 2 : 3;
  };
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int st = threadIdx.x; st < ns; st += blockDim.x) atomicAdd(&cnt[bucket(st)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int b = 0; b < 4; ++b) {
      off[b] = a;
      a += cnt[b];
    }
  }
  __syncthreads();
  for (int st = threadIdx.x; st < ns; st += blockDim.x) order[atomicAdd(&off[bucket(st)], 1)] = st;
}

cudaError_t refine_launch(const RefineParams& p0, int dtype, cudaStream_t st, IcgnRefCache* cache, long ref_key) {
  const bool u8 = dtype == DICB200_U8, f64 = dtype == DICB200_F64;
  if (p0.n_records <= 0) return cudaSuccess;
  RefineParams p = p0;
  p.cache = nullptr;
  if (p.method == 1 && cache && ref_key >= 0) {
    // entries are filled lazily (tag 0 = not yet computed), so a new key only clears them
    const bool same = cache->key == ref_key && cache->ref == p.ref.data && cache->W == p.ref.width &&
                      cache->H == p.ref.height && cache->M == p.M && cache->x0 == p.lat.x0 &&
                      cache->y0 == p.lat.y0 && cache->step == p.lat.step && cache->nx == p.lat.nx &&
                      cache->ny == p.lat.ny;
    const size_t bytes = (size_t)p.lat.nx * p.lat.ny * kIcgnCacheStride * sizeof(double);
    cudaError_t e = cudaSuccess;
    if (!same) {
      cache->key = -1;
      if (cache->cap < bytes) {
        if (cache->data) cudaFreeAsync(cache->data, st);
        cache->data = nullptr;
        cache->cap = 0;
        e = cudaMallocAsync((void**)&cache->data, bytes, st);
        if (e != cudaSuccess) return e;
        cache->cap = bytes;
      }
      e = cudaMemsetAsync(cache->data, 0, bytes, st);
      if (e != cudaSuccess) return e;
      cache->key = ref_key;
      cache->ref = p.ref.data;
      cache->W = p.ref.width;
      cache->H = p.ref.height;
      cache->M = p.M;
      cache->x0 = p.lat.x0;
      cache->y0 = p.lat.y0;
      cache->step = p.lat.step;
      cache->nx = p.lat.nx;
      cache->ny = p.lat.ny;
    }
    p.cache = cache->data;
  }
  p.spc = kWarps;
  while (p.spc > 1 && strip_smem(p.M, p.lat.step, p.spc, p.method) > 110 * 1024) --p.spc;
  size_t smem = strip_smem(p.M, p.lat.step, p.spc, p.method);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  const int rows = p.n_records / p.lat.nx;
  cudaError_t e;
  // fixed-geometry IC-GN kernels for the BASELINE subset / lattice shapes
  // (C4: 41 px subsets every 5 px, C5: every 10 px)
  static const bool generic = std::getenv("DICB200_REFINE_GENERIC") != nullptr;
  TmaPair tm{};
  if (p.method == 1 && p.M == 20 && (p.lat.step == 10 || p.lat.step == 5) && !generic && !f64 &&
      p.interp == DICB200_INTERP_BILINEAR) {
    p.spc = kWarps;
    dim3 grid((p.lat.nx + p.spc - 1) / p.spc, rows);
    // TMA staging of the raw regions (falls back to per-thread loads when the
    // images do not meet the tensor-map layout rules)
    static const bool no_tma = std::getenv("DICB200_NO_TMA") != nullptr;
    const int es = u8 ? 1 : 2;
    auto boxes = [&](int rp, int tp, int rh, int th) {
      const int ae = 16 / es, rbw = ((rp + 2 * ae - 2) / ae) * ae, tbw = ((tp + 2 * ae - 2) / ae) * ae;
      return !no_tma &&
             tma_encode_2d(&tm.ref, p.ref.data, es, p.ref.width, p.ref.height, p.ref.pitch, rbw, rh) &&
             tma_encode_2d(&tm.tgt, p.tgt.data, es, p.tgt.width, p.tgt.height, p.tgt.pitch, tbw, th);
    };
    p.use_tma = p.lat.step == 10 ? boxes(FixedGeom<20, 10>::RP, FixedGeom<20, 10>::TP, FixedGeom<20, 10>::RH,
                                         FixedGeom<20, 10>::TH)
                                 : boxes(FixedGeom<20, 5>::RP, FixedGeom<20, 5>::TP, FixedGeom<20, 5>::RH,
                                         FixedGeom<20, 5>::TH);
    // pre-converted staging images (default; DICB200_REFINE_RAW_TMA=1: the raw
    // boxes converted in shared memory)
    static const bool raw_tma = std::getenv("DICB200_REFINE_RAW_TMA") != nullptr;
    void* own[3] = {nullptr, nullptr, nullptr};
    if (!no_tma && !raw_tma) {
      const int W = p.ref.width, H = p.ref.height, wp = (W + 3) & ~3;
      const size_t px = (size_t)wp * H;
      void *rimg = nullptr, *gimg = nullptr, *timg = nullptr;
      bool ref_ready = false;
      e = cudaSuccess;
      if (cache) {
        if (cache->img_cap < px) {
          for (void** b : {&cache->rimg, &cache->gimg, &cache->timg})
            if (*b) {
              cudaFreeAsync(*b, st);
              *b = nullptr;
            }
          cache->img_cap = 0;
          cache->img_key = -1;
          e = cudaMallocAsync(&cache->rimg, px * 4, st);
          if (e == cudaSuccess) e = cudaMallocAsync(&cache->gimg, px * 8, st);
          if (e == cudaSuccess) e = cudaMallocAsync(&cache->timg, px * 8, st);
          if (e != cudaSuccess) return e;
          cache->img_cap = px;
        }
        rimg = cache->rimg, gimg = cache->gimg, timg = cache->timg;
        ref_ready = ref_key >= 0 && cache->img_key == ref_key && cache->img_ref == p.ref.data;
      } else {
        e = cudaMallocAsync(&own[0], px * 4, st);
        if (e == cudaSuccess) e = cudaMallocAsync(&own[1], px * 8, st);
        if (e == cudaSuccess) e = cudaMallocAsync(&own[2], px * 8, st);
        if (e != cudaSuccess) return e;
        rimg = own[0], gimg = own[1], timg = own[2];
      }
      TmaPair pm{};
      const int rp = p.lat.step == 10 ? FixedGeom<20, 10>::RP : FixedGeom<20, 5>::RP;
      const int tp = p.lat.step == 10 ? FixedGeom<20, 10>::TP : FixedGeom<20, 5>::TP;
      const int rh = FixedGeom<20, 10>::RH, th = FixedGeom<20, 10>::TH;
      if (tma_encode_2d_f(&pm.ref, rimg, 4, W, H, wp, rp, rh) && tma_encode_2d_f(&pm.aux, gimg, 8, W, H, wp, rp, rh) &&
          tma_encode_2d_f(&pm.tgt, timg, 8, W, H, wp, tp, th - 1)) {
        const dim3 ig((wp + 255) / 256, H);
        if (!ref_ready) {
          u8 ? ref_images_kernel<uint8_t><<<ig, 256, 0, st>>>(p.ref, wp, (float*)rimg, (float2*)gimg)
             : ref_images_kernel<uint16_t><<<ig, 256, 0, st>>>(p.ref, wp, (float*)rimg, (float2*)gimg);
          count_launch();
          if (cache) {
            cache->img_key = ref_key;
            cache->img_ref = p.ref.data;
          }
        }
        const dim3 pg((wp / 4 + 255) / 256, H);
        u8 ? pair_image_kernel<uint8_t><<<pg, 256, 0, st>>>(p.tgt, wp, (float2*)timg)
           : pair_image_kernel<uint16_t><<<pg, 256, 0, st>>>(p.tgt, wp, (float2*)timg);
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        tm = pm;
        p.use_tma = 2;
      }
    }
    // DICB200_REFINE_SMEM_PAD (experiments): extra dynamic shared memory per CTA (occupancy study)
    static const size_t smem_pad = std::getenv("DICB200_REFINE_SMEM_PAD") ? std::atoi(std::getenv("DICB200_REFINE_SMEM_PAD")) : 0;
    auto go = [&](auto k, size_t sm) {
      sm += smem_pad;
      e = set_dyn_smem(k, sm);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      if (e == cudaSuccess) k<<<grid, kNT, sm, st>>>(p, tm);
    };
    if (p.lat.step == 10)
      u8 ? go(refine_strip_kernel<uint8_t, 1, 20, 10>, FixedGeom<20, 10>::SMEM)
         : go(refine_strip_kernel<uint16_t, 1, 20, 10>, FixedGeom<20, 10>::SMEM);
    else
      u8 ? go(refine_strip_kernel<uint8_t, 1, 20, 5>, FixedGeom<20, 5>::SMEM)
         : go(refine_strip_kernel<uint16_t, 1, 20, 5>, FixedGeom<20, 5>::SMEM);
    count_launch();
    for (void* b : own)
      if (b) cudaFreeAsync(b, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  dim3 grid((p.lat.nx + p.spc - 1) / p.spc, rows);
  auto go = [&](auto k) {
    e = set_dyn_smem(k, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) k<<<grid, kNT, smem, st>>>(p, tm);
  };
  const bool cubic = p.interp == DICB200_INTERP_BICUBIC;
  int* order = nullptr;
  if (p.method == 0 && grid.x * grid.y > 1 && std::getenv("DICB200_NR_GRID_ORDER") == nullptr) {
    e = cudaMallocAsync((void**)&order, (size_t)grid.x * grid.y * sizeof(int), st);
    if (e != cudaSuccess) return e;
    strip_order_kernel<<<1, 1024, 0, st>>>(p.rec, p.lat.nx, rows, p.spc, order);
    count_launch();
    p.order = order;
  }
  if (f64) {  // fractional gray levels: fp32 gathers of the fp64 images, fp64 sums
    if (p.method == 0)
      cubic ? go(refine_strip_kernel<double, 0, 0, 0, 1>) : go(refine_strip_kernel<double, 0>);
    else
      cubic ? go(refine_strip_kernel<double, 1, 0, 0, 1>) : go(refine_strip_kernel<double, 1>);
  } else if (p.method == 0) {
    if (cubic)
      u8 ? go(refine_strip_kernel<uint8_t, 0, 0, 0, 1>) : go(refine_strip_kernel<uint16_t, 0, 0, 0, 1>);
    else
      u8 ? go(refine_strip_kernel<uint8_t, 0>) : go(refine_strip_kernel<uint16_t, 0>);
  } else {
    if (cubic)
      u8 ? go(refine_strip_kernel<uint8_t, 1, 0, 0, 1>) : go(refine_strip_kernel<uint16_t, 1, 0, 0, 1>);
    else
      u8 ? go(refine_strip_kernel<uint8_t, 1>) : go(refine_strip_kernel<uint16_t, 1>);
  }
  count_launch();
  if (order) cudaFreeAsync(order, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dicb200
