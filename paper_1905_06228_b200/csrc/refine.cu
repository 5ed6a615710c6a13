// K3/K4 — sub-pixel refinement: IC-GN (icgn_precompute + refine_icgn,
// subpixel.cpp:191-222, 301-359) and Newton-Raphson (refine_nr,
// subpixel.cpp:224-299), first-order warp, bilinear interpolation
// (interp_bilinear / grad_bilinear, subpixel.cpp:59-128).
//
// One CTA (8 warps) per POI; every thread owns PPT subset pixels in registers
// for the whole solve. The target neighbourhood of the integer estimate is
// staged once in shared memory as fp32 (taps that drift outside it fall back
// to global loads), so each iteration is ONE pass over the pixels: warp +
// gather + bilinear (+ gradient for NR) in fp32 on subset-local coordinates,
// per-thread fp32 partials of every sum the update needs, one block
// reduction in fp64, and warp 0 doing the 6x6 algebra in fp64.
//
// The reference forms e_k = f_k - (nf/ng)(g_k - gbar) (IC-GN, :331) and
// coeff_k = f_k - (cross/ng^2)(g_k - gbar) (NR, :258) per pixel, which needs
// gbar and ng before the update sums (three passes). Here the update sums are
// expanded exactly,
//   sum e_k sd_k = sum f_k sd_k - (nf/ng) [ sum g'_k sd_k - (gbar - fbar) sum sd_k ],
// with g' = g - fbar, so one pass suffices; the reference-side sums
// (sum f sd, sum sd, and the Hessian) are precomputed in fp64 (the Hessian
// EXACTLY: (2 grad)^2 * {1,dx,dy,dx^2,dxdy,dy^2} are integers < 2^53).
// Convergence test, failure semantics (guard band M+2, domain checks,
// |det| < 1e-8, LDLT failure, non-finite step, degenerate target) and the
// final re-sample + ZNCC follow subpixel.cpp / pipeline.cpp:82-133.
#include "common.cuh"
#include "linalg.cuh"
#include "refine.cuh"

namespace dicb200 {

namespace {

constexpr int kNT = 256;
constexpr int kWarps = kNT / 32;
constexpr int kPad = 4;
constexpr int kRedMax = 40;

template <typename Pix>
__device__ __forceinline__ float gpx(const ImageView& im, int x, int y) {
  return (float)__ldg(reinterpret_cast<const Pix*>(im.data) + (size_t)y * im.pitch + x);
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
  const int lx = x0 - wn.ox, ly = y0 - wn.oy;
  float f00, f10, f01, f11;
  if ((unsigned)lx < (unsigned)(wn.S - 1) && (unsigned)ly < (unsigned)(wn.S - 1)) {
    const float* p = wn.w + ly * wn.P + lx;
    f00 = p[0];
    f10 = p[1];
    f01 = p[wn.P];
    f11 = p[wn.P + 1];
  } else {
    const int x1 = min(x0 + 1, im.width - 1), y1 = min(y0 + 1, im.height - 1);
    f00 = gpx<Pix>(im, x0, y0);
    f10 = gpx<Pix>(im, x1, y0);
    f01 = gpx<Pix>(im, x0, y1);
    f11 = gpx<Pix>(im, x1, y1);
  }
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
  float ax = 0.f, ay = 0.f;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    if (wy[b] == 0.0f) continue;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      if (wx[a] == 0.0f) continue;
      const int i = x0 + a, j = y0 + b;
      const float w = wx[a] * wy[b] * 0.5f;
      ax = fmaf(w, tap<Pix>(wn, im, i + 1, j) - tap<Pix>(wn, im, i - 1, j), ax);
      ay = fmaf(w, tap<Pix>(wn, im, i, j + 1) - tap<Pix>(wn, im, i, j - 1), ay);
    }
  }
  gx = ax;
  gy = ay;
  return true;
}

__device__ __forceinline__ double warp_sum1(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-thread partials -> per-warp sums in rb[warp][base + i] (one value live at a time).
template <int NV, typename T>
__device__ __forceinline__ void block_partials(const T (&v)[NV], double (*rb)[kRedMax], int base = 0) {
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double s = warp_sum1((double)v[i]);
    if ((threadIdx.x & 31) == 0) rb[threadIdx.x >> 5][base + i] = s;
  }
}

// After a __syncthreads: warp 0's lanes total the per-warp sums into tot[0..nv).
__device__ __forceinline__ void warp0_totals(double (*rb)[kRedMax], double* tot, int nv) {
  for (int j = threadIdx.x & 31; j < nv; j += 32) {
    double s = rb[0][j];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) s += rb[w][j];
    tot[j] = s;
  }
  __syncwarp();
}

struct State {
  double p[6];  // u, ux, uy, v, vx, vy (subpixel.hpp:13-16)
  int status, done, iterations, converged;
  double zncc;
  // reference-side constants
  double fbar, nf, scf;   // mean, ||f - fbar||, sum of the fp32 centred values
  double A[6], Ssd[6];    // sum cf*sd, sum sd (IC-GN)
  double Hinv[36];        // IC-GN: H^-1 (H exact)
};

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
  const double i00 = __ddiv_rn(a11, det), i01 = __ddiv_rn(-a01, det);
  const double i10 = __ddiv_rn(-a10, det), i11 = __ddiv_rn(a00, det);
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

// warp 0: finish one iteration from the totals; lane 0 commits the state.
__device__ void finish_step(State& S, const double* step, bool finite, int fail_code, int iter, double tol,
                            bool icgn) {
  int st = finite ? DICB200_POI_OK : fail_code;
  if (st == DICB200_POI_OK) {
    if (icgn) {
      st = compose_with_inverse(S.p, step);
    } else {
      for (int j = 0; j < 6; ++j) S.p[j] += step[j];
    }
  }
  if (st == DICB200_POI_OK && fabs(warp_det(S.p)) < 1e-8) st = DICB200_POI_WARP_NOT_INVERTIBLE;
  S.status = st;
  if (st == DICB200_POI_OK) {
    S.iterations = iter;
    if (fmax(fabs(step[0]), fabs(step[3])) < tol) {
      S.converged = 1;
      S.done = 1;
    }
  } else {
    S.done = 1;
  }
}

// Fast-path bilinear sample from the staged window (no checks: the caller
// proved the whole warped subset lies inside the window and the image).
template <int WP>
__device__ __forceinline__ float sample_fast(const float* w, float wx, float wy) {
  const float flx = floorf(wx), fly = floorf(wy);
  const float fx = wx - flx, fy = wy - fly;
  const float* q = w + (int)fly * WP + (int)flx;
  const float f00 = q[0], f10 = q[1], f01 = q[WP], f11 = q[WP + 1];
  const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f00 + f11) - f10 - f01;
  return fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
}

// Warp-parallel Cholesky of the SPD 6x6 H (lane i < 6 holds row i in h[]),
// then lane c < 6 solves H x = e_c: returns row c of H^-1 in hinv[] (H^-1 is
// symmetric). pd = all pivots > 0. Runs on all 32 lanes of one warp.
__device__ void warp_cholesky_inverse(double (&h)[6], double (&hinv)[6], bool& pd) {
  const int lane = threadIdx.x & 31;
  double L[6][6];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    // pivot on lane j: d = h[j][j] - sum_k<j L[j][k]^2 (lane j's h[k<j] already hold L[j][k])
    double d = h[j];
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) d -= h[k2] * h[k2];
    d = __shfl_sync(0xffffffffu, d, j);
    ok = ok && d > 0.0;
    const double ljj = sqrt(d > 0.0 ? d : 1.0);
    // broadcast row j of L (k < j) and finish column j on lanes i > j
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) L[j][k2] = __shfl_sync(0xffffffffu, h[k2], j);
    L[j][j] = ljj;
    double v = h[j];
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) v -= h[k2] * L[j][k2];
    if (lane > j) h[j] = v / ljj;
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
    y[i] = v / L[i][i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k2 = i + 1; k2 < 6; ++k2) v -= L[k2][i] * hinv[k2];
    hinv[i] = v / L[i][i];
  }
  pd = ok;
}

template <typename Pix, int PPT, int METHOD, int WP>
__global__ void __launch_bounds__(kNT, 3) refine_kernel(RefineParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double rb[kWarps][kRedMax];
  __shared__ double tot[kRedMax];
  __shared__ float rmm[kWarps][2];
  __shared__ double shH[36];
  __shared__ Ldlt6 shL;
  __shared__ State S;
  const int k = blockIdx.x;
  dicb200_poi_record* rec = p.rec + k;
  if (rec->status != DICB200_POI_OK) return;  // integer stage failed: record stays
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = p.M, side = 2 * M + 1, n = side * side;
  const int iy = p.row_begin + k / p.lat.nx, ix = k % p.lat.nx;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy);
  const int idx = rec->integer_dx, idy = rec->integer_dy;
  const int bx = cx + idx, by = cy + idy;

  if (METHOD == 1 && (cx - M - 1 < 0 || cx + M + 1 > p.ref.width - 1 || cy - M - 1 < 0 ||
                      cy + M + 1 > p.ref.height - 1)) {
    if (tid == 0) {
      rec->status = DICB200_POI_BORDER_GRADIENTS;  // subpixel.cpp:193-195
      rec->converged = 0;
    }
    return;
  }

  // ---- stage the target neighbourhood (fp32, pitch WP) ----
  Win wn;
  wn.S = side + 2 * kPad;
  wn.P = WP;
  wn.ox = bx - M - kPad;
  wn.oy = by - M - kPad;
  float* wbuf = reinterpret_cast<float*>(smem_raw);
  for (int i = tid; i < wn.S * WP; i += kNT) {
    const int ly = i / WP, lx = i - ly * WP;
    const int gx = wn.ox + lx, gy = wn.oy + ly;
    float v = 0.f;
    if (lx < wn.S && gx >= 0 && gx < p.tgt.width && gy >= 0 && gy < p.tgt.height) v = gpx<Pix>(p.tgt, gx, gy);
    wbuf[i] = v;
  }
  wn.w = wbuf;

  // ---- reference pixels: registers ----
  float dxf[PPT], dyf[PPT], cf[PPT], gxr[PPT], gyr[PPT];
  {
    double s2[2] = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int kk = tid + i * kNT;
      const int r = kk / side, c = kk - r * side;
      dxf[i] = (float)(c - M);
      dyf[i] = (float)(r - M);
      cf[i] = gxr[i] = gyr[i] = 0.f;
      if (kk < n) {
        const int x = cx + c - M, y = cy + r - M;
        const float f = gpx<Pix>(p.ref, x, y);
        cf[i] = f;
        if (METHOD == 1) {
          gxr[i] = 0.5f * (gpx<Pix>(p.ref, x + 1, y) - gpx<Pix>(p.ref, x - 1, y));
          gyr[i] = 0.5f * (gpx<Pix>(p.ref, x, y + 1) - gpx<Pix>(p.ref, x, y - 1));
        }
        s2[0] += (double)f;
        s2[1] += (double)f * (double)f;
      } else {
        dxf[i] = dyf[i] = 0.f;  // padding slots sample the centre (weight 0 everywhere)
      }
    }
    block_partials<2>(s2, rb);
    __syncthreads();
    if (warp == 0) warp0_totals(rb, tot, 2);
    __syncthreads();
    const int64_t sf = (int64_t)tot[0], sff = (int64_t)tot[1];
    const int64_t vf = (int64_t)n * sff - sf * sf;
    if (vf <= 0) {  // constant subset
      if (tid == 0) {
        rec->status = METHOD == 1 ? DICB200_POI_DEGENERATE_TEXTURE : DICB200_POI_DEGENERATE_SUBSET;
        rec->converged = 0;
      }
      return;
    }
    const double mean = tot[0] / (double)n;  // correlation.cpp:25: exact sum / n
#pragma unroll
    for (int i = 0; i < PPT; ++i) cf[i] = (tid + i * kNT < n) ? (float)((double)cf[i] - mean) : 0.f;
    if (tid == 0) {
      S.fbar = mean;
      S.nf = sqrt((double)vf / (double)n);
    }
  }
  __syncthreads();  // rb reuse + S.fbar/nf visible

  double hinv[6] = {0, 0, 0, 0, 0, 0};  // IC-GN, warp 0 lanes 0..5: row `lane` of H^-1
  if (METHOD == 1) {
    // ---- icgn_precompute: exact Hessian moments, sum f*sd, sum sd ----
#pragma unroll 1
    for (int grp = 0; grp < 3; ++grp) {
      double m6[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        const double ga = 2.0 * gxr[i], gb = 2.0 * gyr[i];  // integers
        const double q = grp == 0 ? ga * ga : (grp == 1 ? ga * gb : gb * gb);
        const double dx = dxf[i], dy = dyf[i];
        m6[0] += q;
        m6[1] = fma(q, dx, m6[1]);
        m6[2] = fma(q, dy, m6[2]);
        m6[3] = fma(q, dx * dx, m6[3]);
        m6[4] = fma(q, dx * dy, m6[4]);
        m6[5] = fma(q, dy * dy, m6[5]);
      }
      block_partials<6>(m6, rb, grp * 6);
    }
    {
      double a7[7] = {0, 0, 0, 0, 0, 0, 0};
      double s6[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        const double c = cf[i], gx = gxr[i], gy = gyr[i], dx = dxf[i], dy = dyf[i];
        const double cgx = c * gx, cgy = c * gy;  // exact (float x float)
        a7[0] += c;
        a7[1] += cgx;
        a7[2] += cgx * dx;
        a7[3] += cgx * dy;
        a7[4] += cgy;
        a7[5] += cgy * dx;
        a7[6] += cgy * dy;
        s6[0] += gx;
        s6[1] += gx * dx;
        s6[2] += gx * dy;
        s6[3] += gy;
        s6[4] += gy * dx;
        s6[5] += gy * dy;
      }
      block_partials<7>(a7, rb, 18);
      block_partials<6>(s6, rb, 25);
    }
    __syncthreads();
    if (warp == 0) {
      warp0_totals(rb, tot, 31);
      // H (exact) row `lane` -> warp Cholesky -> row `lane` of H^-1 in registers
      const int map[6][6][2] = {
          {{0, 0}, {0, 1}, {0, 2}, {1, 0}, {1, 1}, {1, 2}}, {{0, 1}, {0, 3}, {0, 4}, {1, 1}, {1, 3}, {1, 4}},
          {{0, 2}, {0, 4}, {0, 5}, {1, 2}, {1, 4}, {1, 5}}, {{1, 0}, {1, 1}, {1, 2}, {2, 0}, {2, 1}, {2, 2}},
          {{1, 1}, {1, 3}, {1, 4}, {2, 1}, {2, 3}, {2, 4}}, {{1, 2}, {1, 4}, {1, 5}, {2, 2}, {2, 4}, {2, 5}},
      };
      double h[6];
      const int row = lane < 6 ? lane : 0;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < 6; ++r)
          if (r == row) v = tot[map[r][j][0] * 6 + map[r][j][1]] * 0.25;
        h[j] = v;
      }
      double hf2 = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) hf2 += lane < 6 ? h[j] * h[j] : 0.0;
      bool pd;
      warp_cholesky_inverse(h, hinv, pd);
      double if2 = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) if2 += lane < 6 ? hinv[j] * hinv[j] : 0.0;
      hf2 = warp_sum1(hf2);
      if2 = warp_sum1(if2);
      // cond(H) <= ||H||_F ||H^-1||_F; exact eigenvalues only when inconclusive (subpixel.cpp:215-219)
      bool accept = pd && sqrt(hf2) * sqrt(if2) < 1e12;
      if (lane == 0) {
        if (!accept && pd) {
          assemble_hessian(tot, 0.25, shH);
          double lo, hi;
          jacobi6_minmax(shH, &lo, &hi);
          accept = lo > 0.0 && hi / lo < 1e12;
        }
        S.status = accept ? DICB200_POI_OK : DICB200_POI_DEGENERATE_TEXTURE;
        S.scf = tot[18];
        for (int j = 0; j < 6; ++j) {
          S.A[j] = tot[19 + j];
          S.Ssd[j] = tot[25 + j];
        }
      }
    }
  } else {
    double a[1] = {0.0};
#pragma unroll
    for (int i = 0; i < PPT; ++i) a[0] += (double)cf[i];
    block_partials<1>(a, rb);
    __syncthreads();
    if (warp == 0) {
      warp0_totals(rb, tot, 1);
      if (lane == 0) {
        S.scf = tot[0];
        S.status = DICB200_POI_OK;
      }
    }
  }
  if (tid == 0) {
    S.p[0] = (double)idx;
    S.p[1] = S.p[2] = 0.0;
    S.p[3] = (double)idy;
    S.p[4] = S.p[5] = 0.0;
    S.done = 0;
    S.iterations = 0;
    S.converged = 0;
  }
  __syncthreads();
  if (S.status != DICB200_POI_OK) {
    if (tid == 0) {
      rec->status = S.status;
      rec->converged = 0;
    }
    return;
  }

  const double n_d = (double)n;
  const float fbarf = (float)S.fbar;
  const double lim = (double)(M + 2);
  const float wofs = (float)(M + kPad);  // window coords = local coords + wofs

  for (int iter = 1;; ++iter) {
    const bool final_pass = iter > p.max_iter || S.done;
    const double u = S.p[0], ux = S.p[1], uy = S.p[2], v = S.p[3], vx = S.p[4], vy = S.p[5];
    {  // check_guard (subpixel.cpp:134-141), uniform
      const double ccx = cx + u, ccy = cy + v;
      if (!(ccx >= lim && ccx <= p.tgt.width - 1 - lim && ccy >= lim && ccy <= p.tgt.height - 1 - lim)) {
        if (tid == 0) {
          rec->status = DICB200_POI_DRIFTED;
          rec->converged = 0;
        }
        return;
      }
    }
    const float ul = (float)(u - idx), vl = (float)(v - idy);
    const float uxf = (float)ux, uyf = (float)uy, vxf = (float)vx, vyf = (float)vy;
    const bool grads = METHOD == 0 && !final_pass;
    // Fast path iff the warped subset's bounding box (+1 px, +2 px with gradients)
    // sits inside the staged window and the image domain: the affine map attains
    // its extremes at the corners (uniform decision).
    bool fast;
    {
      const float Mf = (float)M;
      const float ex = fabsf(Mf + Mf * uxf) + fabsf(Mf * uyf), ey = fabsf(Mf * vxf) + fabsf(Mf + Mf * vyf);
      const float lo_x = ul - ex, hi_x = ul + ex, lo_y = vl - ey, hi_y = vl + ey;
      const float mg = grads ? 2.0f : 1.0f;
      fast = lo_x - mg >= -wofs && hi_x + mg + 1.0f <= (float)(wn.S - 1) - wofs && lo_y - mg >= -wofs &&
             hi_y + mg + 1.0f <= (float)(wn.S - 1) - wofs && (float)bx + lo_x - mg >= 0.0f &&
             (float)bx + hi_x + mg <= (float)(p.tgt.width - 1) && (float)by + lo_y - mg >= 0.0f &&
             (float)by + hi_y + mg <= (float)(p.tgt.height - 1);
    }
    constexpr int NV = METHOD == 1 ? 9 : 39;
    float acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = 0.f;
    int bad = 0;
    float gmin = 3.0e38f, gmax = -3.0e38f;  // exact "constant subset" test (ng == 0 in the reference)
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const bool valid = tid + i * kNT < n;
      const float xl = fmaf(uyf, dyf[i], fmaf(uxf, dxf[i], dxf[i] + ul));
      const float yl = fmaf(vyf, dyf[i], fmaf(vxf, dxf[i], dyf[i] + vl));
      float g = 0.f, gx = 0.f, gy = 0.f;
      if (fast) {
        g = sample_fast<WP>(wn.w, xl + wofs, yl + wofs);
        if (grads) {
          // grad_bilinear on the window: nodes (x0..x0+1, y0..y0+1), central differences
          const float wx = xl + wofs, wy = yl + wofs;
          const float flx = floorf(wx), fly = floorf(wy);
          const float fx = wx - flx, fy = wy - fly;
          const float* q = wn.w + (int)fly * WP + (int)flx;
          const float dx00 = q[1] - q[-1], dx10 = q[2] - q[0], dx01 = q[WP + 1] - q[WP - 1], dx11 = q[WP + 2] - q[WP];
          const float dy00 = q[WP] - q[-WP], dy10 = q[WP + 1] - q[1 - WP], dy01 = q[2 * WP] - q[0],
                      dy11 = q[2 * WP + 1] - q[1];
          const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
          gx = 0.5f * (w00 * dx00 + w10 * dx10 + w01 * dx01 + w11 * dx11);
          gy = 0.5f * (w00 * dy00 + w10 * dy10 + w01 * dy01 + w11 * dy11);
        }
      } else if (valid) {
        bad |= !bilinear<Pix>(wn, p.tgt, bx, by, xl, yl, g);
        if (grads) bad |= !grad_bilinear<Pix>(wn, p.tgt, bx, by, xl, yl, gx, gy);
      }
      if (!valid) continue;
      gmin = fminf(gmin, g);
      gmax = fmaxf(gmax, g);
      const float gp = g - fbarf;
      acc[0] += gp;
      acc[1] = fmaf(gp, gp, acc[1]);
      if (final_pass || METHOD == 0) acc[2] = fmaf(cf[i], gp, acc[2]);
      if (METHOD == 1) {
        if (!final_pass) {
          const float tx = gp * gxr[i], ty = gp * gyr[i];
          acc[3] += tx;
          acc[4] = fmaf(tx, dxf[i], acc[4]);
          acc[5] = fmaf(tx, dyf[i], acc[5]);
          acc[6] += ty;
          acc[7] = fmaf(ty, dxf[i], acc[7]);
          acc[8] = fmaf(ty, dyf[i], acc[8]);
        }
      } else if (grads) {
        const float dx = dxf[i], dy = dyf[i];
        const float J[6] = {gx, gx * dx, gx * dy, gy, gy * dx, gy * dy};
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          acc[3 + j] = fmaf(cf[i], J[j], acc[3 + j]);
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
    }
    const int nv = final_pass ? 3 : (METHOD == 1 ? 9 : (grads ? 39 : 3));
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if (j < nv) {
        const double s2 = warp_sum1((double)acc[j]);
        if (lane == 0) rb[warp][j] = s2;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gmin = fminf(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
      gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    }
    if (lane == 0) {
      rmm[warp][0] = gmin;
      rmm[warp][1] = gmax;
    }
    const int any_bad = __syncthreads_or(bad);
    if (warp == 0) {
      warp0_totals(rb, tot, nv);
      float mn = rmm[0][0], mx = rmm[0][1];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) {
        mn = fminf(mn, rmm[w][0]);
        mx = fmaxf(mx, rmm[w][1]);
      }
      const double* t = tot;
      int st = DICB200_POI_OK;
      const double delta = t[0] / n_d;                           // gbar - fbar
      const double ng2 = fmax(t[1] - n_d * delta * delta, 0.0);  // sum (g - gbar)^2
      const double ng = sqrt(ng2);
      if (any_bad) st = DICB200_POI_DRIFTED;
      else if (!(mx > mn) || !(ng > 0.0)) st = DICB200_POI_DEGENERATE_TARGET;
      if (final_pass) {
        if (lane == 0) {
          S.status = st;
          S.zncc = (t[2] - delta * S.scf) / (S.nf * ng);  // cross / (nf ng)
          S.done = 2;
        }
      } else if (st != DICB200_POI_OK) {
        if (lane == 0) {
          S.status = st;
          S.done = 1;
        }
      } else if (METHOD == 1) {
        // rhs = sum e_k sd_k (subpixel.cpp:328-333), expanded; step = H^-1 (-rhs), lane i -> step_i
        const double ratio = S.nf / ng;
        double si = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) si = fma(hinv[j], -(S.A[j] - ratio * (t[3 + j] - delta * S.Ssd[j])), si);
        double step[6];
        bool finite = true;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          step[j] = __shfl_sync(0xffffffffu, si, j);
          finite = finite && isfinite(step[j]);
        }
        if (lane == 0) finish_step(S, step, finite, DICB200_POI_DEGENERATE_TEXTURE, iter, p.tol, true);
      } else if (lane == 0) {
        // NR (subpixel.cpp:247-271): gradient = -2/(nf ng) sum coeff J, H = 2/ng^2 sum J J^T
        const double cross = t[2] - delta * S.scf;
        const double kappa = cross / ng2;
        double neg[6], step[6] = {0, 0, 0, 0, 0, 0};
        bool finite = true;
        const double scale = -2.0 / (S.nf * ng);
#pragma unroll
        for (int j = 0; j < 6; ++j) neg[j] = -(scale * (t[3 + j] - kappa * (t[9 + j] - delta * t[15 + j])));
        assemble_hessian(t + 21, 2.0 / ng2, shH);
        ldlt6_compute(shL, shH);
        if (!shL.ok) {
          finite = false;
        } else {
          ldlt6_solve(shL, neg, step);
          for (int j = 0; j < 6; ++j) finite = finite && isfinite(step[j]);
        }
        finish_step(S, step, finite, DICB200_POI_DEGENERATE_SUBSET, iter, p.tol, false);
      }
    }
    __syncthreads();
    if (S.done == 2 || S.status != DICB200_POI_OK) break;
  }
  if (tid == 0) {
    if (S.status == DICB200_POI_OK) {
      rec->u = S.p[0];
      rec->v = S.p[3];
      rec->zncc = S.zncc;
      rec->iterations = S.iterations;
      rec->converged = S.converged;
    } else {
      rec->status = S.status;
      rec->converged = 0;
    }
  }
}

template <typename Pix, int PPT, int WP>
cudaError_t launch_ppt(const RefineParams& p, size_t smem, cudaStream_t st) {
  if (p.method == 0)
    refine_kernel<Pix, PPT, 0, WP><<<p.n_records, kNT, smem, st>>>(p);
  else
    refine_kernel<Pix, PPT, 1, WP><<<p.n_records, kNT, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// (PPT, window pitch) by half-width: n <= 256*PPT and 2M+1+2*kPad <= WP
template <typename Pix>
cudaError_t launch_pix(const RefineParams& p, int ppt, cudaStream_t st) {
  const int S = 2 * p.M + 1 + 2 * kPad;
  switch (ppt) {
    case 2: return launch_ppt<Pix, 2, 32>(p, (size_t)S * 32 * 4, st);
    case 4: return launch_ppt<Pix, 4, 64>(p, (size_t)S * 64 * 4, st);
    case 7: return launch_ppt<Pix, 7, 64>(p, (size_t)S * 64 * 4, st);
    case 10: return launch_ppt<Pix, 10, 64>(p, (size_t)S * 64 * 4, st);
    default: return launch_ppt<Pix, 16, 128>(p, (size_t)S * 128 * 4, st);
  }
}

}  // namespace

bool refine_plan(int M, int* ppt_out, int* nt_out) {
  const int n = (2 * M + 1) * (2 * M + 1);
  const int S = 2 * M + 1 + 2 * kPad;
  const int ppts[] = {2, 4, 7, 10, 16};
  const int pitch[] = {32, 64, 64, 64, 128};
  for (int i = 0; i < 5; ++i)
    if (ppts[i] * kNT >= n && S <= pitch[i]) {
      *ppt_out = ppts[i];
      *nt_out = kNT;
      return true;
    }
  return false;
}

cudaError_t refine_launch(const RefineParams& p, bool u8, cudaStream_t st) {
  if (p.n_records <= 0) return cudaSuccess;
  int ppt = 0, nt = 0;
  if (!refine_plan(p.M, &ppt, &nt)) return cudaErrorInvalidValue;
  return u8 ? launch_pix<uint8_t>(p, ppt, st) : launch_pix<uint16_t>(p, ppt, st);
}

}  // namespace dicb200
