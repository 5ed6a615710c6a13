// K3/K4 — sub-pixel refinement: IC-GN (icgn_precompute + refine_icgn,
// subpixel.cpp:191-222, 301-359) and Newton-Raphson (refine_nr,
// subpixel.cpp:224-299), first-order warp, bilinear interpolation
// (interp_bilinear / grad_bilinear, subpixel.cpp:59-128).
//
// One CTA per POI, NT threads, each thread owns PPT subset pixels in
// registers for the whole solve (reference values, centred values and, for
// IC-GN, the steepest-descent gradients). Per iteration: fused warp + gather
// + bilinear in fp32 on subset-local coordinates (integer base kept apart, so
// coordinates near 2048 px lose nothing), per-thread fp32 partials over
// <= PPT terms, block reductions and the 6x6 algebra in fp64. The reference's
// two-pass structure (mean, then centred sums) is kept per iteration, so each
// e_k / coeff_k is formed exactly as subpixel.cpp:258,331 do.
//
// IC-GN Hessian: with integer gray levels, (2*grad)^2 * {1,dx,dy,dx^2,dxdy,dy^2}
// are integers < 2^53, so the fp64 moment sums are EXACT and the Hessian —
// and its pivoted LDL^T (linalg.cuh) — is bit-identical to the reference's.
// Failure semantics follow pipeline.cpp:82-133: any stage error sets the
// status, clears `converged` and keeps the integer-stage fields.
#include "common.cuh"
#include "linalg.cuh"
#include "refine.cuh"

namespace dicb200 {

namespace {

constexpr int kMaxWarps = 8;
constexpr int kMaxNV = 24;

struct RedBuf {
  double v[2][kMaxWarps][kMaxNV];
};

// Sum NV per-thread doubles over the block; every thread gets the totals.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], RedBuf& rb, int& buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) rb.v[buf][warp][i] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = rb.v[buf][0][i];
    for (int w = 1; w < nw; ++w) s += rb.v[buf][w][i];
    v[i] = s;
  }
  buf ^= 1;
}

template <typename Pix>
__device__ __forceinline__ float px(const ImageView& im, int x, int y) {
  return (float)__ldg(reinterpret_cast<const Pix*>(im.data) + (size_t)y * im.pitch + x);
}

// interp_bilinear (subpixel.cpp:59-102) at global (bx + xl, by + yl).
template <typename Pix>
__device__ __forceinline__ bool bilinear(const ImageView& im, int bx, int by, float xl, float yl, float& g) {
  if (!(xl >= (float)(-bx) && xl <= (float)(im.width - 1 - bx) && yl >= (float)(-by) &&
        yl <= (float)(im.height - 1 - by)))
    return false;
  const float flx = floorf(xl), fly = floorf(yl);
  int x0 = bx + (int)flx, y0 = by + (int)fly;
  if (x0 > im.width - 2) x0 = im.width - 2;
  if (y0 > im.height - 2) y0 = im.height - 2;
  const float fx = xl - (float)(x0 - bx), fy = yl - (float)(y0 - by);
  const int x1 = min(x0 + 1, im.width - 1), y1 = min(y0 + 1, im.height - 1);
  const float f00 = px<Pix>(im, x0, y0), f10 = px<Pix>(im, x1, y0);
  const float f01 = px<Pix>(im, x0, y1), f11 = px<Pix>(im, x1, y1);
  const float a10 = f10 - f00, a01 = f01 - f00, a11 = (f00 + f11) - f10 - f01;
  float v = fmaf(a11 * fx, fy, fmaf(a01, fy, fmaf(a10, fx, f00)));
  const float lo = fminf(fminf(f00, f10), fminf(f01, f11));
  const float hi = fmaxf(fmaxf(f00, f10), fmaxf(f01, f11));
  g = fminf(fmaxf(v, lo), hi);
  return true;
}

// grad_bilinear (subpixel.cpp:104-128): node central differences, bilinearly
// weighted, zero weights skipped (keeps the taps inside the image).
template <typename Pix>
__device__ __forceinline__ bool grad_bilinear(const ImageView& im, int bx, int by, float xl, float yl,
                                              float& gx, float& gy) {
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
      ax = fmaf(w, px<Pix>(im, i + 1, j) - px<Pix>(im, i - 1, j), ax);
      ay = fmaf(w, px<Pix>(im, i, j + 1) - px<Pix>(im, i, j - 1), ay);
    }
  }
  gx = ax;
  gy = ay;
  return true;
}

struct SharedState {
  double p[6];  // u, ux, uy, v, vx, vy (WarpParams order of subpixel.hpp:13-16)
  int status;
  int done;
  int iterations;
  int converged;
  Ldlt6 L;
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
  for (int i = 0; i < 3; ++i)
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

// 18 moment sums m[k*6+w] (k: 0 aa, 1 ab, 2 bb; w: 1,dx,dy,dx^2,dxdy,dy^2) -> symmetric 6x6
// H = sum sd sd^T with sd = [a, a dx, a dy, b, b dx, b dy] (subpixel.cpp:210-212, :261-263).
__device__ void assemble_hessian(const double* mo, double scale, double* H) {
  auto A = [&](int w) { return mo[0 * 6 + w] * scale; };
  auto Bm = [&](int w) { return mo[1 * 6 + w] * scale; };
  auto Cm = [&](int w) { return mo[2 * 6 + w] * scale; };
  // index map of monomials: 0:1 1:dx 2:dy 3:dx^2 4:dxdy 5:dy^2
  const double h[6][6] = {
      {A(0), A(1), A(2), Bm(0), Bm(1), Bm(2)},
      {A(1), A(3), A(4), Bm(1), Bm(3), Bm(4)},
      {A(2), A(4), A(5), Bm(2), Bm(4), Bm(5)},
      {Bm(0), Bm(1), Bm(2), Cm(0), Cm(1), Cm(2)},
      {Bm(1), Bm(3), Bm(4), Cm(1), Cm(3), Cm(4)},
      {Bm(2), Bm(4), Bm(5), Cm(2), Cm(4), Cm(5)},
  };
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) H[i * 6 + j] = h[i][j];
}

template <typename Pix, int PPT, int METHOD>
__global__ void __launch_bounds__(256) refine_kernel(RefineParams p) {
  __shared__ RedBuf rb;
  __shared__ SharedState S;
  const int k = blockIdx.x;
  dicb200_poi_record* rec = p.rec + k;
  if (rec->status != DICB200_POI_OK) return;  // integer stage failed: record stays
  const int tid = threadIdx.x, NT = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int M = p.M, side = 2 * M + 1, n = side * side;
  const int iy = p.row_begin + k / p.lat.nx, ix = k % p.lat.nx;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy);
  const int idx = rec->integer_dx, idy = rec->integer_dy;
  int buf = 0;

  // ---- per-pixel reference data in registers ----
  float dxf[PPT], dyf[PPT], cf[PPT], gxr[PPT], gyr[PPT];
  double mean, nf;
  {
    if (METHOD == 1 && (cx - M - 1 < 0 || cx + M + 1 > p.ref.width - 1 || cy - M - 1 < 0 ||
                        cy + M + 1 > p.ref.height - 1)) {
      if (tid == 0) {
        rec->status = DICB200_POI_BORDER_GRADIENTS;
        rec->converged = 0;
      }
      return;
    }
    double sums[2] = {0.0, 0.0};
    float fv[PPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int kk = tid + i * NT;
      const int r = kk / side, c = kk - r * side;
      dxf[i] = (float)(c - M);
      dyf[i] = (float)(r - M);
      fv[i] = 0.f;
      gxr[i] = gyr[i] = 0.f;
      if (kk < n) {
        const int x = cx + c - M, y = cy + r - M;
        fv[i] = px<Pix>(p.ref, x, y);
        if (METHOD == 1) {
          gxr[i] = 0.5f * (px<Pix>(p.ref, x + 1, y) - px<Pix>(p.ref, x - 1, y));
          gyr[i] = 0.5f * (px<Pix>(p.ref, x, y + 1) - px<Pix>(p.ref, x, y - 1));
        }
        sums[0] += (double)fv[i];
        sums[1] += (double)fv[i] * (double)fv[i];
      }
    }
    block_sum<2>(sums, rb, buf);
    const int64_t sf = (int64_t)sums[0], sff = (int64_t)sums[1];
    const int64_t vf = (int64_t)n * sff - sf * sf;
    mean = sums[0] / (double)n;  // correlation.cpp:25: exact sum / n
    nf = sqrt((double)vf / (double)n);
    if (vf <= 0) {
      if (tid == 0) {
        rec->status = METHOD == 1 ? DICB200_POI_DEGENERATE_TEXTURE : DICB200_POI_DEGENERATE_SUBSET;
        rec->converged = 0;
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < PPT; ++i) cf[i] = (tid + i * NT < n) ? (float)((double)fv[i] - mean) : 0.f;
  }

  if (METHOD == 1) {
    // ---- icgn_precompute: exact Hessian moments, condition test, LDL^T ----
    double mo[18];
#pragma unroll
    for (int j = 0; j < 18; ++j) mo[j] = 0.0;
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const double a = 2.0 * gxr[i], b = 2.0 * gyr[i];  // integers
      const double dx = dxf[i], dy = dyf[i];
      const double w[6] = {1.0, dx, dy, dx * dx, dx * dy, dy * dy};
      const double aa = a * a, ab = a * b, bb = b * b;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        mo[j] = fma(aa, w[j], mo[j]);
        mo[6 + j] = fma(ab, w[j], mo[6 + j]);
        mo[12 + j] = fma(bb, w[j], mo[12 + j]);
      }
    }
    block_sum<18>(mo, rb, buf);
    if (warp == 0) {
      double H[36];
      assemble_hessian(mo, 0.25, H);
      Ldlt6 L;
      ldlt6_compute(L, H);
      bool pd = L.ok != 0;
      for (int i = 0; i < 6; ++i) pd = pd && L.m[i * 7] > 0.0;
      bool accept = false;
      if (pd) {
        // cond <= ||H||_F ||H^-1||_F; exact Jacobi only when the bound is inconclusive
        double col2 = 0.0;
        if (lane < 6) {
          double e[6] = {0, 0, 0, 0, 0, 0}, x[6];
          e[lane] = 1.0;
          ldlt6_solve(L, e, x);
          for (int i = 0; i < 6; ++i) col2 += x[i] * x[i];
        }
        for (int o = 16; o; o >>= 1) col2 += __shfl_xor_sync(0xffffffffu, col2, o);
        double hf2 = 0.0;
        for (int i = 0; i < 36; ++i) hf2 += H[i] * H[i];
        accept = sqrt(hf2) * sqrt(col2) < 1e12;
      }
      if (!accept) {
        double lo, hi;
        jacobi6_minmax(H, &lo, &hi);
        const double cond = lo > 0.0 ? hi / lo : __longlong_as_double(0x7ff0000000000000ULL);
        accept = cond < 1e12;
      }
      if (lane == 0) {
        S.status = accept ? DICB200_POI_OK : DICB200_POI_DEGENERATE_TEXTURE;
        S.L = L;
      }
    }
    __syncthreads();
    if (S.status != DICB200_POI_OK) {
      if (tid == 0) {
        rec->status = S.status;
        rec->converged = 0;
      }
      return;
    }
  }

  if (tid == 0) {
    S.p[0] = (double)idx;
    S.p[1] = S.p[2] = 0.0;
    S.p[3] = (double)idy;
    S.p[4] = S.p[5] = 0.0;
    S.status = DICB200_POI_OK;
    S.done = 0;
    S.iterations = 0;
    S.converged = 0;
  }
  __syncthreads();

  const int bx = cx + idx, by = cy + idy;
  float g[PPT], tgx[PPT], tgy[PPT];
  double zncc_final = 0.0;
  const double lim = (double)(M + 2);

  // sample_through_warp (subpixel.cpp:151-183) for the current S.p; returns
  // status, and (gbar, ng, cross) through the two-pass block sums.
  auto sample = [&](bool with_grad, double& gbar, double& ng, double& cross) -> int {
    const double u = S.p[0], ux = S.p[1], uy = S.p[2], v = S.p[3], vx = S.p[4], vy = S.p[5];
    const double ccx = cx + u, ccy = cy + v;  // check_guard, subpixel.cpp:134-141
    if (!(ccx >= lim && ccx <= p.tgt.width - 1 - lim && ccy >= lim && ccy <= p.tgt.height - 1 - lim))
      return DICB200_POI_DRIFTED;
    const float ul = (float)(u - idx), vl = (float)(v - idy);
    const float uxf = (float)ux, uyf = (float)uy, vxf = (float)vx, vyf = (float)vy;
    double s1[2] = {0.0, 0.0};
    float a1 = 0.f;
    int bad = 0;
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      g[i] = 0.f;
      if (tid + i * NT < n) {
        const float xl = fmaf(uyf, dyf[i], fmaf(uxf, dxf[i], dxf[i] + ul));
        const float yl = fmaf(vyf, dyf[i], fmaf(vxf, dxf[i], dyf[i] + vl));
        bad |= !bilinear<Pix>(p.tgt, bx, by, xl, yl, g[i]);
        if (with_grad) bad |= !grad_bilinear<Pix>(p.tgt, bx, by, xl, yl, tgx[i], tgy[i]);
        a1 += g[i] - (float)mean;
      }
    }
    s1[0] = a1;
    s1[1] = bad;
    block_sum<2>(s1, rb, buf);
    if (s1[1] != 0.0) return DICB200_POI_DRIFTED;
    gbar = mean + s1[0] / (double)n;
    const float gb = (float)gbar;
    float a2 = 0.f, ac = 0.f;
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      if (tid + i * NT < n) {
        const float d = g[i] - gb;
        a2 = fmaf(d, d, a2);
        ac = fmaf(cf[i], d, ac);
      }
    }
    double s2[2] = {a2, ac};
    block_sum<2>(s2, rb, buf);
    ng = sqrt(s2[0]);
    cross = s2[1];
    if (ng <= 0.0) return DICB200_POI_DEGENERATE_TARGET;
    return DICB200_POI_OK;
  };

  int status = DICB200_POI_OK;
  for (int iter = 1; iter <= p.max_iter; ++iter) {
    double gbar, ng, cross;
    status = sample(METHOD == 0, gbar, ng, cross);
    if (status != DICB200_POI_OK) break;
    const float gb = (float)gbar;
    if (METHOD == 1) {
      // rhs = sum_k e_k sd_k, e_k = f_k - (nf/ng)(g_k - gbar) (subpixel.cpp:328-333)
      const float ratio = (float)(nf / ng);
      float r6[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        const float e = cf[i] - ratio * (g[i] - gb);
        const float tx = e * gxr[i], ty = e * gyr[i];
        r6[0] += tx;
        r6[1] = fmaf(tx, dxf[i], r6[1]);
        r6[2] = fmaf(tx, dyf[i], r6[2]);
        r6[3] += ty;
        r6[4] = fmaf(ty, dxf[i], r6[4]);
        r6[5] = fmaf(ty, dyf[i], r6[5]);
      }
      double rhs[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) rhs[j] = r6[j];
      block_sum<6>(rhs, rb, buf);
      if (tid == 0) {
        double neg[6], step[6];
        for (int j = 0; j < 6; ++j) neg[j] = -rhs[j];
        ldlt6_solve(S.L, neg, step);
        bool fin = true;
        for (int j = 0; j < 6; ++j) fin = fin && isfinite(step[j]);
        int st = fin ? DICB200_POI_OK : DICB200_POI_DEGENERATE_TEXTURE;
        if (st == DICB200_POI_OK) st = compose_with_inverse(S.p, step);
        if (st == DICB200_POI_OK && fabs(warp_det(S.p)) < 1e-8) st = DICB200_POI_WARP_NOT_INVERTIBLE;
        S.status = st;
        if (st == DICB200_POI_OK) {
          S.iterations = iter;
          if (fmax(fabs(step[0]), fabs(step[3])) < p.tol) {
            S.converged = 1;
            S.done = 1;
          }
        }
      }
    } else {
      // NR (subpixel.cpp:247-271): coeff_k = c_f - (cross/ng^2) (g_k - gbar);
      // gradient = -2/(nf ng) sum coeff J; H = 2/ng^2 sum J J^T.
      const float kappa = (float)(cross / (ng * ng));
      float a[24];
#pragma unroll
      for (int j = 0; j < 24; ++j) a[j] = 0.f;
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        if (tid + i * NT < n) {
          const float coeff = cf[i] - kappa * (g[i] - gb);
          const float gx = tgx[i], gy = tgy[i];
          const float dx = dxf[i], dy = dyf[i];
          const float tx = coeff * gx, ty = coeff * gy;
          a[0] += tx;
          a[1] = fmaf(tx, dx, a[1]);
          a[2] = fmaf(tx, dy, a[2]);
          a[3] += ty;
          a[4] = fmaf(ty, dx, a[4]);
          a[5] = fmaf(ty, dy, a[5]);
          const float w[6] = {1.f, dx, dy, dx * dx, dx * dy, dy * dy};
          const float aa = gx * gx, ab = gx * gy, bb = gy * gy;
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            a[6 + j] = fmaf(aa, w[j], a[6 + j]);
            a[12 + j] = fmaf(ab, w[j], a[12 + j]);
            a[18 + j] = fmaf(bb, w[j], a[18 + j]);
          }
        }
      }
      double t24[24];
#pragma unroll
      for (int j = 0; j < 24; ++j) t24[j] = a[j];
      block_sum<24>(t24, rb, buf);
      if (tid == 0) {
        const double ng2 = ng * ng;
        const double scale = -2.0 / (nf * ng);
        double H[36], neg[6], step[6];
        assemble_hessian(t24 + 6, 2.0 / ng2, H);
        for (int j = 0; j < 6; ++j) neg[j] = -(t24[j] * scale);
        Ldlt6 L;
        ldlt6_compute(L, H);
        int st = L.ok ? DICB200_POI_OK : DICB200_POI_DEGENERATE_SUBSET;
        if (st == DICB200_POI_OK) {
          ldlt6_solve(L, neg, step);
          bool fin = true;
          for (int j = 0; j < 6; ++j) fin = fin && isfinite(step[j]);
          if (!fin) st = DICB200_POI_DEGENERATE_SUBSET;
        }
        if (st == DICB200_POI_OK) {
          for (int j = 0; j < 6; ++j) S.p[j] += step[j];
          if (fabs(warp_det(S.p)) < 1e-8) st = DICB200_POI_WARP_NOT_INVERTIBLE;
        }
        S.status = st;
        if (st == DICB200_POI_OK) {
          S.iterations = iter;
          if (fmax(fabs(step[0]), fabs(step[3])) < p.tol) {
            S.converged = 1;
            S.done = 1;
          }
        }
      }
    }
    __syncthreads();
    status = S.status;
    if (status != DICB200_POI_OK || S.done) break;
  }
  if (status == DICB200_POI_OK) {
    // final re-sample + ZNCC (subpixel.cpp:288-297, 348-357)
    double gbar, ng, cross;
    status = sample(false, gbar, ng, cross);
    if (status == DICB200_POI_OK) zncc_final = cross / (nf * ng);
  }
  if (tid == 0) {
    if (status == DICB200_POI_OK) {
      rec->u = S.p[0];
      rec->v = S.p[3];
      rec->zncc = zncc_final;
      rec->iterations = S.iterations;
      rec->converged = S.converged;
    } else {
      rec->status = status;
      rec->converged = 0;
    }
  }
}

template <typename Pix, int PPT>
cudaError_t launch_ppt(const RefineParams& p, int nt, cudaStream_t st) {
  if (p.method == 0)
    refine_kernel<Pix, PPT, 0><<<p.n_records, nt, 0, st>>>(p);
  else
    refine_kernel<Pix, PPT, 1><<<p.n_records, nt, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <typename Pix>
cudaError_t launch_pix(const RefineParams& p, int ppt, int nt, cudaStream_t st) {
  switch (ppt) {
    case 4: return launch_ppt<Pix, 4>(p, nt, st);
    case 8: return launch_ppt<Pix, 8>(p, nt, st);
    case 14: return launch_ppt<Pix, 14>(p, nt, st);
    default: return launch_ppt<Pix, 16>(p, nt, st);
  }
}

}  // namespace

bool refine_plan(int M, int* ppt_out, int* nt_out) {
  const int n = (2 * M + 1) * (2 * M + 1);
  const int ppts[] = {4, 8, 14, 16};
  double best = -1.0;
  for (int ppt : ppts) {
    const int nt = (((n + ppt - 1) / ppt) + 31) / 32 * 32;
    if (nt > 256) continue;
    const double util = (double)n / (nt * ppt);
    if (util > best + 1e-9) {
      best = util;
      *ppt_out = ppt;
      *nt_out = nt;
    }
  }
  return best > 0.0;
}

cudaError_t refine_launch(const RefineParams& p, bool u8, cudaStream_t st) {
  if (p.n_records <= 0) return cudaSuccess;
  int ppt = 0, nt = 0;
  if (!refine_plan(p.M, &ppt, &nt)) return cudaErrorInvalidValue;
  return u8 ? launch_pix<uint8_t>(p, ppt, nt, st) : launch_pix<uint16_t>(p, ppt, nt, st);
}

}  // namespace dicb200
