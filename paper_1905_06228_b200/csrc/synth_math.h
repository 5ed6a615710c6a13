/*
 * Per-pixel arithmetic of the synthetic speckle renderer, shared VERBATIM by
 * the host renderer (synth.c, C11) and the device renderer (synth_device.cu),
 * so both produce bit-identical frames by construction:
 *
 *  - only IEEE-754 double +, -, *, /, floor and exact ldexp are used, each
 *    product and sum rounded on its own (SX_MUL / SX_ADD: __dmul_rn /
 *    __dadd_rn on the device, where nvcc would otherwise contract a*b+c into
 *    one FMA; plain operators on the host, built with -ffp-contract=off);
 *  - exp, sin and cos are computed by the polynomials below instead of the
 *    platform libraries (glibc and CUDA's libdevice round differently in the
 *    last ulp).
 *
 * The frames are test/benchmark DATA (BASELINE.json configs);
 * nothing here is on the correlation path.
 */
#ifndef DICB200_SYNTH_MATH_H
#define DICB200_SYNTH_MATH_H

#include <math.h>

#include "synth_internal.h"

#if defined(__CUDACC__)
#define SX_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define SX_MUL(a, b) __dmul_rn((a), (b))
#define SX_ADD(a, b) __dadd_rn((a), (b))
#else
#define SX_MUL(a, b) ((a) * (b))
#define SX_ADD(a, b) ((a) + (b))
#endif
#else
#define SX_HD static inline
#define SX_MUL(a, b) ((a) * (b))
#define SX_ADD(a, b) ((a) + (b))
#endif
#define SX_SUB(a, b) SX_ADD((a), -(b))

/* exp(x): x = k ln2 + r, |r| <= ln2/2 (Cody-Waite split of ln2: k * SX_LN2_HI
 * is exact for |k| < 2^20), degree-13 Taylor polynomial in Horner form
 * (truncation < 4e-18 relative), scaled by the exact ldexp. Arguments here
 * lie in [-12.5, 0]. */
SX_HD double sx_exp(double x) {
  const double ln2_hi = 6.93147180369123816490e-01; /* 0x3fe62e42 fee00000 */
  const double ln2_lo = 1.90821492927058770002e-10;
  const double inv_ln2 = 1.44269504088896338700e+00;
  if (x < -700.0) return 0.0;
  const double k = floor(SX_ADD(SX_MUL(x, inv_ln2), 0.5));
  const double r = SX_SUB(SX_SUB(x, SX_MUL(k, ln2_hi)), SX_MUL(k, ln2_lo));
  /* 1/j! for j = 13 .. 1 */
  const double c[13] = {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
                        2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
                        1.984126984126984e-04,  1.3888888888888889e-03, 8.333333333333333e-03,
                        4.1666666666666664e-02, 1.6666666666666666e-01, 0.5, 1.0};
  double p = c[0];
  for (int j = 1; j < 13; ++j) p = SX_ADD(SX_MUL(p, r), c[j]);
  p = SX_ADD(SX_MUL(p, r), 1.0);
  return ldexp(p, (int)k);
}

/* sin(x), cos(x): x = k pi/2 + r, |r| <= pi/4 (three-part Cody-Waite pi/2,
 * each k * part exact for |k| < 2^20), Taylor polynomials of degree 17 / 18
 * (truncation < 3e-18), quadrant by k mod 4. Arguments here stay below 100. */
SX_HD void sx_sincos(double x, double* s_out, double* c_out) {
  const double pio2_1 = 1.57079632673412561417e+00; /* first 33 bits of pi/2 */
  const double pio2_2 = 6.07710050630396597660e-11; /* next 33 bits */
  const double pio2_3 = 2.02226624871116645580e-21;
  const double two_over_pi = 6.36619772367581382433e-01;
  const double k = floor(SX_ADD(SX_MUL(x, two_over_pi), 0.5));
  const double r =
      SX_SUB(SX_SUB(SX_SUB(x, SX_MUL(k, pio2_1)), SX_MUL(k, pio2_2)), SX_MUL(k, pio2_3));
  const double r2 = SX_MUL(r, r);
  /* sin r = r (1 - r^2/3! + r^4/5! - ...), up to r^17 */
  const double sc[8] = {2.8114572543455206e-15, -7.647163731819816e-13, 1.6059043836821613e-10,
                        -2.505210838544172e-08, 2.7557319223985893e-06, -1.984126984126984e-04,
                        8.333333333333333e-03,  -1.6666666666666666e-01};
  /* cos r = 1 - r^2/2! + r^4/4! - ..., up to r^18 */
  const double cc[9] = {-1.5619206968586225e-16, 4.779477332387385e-14, -1.1470745597729725e-11,
                        2.08767569878681e-09,    -2.755731922398589e-07, 2.48015873015873e-05,
                        -1.3888888888888889e-03, 4.1666666666666664e-02, -0.5};
  double ps = sc[0];
  for (int j = 1; j < 8; ++j) ps = SX_ADD(SX_MUL(ps, r2), sc[j]);
  const double sr = SX_ADD(r, SX_MUL(SX_MUL(ps, r2), r));
  double pc = cc[0];
  for (int j = 1; j < 9; ++j) pc = SX_ADD(SX_MUL(pc, r2), cc[j]);
  const double cr = SX_ADD(1.0, SX_MUL(pc, r2));
  long q = (long)k % 4;
  if (q < 0) q += 4;
  switch (q) {
    case 0: *s_out = sr; *c_out = cr; break;
    case 1: *s_out = cr; *c_out = -sr; break;
    case 2: *s_out = -sr; *c_out = -cr; break;
    default: *s_out = -cr; *c_out = sr; break;
  }
}

#define SX_TWO_PI 6.28318530717958647692

/* d(y) of the spec's field at a reference-frame point (see dicb200_synth.h). */
SX_HD void sx_displacement(const dicb200_synth_spec* sp, double yx, double yy, double* dx, double* dy) {
  const double* a = sp->a;
  if (sp->field == DICB200_FIELD_AFFINE) {
    const double rx = SX_SUB(yx, a[6]), ry = SX_SUB(yy, a[7]);
    *dx = SX_ADD(SX_ADD(a[0], SX_MUL(a[1], rx)), SX_MUL(a[2], ry));
    *dy = SX_ADD(SX_ADD(a[3], SX_MUL(a[4], rx)), SX_MUL(a[5], ry));
  } else if (sp->field == DICB200_FIELD_SINUSOID) {
    double s, c, s2, c2;
    sx_sincos(SX_MUL(SX_TWO_PI, yy) / a[1], &s, &c);
    sx_sincos(SX_MUL(SX_TWO_PI, yx) / a[3], &s2, &c2);
    *dx = SX_MUL(a[0], s);
    *dy = SX_MUL(a[2], c2);
  } else {
    *dx = 0.0;
    *dy = 0.0;
  }
}

/* Preimage y of pixel x under x = y + d(y). */
SX_HD void sx_preimage(const dicb200_synth_spec* sp, double x, double y, double* px, double* py) {
  const double* a = sp->a;
  if (sp->field == DICB200_FIELD_AFFINE) {
    /* x - o = (I + A)(y - o) + t  =>  y = o + (I + A)^-1 (x - o - t) */
    const double m00 = SX_ADD(1.0, a[1]), m01 = a[2], m10 = a[4], m11 = SX_ADD(1.0, a[5]);
    const double det = SX_SUB(SX_MUL(m00, m11), SX_MUL(m01, m10));
    const double bx = SX_SUB(SX_SUB(x, a[6]), a[0]), by = SX_SUB(SX_SUB(y, a[7]), a[3]);
    *px = SX_ADD(a[6], SX_SUB(SX_MUL(m11, bx), SX_MUL(m01, by)) / det);
    *py = SX_ADD(a[7], SX_ADD(SX_MUL(-m10, bx), SX_MUL(m00, by)) / det);
  } else if (sp->field == DICB200_FIELD_SINUSOID) {
    double yx = x, yy = y;
    for (int it = 0; it < 60; ++it) {
      double dx, dy;
      sx_displacement(sp, yx, yy, &dx, &dy);
      const double nx = SX_SUB(x, dx), ny = SX_SUB(y, dy);
      const double ch = SX_ADD(fabs(SX_SUB(nx, yx)), fabs(SX_SUB(ny, yy)));
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

/* One pixel (x, y): blobs of the cells within reach of the preimage, in
 * ascending cell / blob order, summed on the background, clipped to
 * [0, max_value] and rounded half up. */
SX_HD double sx_pixel(const dicb200_synth_spec* sp, const blob_t* blobs, const int* cell_start, const int* items,
                      int gx, int gy, int reach_cells, int x, int y) {
  double qx, qy;
  sx_preimage(sp, (double)x, (double)y, &qx, &qy);
  double v = sp->background;
  const int cx = (int)floor(qx / CELL), cy = (int)floor(qy / CELL);
  for (int by = cy - reach_cells; by <= cy + reach_cells; ++by) {
    if (by < 0 || by >= gy) continue;
    for (int bx = cx - reach_cells; bx <= cx + reach_cells; ++bx) {
      if (bx < 0 || bx >= gx) continue;
      const int c = by * gx + bx;
      for (int i = cell_start[c]; i < cell_start[c + 1]; ++i) {
        const blob_t* b = &blobs[items[i]];
        const double ddx = SX_SUB(qx, b->cx), ddy = SX_SUB(qy, b->cy);
        const double r2 = SX_ADD(SX_MUL(ddx, ddx), SX_MUL(ddy, ddy));
        if (r2 <= b->reach2) v = SX_ADD(v, SX_MUL(b->peak, sx_exp(SX_MUL(-r2, b->inv2s2))));
      }
    }
  }
  const double maxv = (double)sp->max_value;
  if (v < 0.0) v = 0.0;
  if (v > maxv) v = maxv;
  return floor(SX_ADD(v, 0.5));
}

#endif
