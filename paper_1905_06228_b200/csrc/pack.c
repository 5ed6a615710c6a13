/* GrayImage doubles -> u16 gray levels, the host side of the drop-in boundary
 * (the reference stores every image as doubles, image.hpp:14-31). One pass per
 * pixel: convert, check integrality and range, track the maximum. AVX2 when the
 * host has it (8 pixels per trip), scalar otherwise; identical results.
 *
 * dicb200_pack_span: one contiguous span (called per row band).
 * Flags are OR-ed into *frac / *bad, *mx raised to the span's maximum. */
#include <stddef.h>
#include <stdint.h>

#if defined(__x86_64__) && defined(__GNUC__)
#include <immintrin.h>
#define DICB200_HAVE_AVX2_PATH 1
#endif

static void pack_span_scalar(const double* s, size_t n, uint16_t* d, int* frac, int* bad, int* mx) {
  int f = 0, b = 0, m = *mx;
  for (size_t i = 0; i < n; ++i) {
    const double v = s[i];
    const int oob = !(v >= 0.0 && v <= 65535.0); /* also NaN */
    b |= oob;
    const uint16_t q = (uint16_t)(oob ? 0.0 : v);
    f |= (double)q != v;
    d[i] = q;
    m = q > m ? q : m;
  }
  *frac |= f;
  *bad |= b;
  *mx = m;
}

#ifdef DICB200_HAVE_AVX2_PATH
__attribute__((target("avx2"))) static void pack_span_avx2(const double* s, size_t n, uint16_t* d, int* frac,
                                                           int* bad, int* mx) {
  const __m256d lo = _mm256_set1_pd(0.0), hi = _mm256_set1_pd(65535.0);
  __m256d nf = _mm256_setzero_pd(), nb = _mm256_setzero_pd();
  __m128i vmax = _mm_setzero_si128();
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const __m256d a = _mm256_loadu_pd(s + i), b = _mm256_loadu_pd(s + i + 4);
    /* in range (ordered compares: NaN fails both) */
    const __m256d ia = _mm256_and_pd(_mm256_cmp_pd(a, lo, _CMP_GE_OQ), _mm256_cmp_pd(a, hi, _CMP_LE_OQ));
    const __m256d ib = _mm256_and_pd(_mm256_cmp_pd(b, lo, _CMP_GE_OQ), _mm256_cmp_pd(b, hi, _CMP_LE_OQ));
    const __m256d ca = _mm256_and_pd(a, ia), cb = _mm256_and_pd(b, ib); /* out of range -> 0 */
    const __m128i qa = _mm256_cvttpd_epi32(ca), qb = _mm256_cvttpd_epi32(cb);
    nf = _mm256_or_pd(nf, _mm256_cmp_pd(_mm256_cvtepi32_pd(qa), a, _CMP_NEQ_UQ));
    nf = _mm256_or_pd(nf, _mm256_cmp_pd(_mm256_cvtepi32_pd(qb), b, _CMP_NEQ_UQ));
    nb = _mm256_or_pd(nb, _mm256_or_pd(_mm256_andnot_pd(ia, _mm256_castsi256_pd(_mm256_set1_epi64x(-1))),
                                       _mm256_andnot_pd(ib, _mm256_castsi256_pd(_mm256_set1_epi64x(-1)))));
    const __m128i q = _mm_packus_epi32(qa, qb);
    vmax = _mm_max_epu16(vmax, q);
    _mm_storeu_si128((__m128i*)(d + i), q);
  }
  int f = _mm256_movemask_pd(nf) != 0, b = _mm256_movemask_pd(nb) != 0, m = *mx;
  uint16_t t[8];
  _mm_storeu_si128((__m128i*)t, vmax);
  for (int k = 0; k < 8; ++k) m = t[k] > m ? t[k] : m;
  *frac |= f;
  *bad |= b;
  *mx = m;
  if (i < n) pack_span_scalar(s + i, n - i, d + i, frac, bad, mx);
}
#endif

void dicb200_pack_span(const double* s, size_t n, uint16_t* d, int* frac, int* bad, int* mx) {
#ifdef DICB200_HAVE_AVX2_PATH
  static int have = -1;
  if (have < 0) have = __builtin_cpu_supports("avx2") ? 1 : 0;
  if (have) {
    pack_span_avx2(s, n, d, frac, bad, mx);
    return;
  }
#endif
  pack_span_scalar(s, n, d, frac, bad, mx);
}

/* u16 -> u8 in place (front to back), every level known to be <= 255. */
void dicb200_narrow_span(const uint16_t* s, size_t n, uint8_t* d) {
  for (size_t i = 0; i < n; ++i) d[i] = (uint8_t)s[i];
}
