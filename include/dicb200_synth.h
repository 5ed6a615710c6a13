/*
 * dicb200_synth — deterministic synthetic speckle frames for the BASELINE
 * configurations (BASELINE.json "configs"). Plays the role of
 * the reference's synth_speckle / synth_warped_pair (proj/core/src/synth.cpp:51-161)
 * but with the BASELINE recipe: Gaussian blobs (seed-drawn centres, radius
 * sigma ~ U[sigma_min, sigma_max], peak ~ U[peak_min, peak_max]) summed on a
 * background, clipped to [0, max_value] and rounded to integers; deformed
 * frames are ANALYTIC re-renders at the preimage y of each pixel x with
 * y + d(y) = x (no resampling of the reference frame).
 *
 * Not part of the drop-in boundary; host-side data generation only.
 */
#ifndef DICB200_SYNTH_H
#define DICB200_SYNTH_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { DICB200_FIELD_NONE = 0, DICB200_FIELD_AFFINE = 1, DICB200_FIELD_SINUSOID = 2 };

typedef struct {
  int32_t width, height;
  int32_t dtype;      /* DICB200_U8 | DICB200_U16 */
  int32_t max_value;  /* 255 (u8) or 4095 (12-bit u16) */
  uint64_t seed;      /* blob stream seed */
  int32_t blob_count;
  int32_t field;      /* DICB200_FIELD_* */
  double sigma_min, sigma_max;
  double peak_min, peak_max;
  double background;
  /* AFFINE: d(y) = (a[0] + a[1](yx-a[6]) + a[2](yy-a[7]),
   *                 a[3] + a[4](yx-a[6]) + a[5](yy-a[7]))
   * SINUSOID: d(y) = (a[0] sin(2 pi yy / a[1]), a[2] cos(2 pi yx / a[3])) */
  double a[8];
} dicb200_synth_spec;

/* Renders one frame into out (pitch in elements). threads <= 0: all cores. */
int dicb200_synth_render(const dicb200_synth_spec* spec, void* out, int32_t pitch, int32_t threads);

/* Rows [row_begin, row_end) of the same frame into out (out's row 0 = frame
 * row row_begin): identical pixels to the corresponding rows of a full render. */
int dicb200_synth_render_rows(const dicb200_synth_spec* spec, void* out, int32_t pitch, int32_t row_begin,
                              int32_t row_end, int32_t threads);

/* Same frame rendered on the GPU into device memory (pitch in elements);
 * stream is a cudaStream_t (NULL = legacy default). Synchronous. Bit-identical
 * to dicb200_synth_render (shared per-pixel code, synth_math.h). */
int dicb200_synth_render_device(const dicb200_synth_spec* spec, void* out_dev, int32_t pitch, void* stream);

/* Displacement d(y) at a reference-frame point (ground truth helper). */
void dicb200_synth_displacement(const dicb200_synth_spec* spec, double yx, double yy, double* dx,
                                double* dy);

#ifdef __cplusplus
}
#endif
#endif
