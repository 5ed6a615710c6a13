/* Shared between the host (synth.c) and device (synth_device.cu) renderers. */
#ifndef DICB200_SYNTH_INTERNAL_H
#define DICB200_SYNTH_INTERNAL_H
#include "dicb200_synth.h"
#ifdef __cplusplus
extern "C" {
#endif
#define CELL 16
typedef struct {
  double cx, cy, inv2s2, peak, reach2;
} blob_t;
typedef struct {
  blob_t* blobs;
  int n;
  int* cell_start; /* gx*gy+1 */
  int* items;      /* blob index per cell slot */
  int gx, gy, reach_cells;
} synth_blobs_t;
int dicb200_synth_blobs(const dicb200_synth_spec* sp, synth_blobs_t* out);
void dicb200_synth_blobs_free(synth_blobs_t* b);
void dicb200_synth_preimage(const dicb200_synth_spec* sp, double x, double y, double* px, double* py);
#ifdef __cplusplus
}
#endif
#endif
