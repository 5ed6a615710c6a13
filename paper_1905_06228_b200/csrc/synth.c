/*
 * Synthetic speckle frames for the BASELINE configurations (see
 * include/dicb200_synth.h). Host C, multithreaded over row bands; blobs are
 * binned into 16x16 px cells so each pixel only visits nearby blobs.
 */
#define _GNU_SOURCE
#include "dicb200_synth.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "dicb200.h"


#include "synth_internal.h"
#include "synth_math.h"

static uint64_t splitmix_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double u01(uint64_t* s) { return (double)(splitmix_next(s) >> 11) * 0x1.0p-53; }

void dicb200_synth_displacement(const dicb200_synth_spec* sp, double yx, double yy, double* dx,
                                double* dy) {
  sx_displacement(sp, yx, yy, dx, dy);
}

/* Preimage y of pixel x under x = y + d(y). */
void dicb200_synth_preimage(const dicb200_synth_spec* sp, double x, double y, double* px, double* py) {
  sx_preimage(sp, x, y, px, py);
}

typedef struct {
  const dicb200_synth_spec* sp;
  const blob_t* blobs;
  const int* cell_start;
  const int* cell_items;
  int gx, gy;
  void* out;
  int pitch;
  int row0;  /* frame row stored in out's first row */
  int y0, y1;
} job_t;

static void* render_rows(void* arg) {
  const job_t* j = (const job_t*)arg;
  const dicb200_synth_spec* sp = j->sp;
  const int reach_cells = (int)ceil(5.0 * sp->sigma_max / CELL) + 1;
  for (int y = j->y0; y < j->y1; ++y)
    for (int x = 0; x < sp->width; ++x) {
      const double q = sx_pixel(sp, j->blobs, j->cell_start, j->cell_items, j->gx, j->gy, reach_cells, x, y);
      const size_t o = (size_t)(y - j->row0) * j->pitch + x;
      if (sp->dtype == DICB200_U8)
        ((uint8_t*)j->out)[o] = (uint8_t)q;
      else
        ((uint16_t*)j->out)[o] = (uint16_t)q;
    }
  return NULL;
}

int dicb200_synth_blobs(const dicb200_synth_spec* sp, synth_blobs_t* out) {
  const int n = sp->blob_count;
  blob_t* blobs = (blob_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(blob_t));
  uint64_t s = sp->seed;
  for (int i = 0; i < n; ++i) {
    blob_t* b = &blobs[i];
    b->cx = u01(&s) * sp->width;
    b->cy = u01(&s) * sp->height;
    const double sigma = sp->sigma_min + (sp->sigma_max - sp->sigma_min) * u01(&s);
    b->peak = sp->peak_min + (sp->peak_max - sp->peak_min) * u01(&s);
    b->inv2s2 = 1.0 / (2.0 * sigma * sigma);
    b->reach2 = 25.0 * sigma * sigma; /* 5 sigma cut-off */
  }
  /* bin blob centres into CELL x CELL cells */
  const int gx = (sp->width + CELL - 1) / CELL, gy = (sp->height + CELL - 1) / CELL;
  int* cnt = (int*)calloc((size_t)gx * gy + 1, sizeof(int));
  int* cell_of = (int*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
  for (int i = 0; i < n; ++i) {
    int cxx = (int)(blobs[i].cx / CELL), cyy = (int)(blobs[i].cy / CELL);
    if (cxx >= gx) cxx = gx - 1;
    if (cyy >= gy) cyy = gy - 1;
    cell_of[i] = cyy * gx + cxx;
    cnt[cell_of[i] + 1]++;
  }
  for (int c = 0; c < gx * gy; ++c) cnt[c + 1] += cnt[c];
  int* items = (int*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
  int* fill = (int*)malloc((size_t)gx * gy * sizeof(int));
  memcpy(fill, cnt, (size_t)gx * gy * sizeof(int));
  for (int i = 0; i < n; ++i) items[fill[cell_of[i]]++] = i; /* ascending blob order per cell */
  free(fill);
  free(cell_of);
  out->blobs = blobs;
  out->n = n;
  out->cell_start = cnt;
  out->items = items;
  out->gx = gx;
  out->gy = gy;
  out->reach_cells = (int)ceil(5.0 * sp->sigma_max / CELL) + 1;
  return 0;
}

void dicb200_synth_blobs_free(synth_blobs_t* b) {
  free(b->blobs);
  free(b->cell_start);
  free(b->items);
}

int dicb200_synth_render_rows(const dicb200_synth_spec* sp, void* out, int32_t pitch, int32_t row_begin,
                              int32_t row_end, int32_t threads) {
  if (sp->width < 1 || sp->height < 1 || sp->blob_count < 0 || pitch < sp->width) return 1;
  if (row_begin < 0 || row_end > sp->height || row_end <= row_begin) return 1;
  synth_blobs_t B;
  dicb200_synth_blobs(sp, &B);
  const int rows = row_end - row_begin;
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads < 1) threads = 1;
  if (threads > rows) threads = rows;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){sp, B.blobs, B.cell_start, B.items, B.gx, B.gy, out, pitch, row_begin,
                      row_begin + (int)((long)rows * t / threads), row_begin + (int)((long)rows * (t + 1) / threads)};
    if (threads == 1)
      render_rows(&jobs[t]);
    else
      pthread_create(&tid[t], NULL, render_rows, &jobs[t]);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(jobs);
  free(tid);
  dicb200_synth_blobs_free(&B);
  return 0;
}

int dicb200_synth_render(const dicb200_synth_spec* sp, void* out, int32_t pitch, int32_t threads) {
  return dicb200_synth_render_rows(sp, out, pitch, 0, sp->height, threads);
}
