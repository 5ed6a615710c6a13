/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference DIC correlation
 * path (oracle/dic_oracle.c). Loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER, never by the product.
 *
 * Signatures mirror oracle/ref_build/ref_capi.cpp (dicref_*) so tests can run
 * the same case through the reference build and through this restatement.
 * Images are row-major doubles (GrayImage, image.hpp:14-31).
 */
#ifndef DIC_ORACLE_H
#define DIC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#include "dicb200.h"

#ifdef __cplusplus
extern "C" {
#endif

int dco_analyze_pair(const double* ref, const double* tgt, int w, int h,
                     const dicb200_run_config* cfg, uint64_t pair_index, int threads,
                     dicb200_poi_record* out, size_t cap, size_t* count, char* err, size_t errcap);
int dco_analyze_pair_rows(const double* ref, const double* tgt, int w, int h,
                          const dicb200_run_config* cfg, uint64_t pair_index, int threads,
                          int row_begin, int row_end, dicb200_poi_record* out, size_t cap,
                          size_t* count, char* err, size_t errcap);
int dco_grid(int w, int h, int half_width, int spacing, int margin, int32_t* xy, size_t cap,
             size_t* count, char* err, size_t errcap);
int dco_zncc(const double* ref, const double* tgt, int w, int h, int cx, int cy, int m, int dx,
             int dy, double* out, char* err, size_t errcap);
int dco_integer_search(const double* ref, const double* tgt, int w, int h, int cx, int cy, int m,
                       const dicb200_run_config* cfg, uint64_t stream_seed, int32_t* ires,
                       double* zncc, int64_t* evals, char* err, size_t errcap);
int dco_refine(const double* ref, const double* tgt, int w, int h, int cx, int cy, int m,
               int init_dx, int init_dy, int method, double tol, int max_iter, double* out,
               int32_t* iters_conv, char* err, size_t errcap);
int dco_icgn_hessian(const double* ref, int w, int h, int cx, int cy, int m, double* hess,
                     double* condition, char* err, size_t errcap);
double dco_interp_bilinear(const double* img, int w, int h, double x, double y, int* ok);
/* bicubic variant (B200 extension, parity unpinned): value / analytic gradient */
double dco_interp_bicubic(const double* img, int w, int h, double x, double y, int* ok);
int dco_grad_bicubic(const double* img, int w, int h, double x, double y, double* gx, double* gy);
uint64_t dco_derive_stream_seed(uint64_t seed, uint64_t pair, uint64_t subset);
void dco_mt64(uint64_t seed, size_t n, uint64_t* out);
void dco_uniform01(uint64_t seed, size_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
