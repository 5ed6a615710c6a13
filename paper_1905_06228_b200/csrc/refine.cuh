// K3/K4 sub-pixel refinement interface (see refine.cu).
#pragma once
#include "common.cuh"

namespace dicb200 {

struct RefineParams {
  ImageView ref, tgt;
  Lattice lat;
  int row_begin;
  int M;
  int n_records;
  int method;  // 0 = NR, 1 = IC-GN
  double tol;
  int max_iter;
  dicb200_poi_record* rec;
  int spc;  // POIs per CTA strip (<= 8), chosen by refine_launch to fit shared memory
  int interp;   // DICB200_INTERP_BILINEAR | DICB200_INTERP_BICUBIC
  int use_tma;  // fixed-geometry kernels: regions staged by TMA (tensor maps passed beside the params)
  // IC-GN reference-side constants per POI (kIcgnCacheStride doubles, global
  // POI index), reused while the reference frame repeats (fixed_first
  // sequences): [0] tag (0 = not computed, 1 = ok, 1 + status = failed),
  // [1] fbar, [2] nf, [3] scf, [4..9] A, [10..15] S, [16..51] H^-1 rows.
  double* cache;
  // launch order of the strips (CTA b runs strip order[b]; nullptr = grid order)
  const int* order;
};

constexpr int kIcgnCacheStride = 52;

// Device buffer + key of the IC-GN reference-side constants (see RefineParams::cache).
struct IcgnRefCache {
  double* data = nullptr;
  size_t cap = 0;
  long key = -1;
  const void* ref = nullptr;
  int W = 0, H = 0, M = 0, x0 = 0, y0 = 0, step = 0, nx = 0, ny = 0;
  // pre-converted staging images of the fixed-geometry IC-GN kernels: the
  // reference as fp32 and its 2 grad (kept while `img_key` repeats), the
  // target as vertical pairs (rebuilt per pair); row pitch `img_pitch` elements
  void* rimg = nullptr;
  void* gimg = nullptr;
  void* timg = nullptr;
  size_t img_cap = 0;
  long img_key = -1;
  const void* img_ref = nullptr;
  void reset() {
    key = -1;
    img_key = -1;
  }
};

bool refine_plan(int M, int* ppt, int* nt);
// cache/ref_key: reuse the IC-GN reference-side constants across calls with
// the same reference frame (ref_key >= 0, same device pointer, lattice and M).
// dtype: DICB200_U8 | DICB200_U16 | DICB200_F64 (fractional levels, generic kernels)
cudaError_t refine_launch(const RefineParams& p, int dtype, cudaStream_t st, IcgnRefCache* cache = nullptr,
                          long ref_key = -1);
void icgn_cache_free(IcgnRefCache& c, cudaStream_t st = nullptr, bool async = false);

}  // namespace dicb200
