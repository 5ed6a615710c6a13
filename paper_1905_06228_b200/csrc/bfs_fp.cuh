// K1-FP: integer search on fractional (fp64) gray levels in the reference's
// exact evaluation order (see bfs_fp.cu).
#pragma once
#include "bfs.cuh"
#include "common.cuh"

namespace dicb200 {

struct FpParams {
  ImageView ref, tgt;  // fp64 images
  Lattice lat;
  int row_begin;  // first grid row of this launch
  int M, R, whole;
  int subpixel_none;
  int stage_window;          // set by bfs_fp_launch
  dicb200_poi_record* rec;   // records of the launched rows
  double* surface;           // optional [subset][2R+1][2R+1] (swarm walk); records are then not written
};

cudaError_t bfs_fp_launch(FpParams p, int rows, cudaStream_t st);
// f32 image (pitch in elements) -> dense fp64 copy (exact)
cudaError_t widen_f32_to_f64(const float* src, int pitch, double* dst, int w, int h, cudaStream_t st);
// u8 / u16 image (pitch in elements) -> dense fp64 copy (exact)
cudaError_t widen_int_to_f64(const void* src, int elem_size, int pitch, double* dst, int w, int h, cudaStream_t st);

}  // namespace dicb200
