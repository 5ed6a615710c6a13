// K1 BFS-ZNCC tile kernel interface (see bfs.cu).
#pragma once
#include "common.cuh"

namespace dicb200 {

struct BfsParams {
  ImageView ref, tgt;
  Lattice lat;
  int row_begin;   // first grid row of this launch (global row index)
  int M, R, whole, u8, f64;
  int subpixel_none;
  // plan (bfs_plan)
  int EX, EY, DXC, DYC, n_dx_chunks, n_dy_chunks, n_chunks;
  int J, B, QP, CP, TS, tiles_x;
  int RW, RH, region_pitch, ref_pitch, items_max;
  dicb200_poi_record* rec;  // records of the launched rows: index (iy-row_begin)*nx + ix
  BestPartial* partial;     // [subset][n_chunks] when n_chunks > 1
  double* surface;          // optional [subset][EY][EX] ZNCC surface (NaN = no result) for K2
};

struct BfsSmem {
  size_t target, ref, v1, v2, stats, items, total;
};

__host__ __device__ BfsSmem bfs_smem_layout(const BfsParams& p);
__device__ void write_integer_record(dicb200_poi_record& r, int x, int y, const BestPartial& b, int subpixel_none);
bool bfs_plan(BfsParams& p, size_t smem_limit);
cudaError_t bfs_launch(BfsParams& p, int rows, cudaStream_t st);

}  // namespace dicb200
