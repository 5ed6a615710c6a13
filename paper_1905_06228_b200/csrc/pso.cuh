// K2 PSO / modified-PSO integer search interface (see pso.cu).
#pragma once
#include "common.cuh"

namespace dicb200 {

struct PsoParams {
  ImageView ref, tgt;
  Lattice lat;
  int row_begin;
  int M, R, u8, star;
  int P, G;
  double stop, c1, c2;
  uint64_t seed, pair_index;
  int inertia_constant;
  double w_const;
  int subpixel_none;
  dicb200_poi_record* rec;
  int n_records;
  const double* surface;  // [n_records][2R+1][2R+1] ZNCC surface from the BFS kernel (NaN = no result)
  int stage_surface;      // set by pso_walk_launch: copy each surface to shared memory first
};

size_t pso_walk_smem(const PsoParams& p);
dicb200_status pso_walk_launch(PsoParams& p, cudaStream_t st);

}  // namespace dicb200
