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
  // plan
  int wmax;          // window side bound (2R+1)
  int region_pitch;  // bytes (u8) or elements (u16), multiple of 4 bytes
  int QP;            // u8 words per subset row
  size_t smem;
};

dicb200_status pso_launch(PsoParams& p, cudaStream_t st);

}  // namespace dicb200
