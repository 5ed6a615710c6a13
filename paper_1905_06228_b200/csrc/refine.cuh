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
};

bool refine_plan(int M, int* ppt, int* nt);
cudaError_t refine_launch(const RefineParams& p, bool u8, cudaStream_t st);

}  // namespace dicb200
