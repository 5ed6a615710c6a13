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
__device__ inline void write_integer_record(dicb200_poi_record& r, int x, int y, const BestPartial& b, int subpixel_none) {
  r.x = x;
  r.y = y;
  r.iterations = 0;
  r.update_evaluations = 0;
  r.pad = 0;
  if (!b.found) {  // "all positions degenerate" (integer_search.cpp:77): record keeps defaults
    r.u = 0.0;
    r.v = 0.0;
    r.zncc = __longlong_as_double(0x7ff8000000000000ULL);
    r.converged = 0;
    r.evaluations = 0;
    r.status = DICB200_POI_ALL_DEGENERATE;
    r.integer_dx = 0;
    r.integer_dy = 0;
    return;
  }
  r.u = (double)b.dx;
  r.v = (double)b.dy;
  r.zncc = b.c;
  r.evaluations = b.count;
  r.converged = subpixel_none ? 1 : 0;
  r.status = DICB200_POI_OK;
  r.integer_dx = b.dx;
  r.integer_dy = b.dy;
}

bool bfs_plan(BfsParams& p, size_t smem_limit);
cudaError_t bfs_launch(BfsParams& p, int rows, cudaStream_t st);

// ---- K1 on the tensor cores (bfs_tc.cu) ----------------------------------
// Window-mode search as an exact u8 x u8 -> s32 tcgen05 GEMM: M = 128 target
// positions (16 x 8 subset top-left corners), N = the POIs (x byte planes of
// the reference) whose windows touch them, K = the subset pixels. Wider pixels
// are split into hi/lo byte planes and recombined exactly.
struct TcParams {
  ImageView ref, tgt;
  Lattice lat;
  int rb, re;  // POI rows [rb, re)
  int M, R, side, planes, subpixel_none;
  double maxv;  // largest gray level of either image (0 = full dtype range)
  int qx_min, qx_max, qy_min, qy_max, SW, SH;  // position domain (subset top-left corners)
  int ntx, nty, n_tiles;
  int RG, CG, NX, HT, RWB, n_mma;  // K blocking: 8 rows x 4 columns per MMA
  int rem, rem_rows, n_h, NX2, HT2, RWB2;  // row-major remainder stage (last subset rows)
  int nix_max, niy_max, npoi_max, N_max, tmem_cols;
  size_t off_rows, off_B, stage_bytes, smem;  // stage = T | rows | B
  int stages;
  int grid;
  long long* dbg_out;  // optional per-CTA MMA-thread clock breakdown (tools)
  int dbg;  // DICB200_TC_DBG=32: MMA-issuer clock breakdown (tools)
  // buffers (device)
  uint8_t* strips;       // [planes][8][W][strip_h] row-shifted column-major reference byte planes
  int strip_h;
  uint8_t* tail;          // [poi][rem_rows * n_h][planes][32] remainder-row reference blocks
  int64_t* poi_sf;       // [poi] sum f
  double* poi_sqrtvf;    // [poi] sqrt(n Sff - Sf^2)
  uint32_t* S1;          // [SH][SW] window sums of g
  double* SQ;            // [SH][SW] sqrt(n Sgg - Sg^2) (0: constant window)
  float* RSQ;            // [SH][SW] ~1 / SQ (argmax candidate filter)
  int64_t* sfg;          // [poi][2R+1][2R+1] exact cross terms from the tensor cores
  void* tiles;           // [n_tiles] uint4: tx|ty<<16, ix_lo|iy_lo<<16, nix|niy<<16
  double* surface;       // optional [poi][2R+1][2R+1]
  void* slices;          // fused block-sum search: per [poi][dy slice] filter winner (bfs_bs.cu) + flag list
  dicb200_poi_record* rec;
};

// Reference-side inputs of the tensor-core search (strip images, POI moments)
// kept across pairs that share a reference frame (analyze_sequence). `key`
// identifies the frame within one call; reset() between calls.
struct TcRefCache {
  void* strips = nullptr;
  void* psf = nullptr;
  void* pvf = nullptr;
  void* tail = nullptr;
  size_t strips_cap = 0, psf_cap = 0, pvf_cap = 0, tail_cap = 0;
  // per-pair scratch (window sums, cross terms, tile list), reused by every pair
  // on the cache's stream: no allocation per pair, so the memory pool never has
  // to grow (map GBs of fresh pages) in the middle of a sequence
  void* s1 = nullptr;
  void* s2 = nullptr;
  void* sfg = nullptr;
  void* tiles = nullptr;
  void* slices = nullptr;
  size_t s1_cap = 0, s2_cap = 0, sfg_cap = 0, tiles_cap = 0, slices_cap = 0;
  long key = -1;
  const void* data = nullptr;
  int W = 0, H = 0, M = 0, x0 = 0, y0 = 0, step = 0, nx = 0, rb = 0, re = 0;
  int planes = 0;
  bool use_bs = false;  // built for the block-sum kernel (no strip images)
  // declared-width guard (host.cu): device flags {reference, target} and the
  // reference frame flags[0] was computed for (checked once while it repeats)
  int* guard = nullptr;
  long guard_key = -1;
  const void* guard_data = nullptr;
  int guard_bits = -1;
  void reset() { key = -1; guard_key = -1; }
};

// Plans the tensor-core search for POI rows [rb, re); false = not applicable
// (whole-image domain, too many POIs per tile, shared memory).
bool tc_plan(TcParams& p);
// Enqueues stats, reference preparation, the tensor-core kernel and the
// per-POI merge (or only the surface when p.surface is set) on `st`.
cudaError_t tc_launch(TcParams& p, cudaStream_t st, TcRefCache* cache = nullptr, long ref_key = -1);
// ---- K1-BS: shared block sums on CUDA cores (bfs_bs.cu) ----
struct BsGeom {
  int S, RR, q, PX, PY, nbx, nby, nblk, EW, DXC, nchunk, dy_per, nsplit;  // s, r, L / s, POI tile, blocks
  int RWp, RHp, TWp, THp;                                                // staged regions (pixels)
  size_t off_tgt, off_blk, off_state, off_pos, smem;
  int threads;
  int fuse;      // exact argmax fused into the kernel (records via bs_merge_kernel), no cross-term buffer
  int minb;      // CTAs per SM the variant targets
  int async_ok;  // u16 images with 8-byte aligned rows: cp.async staging
  int ws, npw, ncw;  // warp-specialised kernel (bs_ws_kernel): producer / consumer warps
};
bool bs_plan(const TcParams& p, BsGeom& g);
cudaError_t bs_launch(const TcParams& p, const BsGeom& g, cudaStream_t st);
// records from the fused kernel's per-slice results (p.slices)
cudaError_t bs_merge_launch(const TcParams& p, const BsGeom& g, cudaStream_t st);
size_t bs_slices_bytes(size_t npoi, const BsGeom& g);  // p.slices buffer of the fused search

// async: stream-ordered release on `st` (device-resident callers); else cudaFree.
void tc_cache_free(TcRefCache& c, cudaStream_t st = nullptr, bool async = false);

}  // namespace dicb200
