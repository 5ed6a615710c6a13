// K1 on the 5th-generation tensor cores: brute-force ZNCC search over a
// +-R window (bfs_search, integer_search.cpp:52-79; zncc, correlation.cpp:41-72)
// with every cross term Sfg computed EXACTLY by tcgen05.mma kind::i8
// (u8 x u8 -> s32 in TMEM).
//
// GEMM view. A "position" q = (qx, qy) is the top-left corner of a target
// subset. For a POI P with reference subset f_P and a position q,
//   Sfg(P, q) = sum_{r,c} f_P[r][c] * g[qy + r][qx + c].
// One tile = 128 positions (16 in x, 8 in y) = the MMA's M rows; the tile's N
// columns are the POIs whose +-R windows touch it (x the reference byte
// planes); K runs over the subset pixels in blocks of 8 rows x 4 columns.
//
// A operand (positions x K) without an im2col: the target rows are staged as
// 16-pixel windows T[X][y][0..15] = g[Y0 + y][X0 + X + i]. An MN-major,
// no-swizzle UMMA descriptor with SBO = 16 B (next M chunk = next row y) and
// LBO = HT*16 B (next K group = next column offset X) then reads
//   A[(mx, my)][(j, i)] = T[cg*4 + j][rg*8 + my + i][mx]
//                       = g[Y0 + my + rg*8 + i][X0 + mx + cg*4 + j]
// directly: the 8-row core matrices of neighbouring M chunks overlap.
// B operand (K x N, K-major, no swizzle): each POI's 8-row x 4-column
// reference blocks, gathered per stage with 8-byte cp.async from row-shifted
// column-major copies of the reference byte planes (tc_strips_kernel).
//
// 16-bit pixels: g = 256 gh + gl, f = 256 fh + fl; A runs once per g plane
// into its own accumulator, N holds both f planes, and
//   Sfg = 65536 D[gh,fh] + 256 (D[gh,fl] + D[gl,fh]) + D[gl,fl]
// (every partial < 2^31 for side <= 129). Sg and Sgg per position come from a
// separate exact box-sum pass, Sf and Sff per POI from the preparation pass.
// The kernel streams the exact Sfg of every in-window position to HBM; ZNCC,
// the evaluation count and the argmax (or the PSO surface) are then formed
// exactly as in bfs.cu by tc_argmax_kernel / tc_surface_kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bfs.cuh"
#include "common.cuh"

namespace dicb200 {

namespace {

constexpr int kTX = 16, kTY = 8;  // positions per tile: x, y (M = 128)
constexpr int kMaxTilePoi = 128;  // per-tile POI limit (N <= 256 for byte planes)
constexpr int kMaxStages = 8;
// MMA-issuer clock breakdown (DICB200_TC_DBG=32 with -DDICB200_TC_CLOCKS=1; tools)
#ifndef DICB200_TC_CLOCKS
#define DICB200_TC_CLOCKS 0
#endif
constexpr bool kClocks = DICB200_TC_CLOCKS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, SWIZZLE_NONE (16-byte units; version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// Instruction descriptor: kind::i8, D s32, A u8 MN-major, B u8 K-major, M = 128.
__device__ __forceinline__ uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 15) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// Issued by one elected lane of a converged warp (the warp keeps the loop
// state in uniform registers).
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int sleep_ns = 0) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) break;
    if (sleep_ns) __nanosleep(sleep_ns);  // waiting roles yield issue slots to the MMA / working warps
  }
}

// Warp-converged wait: the exit condition is warp-uniform (vote), so the
// caller's loop state stays in uniform registers.
__device__ __forceinline__ void mbar_wait_warp(uint32_t bar, uint32_t parity) {
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (__all_sync(0xffffffffu, done)) break;
  }
}

// int64 -> double without the XU conversion unit (exact for |x| < 2^51: the
// value sits in the mantissa of 1.5 * 2^52 + x); wider values fall back.
__device__ __forceinline__ double i64_to_f64(int64_t x) {
  if (x >= -(1ll << 51) && x < (1ll << 51))
    return __longlong_as_double(0x4338000000000000ll + x) - 6755399441055744.0;
  return (double)x;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// 8-byte async copy; bytes past src_size (0..8) are zero-filled.
__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, int src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_size)
               : "memory");
}

// POIs (lattice index ranges) whose windows intersect the tile rectangle.
__host__ __device__ inline void tile_pois(const TcParams& p, int X0, int Y0, int& ix_lo, int& nix, int& iy_lo,
                                          int& niy) {
  auto ceil_div = [](int a, int b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); };
  auto floor_div = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
  const int s = p.lat.step;
  int lo = ceil_div(X0 + p.M - p.R - p.lat.x0, s), hi = floor_div(X0 + kTX - 1 + p.M + p.R - p.lat.x0, s);
  lo = max(lo, 0);
  hi = min(hi, p.lat.nx - 1);
  ix_lo = lo;
  nix = max(0, hi - lo + 1);
  lo = ceil_div(Y0 + p.M - p.R - p.lat.y0, s);
  hi = floor_div(Y0 + kTY - 1 + p.M + p.R - p.lat.y0, s);
  lo = max(lo, p.rb);
  hi = min(hi, p.re - 1);
  iy_lo = lo;
  niy = max(0, hi - lo + 1);
}

// ---- exact window sums of g and g^2 at every position of the domain ----
// CTA = 64 x ty positions (ty = 64, or 32/16 for large subsets). The target
// region is staged in shared memory by rows (division-free, batched loads);
// row sums over `side` columns go to shared memory (odd pitches: lanes walk
// rows without bank conflicts), then column sums over `side` rows slide down
// each output column, so the global stores of S1/SQ/RSQ are coalesced rows.
// Exact in integers: u32 sums, squares summed in u32 along rows when
// side * maxv^2 < 2^32 (H2 = uint32_t), else u64; u64 along columns.
constexpr int kStatsBX = 64, kStatsSeg = 16, kStatsCh = 16, kStatsHP = kStatsBX + 1;

__host__ __device__ inline int stats_reg_pitch(int side) {  // u16 elements, odd number of 4-byte words
  int rw = (kStatsBX + side - 1 + 1) & ~1;
  if (((rw >> 1) & 1) == 0) rw += 2;
  return rw;
}
__host__ __device__ inline size_t stats_smem_bytes(int side, int ty, bool sq32) {
  const size_t RH = ty + side - 1;
  return ((RH * stats_reg_pitch(side) * 2 + 15) & ~size_t(15)) + ((RH * kStatsHP * 4 + 15) & ~size_t(15)) +
         RH * kStatsHP * (sq32 ? 4 : 8);
}

template <typename Pix, typename H2>
__global__ void __launch_bounds__(256) tc_stats_kernel(TcParams p, int ty) {
  extern __shared__ __align__(16) unsigned char stats_smem[];
  const int side = p.side, RWp = stats_reg_pitch(side), RW = kStatsBX + side - 1;
  const int RH = ty + side - 1;
  uint16_t* reg = reinterpret_cast<uint16_t*>(stats_smem);
  uint32_t* h1 = reinterpret_cast<uint32_t*>(stats_smem + (((size_t)RH * RWp * 2 + 15) & ~size_t(15)));
  H2* h2 = reinterpret_cast<H2*>(reinterpret_cast<unsigned char*>(h1) + (((size_t)RH * kStatsHP * 4 + 15) & ~size_t(15)));
  const int sx0 = blockIdx.x * kStatsBX, sy0 = blockIdx.y * ty;
  const int rows = min(ty, p.SH - sy0), cols = min(kStatsBX, p.SW - sx0);
  const Pix* img = reinterpret_cast<const Pix*>(p.tgt.data);
  const int pitch = p.tgt.pitch, gx0 = p.qx_min + sx0, gy0 = p.qy_min + sy0;
  const int W = p.tgt.width, H = p.tgt.height;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rh = rows + side - 1;  // region rows this CTA needs
  // staging: one warp per region row, 4 independent loads per lane in flight
  for (int r = warp; r < rh; r += 8) {
    const int gy = gy0 + r;
    const Pix* src = img + (size_t)min(gy, H - 1) * pitch;
    uint16_t* dst = reg + r * RWp;
    for (int c0 = 0; c0 < RW; c0 += 128) {
      uint16_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 32 + lane, gx = gx0 + c;
        v[u] = (c < RW && gy < H && gx < W) ? (uint16_t)src[gx] : (uint16_t)0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u * 32 + lane < RW) dst[c0 + u * 32 + lane] = v[u];
    }
  }
  __syncthreads();
  // row sums over `side` columns: h[r][x0 .. x0+15]; lanes take consecutive rows
  constexpr int nseg = kStatsBX / kStatsSeg;
  for (int item = threadIdx.x; item < rh * nseg; item += blockDim.x) {
    const int seg = item / rh, r = item - seg * rh, x0 = seg * kStatsSeg;
    const uint16_t* row = reg + r * RWp + x0;
    uint32_t s1 = 0;
    H2 s2 = 0;
#pragma unroll 8
    for (int c = 0; c < side; ++c) {
      const uint32_t v = row[c];
      s1 += v;
      s2 += (H2)v * v;
    }
    uint32_t* o1 = h1 + r * kStatsHP + x0;
    H2* o2 = h2 + r * kStatsHP + x0;
    o1[0] = s1;
    o2[0] = s2;
#pragma unroll
    for (int x = 1; x < kStatsSeg; ++x) {
      const uint32_t a = row[x + side - 1], b = row[x - 1];
      s1 += a - b;
      s2 += (H2)a * a - (H2)b * b;  // modular: the running sum itself fits H2
      o1[x] = s1;
      o2[x] = s2;
    }
  }
  __syncthreads();
  // column sums over `side` rows, sliding down kStatsCh outputs per item
  const int nch = (rows + kStatsCh - 1) / kStatsCh;
  const int64_t nn = (int64_t)side * side;
  for (int item = threadIdx.x; item < kStatsBX * nch; item += blockDim.x) {
    const int x = item % kStatsBX, t0 = (item / kStatsBX) * kStatsCh;
    if (x >= cols) continue;
    uint32_t s1 = 0;
    uint64_t s2 = 0;
#pragma unroll 8
    for (int r = 0; r < side; ++r) {
      s1 += h1[(t0 + r) * kStatsHP + x];
      s2 += (uint64_t)h2[(t0 + r) * kStatsHP + x];
    }
    size_t o = (size_t)(sy0 + t0) * p.SW + sx0 + x;
    const int t1 = min(t0 + kStatsCh, rows);
    for (int t = t0;;) {
      // sqrt(vg) exactly as zncc_from_moments forms it (0 = degenerate window)
      const int64_t vg = nn * (int64_t)s2 - (int64_t)s1 * (int64_t)s1;
      const double sq = vg > 0 ? sqrt((double)vg) : 0.0;
      p.S1[o] = s1;
      p.SQ[o] = sq;
      p.RSQ[o] = vg > 0 ? (float)(1.0 / sq) : 0.0f;
      if (++t >= t1) break;
      s1 += h1[(t + side - 1) * kStatsHP + x] - h1[(t - 1) * kStatsHP + x];
      s2 += (uint64_t)h2[(t + side - 1) * kStatsHP + x] - (uint64_t)h2[(t - 1) * kStatsHP + x];
      o += p.SW;
    }
  }
}

// tile height and squares width of the stats kernel (largest tile within ~110 KB)
static bool stats_sq32(const TcParams& p) {
  const double maxv = p.maxv > 0 ? p.maxv : (p.planes == 1 ? 255.0 : 65535.0);
  return (double)p.side * maxv * maxv < 4294967296.0;
}
static int stats_ty(const TcParams& p) {
  const bool q = stats_sq32(p);
  for (int ty : {64, 32})
    if (stats_smem_bytes(p.side, ty, q) <= 110 * 1024) return ty;
  return 16;
}

// ---- per POI: exact reference moments (separable window sums at the lattice) ----
// One CTA per POI row: column sums over the subset rows for every column, then
// each POI sums its `side` columns. Exact in integers.
template <typename Pix>
__global__ void __launch_bounds__(256) tc_prep_kernel(TcParams p) {
  extern __shared__ __align__(16) unsigned char prep_smem[];
  const int W = p.ref.width, pitch = p.ref.pitch, M = p.M, side = p.side;
  uint32_t* c1 = reinterpret_cast<uint32_t*>(prep_smem);
  uint64_t* c2 = reinterpret_cast<uint64_t*>(prep_smem + (((size_t)W * 4 + 15) & ~size_t(15)));
  const int iy = p.rb + blockIdx.x, y0 = p.lat.cy(iy) - M;
  const Pix* img = reinterpret_cast<const Pix*>(p.ref.data);
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    uint32_t s1 = 0;
    uint64_t s2 = 0;
    for (int r = 0; r < side; ++r) {
      const uint32_t v = img[(size_t)(y0 + r) * pitch + x];
      s1 += v;
      s2 += (uint64_t)v * v;
    }
    c1[x] = s1;
    c2[x] = s2;
  }
  __syncthreads();
  const int64_t n = (int64_t)side * side;
  for (int ix = threadIdx.x; ix < p.lat.nx; ix += blockDim.x) {
    const int x0 = p.lat.cx(ix) - M;
    uint64_t sf = 0, sff = 0;
    for (int c = 0; c < side; ++c) {
      sf += c1[x0 + c];
      sff += c2[x0 + c];
    }
    const int64_t vf = n * (int64_t)sff - (int64_t)sf * (int64_t)sf;
    const size_t k = (size_t)blockIdx.x * p.lat.nx + ix;
    p.poi_sf[k] = (int64_t)sf;
    p.poi_sqrtvf[k] = vf > 0 ? sqrt((double)vf) : 0.0;
  }
  // remainder-row blocks of every POI of the row: tail[poi][q = ry n_h + h][plane][32 bytes]
  if (p.rem) {
    const int Q = p.rem_rows * p.n_h, r0 = 8 * (p.RG - 1);
    const int per_poi = Q * p.planes * 8;  // words
    for (int e = threadIdx.x; e < p.lat.nx * per_poi; e += blockDim.x) {
      const int ix = e / per_poi, rest = e - ix * per_poi;
      const int w = rest & 7, qp = rest >> 3, pl = qp % p.planes, q = qp / p.planes;
      const int ry = q / p.n_h, h = q - ry * p.n_h;
      const int x0 = p.lat.cx(ix) - M + 32 * h + 4 * w;
      const Pix* row = img + (size_t)(y0 + r0 + ry) * pitch;
      const int shift = (p.planes == 2 && pl == 0) ? 8 : 0;
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = 32 * h + 4 * w + b;
        if (c < side) word |= (((uint32_t)row[x0 + b] >> shift) & 0xffu) << (8 * b);
      }
      reinterpret_cast<uint32_t*>(p.tail)[((size_t)blockIdx.x * p.lat.nx + ix) * per_poi + rest] = word;
    }
  }
}

// ---- reference byte planes as 8 row-shifted strip images ----
// strips[pl][s][y8][x][i] = plane_pl(ref[8 y8 + i + s][x]): the 8-row column
// runs of one 8-row band lie side by side, so the MMA's B block of a POI (8
// subset rows x 4 consecutive columns, K-major = column runs) is 32 contiguous
// bytes of strip s = (first row) % 8 — gathered with cp.async straight from
// here, no per-POI copies of the reference.
template <typename Pix>
__global__ void __launch_bounds__(256) tc_strips_kernel(TcParams p) {
  constexpr int CX = 32, CY = 64;
  __shared__ uint16_t tile[CY + 8][CX + 1];
  const int x0 = blockIdx.x * CX, y0 = blockIdx.y * CY;
  const Pix* img = reinterpret_cast<const Pix*>(p.ref.data);
  const int W = p.ref.width, H = p.ref.height, pitch = p.ref.pitch, Hs = p.strip_h;
  for (int i = threadIdx.x; i < (CY + 8) * CX; i += blockDim.x) {
    const int r = i / CX, c = i - r * CX, gy = y0 + r, gx = x0 + c;
    tile[r][c] = (gy < H && gx < W) ? (uint16_t)img[(size_t)gy * pitch + gx] : (uint16_t)0;
  }
  __syncthreads();
  const int per_plane = 8 * CX * (CY / 4);
  for (int item = threadIdx.x; item < p.planes * per_plane; item += blockDim.x) {
    const int q = item % (CY / 4), c = (item / (CY / 4)) % CX, sft = (item / (CX * (CY / 4))) % 8,
              pl = item / per_plane;
    if (x0 + c >= W) continue;
    const int shift = (p.planes == 2 && pl == 0) ? 8 : 0;
    uint32_t w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) w |= (((uint32_t)tile[q * 4 + e + sft][c] >> shift) & 0xffu) << (8 * e);
    const int yy = y0 + q * 4;  // strip row of the word's first byte
    *reinterpret_cast<uint32_t*>(p.strips + ((size_t)(pl * 8 + sft) * (Hs / 8) + (yy >> 3)) * W * 8 +
                                 (size_t)(x0 + c) * 8 + (yy & 7)) = w;
  }
}

// ---- per tile: position tile coordinates and the POI rectangle it serves ----
__global__ void tc_tiles_kernel(TcParams p) {
  const int tile = blockIdx.x * blockDim.x + threadIdx.x;
  if (tile >= p.n_tiles) return;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  int ix_lo, nix, iy_lo, niy;
  tile_pois(p, p.qx_min + kTX * tx, p.qy_min + kTY * ty, ix_lo, nix, iy_lo, niy);
  reinterpret_cast<uint4*>(p.tiles)[tile] =
      make_uint4((uint32_t)tx | ((uint32_t)ty << 16), (uint32_t)ix_lo | ((uint32_t)iy_lo << 16),
                 (uint32_t)nix | ((uint32_t)niy << 16), 0u);
}

// ---- the tensor-core kernel: persistent, warp-specialised ----
//   warps 0-3 : producers — per K stage (8 subset rows): target rows -> byte
//               planes -> 16-pixel windows (A), reference bytes (B, cp.async)
//   warp  4   : one thread issues the tcgen05.mma stream
//   warps 5-8 : epilogue — TMEM -> exact moments -> ZNCC -> per-POI argmax
// Stages form a ring (full/empty mbarriers); the two TMEM accumulators let the
// epilogue of tile t overlap the MMAs of tile t+1.
constexpr int kGroups = 5, kGroupThreads = 64;  // producer groups = ring slots
constexpr int kProducerWarps = kGroups * kGroupThreads / 32;
constexpr int kProducers = kGroups * kGroupThreads, kEpilogue = 256;
constexpr int kMmaWarps = 2;  // one tcgen05 issuer per byte plane of the target
constexpr int kTcThreads = kProducers + 32 * kMmaWarps + kEpilogue;
constexpr int kStageRows = 16;  // T rows per stage: 8 positions + 8 subset rows - 1, rounded

struct TileInfo {
  int tx, ty, X0, Y0, ix_lo, nix, iy_lo, niy, npoi, N;
};

template <int PLANES>
__device__ __forceinline__ bool tile_info(const TcParams& p, int tile, TileInfo& t) {
  const uint4 q = __ldg(reinterpret_cast<const uint4*>(p.tiles) + tile);  // tc_tiles_kernel
  t.tx = (int)(q.x & 0xffffu);
  t.ty = (int)(q.x >> 16);
  t.X0 = p.qx_min + kTX * t.tx;
  t.Y0 = p.qy_min + kTY * t.ty;
  t.ix_lo = (int)(q.y & 0xffffu);
  t.iy_lo = (int)(q.y >> 16);
  t.nix = (int)(q.z & 0xffffu);
  t.niy = (int)(q.z >> 16);
  t.npoi = t.nix * t.niy;
  t.N = max(16, ((t.npoi * PLANES + 15) / 16) * 16);
  return t.npoi > 0;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// Remainder stage of a tile: subset rows r0 .. r0 + rem_rows - 1 (< 8 of them).
//   T2[pl][y][X][0..15] = plane_pl(g[Y0 + r0 + y][X0 + X + i]), y < HT2, X < NX2
//   B2[q = ry * n_h + h][n][k] = plane(f_n[r0 + ry][32 h + k]) (0 past the subset),
//   copied from the per-POI tails written by tc_prep_kernel
template <int PLANES>
__device__ __forceinline__ void build_remainder_stage(const TcParams& p, const TileInfo& t, const int* poi_idx,
                                                      int r0, uint8_t* T, uint8_t* rows8, uint8_t* Bs, int gt,
                                                      int g) {
  const auto* img = reinterpret_cast<const uint8_t*>(p.tgt.data);
  const int W = p.tgt.width, H = p.tgt.height, pitch = p.tgt.pitch;
  const int NX2 = p.NX2, HT2 = p.HT2, RWB2 = p.RWB2, RW42 = (NX2 + 15 + 3) / 4;
  uint32_t* rows = reinterpret_cast<uint32_t*>(rows8);
  // (a) B2: the POIs' precomputed remainder blocks (tc_prep_kernel), 16 bytes per cp.async
  {
    const int NN = t.npoi * PLANES, Q = p.rem_rows * p.n_h;
    const int items = Q * NN * 2;
    for (int e = gt; e < items; e += kGroupThreads) {
      const int kh = e & 1, rest = e >> 1;
      const int nn = rest % NN, q = rest / NN;
      const int j = nn / PLANES, pl = nn - j * PLANES;
      const uint8_t* src = p.tail + (((size_t)poi_idx[j] * Q + q) * PLANES + pl) * 32 + kh * 16;
      cp_async16(Bs + (size_t)q * t.N * 32 + (nn & 7) * 16 + (nn >> 3) * 256 + kh * 128, src);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // (b) target rows -> byte planes (4 pixels per word)
  for (int e = gt; e < HT2 * RW42; e += kGroupThreads) {
    const int y = e / RW42, w = e - y * RW42;
    const int gy = t.Y0 + r0 + y, gx0 = t.X0 + 4 * w;
    uint32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gx = gx0 + i;
      v[i] = 0;
      if (gy < H && gx < W) {
        if (PLANES == 1)
          v[i] = __ldg(img + (size_t)gy * pitch + gx);
        else
          v[i] = __ldg(reinterpret_cast<const uint16_t*>(img) + (size_t)gy * pitch + gx);
      }
    }
    if (PLANES == 1) {
      rows[y * (RWB2 / 4) + w] = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
    } else {
      rows[y * (RWB2 / 4) + w] = __byte_perm(v[0], v[1], 0x7751) | (__byte_perm(v[2], v[3], 0x5177) & 0xffff0000u);
      rows[(HT2 + y) * (RWB2 / 4) + w] =
          __byte_perm(v[0], v[1], 0x7740) | (__byte_perm(v[2], v[3], 0x4077) & 0xffff0000u);
    }
  }
  named_sync(1 + g, kGroupThreads);
  // (c) row-major 16-pixel windows, four column offsets per item
  const size_t planeT2 = (size_t)HT2 * NX2 * 16;
  (void)g;
  for (int e = gt; e < PLANES * HT2 * (NX2 / 4); e += kGroupThreads) {
    const int X4 = e % (NX2 / 4), rest = e / (NX2 / 4), y = rest % HT2, pl = rest / HT2;
    const uint32_t* rw = rows + (size_t)(pl * HT2 + y) * (RWB2 / 4);
    const uint32_t a0 = rw[X4], a1 = rw[X4 + 1], a2 = rw[X4 + 2], a3 = rw[X4 + 3], a4 = rw[X4 + 4];
    uint8_t* dst = T + pl * planeT2 + ((size_t)y * NX2 + 4 * X4) * 16;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      uint4 o;
      o.x = __funnelshift_r(a0, a1, 8 * s);
      o.y = __funnelshift_r(a1, a2, 8 * s);
      o.z = __funnelshift_r(a2, a3, 8 * s);
      o.w = __funnelshift_r(a3, a4, 8 * s);
      *reinterpret_cast<uint4*>(dst + s * 16) = o;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <int PLANES>
__global__ void __launch_bounds__(kTcThreads, 1) bfs_tc_kernel(TcParams p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base;
  __shared__ int2 prod_poi[kGroups * kMaxTilePoi];
  __shared__ int prod_poi_ix[kGroups * kMaxTilePoi];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int S = kGroups;  // ring slots: one per producer group

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int s = 0; s < kGroups; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&full_bar[s])), "r"(kGroupThreads));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&empty_bar[s])), "r"(PLANES));
    }
    for (int a = 0; a < 2; ++a) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&tfull_bar[a])), "r"(PLANES));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&tempty_bar[a])), "r"(kEpilogue));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int NX = p.NX, RWB = p.RWB, CG = p.CG;
  const size_t planeT = (size_t)NX * kStageRows * 16;

  if (warp < kProducerWarps) {
    // ================= producers =================
    // group g (kGroupThreads threads) owns ring slot g and builds every stage it with it % S == g,
    // so S stages (and their global-load latencies) are in flight at once.
    const int g = tid / kGroupThreads, gt = tid % kGroupThreads;
    const auto* img = reinterpret_cast<const uint8_t*>(p.tgt.data);
    const int W = p.tgt.width, H = p.tgt.height, pitch = p.tgt.pitch;
    const int RW4 = (NX + 15 + 3) / 4;  // words per staged row
    int2* poi_tab = prod_poi + g * kMaxTilePoi;
    int* poi_ix = prod_poi_ix + g * kMaxTilePoi;
    uint32_t ph = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      TileInfo t;
      if (!tile_info<PLANES>(p, tile, t)) continue;
      const int first = (g - it % kGroups + kGroups) % kGroups;  // this group's first stage of the tile
      it += p.RG;
      if (first >= p.RG) continue;
      named_sync(1 + g, kGroupThreads);  // previous tile's readers of poi_tab are done
      for (int j = gt; j < t.npoi; j += kGroupThreads) {
        const int jy = j / t.nix, jx = j - jy * t.nix;
        poi_tab[j] = make_int2(p.lat.cx(t.ix_lo + jx) - p.M, p.lat.cy(t.iy_lo + jy) - p.M);
        poi_ix[j] = (t.iy_lo + jy - p.rb) * p.lat.nx + (t.ix_lo + jx);
      }
      named_sync(1 + g, kGroupThreads);
      const int NN = t.npoi * PLANES;
      unsigned char* base = sm + (size_t)g * p.stage_bytes;
      uint8_t* T = base;
      uint32_t* rows = reinterpret_cast<uint32_t*>(base + p.off_rows);
      uint8_t* Bs = base + p.off_B;
      for (int rg = first; rg < p.RG; rg += kGroups) {
        if (p.rem && rg == p.RG - 1) {
          mbar_wait(smem_u32(&empty_bar[g]), ph ^ 1u, 64);
          // remainder rows (e.g. row 40 of a 41-row subset): row-major stage,
          // K = 32 consecutive columns of one subset row per MMA
          build_remainder_stage<PLANES>(p, t, poi_ix, rg * 8, T, reinterpret_cast<uint8_t*>(rows), Bs, gt, g);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_arrive(smem_u32(&full_bar[g]));
          ph ^= 1u;
          named_sync(1 + g, kGroupThreads);
          continue;
        }
        // (b) target rows (no wait: the MMAs never read the row buffer) [Y0 + 8 rg, +16) x [X0, X0 + 4 RW4): 4 pixels -> one word per byte plane
        {
          const int gy0 = t.Y0 + rg * 8;
          for (int w = gt & 15; w < RW4; w += 16) {
            const int gx0 = t.X0 + 4 * w;
            constexpr int RY = kStageRows * 16 / kGroupThreads;  // rows per thread
            constexpr int YS = kGroupThreads / 16;                // row stride
            uint32_t v[RY][4];
#pragma unroll
            for (int k = 0; k < RY; ++k) {
              const int gy = gy0 + (gt >> 4) + YS * k;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int gx = gx0 + i;
                v[k][i] = 0;
                if (gy < H && gx < W) {
                  if (PLANES == 1)
                    v[k][i] = __ldg(img + (size_t)gy * pitch + gx);
                  else
                    v[k][i] = __ldg(reinterpret_cast<const uint16_t*>(img) + (size_t)gy * pitch + gx);
                }
              }
            }
#pragma unroll
            for (int k = 0; k < RY; ++k) {
              const int y = (gt >> 4) + YS * k;
              if (PLANES == 1) {
                rows[y * (RWB / 4) + w] = v[k][0] | (v[k][1] << 8) | (v[k][2] << 16) | (v[k][3] << 24);
              } else {
                rows[y * (RWB / 4) + w] = __byte_perm(v[k][0], v[k][1], 0x7751) | (__byte_perm(v[k][2], v[k][3], 0x5177) & 0xffff0000u);
                rows[(kStageRows + y) * (RWB / 4) + w] =
                    __byte_perm(v[k][0], v[k][1], 0x7740) | (__byte_perm(v[k][2], v[k][3], 0x4077) & 0xffff0000u);
              }
            }
          }
        }
        mbar_wait(smem_u32(&empty_bar[g]), ph ^ 1u, 64);  // T and B of this slot are free
        // (a) B: the tile's reference blocks (8 subset rows x 4 columns per MMA,
        //     K-major) as 8-byte column runs from the strip images; rows/columns
        //     past the subset are zero-filled (cp.async src-size)
        {
          const int r0 = rg * 8, vrows = min(8, p.side - r0);
          const int W = p.ref.width, Hs = p.strip_h;
          for (int jp = gt >> 2; jp < NN; jp += kGroupThreads / 4) {
            const int jc = gt & 3;
            const int j = jp / PLANES, pl = jp - j * PLANES;
            const int2 o = poi_tab[j];  // subset top-left (x, y) in the reference
            const int ry = o.y + r0, sft = ry & 7;
            const uint8_t* strip = p.strips + ((size_t)(pl * 8 + sft) * (Hs / 8) + (ry >> 3)) * W * 8;
            const uint8_t* src = strip + (size_t)(o.x + jc) * 8;
            const size_t src_step = 32;  // next column group: 4 columns x 8 bytes
            uint8_t* dst = Bs + (jp & 7) * 16 + (jp >> 3) * 256 + (jc >> 1) * 128 + (jc & 1) * 8;
            const size_t dst_step = (size_t)t.N * 32;
            const int cg_full = (p.side - jc + 3) / 4;  // column groups holding column jc + 4 cg < side
            for (int cg = 0; cg < CG; ++cg, src += src_step, dst += dst_step)
              cp_async8_zfill(dst, cg < cg_full ? src : strip, cg < cg_full ? vrows : 0);
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        named_sync(1 + g, kGroupThreads);
        // (c) 16-pixel windows, four column offsets per item:
        //     T[pl][X][y][0..15] = rows[pl][y][X .. X+15], X = 4 X4 + s
        {
          const int y = gt & 15;
          for (int pl = 0; pl < PLANES; ++pl) {
            const uint32_t* rw = rows + (size_t)(pl * kStageRows + y) * (RWB / 4);
            for (int X4 = gt >> 4; X4 < CG; X4 += kGroupThreads / 16) {
              const uint32_t a0 = rw[X4], a1 = rw[X4 + 1], a2 = rw[X4 + 2], a3 = rw[X4 + 3], a4 = rw[X4 + 4];
              uint8_t* dst = T + pl * planeT + ((size_t)(4 * X4) * kStageRows + y) * 16;
#pragma unroll
              for (int s = 0; s < 4; ++s) {
                uint4 o;
                o.x = __funnelshift_r(a0, a1, 8 * s);
                o.y = __funnelshift_r(a1, a2, 8 * s);
                o.z = __funnelshift_r(a2, a3, 8 * s);
                o.w = __funnelshift_r(a3, a4, 8 * s);
                *reinterpret_cast<uint4*>(dst + s * kStageRows * 16) = o;
              }
            }
          }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(smem_u32(&full_bar[g]));
        ph ^= 1u;
        named_sync(1 + g, kGroupThreads);  // rows of this slot are rewritten next round
      }
    }
  } else if (warp < kProducerWarps + kMmaWarps) {
    if (warp - kProducerWarps >= PLANES) {
      // spare issuer (single-plane data)
    } else {
    // ================= MMA issuers =================
    // issuer pl handles target byte plane pl into its own accumulator
    // The whole warp runs the loop (descriptors stay in uniform registers);
    // one elected lane issues each tcgen05.mma / commit.
    {
      int it = 0, tc = 0;
      long long w_full = 0, w_empty = 0, t_issue = 0, t0 = kClocks ? clock64() : 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        TileInfo t;
        if (!tile_info<PLANES>(p, tile, t)) continue;
        const int a = tc & 1;
        const uint32_t aph = (uint32_t)(tc >> 1) & 1u;
        const long long c0 = kClocks ? clock64() : 0;
        mbar_wait_warp(smem_u32(&tempty_bar[a]), aph ^ 1u);
        if (kClocks) w_empty += clock64() - c0;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int pl = warp - kProducerWarps;
        const uint32_t d0 = tmem + (uint32_t)(a * PLANES * p.N_max) + (uint32_t)(pl * t.N);
        const uint32_t idesc = idesc_i8(t.N);
        const uint32_t b_step = (uint32_t)t.N * 2u;  // B block per cg, 16-byte units
        for (int rg = 0; rg < p.RG; ++rg, ++it) {
          const int s = it % S;
          const uint32_t ph = (uint32_t)(it / S) & 1u;
          const long long c1 = kClocks ? clock64() : 0;
          mbar_wait_warp(smem_u32(&full_bar[s]), ph);
          const long long c2 = kClocks ? clock64() : 0;
          if (kClocks) w_full += c2 - c1;
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t base = smem_u32(sm + (size_t)s * p.stage_bytes);
          if (p.rem && rg == p.RG - 1) {
            // row-major remainder stage: M chunks = rows (SBO = NX2 x 16 B),
            // K rows = consecutive columns (16 B), K groups = +8 columns (LBO = 128 B)
            const uint32_t planeT2 = (uint32_t)(p.HT2 * p.NX2 * 16);
            for (int ry = 0; ry < p.rem_rows; ++ry)
              for (int h = 0; h < p.n_h; ++h) {
                const uint64_t da = sdesc(base + pl * planeT2 + (uint32_t)((ry * p.NX2 + 32 * h) * 16), 128,
                                          (uint32_t)(p.NX2 * 16));
                const uint64_t db =
                    sdesc(base + (uint32_t)p.off_B + (uint32_t)((ry * p.n_h + h) * t.N * 32), 128, 256);
                mma_i8_elect(d0, da, db, idesc, 1u);
              }
            umma_commit_elect(smem_u32(&empty_bar[s]));
            if (kClocks) t_issue += clock64() - c2;
            continue;
          }
          uint64_t da = sdesc(base + (uint32_t)(pl * planeT), kStageRows * 16, 16);
          uint64_t db = sdesc(base + (uint32_t)p.off_B, 128, 256);
          for (int cg = 0; cg < CG; ++cg) {
            const uint32_t acc = (rg | cg) != 0;
            mma_i8_elect(d0, da, db, idesc, acc);
            da += (uint64_t)(4 * kStageRows);
            db += (uint64_t)b_step;
          }
          umma_commit_elect(smem_u32(&empty_bar[s]));
          if (kClocks) t_issue += clock64() - c2;
        }
        umma_commit_elect(smem_u32(&tfull_bar[a]));
        ++tc;
      }
      if (kClocks && p.dbg_out && lane == 0 && warp == kProducerWarps) {
        p.dbg_out[blockIdx.x * 4 + 0] = clock64() - t0;
        p.dbg_out[blockIdx.x * 4 + 1] = w_full;
        p.dbg_out[blockIdx.x * 4 + 2] = w_empty;
        p.dbg_out[blockIdx.x * 4 + 3] = t_issue;
      }
    }
    }
  } else if (warp >= kProducerWarps + kMmaWarps) {
    // ================= epilogue =================
    // thread = position (TMEM lane quadrant = warp % 4; the two warps of a
    // quadrant split the POI column groups): the exact cross terms Sfg of every
    // in-window position go to sfg[poi][dy + R][dx + R]; ZNCC and the argmax run
    // in tc_argmax_kernel / tc_surface_kernel.
    const int quad = warp & 3, half = (warp - kProducerWarps - kMmaWarps) >> 2;
    const int m = quad * 32 + lane, mx = m & 15, my = m >> 4;
    const int R = p.R, EW = 2 * R + 1;
    constexpr int PER = 8 / PLANES;  // POIs per 8 accumulator columns
    int tc = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      TileInfo t;
      if (!tile_info<PLANES>(p, tile, t)) continue;
      const int a = tc & 1;
      const uint32_t aph = (uint32_t)(tc >> 1) & 1u;
      ++tc;
      const int qx = t.X0 + mx, qy = t.Y0 + my;
      const bool in_domain = qx <= p.qx_max && qy <= p.qy_max;
      const int rx = qx + p.M - t.ix_lo * p.lat.step - p.lat.x0;  // dx = rx - jx * step
      const int ry = qy + p.M - t.iy_lo * p.lat.step - p.lat.y0;
      const int ngroups = (t.npoi + PER - 1) / PER;
      int jy = 0, jx = half * PER;  // lattice offsets of POI gi * PER
      while (jx >= t.nix) {
        jx -= t.nix;
        ++jy;
      }
      mbar_wait(smem_u32(&tfull_bar[a]), aph, 64);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tl = tmem + (uint32_t)(a * PLANES * p.N_max) + ((uint32_t)(quad * 32) << 16);
      for (int gi = half; gi < ngroups; gi += 2) {
        const int j0 = gi * PER;
        uint32_t d0[8], d1[8];
        tmem_ld8(tl + (uint32_t)(j0 * PLANES), d0);
        if (PLANES == 2) tmem_ld8(tl + (uint32_t)(t.N + j0 * PLANES), d1);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        int ux = jx, uy = jy;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int dx = rx - ux * p.lat.step, dy = ry - uy * p.lat.step;
          if (j0 + u < t.npoi && in_domain && dx >= -R && dx <= R && dy >= -R && dy <= R) {
            int64_t sfg;
            if (PLANES == 1)
              sfg = (int64_t)d0[u];
            else
              sfg = 65536ll * (int64_t)d0[2 * u] + 256ll * ((int64_t)d0[2 * u + 1] + (int64_t)d1[2 * u]) +
                    (int64_t)d1[2 * u + 1];
            const size_t poi = (size_t)(t.iy_lo + uy - p.rb) * p.lat.nx + (t.ix_lo + ux);
            p.sfg[poi * EW * EW + (size_t)(dy + R) * EW + (dx + R)] = sfg;
          }
          if (++ux == t.nix) {
            ux = 0;
            ++uy;
          }
        }
        jx += 2 * PER;
        while (jx >= t.nix) {
          jx -= t.nix;
          ++jy;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(smem_u32(&tempty_bar[a]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(p.tmem_cols));
}

// One candidate's exact numerator n Sfg - Sf Sg from the tensor-core cross
// term and the exact window sums (as zncc_from_moments, common.cuh).
struct Cand {
  int64_t num;
  double sq;   // sqrt(n Sgg - Sg^2), computed once per position by tc_stats_kernel
  float rsq;   // ~1 / sq (candidate filter only)
};

// Position data (Sg, ~1/sqrt(vg)) of the union of a strip's windows, staged in
// shared memory once per CTA (neighbouring POIs share most positions); the
// exact sqrt(vg) is read from global memory for the few near-maximal
// candidates only (tc_argmax_kernel). The surface kernel views global memory.
struct PosView {
  const double* sq;  // surface kernel only
  const uint32_t* s1;
  const float* rsq;
  int x0, y0, W;
};

__host__ __device__ inline size_t pos_smem_bytes(const TcParams& p, int sp) {
  const size_t W = (size_t)(sp - 1) * p.lat.step + 2 * p.R + 1, H = 2 * (size_t)p.R + 1;
  return W * H * 8;
}

__device__ __forceinline__ PosView stage_positions(const TcParams& p, int iy, int ix0, int ts, unsigned char* sm) {
  PosView v;
  const int M = p.M, R = p.R;
  v.x0 = max(p.lat.cx(ix0) - M - R, p.qx_min);
  const int x1 = min(p.lat.cx(ix0 + ts - 1) - M + R, p.qx_max);
  v.y0 = max(p.lat.cy(iy) - M - R, p.qy_min);
  const int y1 = min(p.lat.cy(iy) - M + R, p.qy_max);
  v.W = max(0, x1 - v.x0 + 1);
  const int H = max(0, y1 - v.y0 + 1), N = v.W * H;
  uint32_t* s1 = reinterpret_cast<uint32_t*>(sm);
  float* rsq = reinterpret_cast<float*>(sm + (size_t)N * 4);
  for (int r = threadIdx.x >> 5; r < H; r += blockDim.x >> 5) {
    const size_t o = (size_t)(v.y0 + r - p.qy_min) * p.SW + (v.x0 - p.qx_min);
    for (int c = threadIdx.x & 31; c < v.W; c += 32) {
      s1[r * v.W + c] = p.S1[o + c];
      rsq[r * v.W + c] = p.RSQ[o + c];
    }
  }
  __syncthreads();
  v.sq = nullptr;
  v.s1 = s1;
  v.rsq = rsq;
  return v;
}

// n <= 129^2 and Sf, Sg <= 129^2 * 65535 < 2^31 fit 32 bits, Sfg (>= 0) 64: two
// wide multiplies, exact in wrap-around 64-bit arithmetic.
__device__ __forceinline__ bool tc_candidate_s(const PosView& v, uint32_t n, uint32_t sf, int64_t sfg, int qx, int qy,
                                               Cand& c) {
  const int o = (qy - v.y0) * v.W + (qx - v.x0);
  c.sq = v.sq[o];
  if (!(c.sq > 0.0)) return false;  // constant target window: skipped, not counted
  c.rsq = v.rsq[o];
  c.num = (int64_t)((uint64_t)sfg * n - (uint64_t)sf * v.s1[o]);
  return true;
}

// Filter pass: rsq > 0 exactly when sqrt(vg) > 0 (tc_stats_kernel writes 0 for
// both when vg <= 0, and 1/sqrt(vg) >= 2^-32 is a normal float otherwise).
__device__ __forceinline__ bool tc_candidate_f(const PosView& v, uint32_t n, uint32_t sf, int64_t sfg, int qx, int qy,
                                               int64_t& num, float& rsq) {
  const int o = (qy - v.y0) * v.W + (qx - v.x0);
  rsq = v.rsq[o];
  if (!(rsq > 0.0f)) return false;  // constant target window: skipped, not counted
  num = (int64_t)((uint64_t)sfg * n - (uint64_t)sf * v.s1[o]);
  return true;
}
__device__ __forceinline__ double tc_sq(const TcParams& p, int qx, int qy) {
  return p.SQ[(size_t)(qy - p.qy_min) * p.SW + (qx - p.qx_min)];
}

// Filter value num / (sqrt(vf) sqrt(vg)) in fp32: five roundings of relative
// 2^-24 each (num, 1/sqrt(vf), 1/sqrt(vg), two products) -> absolute error
// < 5.1 * 2^-24 < 2^-21.6 for |zncc| <= 1. No overflow or denormals:
// |num| <= n Sfg < 2^14.1 * 2^46.1, each reciprocal factor >= 2^-30.1.
__device__ __forceinline__ float approx_zncc(int64_t num, float rsvf, float rsq) {
  return __fmul_rn(__fmul_rn(__ll2float_rn(num), rsvf), rsq);
}

// ---- per POI: count, exact argmax in improves() order -> record ----
// One pass finds the maximum of a cheap fp32 quotient num * (1/sqrt(vf)) * rsq
// with rsq the fp32 reciprocal of sqrt(vg) (approx_zncc: absolute error
// < 2^-21.6 as |zncc| <= 1); the EXACT IEEE quotient num / (sqrt(vf) sqrt(vg)) is
// formed only for candidates within 2^-19 of it (a second pass when more than one per lane
// qualifies): the exact argmax, in improves() order, of the correlation formed
// from exact integer moments. The reference accumulates centred doubles with
// rounding, so its values differ from these in the last bits and the two can
// only disagree at ties closer than that (sub-ulp). Warp per POI, lanes across
// the window candidates.
__global__ void __launch_bounds__(256) tc_argmax_kernel(TcParams p, int sp) {
  extern __shared__ __align__(16) unsigned char pos_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int iy = p.rb + blockIdx.y, ix0 = blockIdx.x * sp, ts = min(sp, p.lat.nx - ix0);
  const PosView pv = stage_positions(p, iy, ix0, ts, pos_smem);
  if (w >= ts) return;
  const int ix = ix0 + w, k = (iy - p.rb) * p.lat.nx + ix;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, R = p.R, EW = 2 * R + 1;
  const uint32_t n = (uint32_t)(p.side * p.side);
  const int fx_lo = max(-R, M - cx), fx_hi = min(R, p.tgt.width - 1 - M - cx);   // integer_search.cpp:11-21
  const int fy_lo = max(-R, M - cy), fy_hi = min(R, p.tgt.height - 1 - M - cy);
  const uint32_t sf = (uint32_t)p.poi_sf[k];
  const double svf = p.poi_sqrtvf[k];
  BestPartial b;
  b.c = -2.0;
  b.dx = b.dy = 0;
  b.count = 0;
  b.found = 0;
  if (fx_lo <= fx_hi && fy_lo <= fy_hi && svf > 0.0) {
    const int64_t* buf = p.sfg + (size_t)k * EW * EW;
    const double rsvf = 1.0 / svf;
    const float rsvf_f = (float)rsvf;
    // one pass over memory: count, and each lane's two best candidates by the
    // approximate quotient
    int cnt = 0;
    float a1 = -3.0f, a2 = -3.0f;
    int64_t num1 = 0;
    int x1 = 0, y1 = 0;
    // flattened (dy, dx) walk: lane l takes candidates l, l + 32, ... in row-major order
    const int fw = fx_hi - fx_lo + 1, total = fw * (fy_hi - fy_lo + 1);
    int ry = lane / fw, rx = lane - ry * fw;
    const int jump_y = 32 / fw, jump_x = 32 - jump_y * fw;
    // cross terms U at a time per lane: their loads are issued together
    constexpr int U = 4;
    int64_t pre[U];
    {
      int px = rx, py = ry;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pre[u] = lane + 32 * u < total ? buf[(fy_lo + py + R) * EW + (fx_lo + px + R)] : 0;
        px += jump_x;
        py += jump_y;
        if (px >= fw) {
          px -= fw;
          ++py;
        }
      }
    }
    int ahead_x = rx, ahead_y = ry;  // position of candidate idx + 32 U
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ahead_x += jump_x;
      ahead_y += jump_y;
      if (ahead_x >= fw) {
        ahead_x -= fw;
        ++ahead_y;
      }
    }
    for (int idx = lane; idx < total; idx += 32) {
      {
        const int dx = fx_lo + rx, dy = fy_lo + ry;
        const int64_t sfg_v = pre[0];
#pragma unroll
        for (int u = 0; u < U - 1; ++u) pre[u] = pre[u + 1];
        pre[U - 1] = idx + 32 * U < total ? buf[(fy_lo + ahead_y + R) * EW + (fx_lo + ahead_x + R)] : 0;
        ahead_x += jump_x;
        ahead_y += jump_y;
        if (ahead_x >= fw) {
          ahead_x -= fw;
          ++ahead_y;
        }
        int64_t num;
        float rsq;
        if (tc_candidate_f(pv, n, sf, sfg_v, cx - M + dx, cy - M + dy, num, rsq)) {
          ++cnt;
          const float av = approx_zncc(num, rsvf_f, rsq);
          if (av > a1) {  // a2: the lane's runner-up (only its value is needed)
            a2 = a1;
            a1 = av, num1 = num, x1 = dx, y1 = dy;
          } else if (av > a2) {
            a2 = av;
          }
        }
      }
      rx += jump_x;
      ry += jump_y;
      if (rx >= fw) {
        rx -= fw;
        ++ry;
      }
    }
    float amax = a1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    const float thr = amax - 0x1p-19f;  // twice the filter's error bound (< 2^-21.6), see approx_zncc
    if (!__any_sync(0xffffffffu, a2 >= thr)) {
      // every near-maximal candidate is some lane's best: exact quotients for those
      if (a1 >= thr) {
        const double z = i64_to_f64(num1) / (svf * tc_sq(p, cx - M + x1, cy - M + y1));  // exact (zncc_from_moments)
        b.found = 1;
        b.c = z;
        b.dx = x1;
        b.dy = y1;
      }
    } else {
      // near-ties beyond two per lane: second pass over the window
      for (int dy = fy_lo; dy <= fy_hi; ++dy)
        for (int dx = fx_lo + lane; dx <= fx_hi; dx += 32) {
          int64_t num;
          float rsq;
          if (tc_candidate_f(pv, n, sf, buf[(dy + R) * EW + (dx + R)], cx - M + dx, cy - M + dy, num, rsq)) {
            if (approx_zncc(num, rsvf_f, rsq) >= thr) {
              const double z = i64_to_f64(num) / (svf * tc_sq(p, cx - M + dx, cy - M + dy));
              if (!b.found || improves(z, dx, dy, b.c, b.dx, b.dy)) {
                b.found = 1;
                b.c = z;
                b.dx = dx;
                b.dy = dy;
              }
            }
          }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      BestPartial q;
      q.c = __shfl_xor_sync(0xffffffffu, b.c, o);
      q.dx = __shfl_xor_sync(0xffffffffu, b.dx, o);
      q.dy = __shfl_xor_sync(0xffffffffu, b.dy, o);
      q.count = 0;
      q.found = __shfl_xor_sync(0xffffffffu, b.found, o);
      merge_best(b, q);
    }
    b.count = cnt;
  }
  if (lane == 0) write_integer_record(p.rec[k], cx, cy, b, p.subpixel_none);
}

// ---- per POI: the full exact ZNCC surface over the +-R window (NaN = no result) ----
__global__ void __launch_bounds__(256) tc_surface_kernel(TcParams p) {
  // every candidate is written: position data read straight from global memory (L2)
  const int lane = threadIdx.x & 31;
  const int k = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (k >= (p.re - p.rb) * p.lat.nx) return;
  const int iy = p.rb + k / p.lat.nx, ix = k % p.lat.nx;
  PosView pv;
  pv.sq = p.SQ;
  pv.s1 = p.S1;
  pv.rsq = p.RSQ;
  pv.x0 = p.qx_min;
  pv.y0 = p.qy_min;
  pv.W = p.SW;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, R = p.R, EW = 2 * R + 1;
  const uint32_t n = (uint32_t)(p.side * p.side);
  const int fx_lo = max(-R, M - cx), fx_hi = min(R, p.tgt.width - 1 - M - cx);
  const int fy_lo = max(-R, M - cy), fy_hi = min(R, p.tgt.height - 1 - M - cy);
  const uint32_t sf = (uint32_t)p.poi_sf[k];
  const double svf = p.poi_sqrtvf[k];
  const int64_t* buf = p.sfg + (size_t)k * EW * EW;
  double* out = p.surface + (size_t)k * EW * EW;
  const double qnan = __longlong_as_double(0x7ff8000000000000ULL);
  for (int idx = lane; idx < EW * EW; idx += 32) {
    const int ry = idx / EW, dx = idx - ry * EW - R, dy = ry - R;
    double z = qnan;
    Cand c;
    if (svf > 0.0 && dx >= fx_lo && dx <= fx_hi && dy >= fy_lo && dy <= fy_hi &&
        tc_candidate_s(pv, n, sf, buf[idx], cx - M + dx, cy - M + dy, c))
      z = i64_to_f64(c.num) / (svf * c.sq);  // exact, as bfs.cu
    out[idx] = z;
  }
}

template <typename K>
cudaError_t set_smem(K kern, size_t bytes) {
  cudaError_t e = set_dyn_smem(kern, bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

}  // namespace

bool tc_plan(TcParams& p) {
  if (std::getenv("DICB200_BFS_LEGACY")) return false;  // A/B switch: CUDA-core kernel
  // DICB200_TC_DBG=32: per-CTA clock breakdown of the MMA issuer (tools)
  p.dbg = std::getenv("DICB200_TC_DBG") ? std::atoi(std::getenv("DICB200_TC_DBG")) : 0;
  if (p.R < 0 || p.M < 0) return false;
  p.side = 2 * p.M + 1;
  if (p.side > 129) return false;
  if ((size_t)p.ref.width * 12 + 16 > 200 * 1024) return false;  // tc_prep_kernel column sums
  if (stats_smem_bytes(p.side, 16, false) > 200 * 1024) return false;
  if (pos_smem_bytes(p, 1) > 200 * 1024) return false;
  const int side = p.side, W = p.tgt.width, H = p.tgt.height;
  const int rows = p.re - p.rb;
  if (rows <= 0 || p.lat.nx <= 0) return false;
  if ((size_t)rows * p.lat.nx < 1024) return false;  // tiny grids: the single-launch CUDA-core kernel wins
  p.qx_min = std::max(0, p.lat.cx(0) - p.M - p.R);
  p.qx_max = std::min(W - side, p.lat.cx(p.lat.nx - 1) - p.M + p.R);
  p.qy_min = std::max(0, p.lat.cy(p.rb) - p.M - p.R);
  p.qy_max = std::min(H - side, p.lat.cy(p.re - 1) - p.M + p.R);
  if (p.qx_min > p.qx_max || p.qy_min > p.qy_max) {
    p.SW = p.SH = p.ntx = p.nty = p.n_tiles = 0;
  } else {
    p.SW = p.qx_max - p.qx_min + 1;
    p.SH = p.qy_max - p.qy_min + 1;
    p.ntx = (p.SW + kTX - 1) / kTX;
    p.nty = (p.SH + kTY - 1) / kTY;
    p.n_tiles = p.ntx * p.nty;
  }
  p.RG = (side + 7) / 8;
  p.CG = (side + 3) / 4;
  p.NX = 4 * p.CG;
  p.HT = 16;
  int rwb = ((p.NX + 16 + 3) / 4) * 4 + 4;  // +1 word for the funnel shift reads
  if (((rwb / 4) & 1) == 0) rwb += 4;      // odd word pitch
  p.RWB = rwb;
  p.n_mma = p.RG * p.CG;
  // remainder rows (side = 8 (RG - 1) + rem_rows): a row-major last stage with
  // K = 32 columns per MMA when that needs fewer MMAs than CG (e.g. side 41: 2 vs 11)
  p.rem_rows = side - 8 * (p.RG - 1);
  p.n_h = (side + 31) / 32;
  p.NX2 = 32 * p.n_h;
  p.HT2 = 8 + p.rem_rows - 1;
  {
    int rwb2 = ((p.NX2 + 16 + 3) / 4) * 4 + 4;
    if (((rwb2 / 4) & 1) == 0) rwb2 += 4;
    p.RWB2 = rwb2;
  }
  p.rem = p.RG >= 2 && p.rem_rows * p.n_h < p.CG && !std::getenv("DICB200_TC_NOREM");
  const int s = p.lat.step;
  p.nix_max = std::min(p.lat.nx, (kTX - 1 + 2 * p.R) / s + 1);
  p.niy_max = std::min(rows, (kTY - 1 + 2 * p.R) / s + 1);
  p.npoi_max = p.nix_max * p.niy_max;
  if (p.npoi_max > kMaxTilePoi) return false;
  p.N_max = std::max(16, ((p.npoi_max * p.planes + 15) / 16) * 16);
  if (p.N_max > 256) return false;
  int cols = 32;
  while (cols < 2 * p.planes * p.N_max) cols *= 2;  // two accumulators
  if (cols > 512) return false;
  p.tmem_cols = cols;
  // shared memory: a ring of K stages (T | rows | B), one per producer group
  auto al = [](size_t v, size_t a) { return (v + a - 1) & ~(a - 1); };
  p.off_rows = al((size_t)p.planes * p.NX * 16 * 16, 128);
  p.off_B = al(p.off_rows + (size_t)p.planes * 16 * p.RWB, 128);
  p.stage_bytes = al(p.off_B + (size_t)p.CG * p.N_max * 32, 1024);
  if (p.rem && ((size_t)p.planes * p.HT2 * p.NX2 * 16 > p.off_rows ||
                (size_t)p.planes * p.HT2 * p.RWB2 > p.off_B - p.off_rows ||
                (size_t)p.rem_rows * p.n_h * p.N_max * 32 > p.stage_bytes - p.off_B))
    p.rem = 0;
  p.stages = kGroups;
  p.smem = (size_t)p.stages * p.stage_bytes;
  // 227 KB per CTA on sm_100a, less the kernel's 9 KB of static shared memory (barriers, tile lists):
  // the former 220 KB bound let a 220 KB ring through, which the launch rejected (found by the
  // randomised sweep: side 25, R 9, step 4, two planes)
  if (p.smem > (227 - 10) * 1024) return false;
  // cross-term buffer: one window per POI of the launch
  const size_t EW = 2 * (size_t)p.R + 1;
  if ((size_t)rows * p.lat.nx * EW * EW * 8 > ((size_t)3 << 30)) return false;
  p.grid = std::max(1, std::min(p.n_tiles, sm_count()));
  return true;
}

namespace {
cudaError_t grow(void*& ptr, size_t& cap, size_t bytes, cudaStream_t st) {
  if (cap >= bytes) return cudaSuccess;
  if (ptr) cudaFreeAsync(ptr, st);
  ptr = nullptr;
  cap = 0;
  cudaError_t e = cudaMallocAsync(&ptr, bytes, st);
  if (e == cudaSuccess) cap = bytes;
  return e;
}
}  // namespace

void tc_cache_free(TcRefCache& c, cudaStream_t st, bool async) {
  for (void* q : {c.tail, c.strips, c.psf, c.pvf, c.s1, c.s2, c.sfg, c.tiles, (void*)c.guard})
    if (q) async ? cudaFreeAsync(q, st) : cudaFree(q);
  c = TcRefCache{};
}

cudaError_t tc_launch(TcParams& p, cudaStream_t st, TcRefCache* cache, long ref_key) {
  const int rows = p.re - p.rb;
  const size_t npoi = (size_t)rows * p.lat.nx;
  cudaError_t e = cudaSuccess;
  void *bprep = nullptr, *psf = nullptr, *pvf = nullptr, *s1 = nullptr, *s2 = nullptr, *part = nullptr,
       *tiles = nullptr, *tailb = nullptr;
  const size_t tail_bytes = p.rem ? npoi * (size_t)p.rem_rows * p.n_h * p.planes * 32 : 0;
  auto cleanup = [&]() {
    for (void* q : {bprep, psf, pvf, s1, s2, part, tiles, tailb})
      if (q) cudaFreeAsync(q, st);
  };
  const size_t sbytes = (size_t)std::max(1, p.SW) * std::max(1, p.SH);
  p.strip_h = ((p.ref.height + 63) / 64) * 64;
  const size_t strip_bytes = (size_t)p.planes * 8 * p.ref.width * p.strip_h;
  // Block-sum or tensor-core search: decided per pair from the pair's pixel range
  // (p.maxv), so a reference frame cached for one kernel may be reused by the
  // other — the cache key includes the choice (only the tensor kernel needs the
  // strip images).
  BsGeom bsg{};
  const bool use_bs = bs_plan(p, bsg);
  // reference-side inputs: from the cache when this reference frame's were built already
  bool ref_ready = false;
  if (cache && ref_key >= 0) {
    ref_ready = cache->key == ref_key && cache->data == p.ref.data && cache->W == p.ref.width &&
                cache->H == p.ref.height && cache->M == p.M && cache->x0 == p.lat.x0 && cache->y0 == p.lat.y0 &&
                cache->step == p.lat.step && cache->nx == p.lat.nx && cache->rb == p.rb && cache->re == p.re &&
                cache->planes == p.planes && cache->use_bs == use_bs;
    if (!ref_ready) {
      cache->key = -1;
      e = grow(cache->strips, cache->strips_cap, strip_bytes, st);
      if (e == cudaSuccess) e = grow(cache->psf, cache->psf_cap, npoi * 8, st);
      if (e == cudaSuccess) e = grow(cache->pvf, cache->pvf_cap, npoi * 8, st);
      if (e == cudaSuccess) e = grow(cache->tail, cache->tail_cap, std::max<size_t>(16, tail_bytes), st);
      if (e != cudaSuccess) return e;
    }
    p.strips = (uint8_t*)cache->strips;
    p.poi_sf = (int64_t*)cache->psf;
    p.poi_sqrtvf = (double*)cache->pvf;
    p.tail = (uint8_t*)cache->tail;
  } else {
    e = cudaMallocAsync(&bprep, strip_bytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&psf, npoi * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&pvf, npoi * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&tailb, std::max<size_t>(16, tail_bytes), st);
    p.tail = (uint8_t*)tailb;
    p.strips = (uint8_t*)bprep;
    p.poi_sf = (int64_t*)psf;
    p.poi_sqrtvf = (double*)pvf;
  }
  const size_t EW = 2 * (size_t)p.R + 1;
  const size_t s1_bytes = sbytes * 4, s2_bytes = sbytes * 12;  // S1 (u32); SQ (double) + RSQ (float)
  // the fused block-sum search keeps its cross terms on chip: per-slice
  // results instead of the [poi][2R+1][2R+1] buffer
  const bool fused = use_bs && bsg.fuse;
  const size_t sfg_bytes = fused ? bs_slices_bytes(npoi, bsg) : npoi * EW * EW * sizeof(int64_t);
  const size_t tiles_bytes = (size_t)std::max(1, p.n_tiles) * 16;
  void *S1 = nullptr, *S2 = nullptr, *SFG = nullptr, *TILES = nullptr;
  if (cache) {
    if (e == cudaSuccess) e = grow(cache->s1, cache->s1_cap, s1_bytes, st);
    if (e == cudaSuccess) e = grow(cache->s2, cache->s2_cap, s2_bytes, st);
    if (e == cudaSuccess) e = grow(cache->sfg, cache->sfg_cap, sfg_bytes, st);
    if (e == cudaSuccess) e = grow(cache->tiles, cache->tiles_cap, tiles_bytes, st);
    S1 = cache->s1, S2 = cache->s2, SFG = cache->sfg, TILES = cache->tiles;
  } else {
    if (e == cudaSuccess) e = cudaMallocAsync(&s1, s1_bytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&s2, s2_bytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&part, sfg_bytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&tiles, tiles_bytes, st);
    S1 = s1, S2 = s2, SFG = part, TILES = tiles;
  }
  if (e != cudaSuccess) {
    cleanup();
    return e;
  }
  host_trace("tc mallocs");
  p.S1 = (uint32_t*)S1;
  p.SQ = (double*)S2;
  p.RSQ = (float*)((char*)S2 + sbytes * 8);
  p.sfg = fused ? nullptr : (int64_t*)SFG;
  p.slices = fused ? SFG : nullptr;
  p.tiles = TILES;
  const bool u8 = p.planes == 1;
  // (a) window sums of the target
  if (e == cudaSuccess && p.n_tiles > 0) {
    const bool q = stats_sq32(p);
    const int ty = stats_ty(p);
    const size_t sm = stats_smem_bytes(p.side, ty, q);
    dim3 grid((p.SW + kStatsBX - 1) / kStatsBX, (p.SH + ty - 1) / ty);
    auto go = [&](auto kern) {
      e = set_smem(kern, sm);
      if (e == cudaSuccess) kern<<<grid, 256, sm, st>>>(p, ty);
    };
    if (u8)
      q ? go(tc_stats_kernel<uint8_t, uint32_t>) : go(tc_stats_kernel<uint8_t, uint64_t>);
    else
      q ? go(tc_stats_kernel<uint16_t, uint32_t>) : go(tc_stats_kernel<uint16_t, uint64_t>);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  int failed_stage = e != cudaSuccess ? 1 : 0;  // first failing stage, named in the error trace below
  host_trace("tc stats");
  // (b) reference moments + strip images (skipped when cached; the block-sum
  //     kernel reads the reference directly and needs no strips)
  if (e == cudaSuccess && !ref_ready) {
    if (!use_bs) {
      dim3 sg((p.ref.width + 31) / 32, p.strip_h / 64);
      if (u8)
        tc_strips_kernel<uint8_t><<<sg, 256, 0, st>>>(p);
      else
        tc_strips_kernel<uint16_t><<<sg, 256, 0, st>>>(p);
      count_launch();
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      const size_t sm = (((size_t)p.ref.width * 4 + 15) & ~size_t(15)) + (size_t)p.ref.width * 8;
      if (u8) {
        e = set_smem(tc_prep_kernel<uint8_t>, sm);
        if (e == cudaSuccess) tc_prep_kernel<uint8_t><<<rows, 256, sm, st>>>(p);
      } else {
        e = set_smem(tc_prep_kernel<uint16_t>, sm);
        if (e == cudaSuccess) tc_prep_kernel<uint16_t><<<rows, 256, sm, st>>>(p);
      }
      count_launch();
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e == cudaSuccess && cache && ref_key >= 0) {
      cache->key = ref_key;
      cache->data = p.ref.data;
      cache->W = p.ref.width;
      cache->H = p.ref.height;
      cache->M = p.M;
      cache->x0 = p.lat.x0;
      cache->y0 = p.lat.y0;
      cache->step = p.lat.step;
      cache->nx = p.lat.nx;
      cache->rb = p.rb;
      cache->re = p.re;
      cache->planes = p.planes;
      cache->use_bs = use_bs;
    }
  }
  if (e != cudaSuccess && !failed_stage) failed_stage = 2;
  host_trace("tc prep");
  // (c) tensor-core search
  if (e == cudaSuccess && use_bs) {
    StageTimer tm(6, st);
    e = bs_launch(p, bsg, st);
    host_trace("bs");
  }
  if (e == cudaSuccess && p.n_tiles > 0 && !use_bs) {
    tc_tiles_kernel<<<(p.n_tiles + 255) / 256, 256, 0, st>>>(p);
    count_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && p.n_tiles > 0 && !use_bs) {
    long long* dbg_buf = nullptr;
    if (p.dbg & 32) {  // tools: MMA-thread clock breakdown
      cudaMalloc(&dbg_buf, (size_t)p.grid * 8 * sizeof(long long));
      cudaMemsetAsync(dbg_buf, 0, (size_t)p.grid * 8 * sizeof(long long), st);
      p.dbg_out = dbg_buf;
    }
    {
      StageTimer tm(4, st);
      if (u8) {
        e = set_smem(bfs_tc_kernel<1>, p.smem);
        if (e == cudaSuccess) bfs_tc_kernel<1><<<p.grid, kTcThreads, p.smem, st>>>(p);
      } else {
        e = set_smem(bfs_tc_kernel<2>, p.smem);
        if (e == cudaSuccess) bfs_tc_kernel<2><<<p.grid, kTcThreads, p.smem, st>>>(p);
      }
    }
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (dbg_buf) {
      std::vector<long long> h((size_t)p.grid * 8);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), dbg_buf, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      double a[4] = {0, 0, 0, 0};
      for (int b = 0; b < p.grid; ++b)
        for (int k = 0; k < 4; ++k) a[k] += (double)h[(size_t)b * 4 + k] / p.grid;
      fprintf(stderr, "[tc dbg] clk total %.0f  wait_full %.0f  wait_tmem %.0f  mma-loop %.0f  (tiles/cta %.1f)\n", a[0],
              a[1], a[2], a[3], (double)p.n_tiles / p.grid);
      cudaFree(dbg_buf);
      p.dbg_out = nullptr;
    }
  }
  if (e != cudaSuccess && !failed_stage) failed_stage = 3;
  // (d) per POI: exact ZNCC -> argmax record, or the full surface for the swarm walk
  if (e == cudaSuccess && fused) {
    StageTimer tm(5, st);
    e = bs_merge_launch(p, bsg, st);
  } else if (e == cudaSuccess) {
    int sp = 8;  // POIs per CTA strip (one warp each), sharing the staged position data
    while (sp > 1 && pos_smem_bytes(p, sp) > 96 * 1024) sp /= 2;
    const size_t sm = pos_smem_bytes(p, sp);
    dim3 grid((p.lat.nx + sp - 1) / sp, rows);
    StageTimer tm(5, st);
    if (p.surface) {
      tc_surface_kernel<<<(int)((npoi * 32 + 255) / 256), 256, 0, st>>>(p);
    } else {
      e = set_smem(tc_argmax_kernel, sm);
      if (e == cudaSuccess) tc_argmax_kernel<<<grid, 256, sm, st>>>(p, sp);
    }
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e != cudaSuccess && !failed_stage) failed_stage = 4;
  if (e != cudaSuccess)
    fprintf(stderr, "[dicb200] tc_launch: stage %d (1 window sums, 2 reference prep, 3 search, 4 argmax / surface) failed: %s "
            "(side %d R %d step %d planes %d SW %d SH %d tiles %d grid %d smem %zu)\n", failed_stage, cudaGetErrorString(e),
            p.side, p.R, p.lat.step, p.planes, p.SW, p.SH, p.n_tiles, p.grid, p.smem);
  cleanup();
  return e;
}

}  // namespace dicb200
