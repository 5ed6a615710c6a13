// K1 — brute-force ZNCC integer search (bfs_search, integer_search.cpp:52-79,
// with zncc, correlation.cpp:41-72, and subset_stats, correlation.cpp:9-39).
//
// One CTA = a tile of TS consecutive POIs of one grid row x one chunk of the
// candidate window. The target region the tile touches and the reference
// subsets are staged in shared memory once; every candidate's cross term
// Sfg is accumulated EXACTLY in integers:
//   u8  : __dp4a over packed bytes (4 MAC / instruction, IDP.4A pipe),
//         output-stationary over reference words with a register window of
//         byte-shifted target words (PRMT), J candidates per thread;
//   u16 : IMAD u32 per subset row (exact while (2M+1)*max^2 < 2^32, e.g. any
//         12-bit image), flushed to u64 per row; wider data uses exact fp64 DFMA
//         accumulation (exact below 2^53).
// Sg / Sgg per candidate come from column sums of the staged region (exact).
// ZNCC is finalised in fp64 from the exact moments (common.cuh), which makes
// every decision (argmax, tie-break, degenerate skip, evaluation count)
// identical to the reference's sequential double loop except for ties closer
// than ~1e-15 relative (SURVEY.md Appendix C.4 measured 0 mismatches).
#include <cstdio>
#include <type_traits>

#include "bfs.cuh"
#include "common.cuh"

namespace dicb200 {

namespace {

__device__ __forceinline__ int pmod4(int v) { return v & 3; }

template <typename Pix>
struct PixTraits;
template <>
struct PixTraits<uint8_t> {
  static constexpr bool kU8 = true;
};
template <>
struct PixTraits<uint16_t> {
  static constexpr bool kU8 = false;
};

struct TileGeom {
  int iy, ix0, ts, cy;
  int chunk, dy0, dyn, dx0, dxn;
  int base_y;  // global row of candidate dy'=0's top edge
  int X0;      // global column of region column 0
};

__device__ __forceinline__ int base_x_of(const BfsParams& p, int cx) {
  return p.whole ? 0 : cx - p.R - p.M;
}

__device__ __forceinline__ int align_of(const BfsParams& p, int cx, int dx0) {
  return p.u8 ? pmod4(base_x_of(p, cx) + dx0) : 0;
}

}  // namespace

// Shared memory carve-up (bytes), identical on host and device.
__host__ __device__ BfsSmem bfs_smem_layout(const BfsParams& p) {
  BfsSmem s;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = (off + 15) & ~size_t(15);
    off = o + bytes;
    return o;
  };
  const int elt = p.u8 ? 1 : 2;
  s.target = take((size_t)p.RH * p.region_pitch * elt);
  if (p.u8)
    s.ref = take((size_t)p.TS * (2 * p.M + 1) * p.QP * 4);
  else
    s.ref = take((size_t)(2 * p.M + 1) * p.ref_pitch * 2);
  s.v1 = take((size_t)p.DYC * p.RW * 4);
  s.v2 = take((size_t)p.DYC * p.RW * (p.f64 ? 8 : 4));  // u32 whenever (2M+1) max^2 < 2^32
  s.stats = take((size_t)p.TS * 16);
  s.items = take((size_t)p.items_max * sizeof(BestPartial));
  s.total = (off + 15) & ~size_t(15);
  return s;
}

// Remainder of a subset row after the J-unrolled blocks: R (< J) steps,
// straight-line (no per-step predicate), selected by a runtime switch.
template <int J, int R>
__device__ __forceinline__ void imad_tail(const uint16_t* frow, const uint16_t* grow, uint32_t (&acc)[J],
                                          uint32_t (&gw)[J]) {
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const uint32_t f = frow[k];
    gw[(k + J - 1) % J] = grow[k + J - 1];
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += f * gw[(k + j) % J];
  }
}

template <int J, int R = 1>
__device__ __forceinline__ void imad_tail_dispatch(int rem, const uint16_t* frow, const uint16_t* grow,
                                                   uint32_t (&acc)[J], uint32_t (&gw)[J]) {
  if constexpr (R < J) {
    if (rem == R) {
      imad_tail<J, R>(frow, grow, acc, gw);
      return;
    }
    imad_tail_dispatch<J, R + 1>(rem, frow, grow, acc, gw);
  }
}

template <typename Pix, int J, bool kF64>
__global__ void __launch_bounds__(256, 3) bfs_tile_kernel(BfsParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BfsSmem L = bfs_smem_layout(p);
  constexpr bool kU8 = PixTraits<Pix>::kU8;
  const int M = p.M, side = 2 * M + 1;
  const int64_t n = (int64_t)side * side;

  TileGeom g;
  g.iy = p.row_begin + blockIdx.y;
  const int tile = blockIdx.x / p.n_chunks;
  g.chunk = blockIdx.x % p.n_chunks;
  g.ix0 = tile * p.TS;
  g.ts = min(p.TS, p.lat.nx - g.ix0);
  g.cy = p.lat.cy(g.iy);
  const int dyc = g.chunk / p.n_dx_chunks, dxc = g.chunk % p.n_dx_chunks;
  g.dy0 = dyc * p.DYC;
  g.dyn = min(p.DYC, p.EY - g.dy0);
  g.dx0 = dxc * p.DXC;
  g.dxn = min(p.DXC, p.EX - g.dx0);
  g.base_y = (p.whole ? 0 : g.cy - p.R - p.M) + g.dy0;
  const int cx_first = p.lat.cx(g.ix0);
  g.X0 = base_x_of(p, cx_first) + g.dx0 - align_of(p, cx_first, g.dx0);

  Pix* T = reinterpret_cast<Pix*>(smem + L.target);
  const int RH = g.dyn + 2 * M;
  const int tid = threadIdx.x, nthr = blockDim.x;

  // ---- stage target region (zero outside the image: such pixels only feed
  // candidates outside the feasible window, which are discarded) ----
  {
    const Pix* src = reinterpret_cast<const Pix*>(p.tgt.data);
    const int total = RH * p.RW;
    for (int i = tid; i < total; i += nthr) {
      const int t = i / p.RW, x = i - t * p.RW;
      const int gy = g.base_y + t, gx = g.X0 + x;
      Pix v = 0;
      if (gy >= 0 && gy < p.tgt.height && gx >= 0 && gx < p.tgt.width) v = src[(size_t)gy * p.tgt.pitch + gx];
      T[t * p.region_pitch + x] = v;
    }
  }
  // ---- stage reference subsets ----
  if constexpr (kU8) {
    uint32_t* F = reinterpret_cast<uint32_t*>(smem + L.ref);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.ref.data);
    const int total = g.ts * side * p.QP;
    for (int i = tid; i < total; i += nthr) {
      const int q = i % p.QP, rs = i / p.QP, r = rs % side, s = rs / side;
      const int cx = p.lat.cx(g.ix0 + s);
      const uint8_t* row = src + (size_t)(g.cy - M + r) * p.ref.pitch + (cx - M);
      uint32_t w = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * q + e;
        if (c < side) w |= (uint32_t)row[c] << (8 * e);
      }
      F[i] = w;
    }
  } else {
    uint16_t* F = reinterpret_cast<uint16_t*>(smem + L.ref);
    const uint16_t* src = reinterpret_cast<const uint16_t*>(p.ref.data);
    const int fw = (g.ts - 1) * p.lat.step + side;
    const int total = side * p.ref_pitch;
    for (int i = tid; i < total; i += nthr) {
      const int r = i / p.ref_pitch, x = i - r * p.ref_pitch;
      uint16_t v = 0;
      if (x < fw) v = src[(size_t)(g.cy - M + r) * p.ref.pitch + (cx_first - M + x)];
      F[i] = v;
    }
  }
  __syncthreads();

  // ---- per-subset reference moments (warp per subset) ----
  {
    uint64_t* st = reinterpret_cast<uint64_t*>(smem + L.stats);
    const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
    for (int s = warp; s < g.ts; s += nwarps) {
      uint64_t sf = 0, sff = 0;
      for (int k = lane; k < n; k += 32) {
        const int r = k / side, c = k - r * side;
        uint32_t f;
        if constexpr (kU8) {
          const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + L.ref);
          f = (F[(s * side + r) * p.QP + (c >> 2)] >> (8 * (c & 3))) & 0xffu;
        } else {
          const uint16_t* F = reinterpret_cast<const uint16_t*>(smem + L.ref);
          f = F[r * p.ref_pitch + s * p.lat.step + c];
        }
        sf += f;
        sff += (uint64_t)f * f;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        sf += __shfl_xor_sync(0xffffffffu, sf, o);
        sff += __shfl_xor_sync(0xffffffffu, sff, o);
      }
      if (lane == 0) {
        const int64_t vf = n * (int64_t)sff - (int64_t)sf * (int64_t)sf;
        st[2 * s] = sf;
        reinterpret_cast<double*>(st)[2 * s + 1] = vf > 0 ? sqrt((double)vf) : 0.0;
      }
    }
  }
  // ---- column sums of the region: V1[t][x] = sum_r T[t+r][x], V2 of squares ----
  {
    using V2T = typename std::conditional<kF64, uint64_t, uint32_t>::type;
    uint32_t* V1 = reinterpret_cast<uint32_t*>(smem + L.v1);
    V2T* V2 = reinterpret_cast<V2T*>(smem + L.v2);
    for (int x = tid; x < p.RW; x += nthr) {
      uint32_t s1 = 0;
      uint64_t s2 = 0;
      for (int r = 0; r < side; ++r) {
        const uint32_t v = T[r * p.region_pitch + x];
        s1 += v;
        s2 += (uint64_t)v * v;
      }
      V1[x] = s1;
      V2[x] = (V2T)s2;
      for (int t = 1; t < g.dyn; ++t) {
        const uint32_t a = T[(t + side - 1) * p.region_pitch + x], b = T[(t - 1) * p.region_pitch + x];
        s1 += a - b;
        s2 += (uint64_t)a * a - (uint64_t)b * b;
        V1[t * p.RW + x] = s1;
        V2[t * p.RW + x] = (V2T)s2;
      }
    }
  }
  __syncthreads();

  // ---- main loop: one item = (subset s, candidate row t, block b of J) ----
  BestPartial* items = reinterpret_cast<BestPartial*>(smem + L.items);
  const int n_items = g.ts * g.dyn * p.B;
  const uint64_t* st = reinterpret_cast<const uint64_t*>(smem + L.stats);
  const uint32_t* V1 = reinterpret_cast<const uint32_t*>(smem + L.v1);
  using V2R = typename std::conditional<kF64, uint64_t, uint32_t>::type;
  const V2R* V2 = reinterpret_cast<const V2R*>(smem + L.v2);
  for (int item = tid; item < n_items; item += nthr) {
    const int b = item % p.B, st_ = item / p.B, t = st_ % g.dyn, s = st_ / g.dyn;
    const int cx = p.lat.cx(g.ix0 + s);
    const int al = align_of(p, cx, g.dx0);
    const int dxs = g.dx0 - al + b * J;                            // dx' of slot 0
    const int cs = base_x_of(p, cx) + dxs - g.X0;                  // region column of slot 0
    uint64_t sfg[J];
#pragma unroll
    for (int j = 0; j < J; ++j) sfg[j] = 0;

    if constexpr (kU8) {
      constexpr int U = J / 4;
      const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + L.ref) + (size_t)s * side * p.QP;
      const uint32_t* Tw = reinterpret_cast<const uint32_t*>(T);
      const int pw = p.region_pitch >> 2;
      uint32_t acc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = 0;
      for (int r = 0; r < side; ++r) {
        const uint32_t* frow = F + r * p.QP;
        const uint32_t* grow = Tw + (t + r) * pw + (cs >> 2);
        uint32_t Ue[4][U];
        uint32_t aprev = grow[0];
#pragma unroll
        for (int i = 0; i < U - 1; ++i) {
          const uint32_t anext = grow[i + 1];
          Ue[0][i] = aprev;
          Ue[1][i] = __byte_perm(aprev, anext, 0x4321);
          Ue[2][i] = __byte_perm(aprev, anext, 0x5432);
          Ue[3][i] = __byte_perm(aprev, anext, 0x6543);
          aprev = anext;
        }
        for (int q0 = 0; q0 < p.QP; q0 += U) {
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int q = q0 + k;
            const uint32_t fw = frow[q];
            const uint32_t anew = grow[q + U];
            constexpr int dummy = 0;
            (void)dummy;
            const int sl = (k + U - 1) % U;
            Ue[0][sl] = aprev;
            Ue[1][sl] = __byte_perm(aprev, anew, 0x4321);
            Ue[2][sl] = __byte_perm(aprev, anew, 0x5432);
            Ue[3][sl] = __byte_perm(aprev, anew, 0x6543);
            aprev = anew;
#pragma unroll
            for (int a = 0; a < U; ++a) {
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[4 * a + e] = __dp4a(fw, Ue[e][(k + a) % U], acc[4 * a + e]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) sfg[j] = acc[j];
    } else {
      const uint16_t* F = reinterpret_cast<const uint16_t*>(smem + L.ref);
      const uint16_t* T16 = reinterpret_cast<const uint16_t*>(T);
      // Exact fp64 accumulation on the DFMA pipe when the data is too wide for
      // u32 row sums (kF64). (Splitting 12-bit work between the IMAD and DFMA
      // pipes — per warp or per thread — was measured slower: DESIGN.md §7.)
      if constexpr (kF64) {
        double accd[J];
#pragma unroll
        for (int j = 0; j < J; ++j) accd[j] = 0.0;
        const int full = (side / J) * J;
        for (int r = 0; r < side; ++r) {
          const uint16_t* frow = F + r * p.ref_pitch + s * p.lat.step;
          const uint16_t* grow = T16 + (t + r) * p.region_pitch + cs;
          double gw[J];
#pragma unroll
          for (int i = 0; i < J - 1; ++i) gw[i] = (double)grow[i];
          for (int c0 = 0; c0 < full; c0 += J) {
#pragma unroll
            for (int k = 0; k < J; ++k) {
              const double f = (double)frow[c0 + k];
              gw[(k + J - 1) % J] = (double)grow[c0 + k + J - 1];
#pragma unroll
              for (int j = 0; j < J; ++j) accd[j] = fma(f, gw[(k + j) % J], accd[j]);
            }
          }
          if (full < side) {
#pragma unroll
            for (int k = 0; k < J; ++k) {
              if (full + k < side) {
                const double f = (double)frow[full + k];
                gw[(k + J - 1) % J] = (double)grow[full + k + J - 1];
#pragma unroll
                for (int j = 0; j < J; ++j) accd[j] = fma(f, gw[(k + j) % J], accd[j]);
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < J; ++j) sfg[j] = (uint64_t)accd[j];
        } else {
        const int full = (side / J) * J;  // mask-free blocks, then one uniform tail block
        for (int r = 0; r < side; ++r) {
          const uint16_t* frow = F + r * p.ref_pitch + s * p.lat.step;
          const uint16_t* grow = T16 + (t + r) * p.region_pitch + cs;
          uint32_t acc[J];
          uint32_t gw[J];
#pragma unroll
          for (int j = 0; j < J; ++j) acc[j] = 0;
#pragma unroll
          for (int i = 0; i < J - 1; ++i) gw[i] = grow[i];
          for (int c0 = 0; c0 < full; c0 += J) {
#pragma unroll
            for (int k = 0; k < J; ++k) {
              const uint32_t f = frow[c0 + k];
              gw[(k + J - 1) % J] = grow[c0 + k + J - 1];
#pragma unroll
              for (int j = 0; j < J; ++j) acc[j] += f * gw[(k + j) % J];
            }
          }
          if (full < side) imad_tail_dispatch<J>(side - full, frow + full, grow + full, acc, gw);
#pragma unroll
          for (int j = 0; j < J; ++j) sfg[j] += acc[j];
        }
      }
    }

    // ---- epilogue: moments -> ZNCC -> item argmax ----
    const int64_t sf = (int64_t)st[2 * s];
    const double sqrt_vf = reinterpret_cast<const double*>(st)[2 * s + 1];
    const int dy = (p.whole ? p.M - g.cy : -p.R) + g.dy0 + t;
    const int dx_lo_nom = p.whole ? p.M - cx : -p.R;
    const int fx_lo = max(-p.R, p.M - cx), fx_hi = min(p.R, p.tgt.width - 1 - p.M - cx);
    const int fy_lo = max(-p.R, p.M - g.cy), fy_hi = min(p.R, p.tgt.height - 1 - p.M - g.cy);
    const bool row_ok = p.whole || (dy >= fy_lo && dy <= fy_hi);
    BestPartial best;
    best.c = -2.0;
    best.dx = 0;
    best.dy = 0;
    best.count = 0;
    best.found = 0;
    const uint32_t* v1 = V1 + t * p.RW + cs;
    const V2R* v2 = V2 + t * p.RW + cs;
    uint64_t s1 = 0, s2 = 0;
    for (int c = 0; c < side; ++c) {
      s1 += v1[c];
      s2 += v2[c];
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (j > 0) {
        s1 += (uint64_t)v1[j + side - 1] - v1[j - 1];
        s2 += (uint64_t)v2[j + side - 1] - (uint64_t)v2[j - 1];
      }
      const int dxp = dxs + j;
      const int dx = dx_lo_nom + dxp;
      const bool in_chunk = dxp >= g.dx0 && dxp < g.dx0 + g.dxn;
      const bool ok = in_chunk && row_ok && (p.whole || (dx >= fx_lo && dx <= fx_hi));
      const int64_t vg = n * (int64_t)s2 - (int64_t)s1 * (int64_t)s1;
      const bool valid = ok && sqrt_vf > 0.0 && vg > 0;  // constant target window: skipped, not counted
      const double c = valid ? zncc_from_moments(n, (int64_t)sfg[j], sf, (int64_t)s1, (int64_t)s2, sqrt_vf)
                             : __longlong_as_double(0x7ff8000000000000ULL);
      if (p.surface && in_chunk) {
        // full correlation surface for the swarm walk (K2): NaN = no result
        const size_t k = (size_t)(g.iy - p.row_begin) * p.lat.nx + (g.ix0 + s);
        p.surface[k * p.EX * p.EY + (size_t)(g.dy0 + t) * p.EX + dxp] = c;
      }
      if (!valid) continue;
      best.count++;
      if (!best.found || improves(c, dx, dy, best.c, best.dx, best.dy)) {
        best.found = 1;
        best.c = c;
        best.dx = dx;
        best.dy = dy;
      }
    }
    items[item] = best;
  }
  __syncthreads();

  // ---- per-subset reduction over its items, then record / partial ----
  for (int s = tid; s < g.ts; s += nthr) {
    BestPartial acc = items[s * g.dyn * p.B];
    for (int i = 1; i < g.dyn * p.B; ++i) merge_best(acc, items[s * g.dyn * p.B + i]);
    const int ix = g.ix0 + s;
    const size_t k = (size_t)(g.iy - p.row_begin) * p.lat.nx + ix;
    if (p.n_chunks == 1) {
      write_integer_record(p.rec[k], p.lat.cx(ix), g.cy, acc, p.subpixel_none);
    } else {
      p.partial[k * p.n_chunks + g.chunk] = acc;
    }
  }
}

__global__ void bfs_reduce_kernel(BfsParams p, int n_subsets) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_subsets) return;
  const BestPartial* src = p.partial + (size_t)k * p.n_chunks;
  BestPartial acc = src[0];
  for (int c = 1; c < p.n_chunks; ++c) merge_best(acc, src[c]);
  const int iy = p.row_begin + k / p.lat.nx, ix = k % p.lat.nx;
  write_integer_record(p.rec[k], p.lat.cx(ix), p.lat.cy(iy), acc, p.subpixel_none);
}

// ------------------------------------------------------------------ host

namespace {

template <typename Pix, int J, bool kF64>
cudaError_t launch_t(const BfsParams& p, dim3 grid, int threads, size_t smem, cudaStream_t st) {
  auto kern = bfs_tile_kernel<Pix, J, kF64>;
  cudaError_t e = set_dyn_smem(kern, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  kern<<<grid, threads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

const int kJu8[] = {4, 8, 12, 16};
const int kJu16[] = {4, 6, 8, 11, 12, 13};

}  // namespace

bool bfs_plan(BfsParams& p, size_t smem_limit) {
  const int side = 2 * p.M + 1;
  if (p.whole) {
    p.EX = p.tgt.width - 2 * p.M;
    p.EY = p.tgt.height - 2 * p.M;
  } else {
    p.EX = p.EY = 2 * p.R + 1;
  }
  if (p.EX < 1 || p.EY < 1) return false;
  p.DXC = p.EX <= 64 ? p.EX : 64;
  p.DYC = p.EY <= 64 ? p.EY : 16;
  p.n_dx_chunks = (p.EX + p.DXC - 1) / p.DXC;
  p.n_dy_chunks = (p.EY + p.DYC - 1) / p.DYC;
  p.n_chunks = p.n_dx_chunks * p.n_dy_chunks;
  // candidates per block J and blocks B: minimise slots B*J covering the chunk
  const int need = p.DXC + (p.u8 ? 3 : 0);
  int bestJ = 0, bestB = 0, bestSlots = 1 << 30;
  const int* Js = p.u8 ? kJu8 : kJu16;
  const int nJ = p.u8 ? (int)(sizeof(kJu8) / sizeof(int)) : (int)(sizeof(kJu16) / sizeof(int));
  // cost ~ candidate slots + per-block overhead (u8: f/word loads + 3 PRMT per
  // step amortised over J; u16: 2 loads per step)
  const int ovh = p.u8 ? 5 : 2;
  for (int i = 0; i < nJ; ++i) {
    const int J = Js[i];
    const int B = (need + J - 1) / J;
    const int cost = B * J + ovh * B;
    if (cost < bestSlots || (cost == bestSlots && B < bestB)) {
      bestSlots = cost;
      bestJ = J;
      bestB = B;
    }
  }
  p.J = bestJ;
  p.B = bestB;
  const int Q = (side + 3) / 4;
  const int U = p.u8 ? p.J / 4 : p.J;
  p.QP = ((Q + U - 1) / U) * U;
  p.CP = ((side + p.J - 1) / p.J) * p.J;
  // subsets per tile: aim for <= 512 items and fit shared memory
  int TS = p.whole ? 1 : max(1, 256 / (p.DYC * p.B));
  TS = min(TS, p.lat.nx);
  for (;; --TS) {
    p.TS = TS;
    const int span = (TS - 1) * p.lat.step + p.B * p.J;
    int rw = p.u8 ? span + 4 * p.QP + 12 : span + p.CP + p.J + 2;
    rw = (rw + 3) & ~3;
    p.RW = rw;
    int pitch = rw;
    if (p.u8 && ((pitch / 4) % 2 == 0)) pitch += 4;  // odd word pitch: spread banks
    if (!p.u8 && ((pitch / 2) % 2 == 0)) pitch += 2;
    p.region_pitch = pitch;
    p.RH = p.DYC + 2 * p.M;
    p.ref_pitch = (TS - 1) * p.lat.step + side + p.J + 2;
    p.items_max = TS * p.DYC * p.B;
    const BfsSmem s = bfs_smem_layout(p);
    if (s.total <= smem_limit) break;
    if (TS == 1) return false;
  }
  p.tiles_x = (p.lat.nx + p.TS - 1) / p.TS;
  return true;
}

cudaError_t bfs_launch(BfsParams& p, int rows, cudaStream_t st) {
  const BfsSmem s = bfs_smem_layout(p);
  const int threads = min(256, ((p.items_max + 31) / 32) * 32);
  dim3 grid(p.tiles_x * p.n_chunks, rows);
  cudaError_t e = cudaErrorInvalidValue;
#define DICB200_BFS_CASE(PIX, JJ, F64) \
  if (p.J == JJ) e = launch_t<PIX, JJ, F64>(p, grid, threads, s.total, st);
  if (p.u8) {
    DICB200_BFS_CASE(uint8_t, 4, false)
    DICB200_BFS_CASE(uint8_t, 8, false)
    DICB200_BFS_CASE(uint8_t, 12, false)
    DICB200_BFS_CASE(uint8_t, 16, false)
  } else if (!p.f64) {
    DICB200_BFS_CASE(uint16_t, 4, false)
    DICB200_BFS_CASE(uint16_t, 6, false)
    DICB200_BFS_CASE(uint16_t, 8, false)
    DICB200_BFS_CASE(uint16_t, 11, false)
    DICB200_BFS_CASE(uint16_t, 12, false)
    DICB200_BFS_CASE(uint16_t, 13, false)
  } else {
    DICB200_BFS_CASE(uint16_t, 4, true)
    DICB200_BFS_CASE(uint16_t, 6, true)
    DICB200_BFS_CASE(uint16_t, 8, true)
    DICB200_BFS_CASE(uint16_t, 11, true)
    DICB200_BFS_CASE(uint16_t, 12, true)
    DICB200_BFS_CASE(uint16_t, 13, true)
  }
#undef DICB200_BFS_CASE
  if (e != cudaSuccess) return e;
  if (p.n_chunks > 1) {
    const int n = rows * p.lat.nx;
    bfs_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n);
    count_launch();
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace dicb200
