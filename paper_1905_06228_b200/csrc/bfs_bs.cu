// K1-BS: the window-mode cross terms Sfg(P, d) of every POI P and displacement
// d in [-R, R]^2 from SHARED block sums (CUDA cores, exact u32/u64 integers).
//
// The POIs sit on a regular lattice of spacing s (grid_subsets, image.cpp:140-158)
// and their subsets (side L = 2M+1) overlap whenever s < L: neighbouring POIs
// correlate largely the same reference pixels against the same target pixels.
// Write L = q s + r (0 <= r < s) and cut the reference into s x s blocks aligned
// with the lattice: the box of POI (i, j) is exactly
//     q x q full blocks (i + a, j + b),              a, b < q
//   + the first r columns of blocks (i + q, j + b),  b < q
//   + the first r rows    of blocks (i + a, j + q),  a < q
//   + the r x r corner    of block  (i + q, j + q),
// so, per displacement d, each block's four partial sums
//   F = sum_block f g_d,  C = first r columns,  W = first r rows,  K = corner
// are computed ONCE and shared by the (up to) (q+1)^2 POIs whose boxes contain
// them. For BASELINE c5 (L = 41, s = 10) that is 16.8x fewer multiply-adds than
// correlating every subset on its own (the tensor-core kernel's formulation).
//
// Integer path, bit-exact: F < s^2 maxv^2 < 2^32 (checked by bs_plan), the box
// sums are u64. The results land in the same per-POI cross-term buffer as the
// tensor-core kernel's (TcParams::sfg), so the exact ZNCC / argmax / surface
// kernels downstream are shared (bfs_tc.cu).
//
// CTA = PX x PY POIs (all of them, or a slice of the dy range). Both image
// regions are staged once in shared memory; then per dy:
//   phase A: one thread per (block, dx chunk) walks the block's s rows, holding
//            F, C, W, K for DXC displacements in registers (s * DXC IMADs/row);
//   phase B: one thread per (POI, dx) adds the (q+1)^2 block partials (u64)
//            and stores Sfg.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <cstdio>
#include <vector>

#include "bfs.cuh"

namespace dicb200 {

namespace {

// 8-byte global -> shared async copy; bytes past src_bytes (0..8) are zero-filled.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}

// ---- fused exact argmax (FUSE): the cross terms never leave the SM ----
// Phase B maps one warp (or a 16-lane half for 2R+1 <= 16) to a POI column,
// lanes = dx. For every Sfg it forms the candidate exactly as tc_argmax_kernel
// does: the fp32 filter quotient num * (1/sqrt(vf)) * (1/sqrt(vg)) (absolute
// error < 2^-21.6), a running per-POI maximum, and the EXACT IEEE quotient
// num / (sqrt(vf) sqrt(vg)) only for candidates within 2^-19 of the running
// maximum at their row — a superset of the candidates within 2^-19 of the
// final maximum, which contains every possible winner. Each POI keeps its
// exact best in improves() order (integer_search.cpp:43-48) and its count of
// non-degenerate candidates in shared memory; a CTA covers one slice of the dy
// range, and bs_merge_kernel combines the slices into the record.
__device__ __forceinline__ uint32_t fkey(float a) {  // monotonic float -> u32 (0 = none)
  const uint32_t b = __float_as_uint(a);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ double bs_i64_to_f64(int64_t x) {  // exact for |x| < 2^51 without the XU unit
  if (x >= -(1ll << 51) && x < (1ll << 51))
    return __longlong_as_double(0x4338000000000000ll + x) - 6755399441055744.0;
  return (double)x;
}

constexpr int kBsMaxPY = 8;

// One dy slice's result for one POI (fused block-sum search).
struct BsSlice {
  long long num;  // exact numerator of the slice's best filter value
  float a1, a2;   // best / runner-up filter values (-3 = none)
  int cnt;        // non-degenerate candidates
  short dx, dy;
};  // POI rows per CTA tile (bs_plan starts at 8 and only shrinks)

struct BsPoiState {
  long long num;  // exact numerator n Sfg - Sf Sg of the slice's best filter value
  float a1, a2;   // best and runner-up filter values of the slice (-3 = none)
  int cnt;        // non-degenerate candidates of the slice
  short dx, dy;   // the best candidate
  float rsvf;     // POI constants: 1 / sqrt(vf), Sf (staged once per CTA)
  uint32_t sf;
};

// Stage the CTA's reference blocks and the target rows of its dy slice as u16
// (0 outside the images). u16 images: 8-byte cp.async from 4-pixel-aligned
// global columns (zero-filled past the borders); the staged rows then start
// `sh` pixels before the region. Phase A reads g.nchunk * dxc columns past
// each block (dx past R: zero).
template <typename Pix, int NT>
__device__ __forceinline__ void bs_stage(const TcParams& p, const BsGeom& g, uint16_t* Rf, uint16_t* Tg, int RX0,
                                         int RY0, int TX0, int TY0, int dy_lo, int dy_hi, int dxc, int& shR,
                                         int& shT) {
  const int R = p.R, RP = g.RWp, TP = g.TWp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (sizeof(Pix) == 2 && g.async_ok) {
    shR = RX0 & 3;
    shT = TX0 & 3;
    const int XR = RX0 - shR, XT = TX0 - shT;
    const uint16_t* ref = static_cast<const uint16_t*>(p.ref.data);
    const int cr = (shR + g.nbx * g.S + 3) / 4;  // 4-pixel chunks per staged row
    for (int i = threadIdx.x; i < g.RHp * cr; i += NT) {
      const int y = i / cr, c = i - y * cr, gy = RY0 + y, gx = XR + 4 * c;
      const int valid = (gy >= 0 && gy < p.ref.height && gx >= 0) ? max(0, min(4, p.ref.width - gx)) : 0;
      const uint16_t* src = valid ? ref + (size_t)gy * p.ref.pitch + gx : ref;
      cp_async8(Rf + y * RP + 4 * c, src, 2 * valid);
    }
    const uint16_t* tgt = static_cast<const uint16_t*>(p.tgt.data);
    const int ct = (shT + g.nbx * g.S + g.nchunk * dxc + 3) / 4;
    const int y_lo = dy_lo + R, nrow = dy_hi - dy_lo + g.RHp;
    for (int i = threadIdx.x; i < nrow * ct; i += NT) {
      const int yy = i / ct, c = i - yy * ct, y = y_lo + yy, gy = TY0 + y, gx = XT + 4 * c;
      const int valid = (gy >= 0 && gy < p.tgt.height && gx >= 0) ? max(0, min(4, p.tgt.width - gx)) : 0;
      const uint16_t* src = valid ? tgt + (size_t)gy * p.tgt.pitch + gx : tgt;
      cp_async8(Tg + y * TP + 4 * c, src, 2 * valid);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {
    const Pix* ref = static_cast<const Pix*>(p.ref.data);
    const int w = g.nbx * g.S;
    for (int y = warp; y < g.RHp; y += NT / 32) {
      const int gy = RY0 + y;
      const bool rowok = gy >= 0 && gy < p.ref.height;
      const Pix* src = ref + (size_t)(rowok ? gy : 0) * p.ref.pitch;
      for (int x = lane; x < w; x += 32) {
        const int gx = RX0 + x;
        Rf[y * RP + x] = (rowok && gx >= 0 && gx < p.ref.width) ? (uint16_t)src[gx] : (uint16_t)0;
      }
    }
    const Pix* tgt = static_cast<const Pix*>(p.tgt.data);
    const int tw = w + g.nchunk * dxc;  // columns read by phase A (dx past R: zero)
    for (int y = dy_lo + R + warp; y < dy_hi + R + g.RHp; y += NT / 32) {
      const int gy = TY0 + y;
      const bool rowok = gy >= 0 && gy < p.tgt.height;
      const Pix* src = tgt + (size_t)(rowok ? gy : 0) * p.tgt.pitch;
      for (int x = lane; x < tw; x += 32) {
        const int gx = TX0 + x;
        Tg[y * TP + x] = (rowok && x < w + 2 * R && gx >= 0 && gx < p.tgt.width) ? (uint16_t)src[gx] : (uint16_t)0;
      }
    }
  }
}

template <int S, int RR, int Q, int DXC, int NT, int MINB, typename Pix, bool FUSE = false>
__global__ void __launch_bounds__(NT, MINB) bs_kernel(TcParams p, BsGeom g) {
  extern __shared__ __align__(16) unsigned char bs_smem[];
  // both images staged as u16 whatever the pixel type (u8 operands made the
  // compiler keep packed bytes live and spill)
  uint16_t* Rf = reinterpret_cast<uint16_t*>(bs_smem);              // [RHp][RP]
  uint16_t* Tg = reinterpret_cast<uint16_t*>(bs_smem + g.off_tgt);  // [THp][TP]
  uint32_t* blk = reinterpret_cast<uint32_t*>(bs_smem + g.off_blk);  // [nblk][4][EW]
  const int M = p.M, R = p.R, EW = g.EW, RP = g.RWp, TP = g.TWp;
  const int ix0 = blockIdx.x * g.PX, iy0 = p.rb + blockIdx.y * g.PY;
  const int dy_lo = -R + (int)blockIdx.z * g.dy_per, dy_hi = min(R, dy_lo + g.dy_per - 1);
  const int RX0 = p.lat.cx(ix0) - M, RY0 = p.lat.cy(iy0) - M;  // block (0, 0) origin
  const int TX0 = RX0 - R, TY0 = RY0 - R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- stage the reference blocks and the target rows of this dy slice (0 outside)
  int shR = 0, shT = 0;
  bs_stage<Pix, NT>(p, g, Rf, Tg, RX0, RY0, TX0, TY0, dy_lo, dy_hi, DXC, shR, shT);
  __syncthreads();
  const int nx_here = min(g.PX, p.lat.nx - ix0), ny_here = min(g.PY, p.re - iy0);
  BsPoiState* st = reinterpret_cast<BsPoiState*>(bs_smem + g.off_state);  // FUSE: [PY][PX]
  if (FUSE) {
    for (int i = threadIdx.x; i < g.PX * g.PY; i += NT) {
      const int pi = i % g.PX, pj = i / g.PX;
      st[i].num = 0;
      st[i].a1 = st[i].a2 = -3.0f;
      st[i].cnt = 0;
      st[i].dx = st[i].dy = 0;
      st[i].rsvf = 0.0f;
      st[i].sf = 0;
      if (pi < nx_here && pj < ny_here) {
        const size_t k = (size_t)(iy0 + pj - p.rb) * p.lat.nx + (ix0 + pi);
        const double svf = p.poi_sqrtvf[k];
        st[i].rsvf = svf > 0.0 ? (float)(1.0 / svf) : 0.0f;  // 0: degenerate reference subset, no candidates
        st[i].sf = (uint32_t)p.poi_sf[k];
      }
    }
  }
  const int nbx = g.nbx;  // block-record row stride
  const int nbx_here = nx_here + Q - (RR == 0 ? 1 : 0), nby = ny_here + Q - (RR == 0 ? 1 : 0);  // blocks needed
  const int BS = 4 * EW + 1;  // words per block record (odd: conflict-free stores across blocks)
  const size_t ew2 = (size_t)EW * EW;
  for (int dy = dy_lo; dy <= dy_hi; ++dy) {
    // ---- phase A: block partials, DXC displacements per thread
    for (int task = threadIdx.x; task < nbx_here * nby * g.nchunk; task += NT) {
      const int c = task / (nbx_here * nby), bb = task - c * (nbx_here * nby);
      const int by = bb / nbx_here, bx = bb - by * nbx_here, b = by * nbx + bx;
      const int dx0 = c * DXC;  // chunk start, as an index dx + R
      const uint16_t* fr = Rf + (by * S) * RP + shR + bx * S;
      const uint16_t* gr = Tg + (by * S + dy + R) * TP + shT + bx * S + dx0;
      uint32_t* o = blk + b * BS + dx0;
      const int nd = min(DXC, EW - dx0);
      uint32_t F[DXC], Cc[DXC], Wr[DXC], Kc[DXC];
#pragma unroll
      for (int j = 0; j < DXC; ++j) F[j] = Cc[j] = Wr[j] = Kc[j] = 0u;
#pragma unroll
      for (int yy = 0; yy < S; ++yy) {
        uint32_t f[S], gg[S + DXC - 1];
#pragma unroll
        for (int k = 0; k < S; ++k) f[k] = fr[yy * RP + k];
#pragma unroll
        for (int k = 0; k < S + DXC - 1; ++k) gg[k] = gr[yy * TP + k];
        // k outer, j inner: DXC independent multiply-add chains per pixel column
        uint32_t part[DXC], full[DXC];
#pragma unroll
        for (int j = 0; j < DXC; ++j) part[j] = RR > 0 ? f[0] * gg[j] : 0u;
#pragma unroll
        for (int k = 1; k < RR; ++k)
#pragma unroll
          for (int j = 0; j < DXC; ++j) part[j] += f[k] * gg[k + j];
#pragma unroll
        for (int j = 0; j < DXC; ++j) full[j] = part[j];
#pragma unroll
        for (int k = RR; k < S; ++k)
#pragma unroll
          for (int j = 0; j < DXC; ++j) full[j] += f[k] * gg[k + j];
#pragma unroll
        for (int j = 0; j < DXC; ++j) {
          F[j] += full[j];
          if (RR > 0) {
            Cc[j] += part[j];
            if (yy < RR) {
              Wr[j] += full[j];
              Kc[j] += part[j];
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < DXC; ++j)
        if (j < nd) {
          o[j] = F[j];
          if (RR > 0) {
            o[EW + j] = Cc[j];
            o[2 * EW + j] = Wr[j];
            o[3 * EW + j] = Kc[j];
          }
        }
    }
    __syncthreads();
    if (FUSE) {
      // ---- phase B + exact argmax: a warp segment per POI column, lanes = dx ----
      // The candidates' window data (Sg, ~1/sqrt(vg)) of all the column's POI
      // rows are loaded up front (independent loads, one latency), the block-row
      // walk is unrolled so they stay in registers.
      constexpr int PYM = kBsMaxPY;
      const int seg = EW <= 16 ? 16 : 32, per_warp = 32 / seg;
      const int sub = lane / seg, dxi = lane - sub * seg;
      const unsigned segmask = seg == 32 ? 0xffffffffu : (0xffffu << (16 * sub));
      const uint32_t n = (uint32_t)(p.side * p.side);
      const int dy_ = dy;
      for (int col0 = warp * per_warp; col0 < nx_here; col0 += (NT / 32) * per_warp) {
        const int pi = col0 + sub;
        const bool act = dxi < EW && pi < nx_here;
        const int pic = act ? pi : 0;
        const uint32_t* col = blk + pic * BS + (act ? dxi : 0);
        const int cxp = p.lat.cx(ix0 + pic);
        const int dx = dxi - R;
        const bool xin = act && dx >= max(-R, M - cxp) && dx <= min(R, p.tgt.width - 1 - M - cxp);
        float rsq[PYM];
        uint32_t s1[PYM];
#pragma unroll
        for (int j = 0; j < PYM; ++j) {
          rsq[j] = 0.0f;
          s1[j] = 0;
          if (j < ny_here) {
            const int cyp = p.lat.cy(iy0 + j);
            if (xin && st[j * g.PX + pic].rsvf > 0.0f && dy_ >= max(-R, M - cyp) &&
                dy_ <= min(R, p.tgt.height - 1 - M - cyp)) {
              const size_t o = (size_t)(cyp - M + dy_ - p.qy_min) * p.SW + (cxp - M + dx - p.qx_min);
              rsq[j] = p.RSQ[o];
              s1[j] = p.S1[o];
            }
          }
        }
        uint64_t ring[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) ring[b] = 0;
#pragma unroll
        for (int by = 0; by < PYM + Q; ++by) {
          if (by >= nby) break;  // uniform
          uint64_t h = 0, hw = 0;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            h += col[a * BS];
            if (RR > 0) hw += col[a * BS + 2 * EW];
          }
          if (RR > 0) {
            h += col[Q * BS + EW];
            hw += col[Q * BS + 3 * EW];
          }
          col += nbx * BS;
          constexpr int sh = RR == 0 ? 1 : 0;
          uint64_t sfg = 0;
          if (RR > 0) {
            sfg = hw;
#pragma unroll
            for (int b = 0; b < Q; ++b) sfg += ring[b];
          }
#pragma unroll
          for (int b = 0; b < Q - 1; ++b) ring[b] = ring[b + 1];
          ring[Q - 1] = h;
          if (RR == 0) {
            sfg = 0;
#pragma unroll
            for (int b = 0; b < Q; ++b) sfg += ring[b];
          }
          const int pj = by - Q + sh;  // the POI row whose box ends here (compile-time per unrolled step)
          if (pj < 0 || pj >= PYM) continue;
          if (pj >= ny_here) break;  // uniform
          // ---- candidate (POI (ix0+pi, iy0+pj), displacement (dx, dy)) ----
          BsPoiState& ps = st[pj * g.PX + pic];
          const bool valid = rsq[pj] > 0.0f;  // outside the window / constant target window: skipped, not counted
          const int64_t num = (int64_t)(sfg * n - (uint64_t)ps.sf * s1[pj]);
          const float a = __fmul_rn(__fmul_rn(__ll2float_rn(num), ps.rsvf), rsq[pj]);
          // the row's best (first lane on equal values) and runner-up filter values
          const uint32_t key = valid ? fkey(a) : 0u;
          uint32_t km = key;
#pragma unroll
          for (int o2 = 8; o2; o2 >>= 1) km = max(km, __shfl_xor_sync(0xffffffffu, km, o2));
          if (seg == 32) km = max(km, __shfl_xor_sync(0xffffffffu, km, 16));
          const unsigned top = __ballot_sync(0xffffffffu, key == km && km != 0u) & segmask;
          const int wl = top ? __ffs(top) - 1 : -1;  // winning lane of the segment
          uint32_t k2 = lane == wl ? 0u : key;
#pragma unroll
          for (int o2 = 8; o2; o2 >>= 1) k2 = max(k2, __shfl_xor_sync(0xffffffffu, k2, o2));
          if (seg == 32) k2 = max(k2, __shfl_xor_sync(0xffffffffu, k2, 16));
          const unsigned vb = __ballot_sync(0xffffffffu, valid) & segmask;
          const float a1o = ps.a1, a2o = ps.a2;
          __syncwarp();
          if (km) {
            const float r1 = funkey(km), r2 = k2 ? funkey(k2) : -3.0f;
            if (r1 > a1o) {  // new best from this row (equal values: a near tie, see bs_merge_kernel)
              if (lane == wl) {
                ps.a2 = fmaxf(a1o, r2);
                ps.a1 = r1;
                ps.num = num;
                ps.dx = (short)dx;
                ps.dy = (short)dy_;
              }
            } else if (dxi == 0) {
              ps.a2 = fmaxf(a2o, r1);
            }
          }
          if (dxi == 0 && pi < nx_here) ps.cnt += __popc(vb);
          __syncwarp();
        }
      }
      __syncthreads();
      continue;
    }
    // ---- phase B: one (POI column, dx) per thread, sliding down the block rows:
    //   h(by)  = sum_{a<Q} F(i+a, by) + C(i+Q, by)    (the POI column's row of blocks)
    //   hw(by) = sum_{a<Q} W(i+a, by) + K(i+Q, by)    (its first-r-rows strip)
    //   Sfg(i, j) = sum_{b<Q} h(j+b) + hw(j+Q)
    for (int t = threadIdx.x; t < nx_here * EW; t += NT) {
      const int pi = t / EW, dxi = t - pi * EW;
      const uint32_t* col = blk + pi * BS + dxi;
      uint64_t ring[Q];
#pragma unroll
      for (int b = 0; b < Q; ++b) ring[b] = 0;
      int64_t* out = p.sfg + ((size_t)(iy0 - p.rb) * p.lat.nx + (ix0 + pi)) * ew2 + (size_t)(dy + R) * EW + dxi;
      const size_t out_step = (size_t)p.lat.nx * ew2;
      for (int by = 0; by < nby; ++by, col += nbx * BS) {
        uint64_t h = 0, hw = 0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          h += col[a * BS];
          if (RR > 0) hw += col[a * BS + 2 * EW];
        }
        if (RR > 0) {
          h += col[Q * BS + EW];
          hw += col[Q * BS + 3 * EW];
        }
        const int pj = by - Q + (RR == 0 ? 1 : 0);  // the POI row whose box ends here
        if (RR > 0) {
          if (pj >= 0) {
            uint64_t s = hw;
#pragma unroll
            for (int b = 0; b < Q; ++b) s += ring[b];
            out[(size_t)pj * out_step] = (int64_t)s;
          }
        }
#pragma unroll
        for (int b = 0; b < Q - 1; ++b) ring[b] = ring[b + 1];
        ring[Q - 1] = h;
        if (RR == 0 && pj >= 0) {
          uint64_t s = 0;
#pragma unroll
          for (int b = 0; b < Q; ++b) s += ring[b];
          out[(size_t)pj * out_step] = (int64_t)s;
        }
      }
    }
    __syncthreads();
  }
  if (FUSE) {  // this dy slice's result per POI
    for (int i = threadIdx.x; i < nx_here * ny_here; i += NT) {
      const int pi = i % nx_here, pj = i / nx_here;
      const BsPoiState& ps = st[pj * g.PX + pi];
      BsSlice b;
      b.num = ps.num;
      b.a1 = ps.a1;
      b.a2 = ps.a2;
      b.cnt = ps.cnt;
      b.dx = ps.dx;
      b.dy = ps.dy;
      const size_t k = (size_t)(iy0 + pj - p.rb) * p.lat.nx + (ix0 + pi);
      reinterpret_cast<BsSlice*>(p.slices)[k * g.nsplit + blockIdx.z] = b;
    }
  }
}

// ---- K1-BS-WS: the same block sums, warp-specialised ----
// The single-role kernel above alternates phase A (IMAD-bound) and phase B
// (loads and u64 adds) behind CTA barriers, so the IMAD pipe idles during
// every phase B (ncu C5: fmaheavy 51 %, 8 warps/SM, 255 registers). Here the
// dx range is cut into chunks of DXC (registers <= 128), phase A of item
// (dy, chunk) runs on NPW producer warps (one block per thread, partials in
// registers) while NCW consumer warps run phase B of the previous item; the
// producers store into the single block-partial buffer once the consumers have
// released it (named barriers: FULL = 1, producers arrive / consumers wait;
// EMPTY = 2, the reverse), so the buffer costs one item of shared memory and
// the tile can be taller (less halo). Same partials, same u64 box sums, same
// cross-term buffer: the records are bit-identical to bs_kernel's.
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 4-byte global -> shared async copy.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// Fused bs_ws_kernel: stage the window data (1/sqrt(vg) filter factor, Sg) of
// every position the tile's candidates at displacement row dy can touch:
// [PYM rows][XW] with XW = (PX-1) step + 2R + 1 (0 outside the position domain:
// such candidates are outside their windows anyway). Issued by the consumers
// one dy ahead (cp.async, one commit group per dy).
__device__ __forceinline__ void bs_stage_positions(const TcParams& p, const BsGeom& g, int ix0, int iy0, int ny_here,
                                                   int dy, int XW, int PYM, float* rsq, uint32_t* s1, int t, int nt) {
  const int x0 = p.lat.cx(ix0) - p.M - p.R - p.qx_min;
  for (int xo = t; xo < XW; xo += nt) {
    const int qx = x0 + xo;
    const bool xok = qx >= 0 && qx < p.SW;
    for (int j = 0; j < ny_here; ++j) {
      const int qy = p.lat.cy(iy0 + j) - p.M + dy - p.qy_min;
      float* dr = rsq + j * XW + xo;
      uint32_t* ds = s1 + j * XW + xo;
      if (xok && qy >= 0 && qy < p.SH) {
        const size_t o = (size_t)qy * p.SW + qx;
        cp_async4(dr, p.RSQ + o);
        cp_async4(ds, p.S1 + o);
      } else {
        *dr = 0.0f;
        *ds = 0u;
      }
    }
  }
  (void)PYM;
  (void)g;
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// One dx lane's slice result for one POI (fused bs_ws_kernel, end-of-tile reduction).
struct BsLane {
  long long num;
  float a1, a2;
  uint32_t dc;
  uint32_t pad;
};

// Cycle counters of one interior CTA (DICB200_BS_PROF=1, PROF instantiation):
// [0..3] producer warp 0: compute, wait for the buffer, store, items;
// [4..7] consumer warp 0: wait for the partials, phase B, window staging, items.
__device__ unsigned long long g_bs_prof[8];

template <int S, int RR, int Q, int DXC, int NPW, int NCW, typename Pix, bool FUSE = false, int PYM = 1, int PV = 0,
          bool PROF = false>
__global__ void __launch_bounds__(32 * (NPW + NCW), 1) bs_ws_kernel(TcParams p, BsGeom g) {
  constexpr int NT = 32 * (NPW + NCW), NP = 32 * NPW, NC = 32 * NCW;
  constexpr int BS = 4 * DXC + 1;  // words per block record (odd: conflict-free stores across blocks)
  extern __shared__ __align__(16) unsigned char bs_smem[];
  uint16_t* Rf = reinterpret_cast<uint16_t*>(bs_smem);              // [RHp][RP]
  uint16_t* Tg = reinterpret_cast<uint16_t*>(bs_smem + g.off_tgt);  // [THp][TP]
  uint32_t* blk0 = reinterpret_cast<uint32_t*>(bs_smem + g.off_blk);  // [nblk][F|C|W|K x DXC]
  const int M = p.M, R = p.R, EW = g.EW, RP = g.RWp, TP = g.TWp;
  const int ix0 = blockIdx.x * g.PX, iy0 = p.rb + blockIdx.y * g.PY;
  const int dy_lo = -R + (int)blockIdx.z * g.dy_per, dy_hi = min(R, dy_lo + g.dy_per - 1);
  const int RX0 = p.lat.cx(ix0) - M, RY0 = p.lat.cy(iy0) - M;  // block (0, 0) origin
  const int TX0 = RX0 - R, TY0 = RY0 - R;
  int shR = 0, shT = 0;
  bs_stage<Pix, NT>(p, g, Rf, Tg, RX0, RY0, TX0, TY0, dy_lo, dy_hi, DXC, shR, shT);
  const int nx_here = min(g.PX, p.lat.nx - ix0), ny_here = min(g.PY, p.re - iy0);
  if (FUSE) {  // POI constants of the tile: 1 / sqrt(vf) (0: degenerate subset), Sf
    float* prs = reinterpret_cast<float*>(bs_smem + g.off_state);
    uint32_t* psf = reinterpret_cast<uint32_t*>(prs + g.PX * g.PY);
    for (int i = threadIdx.x; i < g.PX * g.PY; i += NT) {
      const int qi = i % g.PX, qj = i / g.PX;
      float r = 0.0f;
      uint32_t sf = 0;
      if (qi < nx_here && qj < ny_here) {
        const size_t k = (size_t)(iy0 + qj - p.rb) * p.lat.nx + (ix0 + qi);
        const double svf = p.poi_sqrtvf[k];
        r = svf > 0.0 ? (float)(1.0 / svf) : 0.0f;
        sf = (uint32_t)p.poi_sf[k];
      }
      prs[i] = r;
      psf[i] = sf;
    }
  }
  __syncthreads();
  const int nbx = g.nbx;
  const int nbx_here = nx_here + Q - (RR == 0 ? 1 : 0), nby = ny_here + Q - (RR == 0 ? 1 : 0);
  const int nchunk = g.nchunk, n_items = (dy_hi - dy_lo + 1) * nchunk;
  // PV 1, fused: the consumer warps past the (POI column, dx lane) threads of
  // phase B are dedicated stagers of the window data (see below) and stay out of
  // the item barriers
  const int nbw = (g.PX * DXC + 31) >> 5;
  const bool ded = FUSE && PV == 1 && nbw < NCW;
  const int NTB = ded ? NP + 32 * nbw : NT;
  if (threadIdx.x < NP) {
    // ---- producers: phase A of item it in registers (one block per thread),
    // then, once the consumers have released the buffer, the store
    // blocks spread evenly over the four SM sub-partitions (warp w issues on
    // SMSP w % 4): each takes a contiguous quarter of the block list
    const int w = threadIdx.x >> 5, per_smsp = (nbx_here * nby + 3) / 4, slot = (w >> 2) * 32 + (threadIdx.x & 31);
    const int task = (w & 3) * per_smsp + slot;
    const bool active = slot < per_smsp && task < nbx_here * nby;
    const int by = active ? task / nbx_here : 0, bx = active ? task - by * nbx_here : 0, bi = by * nbx + bx;
    const uint16_t* fr = Rf + (by * S) * RP + shR + bx * S;
    uint32_t* o = blk0 + bi * BS;
    const bool prof = PROF && blockIdx.x == 1 && blockIdx.y == 1 && blockIdx.z == 0 && threadIdx.x == 0;
    unsigned long long pc0 = 0, pc1 = 0, pc2 = 0;
    for (int it = 0; it < n_items; ++it) {
      const int dy = dy_lo + it / nchunk, dx0 = (it % nchunk) * DXC;
      const uint16_t* gr = Tg + (by * S + dy + R) * TP + shT + bx * S + dx0;
      long long t0 = 0, t1 = 0, t2 = 0;
      if (PROF) t0 = clock64();
      uint32_t F[DXC], Cc[DXC], Wr[DXC], Kc[DXC];
#pragma unroll
      for (int j = 0; j < DXC; ++j) F[j] = Cc[j] = Wr[j] = Kc[j] = 0u;
      if (PV == 1) {
        // rows >= RR accumulate straight into F (columns >= RR) and Cc (columns
        // < RR), the first RR rows — walked last, so their accumulators are
        // short-lived — into Wr / Kc; the four stored partials are sums of those
        if (active) {
#pragma unroll
          for (int y2 = 0; y2 < S; ++y2) {
            const int yy = y2 < S - RR ? y2 + RR : y2 - (S - RR);  // RR .. S-1, then 0 .. RR-1
            uint32_t f[S], gg[S + DXC - 1];
#pragma unroll
            for (int k = 0; k < S; ++k) f[k] = fr[yy * RP + k];
#pragma unroll
            for (int k = 0; k < S + DXC - 1; ++k) gg[k] = gr[yy * TP + k];
#pragma unroll
            for (int k = 0; k < S; ++k)
#pragma unroll
              for (int j = 0; j < DXC; ++j) {
                if (yy >= RR) {
                  if (k >= RR)
                    F[j] += f[k] * gg[k + j];
                  else
                    Cc[j] += f[k] * gg[k + j];
                } else {
                  if (k >= RR)
                    Wr[j] += f[k] * gg[k + j];
                  else
                    Kc[j] += f[k] * gg[k + j];
                }
              }
          }
#pragma unroll
          for (int j = 0; j < DXC; ++j) {
            if (RR > 0) {
              F[j] += Cc[j] + Wr[j] + Kc[j];
              Cc[j] += Kc[j];
              Wr[j] += Kc[j];
            }
          }
        }
      } else if (active) {
#pragma unroll
        for (int yy = 0; yy < S; ++yy) {
          uint32_t f[S], gg[S + DXC - 1];
#pragma unroll
          for (int k = 0; k < S; ++k) f[k] = fr[yy * RP + k];
#pragma unroll
          for (int k = 0; k < S + DXC - 1; ++k) gg[k] = gr[yy * TP + k];
          uint32_t part[DXC], full[DXC];
#pragma unroll
          for (int j = 0; j < DXC; ++j) part[j] = RR > 0 ? f[0] * gg[j] : 0u;
#pragma unroll
          for (int k = 1; k < RR; ++k)
#pragma unroll
            for (int j = 0; j < DXC; ++j) part[j] += f[k] * gg[k + j];
#pragma unroll
          for (int j = 0; j < DXC; ++j) full[j] = part[j];
#pragma unroll
          for (int k = RR; k < S; ++k)
#pragma unroll
            for (int j = 0; j < DXC; ++j) full[j] += f[k] * gg[k + j];
#pragma unroll
          for (int j = 0; j < DXC; ++j) {
            F[j] += full[j];
            if (RR > 0) {
              Cc[j] += part[j];
              if (yy < RR) {
                Wr[j] += full[j];
                Kc[j] += part[j];
              }
            }
          }
        }
      }
      if (PROF) t1 = clock64();
      if (it >= 1) named_bar_sync(2, NTB);  // consumers are done with item it - 1
      if (PROF) t2 = clock64();
      // columns past the chunk's last dx hold products with zero padding or
      // the next chunk's dx: stored anyway (never read)
      if (active) {
#pragma unroll
        for (int j = 0; j < DXC; ++j) {
          o[j] = F[j];
          if (RR > 0) {
            o[DXC + j] = Cc[j];
            o[2 * DXC + j] = Wr[j];
            o[3 * DXC + j] = Kc[j];
          }
        }
      }
      named_bar_arrive(1, NTB);
      if (PROF) {
        const long long t3 = clock64();
        pc0 += (unsigned long long)(t1 - t0);
        pc1 += (unsigned long long)(t2 - t1);
        pc2 += (unsigned long long)(t3 - t2);
      }
    }
    if (prof) {
      g_bs_prof[0] = pc0;
      g_bs_prof[1] = pc1;
      g_bs_prof[2] = pc2;
      g_bs_prof[3] = (unsigned long long)n_items;
    }
  } else if (FUSE) {
    // ---- fused consumers: phase B and the exact-argmax filter. Thread
    // (POI column pi, dx lane dxi) handles dx = c DXC + dxi of every chunk c and
    // keeps, per POI row of the tile, its best filter value, runner-up, the
    // best's exact numerator and dx/dy, and its candidate count in registers;
    // the tile's slice result per POI is reduced over the dx lanes at the end
    // (bs_merge_kernel then combines the dy slices exactly, near ties included).
    const int tc = threadIdx.x - NP;
    const bool act = tc < nx_here * DXC;
    const int pi = act ? tc / DXC : 0, dxi = act ? tc - pi * DXC : 0;
    const float* poi_rsvf = reinterpret_cast<const float*>(bs_smem + g.off_state);            // [PY][PX]
    const uint32_t* poi_sf = reinterpret_cast<const uint32_t*>(poi_rsvf + g.PX * g.PY);        // [PY][PX]
    const uint32_t n = (uint32_t)(p.side * p.side);
    const int cxp = p.lat.cx(ix0 + pi);
    const int fx_lo = max(-R, M - cxp), fx_hi = min(R, p.tgt.width - 1 - M - cxp);
    float a1[PYM], a2[PYM];
    long long num1[PYM];
    uint32_t dc[PYM];  // count (bits 0-15) | dx index (16-23) | dy index (24-31) of the best
#pragma unroll
    for (int j = 0; j < PYM; ++j) {
      a1[j] = a2[j] = -3.0f;
      num1[j] = 0;
      dc[j] = 0;
    }
    const int XW = (g.PX - 1) * p.lat.step + 2 * R + 1;
    float* pos_rsq = reinterpret_cast<float*>(bs_smem + g.off_pos);  // [2][PYM][XW]
    uint32_t* pos_s1 = reinterpret_cast<uint32_t*>(pos_rsq + 2 * PYM * XW);
    const bool cprof = PROF && blockIdx.x == 1 && blockIdx.y == 1 && blockIdx.z == 0 && tc == 0;
    unsigned long long cc0 = 0, cc1 = 0, cc2 = 0;
    if (ded && tc >= 32 * nbw) {
      // ---- dedicated stagers: the window data of dy go into buffer (dy - dy_lo) & 1
      // once the phase-B warps have released it (they were done with dy - 2),
      // a whole displacement row ahead of its use. Named barriers by buffer
      // parity: 3 / 4 = data landed (stagers arrive, phase B waits), 5 / 6 =
      // buffer released (the reverse); a generation of either can only start
      // after the previous one of the same parity completed.
      const int ts = tc - 32 * nbw, ns = NC - 32 * nbw;
      for (int dy = dy_lo; dy <= dy_hi; ++dy) {
        const int pb = (dy - dy_lo) & 1;
        if (dy >= dy_lo + 2) named_bar_sync(5 + pb, NC);
        bs_stage_positions(p, g, ix0, iy0, ny_here, dy, XW, PYM, pos_rsq + pb * PYM * XW, pos_s1 + pb * PYM * XW, ts,
                           ns);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        named_bar_arrive(3 + pb, NC);
      }
    } else {
    if (!ded) bs_stage_positions(p, g, ix0, iy0, ny_here, dy_lo, XW, PYM, pos_rsq, pos_s1, tc, NC);
    for (int it = 0; it < n_items; ++it) {
      const int dy = dy_lo + it / nchunk, dxv = (it % nchunk) * DXC + dxi - R;
      const int pb = (dy - dy_lo) & 1;
      long long c0 = 0, c1 = 0, c2 = 0;
      if (PROF) c0 = clock64();
      if (ded) {
        if (it % nchunk == 0) named_bar_sync(3 + pb, NC);  // the stagers' data of dy landed
      } else if (it % nchunk == 0) {  // new dy: its window data landed, the next dy's starts
        named_bar_sync(3, NC);   // every consumer is done with dy - 1: its buffer is free
        if (dy < dy_hi) {
          bs_stage_positions(p, g, ix0, iy0, ny_here, dy + 1, XW, PYM, pos_rsq + (pb ^ 1) * PYM * XW,
                             pos_s1 + (pb ^ 1) * PYM * XW, tc, NC);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        named_bar_sync(3, NC);
      }
      if (PROF) c1 = clock64();
      named_bar_sync(1, NTB);  // producers stored item it
      if (PROF) c2 = clock64();
      const bool xin = act && dxv <= R && dxv >= fx_lo && dxv <= fx_hi;
      if (__any_sync(0xffffffffu, xin)) {
        const uint32_t* col = blk0 + pi * BS + dxi;
        const int xo = pi * p.lat.step + dxv + R;
        const float* prow = pos_rsq + pb * PYM * XW + xo;
        const uint32_t* srow = pos_s1 + pb * PYM * XW + xo;
        uint64_t ring[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) ring[q] = 0;
#pragma unroll
        for (int by = 0; by < PYM + Q; ++by) {
          if (by >= nby) break;  // uniform
          uint64_t h = 0, hw = 0;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            h += col[a * BS];
            if (RR > 0) hw += col[a * BS + 2 * DXC];
          }
          if (RR > 0) {
            h += col[Q * BS + DXC];
            hw += col[Q * BS + 3 * DXC];
          }
          col += nbx * BS;
          constexpr int sh = RR == 0 ? 1 : 0;
          uint64_t sfg = 0;
          if (RR > 0) {
            sfg = hw;
#pragma unroll
            for (int q = 0; q < Q; ++q) sfg += ring[q];
          }
#pragma unroll
          for (int q = 0; q < Q - 1; ++q) ring[q] = ring[q + 1];
          ring[Q - 1] = h;
          if (RR == 0) {
            sfg = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) sfg += ring[q];
          }
          const int pj = by - Q + sh;  // the POI row whose box ends here (compile-time per step)
          if (pj < 0 || pj >= PYM) continue;
          const int cyp = p.lat.cy(iy0 + pj);
          const float rsvf = poi_rsvf[pj * g.PX + pi];  // (pj >= ny_here: 0)
          // integer_search.cpp:11-21 window; degenerate reference subset (rsvf 0): no candidates
          // branch-free: an invalid candidate gets filter value -3 (never kept) and counts 0
          const float rsq = prow[pj * XW];
          // constant target window (rsq 0): skipped, not counted (tc_candidate_f)
          const bool valid = xin && pj < ny_here && rsvf > 0.0f && rsq > 0.0f && dy >= max(-R, M - cyp) &&
                             dy <= min(R, p.tgt.height - 1 - M - cyp);
          const int64_t num = (int64_t)(sfg * n - (uint64_t)poi_sf[pj * g.PX + pi] * srow[pj * XW]);
          const float a = valid ? __fmul_rn(__fmul_rn(__ll2float_rn(num), rsvf), rsq) : -3.0f;  // approx_zncc
          const bool better = a > a1[pj];
          a2[pj] = fmaxf(a2[pj], fminf(a, a1[pj]));  // runner-up (equal values: a near tie)
          a1[pj] = fmaxf(a1[pj], a);
          num1[pj] = better ? num : num1[pj];
          dc[pj] = (better ? (((uint32_t)(dxv + R) << 16) | ((uint32_t)(dy + R) << 24)) : (dc[pj] & 0xffff0000u)) |
                   ((dc[pj] & 0xffffu) + (valid ? 1u : 0u));
        }
      }
      if (it + 1 < n_items) named_bar_arrive(2, NTB);  // buffer free for item it + 1
      if (ded && it % nchunk == nchunk - 1 && dy + 2 <= dy_hi) named_bar_arrive(5 + pb, NC);  // done with dy
      if (PROF) {
        const long long c3 = clock64();
        cc0 += (unsigned long long)(c2 - c1);
        cc1 += (unsigned long long)(c3 - c2);
        cc2 += (unsigned long long)(c1 - c0);
      }
    }
    }
    if (cprof) {
      g_bs_prof[4] = cc0;
      g_bs_prof[5] = cc1;
      g_bs_prof[6] = cc2;
      g_bs_prof[7] = (unsigned long long)n_items;
    }
    // ---- slice result per POI: reduce the DXC dx lanes (through the free block buffer)
    named_bar_sync(7, NC);  // every consumer is past its last read of the block buffer
    BsLane* lanes = reinterpret_cast<BsLane*>(blk0);  // [PY][PX][DXC]
    if (act) {
#pragma unroll
      for (int j = 0; j < PYM; ++j) {
        if (j < ny_here) {
          BsLane& l = lanes[(j * g.PX + pi) * DXC + dxi];
          l.num = num1[j];
          l.a1 = a1[j];
          l.a2 = a2[j];
          l.dc = dc[j];
        }
      }
    }
    named_bar_sync(7, NC);
    for (int i = tc; i < nx_here * ny_here; i += NC) {
      const int qi = i % nx_here, qj = i / nx_here;
      const BsLane* l = lanes + (qj * g.PX + qi) * DXC;
      BsSlice b;
      b.num = 0;
      b.a1 = b.a2 = -3.0f;
      b.cnt = 0;
      b.dx = b.dy = 0;
      for (int d = 0; d < DXC; ++d) {
        const BsLane v = l[d];
        b.cnt += (int)(v.dc & 0xffffu);
        if (v.a1 > b.a1) {
          b.a2 = fmaxf(b.a1, v.a2);
          b.a1 = v.a1;
          b.num = v.num;
          b.dx = (short)((int)((v.dc >> 16) & 0xffu) - R);
          b.dy = (short)((int)(v.dc >> 24) - R);
        } else {
          b.a2 = fmaxf(b.a2, v.a1);  // equal values: a near tie, see bs_merge_kernel
        }
        b.a2 = fmaxf(b.a2, v.a2);
      }
      const size_t k = (size_t)(iy0 + qj - p.rb) * p.lat.nx + (ix0 + qi);
      reinterpret_cast<BsSlice*>(p.slices)[k * g.nsplit + blockIdx.z] = b;
    }
  } else {
    // ---- consumers: phase B, one (POI column, dx of the chunk) per thread
    const int tc = threadIdx.x - NP;
    const size_t ew2 = (size_t)EW * EW;
    const size_t out_step = (size_t)p.lat.nx * ew2;
    for (int it = 0; it < n_items; ++it) {
      named_bar_sync(1, NT);  // producers stored item it
      const int dy = dy_lo + it / nchunk, dx0 = (it % nchunk) * DXC, nd = min(DXC, EW - dx0);
      const uint32_t* blk = blk0;
      for (int t = tc; t < nx_here * nd; t += NC) {
        const int pi = t / nd, dxi = t - pi * nd;
        const uint32_t* col = blk + pi * BS + dxi;
        uint64_t ring[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) ring[q] = 0;
        int64_t* out = p.sfg + ((size_t)(iy0 - p.rb) * p.lat.nx + (ix0 + pi)) * ew2 + (size_t)(dy + R) * EW + dx0 + dxi;
        for (int by = 0; by < nby; ++by, col += nbx * BS) {
          uint64_t h = 0, hw = 0;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            h += col[a * BS];
            if (RR > 0) hw += col[a * BS + 2 * DXC];
          }
          if (RR > 0) {
            h += col[Q * BS + DXC];
            hw += col[Q * BS + 3 * DXC];
          }
          const int pj = by - Q + (RR == 0 ? 1 : 0);  // the POI row whose box ends here
          if (RR > 0 && pj >= 0) {
            uint64_t s = hw;
#pragma unroll
            for (int q = 0; q < Q; ++q) s += ring[q];
            out[(size_t)pj * out_step] = (int64_t)s;
          }
#pragma unroll
          for (int q = 0; q < Q - 1; ++q) ring[q] = ring[q + 1];
          ring[Q - 1] = h;
          if (RR == 0 && pj >= 0) {
            uint64_t s = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) s += ring[q];
            out[(size_t)pj * out_step] = (int64_t)s;
          }
        }
      }
      if (it + 1 < n_items) named_bar_arrive(2, NT);  // buffer free for item it + 1
    }
  }
}

// Per POI: the dy slices' filter winners -> the record (tc_argmax_kernel's
// output, including "all positions degenerate"). Every candidate that can be
// the exact maximum has a filter value within 2^-19 of the largest one (filter
// error < 2^-21.6, approx_zncc): when those are exactly the slices' stored
// winners, their exact quotients decide in improves() order; when a runner-up
// also lies that close (a near tie the slices did not keep), the POI is
// flagged and bs_exact_kernel searches it exactly.
__global__ void __launch_bounds__(256) bs_merge_kernel(TcParams p, int nsplit, int* flagged, int* n_flagged) {
  const size_t npoi = (size_t)(p.re - p.rb) * p.lat.nx;
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npoi) return;
  const int ix = (int)(k % p.lat.nx), iy = p.rb + (int)(k / p.lat.nx);
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, R = p.R;
  const int fx_lo = max(-R, M - cx), fx_hi = min(R, p.tgt.width - 1 - M - cx);
  const int fy_lo = max(-R, M - cy), fy_hi = min(R, p.tgt.height - 1 - M - cy);
  BestPartial b;
  b.c = -2.0;
  b.dx = b.dy = 0;
  b.count = 0;
  b.found = 0;
  const double svf = p.poi_sqrtvf[k];
  if (fx_lo <= fx_hi && fy_lo <= fy_hi && svf > 0.0) {
    const BsSlice* sl = reinterpret_cast<const BsSlice*>(p.slices) + k * nsplit;
    float amax = -3.0f;
    for (int s = 0; s < nsplit; ++s) {
      b.count += sl[s].cnt;
      amax = fmaxf(amax, sl[s].a1);
    }
    const float thr = amax - 0x1p-19f;
    bool near_tie = false;
    for (int s = 0; s < nsplit; ++s) {
      if (sl[s].cnt == 0) continue;
      near_tie |= sl[s].a2 >= thr;
      if (sl[s].a1 >= thr) {
        const int qx = cx - M + sl[s].dx, qy = cy - M + sl[s].dy;
        const double z = bs_i64_to_f64(sl[s].num) /
                         (svf * p.SQ[(size_t)(qy - p.qy_min) * p.SW + (qx - p.qx_min)]);  // exact
        if (!b.found || improves(z, sl[s].dx, sl[s].dy, b.c, b.dx, b.dy)) {
          b.found = 1;
          b.c = z;
          b.dx = sl[s].dx;
          b.dy = sl[s].dy;
        }
      }
    }
    if (near_tie) {
      flagged[atomicAdd(n_flagged, 1)] = (int)k;
      return;  // bs_exact_kernel writes this record
    }
  }
  write_integer_record(p.rec[k], cx, cy, b, p.subpixel_none);
}

// Flagged POIs (near ties of the filter): the reference's bfs_search over the
// window, exactly — CTA per POI, the reference subset and the target window
// staged in shared memory, exact u64 cross terms per candidate (thread per
// candidate), exact quotients, block argmax in improves() order.
constexpr int kExactMaxSide = 64, kExactMaxWin = 96;
// Flagged POIs, fast path: CTA (slot, candidate row) computes the exact cross
// terms of one displacement row of one flagged POI — warp per dx, lanes across
// the subset columns (u32 per lane: < 2 x side x 2^24 products, then u64 warp
// sums) — and its row argmax / count; the last CTA of a POI (arrival counter)
// merges the rows in improves() order and writes the record. A flagged POI is
// 1 M exact MACs (C5): spread over 2R+1 CTAs instead of one (measured: the
// single-CTA search cost ~70 us per pair with one or two flagged POIs; the
// single-CTA bs_exact_kernel below takes the slots past kExactSlots).
constexpr int kExactSlots = 256;
constexpr int kExactRowWarps = 8;  // warps per CTA, dx strided over them (2R+1 <= 32)
template <typename Pix>
__global__ void __launch_bounds__(32 * kExactRowWarps) bs_exact_rows_kernel(TcParams p, const int* flagged,
                                                                           const int* n_flagged, BestPartial* part,
                                                                           int* arrivals) {
  __shared__ uint16_t fs[kExactMaxSide * kExactMaxSide];
  __shared__ uint16_t gs[kExactMaxSide * kExactMaxWin];
  __shared__ double red_c[kExactRowWarps];
  __shared__ int red_d[kExactRowWarps][3];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = min(*n_flagged, kExactSlots);
  const int ry = blockIdx.x;  // rows fastest: the CTAs of the first slots come first in launch order
  for (int i = blockIdx.y; i < nf; i += gridDim.y) {
  const size_t k = (size_t)flagged[i];
  const int ix = (int)(k % p.lat.nx), iy = p.rb + (int)(k / p.lat.nx);
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, R = p.R, side = p.side;
  const int fx_lo = max(-R, M - cx), fx_hi = min(R, p.tgt.width - 1 - M - cx);
  const int fy_lo = max(-R, M - cy), fy_hi = min(R, p.tgt.height - 1 - M - cy);
  const int fw = fx_hi - fx_lo + 1, fh = fy_hi - fy_lo + 1, ww = fw + side - 1;
  if (ry >= fh) continue;  // rows past the feasible window: no CTA work, no arrival (uniform)
  // u32 partial sums of at most flush_every products (< 2^32 for the pair's pixel range)
  // (2R+1 <= kExactRowWarps * kExactDx dx lanes per CTA: rows_ok)
  const double mv = p.maxv > 0 ? p.maxv : 65535.0;
  const int flush_every = (int)fmax(1.0, fmin(64.0, floor(4294967295.0 / fmax(1.0, mv * mv))));
  const int dy = fy_lo + ry;
  const Pix* f = static_cast<const Pix*>(p.ref.data);
  const Pix* g = static_cast<const Pix*>(p.tgt.data);
  __syncthreads();  // the previous slot's reduction is done with the staged data
  // warp per row, lanes across columns: the loads of a warp's rows are independent
  for (int r = warp; r < side; r += kExactRowWarps) {
    const Pix* fr = f + (size_t)(cy - M + r) * p.ref.pitch + (cx - M);
    const Pix* gr = g + (size_t)(cy - M + dy + r) * p.tgt.pitch + (cx - M + fx_lo);
    for (int c = lane; c < side; c += 32) fs[r * side + c] = (uint16_t)fr[c];
    for (int c = lane; c < ww; c += 32) gs[r * ww + c] = (uint16_t)gr[c];
  }
  __syncthreads();
  BestPartial b;
  b.c = -2.0;
  b.dx = b.dy = 0;
  b.count = 0;
  b.found = 0;
  // warp w takes dx lanes w, w + 8, w + 16, w + 24 (kExactDx per warp, all
  // at once: one reference load per pixel feeds them all); lanes across the
  // subset columns (c and c + 32), rows in order; u32 runs of at most
  // flush_every rows' products, flushed to u64 (exact)
  constexpr int kExactDx = 4;
  uint64_t acc64[kExactDx] = {0, 0, 0, 0};
  uint32_t acc[kExactDx] = {0, 0, 0, 0};
  const int c0 = lane, c1 = lane + 32;
  const bool two = c1 < side;
  int run = 0;
  const bool wide = flush_every < 2;
  const int rows_per_flush = max(1, flush_every / 2);
  for (int r = 0; r < side; ++r) {
    const uint16_t* fr = fs + r * side;
    const uint16_t* gr = gs + r * ww + warp;
    const uint32_t fa = c0 < side ? fr[c0] : 0u, fb = two ? fr[c1] : 0u;
#pragma unroll
    for (int j = 0; j < kExactDx; ++j) {
      const int wx = j * kExactRowWarps;  // + warp (in gr)
      if (warp + wx < fw) {
        const uint32_t va = c0 < side ? fa * gr[wx + c0] : 0u, vb = two ? fb * gr[wx + c1] : 0u;
        if (wide)  // products near 2^32 (16-bit pixels): straight into u64
          acc64[j] += (uint64_t)va + vb;
        else
          acc[j] += va + vb;
      }
    }
    if (++run == rows_per_flush) {
#pragma unroll
      for (int j = 0; j < kExactDx; ++j) {
        acc64[j] += acc[j];
        acc[j] = 0;
      }
      run = 0;
    }
  }
#pragma unroll
  for (int j = 0; j < kExactDx; ++j) {
    acc64[j] += acc[j];
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) acc64[j] += __shfl_xor_sync(0xffffffffu, acc64[j], o2);
  }
  const uint32_t n = (uint32_t)(side * side), sf = (uint32_t)p.poi_sf[k];
#pragma unroll
  for (int j = 0; j < kExactDx; ++j) {  // dx ascending within the warp
    const int wx = warp + j * kExactRowWarps;
    if (wx >= fw) continue;
    const int dx = fx_lo + wx;
    const size_t o = (size_t)(cy - M + dy - p.qy_min) * p.SW + (cx - M + dx - p.qx_min);
    const double sq = p.SQ[o];
    if (!(sq > 0.0)) continue;  // constant target window: skipped, not counted
    const int64_t num = (int64_t)(acc64[j] * n - (uint64_t)sf * p.S1[o]);
    BestPartial q;
    q.c = bs_i64_to_f64(num) / (p.poi_sqrtvf[k] * sq);
    q.dx = dx;
    q.dy = dy;
    q.count = 1;
    q.found = 1;
    merge_best(b, q);
  }
  if (lane == 0) {
    red_c[warp] = b.found ? b.c : -3.0;
    red_d[warp][0] = b.found ? b.dx : 0x7fff;
    red_d[warp][1] = b.found ? b.dy : 0x7fff;
    red_d[warp][2] = b.count;
  }
  __syncthreads();
  if (tid == 0) {
    BestPartial t;
    t.c = -2.0;
    t.dx = t.dy = 0;
    t.count = 0;
    t.found = 0;
    for (int w2 = 0; w2 < kExactRowWarps; ++w2) {
      BestPartial q;
      q.c = red_c[w2];
      q.dx = red_d[w2][0];
      q.dy = red_d[w2][1];
      q.count = red_d[w2][2];
      q.found = red_d[w2][0] != 0x7fff;
      merge_best(t, q);
    }
    part[(size_t)i * kExactMaxWin + ry] = t;
    __threadfence();
    s_last = atomicAdd(&arrivals[i], 1) == fh - 1;
  }
  __syncthreads();
  if (s_last && warp == 0) {  // every row of this POI is in: merge (improves() decides, any order)
    __threadfence();
    BestPartial t;
    t.c = -2.0;
    t.dx = t.dy = 0;
    t.count = 0;
    t.found = 0;
    for (int r = lane; r < fh; r += 32) {  // rows loaded together, one per lane
      const BestPartial* src = part + (size_t)i * kExactMaxWin + r;  // written by other CTAs: read through L2
      BestPartial q;
      q.c = __ldcg(&src->c);
      q.dx = __ldcg(&src->dx);
      q.dy = __ldcg(&src->dy);
      q.count = __ldcg(&src->count);
      q.found = __ldcg(&src->found);
      merge_best(t, q);
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
      BestPartial q;
      q.c = __shfl_xor_sync(0xffffffffu, t.c, o2);
      q.dx = __shfl_xor_sync(0xffffffffu, t.dx, o2);
      q.dy = __shfl_xor_sync(0xffffffffu, t.dy, o2);
      q.count = __shfl_xor_sync(0xffffffffu, t.count, o2);
      q.found = __shfl_xor_sync(0xffffffffu, t.found, o2);
      merge_best(t, q);
    }
    if (lane == 0) {
      arrivals[i] = 0;
      write_integer_record(p.rec[k], cx, cy, t, p.subpixel_none);
    }
  }
  }
}

template <typename Pix>
__global__ void __launch_bounds__(256) bs_exact_kernel(TcParams p, const int* flagged, const int* n_flagged,
                                                       int first_slot) {
  __shared__ uint16_t fs[kExactMaxSide * kExactMaxSide];
  __shared__ uint16_t gs[kExactMaxWin * kExactMaxWin];
  __shared__ double red_c[8];
  __shared__ int red_d[8][3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = *n_flagged;
  for (int i = first_slot + blockIdx.x; i < nf; i += gridDim.x) {  // earlier slots: bs_exact_rows_kernel
    const size_t k = (size_t)flagged[i];
    const int ix = (int)(k % p.lat.nx), iy = p.rb + (int)(k / p.lat.nx);
    const int cx = p.lat.cx(ix), cy = p.lat.cy(iy), M = p.M, R = p.R, side = p.side;
    const int fx_lo = max(-R, M - cx), fx_hi = min(R, p.tgt.width - 1 - M - cx);
    const int fy_lo = max(-R, M - cy), fy_hi = min(R, p.tgt.height - 1 - M - cy);
    const int fw = fx_hi - fx_lo + 1, fh = fy_hi - fy_lo + 1, ww = fw + side - 1, wh = fh + side - 1;
    const Pix* f = static_cast<const Pix*>(p.ref.data);
    const Pix* g = static_cast<const Pix*>(p.tgt.data);
    __syncthreads();  // previous POI's reduction done
    for (int t = tid; t < side * side; t += 256) {
      const int r = t / side, c = t - r * side;
      fs[t] = (uint16_t)f[(size_t)(cy - M + r) * p.ref.pitch + (cx - M + c)];
    }
    for (int t = tid; t < ww * wh; t += 256) {
      const int r = t / ww, c = t - r * ww;
      gs[t] = (uint16_t)g[(size_t)(cy - M + fy_lo + r) * p.tgt.pitch + (cx - M + fx_lo + c)];
    }
    __syncthreads();
    const uint32_t n = (uint32_t)(side * side), sf = (uint32_t)p.poi_sf[k];
    const double svf = p.poi_sqrtvf[k];
    BestPartial b;
    b.c = -2.0;
    b.dx = b.dy = 0;
    b.count = 0;
    b.found = 0;
    for (int t = tid; t < fw * fh; t += 256) {
      const int ry = t / fw, rx = t - ry * fw, dx = fx_lo + rx, dy = fy_lo + ry;
      const size_t o = (size_t)(cy - M + dy - p.qy_min) * p.SW + (cx - M + dx - p.qx_min);
      const double sq = p.SQ[o];
      if (!(sq > 0.0)) continue;  // constant target window: skipped, not counted
      uint64_t sfg = 0;
      for (int r = 0; r < side; ++r) {
        const uint16_t* fr = fs + r * side;
        const uint16_t* gr = gs + (ry + r) * ww + rx;
        for (int c = 0; c < side; ++c) sfg += (uint64_t)((uint32_t)fr[c] * gr[c]);  // each product < 2^32
      }
      const int64_t num = (int64_t)(sfg * n - (uint64_t)sf * p.S1[o]);
      const double z = bs_i64_to_f64(num) / (svf * sq);
      ++b.count;
      if (!b.found || improves(z, dx, dy, b.c, b.dx, b.dy)) {
        b.found = 1;
        b.c = z;
        b.dx = dx;
        b.dy = dy;
      }
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
      BestPartial q;
      q.c = __shfl_xor_sync(0xffffffffu, b.c, o2);
      q.dx = __shfl_xor_sync(0xffffffffu, b.dx, o2);
      q.dy = __shfl_xor_sync(0xffffffffu, b.dy, o2);
      q.count = __shfl_xor_sync(0xffffffffu, b.count, o2);
      q.found = __shfl_xor_sync(0xffffffffu, b.found, o2);
      merge_best(b, q);
    }
    if (lane == 0) {
      red_c[warp] = b.found ? b.c : -3.0;
      red_d[warp][0] = b.found ? b.dx : 0x7fff;
      red_d[warp][1] = b.found ? b.dy : 0x7fff;
      red_d[warp][2] = b.count;
    }
    __syncthreads();
    if (tid == 0) {
      BestPartial t;
      t.c = -2.0;
      t.dx = t.dy = 0;
      t.count = 0;
      t.found = 0;
      for (int w2 = 0; w2 < 8; ++w2) {
        BestPartial q;
        q.c = red_c[w2];
        q.dx = red_d[w2][0];
        q.dy = red_d[w2][1];
        q.count = red_d[w2][2];
        q.found = red_d[w2][0] != 0x7fff;
        merge_best(t, q);
      }
      write_integer_record(p.rec[k], cx, cy, t, p.subpixel_none);
    }
  }
}

// Instantiations: (s, r, DXC, threads). A configuration runs on the block-sum
// kernel when one of them matches its lattice spacing and remainder.
struct BsVariant {
  int S, RR, Q, DXC, NT, MINB;  // MINB: CTAs per SM the variant is sized for (shared memory, registers)
  int NPW, NCW;                 // warp-specialised (bs_ws_kernel): producer / consumer warps; 0 = bs_kernel
  int PX0, PY0;                 // POI tile tried first (bs_plan halves it until it fits)
};
constexpr BsVariant kVariants[] = {
    {10, 1, 4, 25, 256, 1, 0, 0, 16, 8},    // c5: L 41, s 10, R 12
    {10, 1, 3, 31, 256, 1, 0, 0, 16, 8},    // c2: L 31, s 10, R 15
    {5, 1, 8, 11, 384, 1, 0, 0, 16, 8},     // c4: L 41, s 5, R 5
    {8, 7, 3, 41, 256, 1, 0, 0, 16, 8},     // c3: L 31, s 8, R 20
    // warp-specialised: producer blocks fill whole warps on every SM sub-partition
    {10, 1, 4, 13, 512, 1, 8, 8, 12, 12},   // c5: 2 dx chunks, 12 x 12 POI tiles = 16 x 16 blocks
    {5, 1, 8, 11, 512, 1, 12, 4, 11, 8},    // c4: 11 x 8 POI tiles = 19 x 16 blocks; 121 (POI column, dx) consumer threads: fused argmax
};
// Measured and dropped (C5, B200): two CTAs per SM with dx chunks of 13 / 9
// (127 registers, 16 x 4 POI tiles to fit 110 KB): 0.93 / 0.98 ms against
// 0.57 ms for {10, 1, 4, 25, 256, 1} — the taller halo and the per-chunk
// target reloads cost more than the second CTA's latency hiding recovers.

template <int S, int RR, int Q, int DXC, int NT, int MINB>
cudaError_t launch_variant(const TcParams& p, const BsGeom& g, dim3 grid, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  auto go = [&](auto k) {
    e = set_dyn_smem(k, g.smem);
    if (e == cudaSuccess) k<<<grid, NT, g.smem, st>>>(p, g);
  };
  if (p.planes == 1)
    g.fuse ? go(bs_kernel<S, RR, Q, DXC, NT, MINB, uint8_t, true>) : go(bs_kernel<S, RR, Q, DXC, NT, MINB, uint8_t>);
  else
    g.fuse ? go(bs_kernel<S, RR, Q, DXC, NT, MINB, uint16_t, true>) : go(bs_kernel<S, RR, Q, DXC, NT, MINB, uint16_t>);
  return e;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// Geometry of the block-sum search for a planned TcParams; false = not applicable.
bool bs_plan(const TcParams& p, BsGeom& g) {
  if (std::getenv("DICB200_BFS_TC")) return false;  // A/B switch: tensor-core kernel
  const int s = p.lat.step, L = p.side;
  if (s < 2 || s >= L) return false;  // no overlap to share
  // u8 data: one byte plane keeps the tensor-core kernel ahead (measured on
  // c2 / c3); the block sums win for two-plane (wide) pixels
  if (p.planes != 2 && !std::getenv("DICB200_BFS_BS")) return false;
  const double maxv = p.maxv > 0 ? p.maxv : (p.planes == 1 ? 255.0 : 65535.0);
  if ((double)s * s * maxv * maxv >= 4294967296.0) return false;  // block sums must fit u32
  g.S = s;
  g.q = L / s;
  g.RR = L - g.q * s;
  g.EW = 2 * p.R + 1;
  int best = -1, waste = 1 << 30;
  const char* force = std::getenv("DICB200_BS_VARIANT");
  const int nvar = (int)(sizeof(kVariants) / sizeof(kVariants[0]));
  // warp-specialised variants first (DICB200_BS_CLASSIC=1: the single-role kernel)
  for (int pass = std::getenv("DICB200_BS_CLASSIC") ? 1 : 0; pass < 2 && best < 0; ++pass) {
    for (int v = 0; v < nvar; ++v) {
      if (kVariants[v].S != s || kVariants[v].RR != g.RR || kVariants[v].Q != g.q) continue;
      if (force ? v != std::atoi(force) : (kVariants[v].MINB != 1 || (kVariants[v].NPW > 0) != (pass == 0)))
        continue;
      const int nch = (g.EW + kVariants[v].DXC - 1) / kVariants[v].DXC;
      const int w = nch * kVariants[v].DXC - g.EW;
      if (w < waste) {
        waste = w;
        best = v;
      }
    }
  }
  if (best < 0) return false;
  g.ws = kVariants[best].NPW > 0;
  g.npw = kVariants[best].NPW;
  g.ncw = kVariants[best].NCW;
  g.async_ok = p.planes == 2 && ((uintptr_t)p.ref.data % 8) == 0 && ((uintptr_t)p.tgt.data % 8) == 0 &&
               (p.ref.pitch % 4) == 0 && (p.tgt.pitch % 4) == 0;
  // fused argmax (opt-in, DICB200_BS_FUSE=1): record mode (not the swarm's
  // surface), window of <= 32 dx. Bit-identical records without the cross-term
  // buffer (DRAM traffic ~ the two frames), but measured slower on C5 (B200):
  // 1.01 ms + 0.08 ms merge against 0.57 ms + 0.136 ms argmax — the warp-per-
  // POI-column phase B with its per-row reductions costs more than the HBM
  // round trip it removes (the unfused kernel writes the buffer while the IMAD
  // pipe is busy, and the argmax pass runs at 70% issue).
  g.fuse = g.ws ? (!p.surface && L <= 64 && L + g.EW - 1 <= 96 && std::getenv("DICB200_BS_UNFUSED") == nullptr)
               : !p.surface && g.EW <= 32 && L <= 64 && L + g.EW - 1 <= 96 && std::getenv("DICB200_BS_FUSE") != nullptr;
  g.DXC = kVariants[best].DXC;
  // fused ws: one consumer thread per (POI column, dx lane) of the widest tile
  if (g.ws && g.fuse && kVariants[best].PX0 * g.DXC > 32 * g.ncw) g.fuse = 0;
  g.threads = kVariants[best].NT;
  g.minb = kVariants[best].MINB;
  const size_t smem_cap = g.minb > 1 ? (size_t)(227 * 1024 / g.minb - 1024) : (size_t)220 * 1024;
  g.nchunk = (g.EW + g.DXC - 1) / g.DXC;
  const size_t pix = 2;  // staged as u16
  const int rows = p.re - p.rb;
  for (g.PX = kVariants[best].PX0, g.PY = kVariants[best].PY0;; ) {
    g.nbx = g.PX + g.q - (g.RR == 0 ? 1 : 0);
    g.nby = g.PY + g.q - (g.RR == 0 ? 1 : 0);
    g.nblk = g.nbx * g.nby;
    // row pitches: multiples of 4 pixels (8-byte cp.async rows) and, when nbx
    // allows it, the block row below starts where a 33rd block of the row would,
    // modulo the 128-byte bank period (s * pix * (pitch - nbx) = 0 mod 128), so
    // any 32 consecutive blocks read distinct banks
    const int per = 128 / std::gcd(128, (int)(s * pix));
    auto pitch_for = [&](int need) {
      need = (need + 3) & ~3;
      if (g.nbx % 4 == 0 && per % 4 == 0)
        return need + (((g.nbx - need) % per) + per) % per;
      return need;
    };
    g.RWp = pitch_for(g.nbx * s + 3);
    g.RHp = g.nby * s;
    g.TWp = pitch_for(g.nbx * s + g.nchunk * g.DXC + 3);  // phase A reads run DXC - 1 past a chunk start
    g.THp = g.RHp + 2 * p.R;
    auto al = [](size_t v) { return (v + 15) & ~(size_t)15; };
    g.off_tgt = al((size_t)g.RWp * g.RHp * pix);
    g.off_blk = al(g.off_tgt + (size_t)g.TWp * g.THp * pix);
    g.off_state = g.ws ? al(g.off_blk + (size_t)g.nblk * (4 * g.DXC + 1) * 4)  // one chunk buffer
                       : al(g.off_blk + (size_t)g.nblk * (4 * g.EW + 1) * 4);
    g.smem = g.off_state + (g.fuse ? (size_t)g.PX * g.PY * (g.ws ? 8 : sizeof(BsPoiState)) : 0);
    g.off_pos = al(g.smem);
    if (g.ws && g.fuse)  // window data of two dy rows: [2][PY][XW] x (1/sqrt(vg), Sg)
      g.smem = g.off_pos + 2 * (size_t)g.PY * ((g.PX - 1) * s + g.EW) * 8 + 4 * g.DXC;  // + the unused lanes' overrun
    // ws: at most one block per producer thread on each SM sub-partition
    // fused ws: the end-of-tile lane reduction reuses the block buffer
    const bool lanes_fit = !(g.ws && g.fuse) || (size_t)g.PX * g.PY * g.DXC * sizeof(BsLane) <=
                                                     (size_t)g.nblk * (4 * g.DXC + 1) * 4;
    if (g.smem <= smem_cap && lanes_fit && (!g.ws || (g.nblk + 3) / 4 <= 8 * g.npw)) break;
    if (g.PY > 2)
      g.PY /= 2;
    else if (g.PX > 4)
      g.PX /= 2;
    else
      return false;
  }
  // dy slices so that the grid covers the SMs several times (tail balance)
  const long tiles = (long)((p.lat.nx + g.PX - 1) / g.PX) * ((rows + g.PY - 1) / g.PY);
  g.nsplit = (int)std::min<long>(g.EW, std::max<long>(1, (4L * num_sms() + tiles - 1) / tiles));
  if (g.ws) {
    // whole waves: per CTA ~ (dy rows + staging) units, ceil(CTAs / SMs) waves
    double best_cost = 1e30;
    for (int ns = std::max(1, (int)((2L * num_sms() + tiles - 1) / tiles)); ns <= g.EW; ++ns) {
      const int per = (g.EW + ns - 1) / ns, ns2 = (g.EW + per - 1) / per;
      const double cost = (double)((tiles * ns2 + num_sms() - 1) / num_sms()) * (per + 0.7);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        g.nsplit = ns2;
      }
    }
  }
  if (const char* e = std::getenv("DICB200_BS_NSPLIT")) g.nsplit = std::max(1, std::min(g.EW, std::atoi(e)));
  g.dy_per = (g.EW + g.nsplit - 1) / g.nsplit;
  g.nsplit = (g.EW + g.dy_per - 1) / g.dy_per;
  return tiles > 0;
}

cudaError_t bs_merge_launch(const TcParams& p, const BsGeom& g, cudaStream_t st) {
  const size_t npoi = (size_t)(p.re - p.rb) * p.lat.nx;
  // scratch after the slice records: [n_flagged][flagged POIs][row arrivals x
  // kExactSlots][row partials x kExactSlots x kExactMaxWin] (bs_slices_bytes)
  int* n_flagged = reinterpret_cast<int*>(reinterpret_cast<BsSlice*>(p.slices) + npoi * g.nsplit);
  int* flagged = n_flagged + 1;
  int* arrivals = flagged + npoi;
  BestPartial* part = reinterpret_cast<BestPartial*>(
      (reinterpret_cast<uintptr_t>(arrivals + kExactSlots) + 15) & ~(uintptr_t)15);
  cudaError_t e = cudaMemsetAsync(n_flagged, 0, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(arrivals, 0, kExactSlots * sizeof(int), st);
  if (e != cudaSuccess) return e;
  bs_merge_kernel<<<(unsigned)((npoi + 255) / 256), 256, 0, st>>>(p, g.nsplit, flagged, n_flagged);
  count_launch();
  if (std::getenv("DICB200_BS_DEBUG")) {
    int nf = 0;
    cudaMemcpyAsync(&nf, n_flagged, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::vector<BsSlice> h(std::min<size_t>(npoi * g.nsplit, 64));
    cudaMemcpy(h.data(), p.slices, h.size() * sizeof(BsSlice), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[bs debug] flagged %d of %zu POIs (nsplit %d)\n", nf, npoi, g.nsplit);
    if (nf > 0) {  // the first flagged POIs' slices
      std::vector<int> fl(std::min(nf, 4));
      cudaMemcpy(fl.data(), flagged, fl.size() * sizeof(int), cudaMemcpyDeviceToHost);
      for (int k : fl) {
        std::vector<BsSlice> sl(g.nsplit);
        cudaMemcpy(sl.data(), reinterpret_cast<BsSlice*>(p.slices) + (size_t)k * g.nsplit, g.nsplit * sizeof(BsSlice),
                   cudaMemcpyDeviceToHost);
        for (int q = 0; q < g.nsplit; ++q)
          fprintf(stderr, "  flagged poi %d slice %d: a1 %.9g a2 %.9g cnt %d d (%d,%d)\n", k, q, sl[q].a1, sl[q].a2,
                  sl[q].cnt, sl[q].dx, sl[q].dy);
      }
    }
    for (size_t i = 0; i < h.size() && i < 16; ++i)
      fprintf(stderr, "  slice %zu: a1 %.9g a2 %.9g cnt %d d (%d,%d)\n", i, h[i].a1, h[i].a2, h[i].cnt, h[i].dx, h[i].dy);
  }
  // flagged POIs (near ties are rare: idle CTAs exit at once): a CTA per
  // (slot, displacement row), slots strided over 16 CTA rows; past
  // kExactSlots, one CTA per POI
  const int ew = 2 * p.R + 1;
  const bool rows_ok = ew <= 32 && p.side <= kExactMaxSide && p.side + ew - 1 <= kExactMaxWin;
  if (rows_ok) {
    const dim3 grid(ew, 16);
    if (p.planes == 1)
      bs_exact_rows_kernel<uint8_t><<<grid, 32 * kExactRowWarps, 0, st>>>(p, flagged, n_flagged, part, arrivals);
    else
      bs_exact_rows_kernel<uint16_t><<<grid, 32 * kExactRowWarps, 0, st>>>(p, flagged, n_flagged, part, arrivals);
    count_launch();
  }
  const unsigned ctas = (unsigned)std::min<size_t>(npoi, 148);
  if (p.planes == 1)
    bs_exact_kernel<uint8_t><<<ctas, 256, 0, st>>>(p, flagged, n_flagged, rows_ok ? kExactSlots : 0);
  else
    bs_exact_kernel<uint16_t><<<ctas, 256, 0, st>>>(p, flagged, n_flagged, rows_ok ? kExactSlots : 0);
  count_launch();
  return cudaGetLastError();
}

size_t bs_slices_bytes(size_t npoi, const BsGeom& g) {
  return npoi * (size_t)g.nsplit * sizeof(BsSlice) + (npoi + 1 + kExactSlots) * sizeof(int) + 16 +
         (size_t)kExactSlots * kExactMaxWin * sizeof(BestPartial);
}

template <int S, int RR, int Q, int DXC, int NPW, int NCW, int PYM>
cudaError_t launch_ws(const TcParams& p, const BsGeom& g, dim3 grid, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  auto go = [&](auto k) {
    e = set_dyn_smem(k, g.smem);
    if (e == cudaSuccess) k<<<grid, 32 * (NPW + NCW), g.smem, st>>>(p, g);
  };
  if (g.PY > PYM) return cudaErrorInvalidValue;
  // producer / staging variant: 1 (default) = direct accumulation + dedicated stager warps, 0 = round-2a kernel (A/B)
  static const int pv = std::getenv("DICB200_BS_PV") ? std::atoi(std::getenv("DICB200_BS_PV")) : 1;
  static const bool prof = std::getenv("DICB200_BS_PROF") != nullptr;
  if (p.planes == 1)
    g.fuse ? go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint8_t, true, PYM>) : go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint8_t>);
  else if (!g.fuse)
    go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint16_t>);
  else if (prof) {
    pv == 1 ? go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint16_t, true, PYM, 1, true>)
            : go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint16_t, true, PYM, 0, true>);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    unsigned long long h[8] = {0};
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h, g_bs_prof, sizeof(h));
    fprintf(stderr,
            "[bs prof] pv %d items %llu producer: compute %llu wait %llu store %llu | consumer: wait %llu phaseB %llu "
            "staging %llu (cycles, CTA (1,1,0))\n",
            pv, h[3], h[0], h[1], h[2], h[4], h[5], h[6]);
  } else
    pv == 1 ? go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint16_t, true, PYM, 1>)
            : go(bs_ws_kernel<S, RR, Q, DXC, NPW, NCW, uint16_t, true, PYM>);
  return e;
}

cudaError_t bs_launch(const TcParams& p, const BsGeom& g, cudaStream_t st) {
  const int rows = p.re - p.rb;
  dim3 grid((p.lat.nx + g.PX - 1) / g.PX, (rows + g.PY - 1) / g.PY, g.nsplit);
  cudaError_t e = cudaErrorInvalidValue;
  if (g.ws) {
    if (g.S == 10 && g.RR == 1 && g.q == 4 && g.DXC == 13 && g.npw == 8 && g.ncw == 8)
      e = launch_ws<10, 1, 4, 13, 8, 8, 12>(p, g, grid, st);
    if (g.S == 5 && g.RR == 1 && g.q == 8 && g.DXC == 11 && g.npw == 12 && g.ncw == 4)
      e = launch_ws<5, 1, 8, 11, 12, 4, 8>(p, g, grid, st);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  if (g.S == 10 && g.RR == 1 && g.q == 4 && g.DXC == 25) e = launch_variant<10, 1, 4, 25, 256, 1>(p, g, grid, st);
  if (g.S == 10 && g.RR == 1 && g.q == 3 && g.DXC == 31) e = launch_variant<10, 1, 3, 31, 256, 1>(p, g, grid, st);
  if (g.S == 5 && g.RR == 1 && g.q == 8 && g.DXC == 11) e = launch_variant<5, 1, 8, 11, 384, 1>(p, g, grid, st);
  if (g.S == 8 && g.RR == 7 && g.q == 3 && g.DXC == 41) e = launch_variant<8, 7, 3, 41, 256, 1>(p, g, grid, st);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dicb200
