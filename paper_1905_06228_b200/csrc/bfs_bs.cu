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

#include "bfs.cuh"

namespace dicb200 {

namespace {

// 8-byte global -> shared async copy; bytes past src_bytes (0..8) are zero-filled.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}

template <int S, int RR, int Q, int DXC, int NT, int MINB, typename Pix>
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
  // ---- stage the reference blocks and the target rows of this dy slice (0 outside).
  // u16 images: 8-byte cp.async from 4-pixel-aligned global columns (zero-filled
  // past the borders); the staged rows then start `sh` pixels before the region.
  int shR = 0, shT = 0;
  if (sizeof(Pix) == 2 && g.async_ok) {
    shR = RX0 & 3;
    shT = TX0 & 3;
    const int XR = RX0 - shR, XT = TX0 - shT;
    const uint16_t* ref = static_cast<const uint16_t*>(p.ref.data);
    const int cr = (shR + g.nbx * S + 3) / 4;  // 4-pixel chunks per staged row
    for (int i = threadIdx.x; i < g.RHp * cr; i += NT) {
      const int y = i / cr, c = i - y * cr, gy = RY0 + y, gx = XR + 4 * c;
      const int valid = (gy >= 0 && gy < p.ref.height && gx >= 0) ? max(0, min(4, p.ref.width - gx)) : 0;
      const uint16_t* src = valid ? ref + (size_t)gy * p.ref.pitch + gx : ref;
      cp_async8(Rf + y * RP + 4 * c, src, 2 * valid);
    }
    const uint16_t* tgt = static_cast<const uint16_t*>(p.tgt.data);
    const int ct = (shT + g.nbx * S + g.nchunk * DXC + 3) / 4;
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
    const int w = g.nbx * S;
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
    const int tw = w + g.nchunk * DXC;  // columns read by phase A (dx past R: zero)
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
  __syncthreads();
  const int nx_here = min(g.PX, p.lat.nx - ix0), ny_here = min(g.PY, p.re - iy0);
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
}

// Instantiations: (s, r, DXC, threads). A configuration runs on the block-sum
// kernel when one of them matches its lattice spacing and remainder.
struct BsVariant {
  int S, RR, Q, DXC, NT, MINB;  // MINB: CTAs per SM the variant is sized for (shared memory, registers)
};
constexpr BsVariant kVariants[] = {
    {10, 1, 4, 25, 256, 1},  // c5: L 41, s 10, R 12
    {10, 1, 3, 31, 256, 1},  // c2: L 31, s 10, R 15
    {5, 1, 8, 11, 384, 1},   // c4: L 41, s 5, R 5
    {8, 7, 3, 41, 256, 1},   // c3: L 31, s 8, R 20
};
// Measured and dropped (C5, B200): two CTAs per SM with dx chunks of 13 / 9
// (127 registers, 16 x 4 POI tiles to fit 110 KB): 0.93 / 0.98 ms against
// 0.57 ms for {10, 1, 4, 25, 256, 1} — the taller halo and the per-chunk
// target reloads cost more than the second CTA's latency hiding recovers.

template <int S, int RR, int Q, int DXC, int NT, int MINB>
cudaError_t launch_variant(const TcParams& p, const BsGeom& g, dim3 grid, cudaStream_t st) {
  cudaError_t e;
  if (p.planes == 1) {
    auto k = bs_kernel<S, RR, Q, DXC, NT, MINB, uint8_t>;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e == cudaSuccess) k<<<grid, NT, g.smem, st>>>(p, g);
  } else {
    auto k = bs_kernel<S, RR, Q, DXC, NT, MINB, uint16_t>;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e == cudaSuccess) k<<<grid, NT, g.smem, st>>>(p, g);
  }
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
  for (int v = 0; v < nvar; ++v) {
    if (kVariants[v].S != s || kVariants[v].RR != g.RR || kVariants[v].Q != g.q) continue;
    if (force ? v != std::atoi(force) : kVariants[v].MINB != 1) continue;
    const int nch = (g.EW + kVariants[v].DXC - 1) / kVariants[v].DXC;
    const int w = nch * kVariants[v].DXC - g.EW;
    if (w < waste) {
      waste = w;
      best = v;
    }
  }
  if (best < 0) return false;
  g.async_ok = p.planes == 2 && ((uintptr_t)p.ref.data % 8) == 0 && ((uintptr_t)p.tgt.data % 8) == 0 &&
               (p.ref.pitch % 4) == 0 && (p.tgt.pitch % 4) == 0;
  g.DXC = kVariants[best].DXC;
  g.threads = kVariants[best].NT;
  g.minb = kVariants[best].MINB;
  const size_t smem_cap = g.minb > 1 ? (size_t)(227 * 1024 / g.minb - 1024) : (size_t)220 * 1024;
  g.nchunk = (g.EW + g.DXC - 1) / g.DXC;
  const size_t pix = 2;  // staged as u16
  const int rows = p.re - p.rb;
  for (g.PX = 16, g.PY = 8;; ) {
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
    g.smem = g.off_blk + (size_t)g.nblk * (4 * g.EW + 1) * 4;
    if (g.smem <= smem_cap) break;
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
  g.dy_per = (g.EW + g.nsplit - 1) / g.nsplit;
  g.nsplit = (g.EW + g.dy_per - 1) / g.dy_per;
  return tiles > 0;
}

cudaError_t bs_launch(const TcParams& p, const BsGeom& g, cudaStream_t st) {
  const int rows = p.re - p.rb;
  dim3 grid((p.lat.nx + g.PX - 1) / g.PX, (rows + g.PY - 1) / g.PY, g.nsplit);
  cudaError_t e = cudaErrorInvalidValue;
  if (g.S == 10 && g.RR == 1 && g.q == 4 && g.DXC == 25) e = launch_variant<10, 1, 4, 25, 256, 1>(p, g, grid, st);
  if (g.S == 10 && g.RR == 1 && g.q == 3 && g.DXC == 31) e = launch_variant<10, 1, 3, 31, 256, 1>(p, g, grid, st);
  if (g.S == 5 && g.RR == 1 && g.q == 8 && g.DXC == 11) e = launch_variant<5, 1, 8, 11, 384, 1>(p, g, grid, st);
  if (g.S == 8 && g.RR == 7 && g.q == 3 && g.DXC == 41) e = launch_variant<8, 7, 3, 41, 256, 1>(p, g, grid, st);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dicb200
