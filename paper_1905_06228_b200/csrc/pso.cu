// K2 — particle-swarm integer search: pso_search / mpso_search
// (swarm_search, integer_search.cpp:107-201; star_best :205-225) with the
// per-subset std::mt19937_64 stream keyed by derive_stream_seed(seed, pair,
// subset) (rng.hpp:20-55, pipeline.cpp:84).
//
// Two stages. (1) The K1 BFS kernel writes each POI's full ZNCC surface over
// the +-R window (exact integer moments, fp64 finalisation — the very values
// a probe would return; NaN = degenerate target = "no result"). That costs
// ~3x the MACs of the distinct probes a swarm makes, but at the dense
// kernel's DP4A/IMAD efficiency instead of one serial probe at a time.
// (2) This kernel walks the swarm, ONE WARP PER POI, particles in lanes.
// The reference updates g_best asynchronously inside a generation
// (integer_search.cpp:128-137,165): particle i's velocity uses the g_best
// left by particles < i. Each round speculates every not-yet-committed
// particle from the current g_best (the RNG draws do not depend on it), finds
// by ballot the first particle whose star/probe result improves g_best (in
// the reference's improves() order), commits everything up to it, adopts its
// result as g_best, and re-speculates the rest. `evaluations` counts exactly
// the reference's memo misses: a visited bitmap marked only by committed
// probes (atomicOr returns whether the bit was new). Particle arithmetic is
// fp64 with explicit _rn intrinsics (no FMA), rounding is llround (half away
// from zero) as std::lround, clamps are std::clamp.
#include <cstdlib>

#include "common.cuh"
#include "pso.cuh"

namespace dicb200 {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kMaxPC = 4;  // particles per lane -> particle_count <= 128

struct Ctl {
  int mt_idx;
};

// ---------------------------------------------------------------- rng.hpp

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t derive_stream_seed(uint64_t master, uint64_t pair, uint64_t subset) {
  uint64_t s = mix64(master);
  s = mix64(s ^ (pair * 0xd6e8feb86659fd93ULL + 1));
  s = mix64(s ^ (subset * 0xa0761d6478bd642fULL + 1));
  return s;
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
  return c ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// std::mt19937_64 generation step, warp-parallel in three dependency phases.
__device__ void mt_twist_warp(uint64_t* mt) {
  const int lane = threadIdx.x & 31;
  uint64_t nv[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int i = lane + 32 * j;
    if (i < 156) nv[j] = mt_mix(mt[i], mt[i + 1], mt[i + 156]);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int i = lane + 32 * j;
    if (i < 156) mt[i] = nv[j];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int i = 156 + lane + 32 * j;
    if (i < 311) nv[j] = mt_mix(mt[i], mt[i + 1], mt[i - 156]);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int i = 156 + lane + 32 * j;
    if (i < 311) mt[i] = nv[j];
  }
  __syncwarp();
  if (lane == 0) mt[311] = mt_mix(mt[311], mt[0], mt[155]);
  __syncwarp();
}

// StreamRng::uniform01 (rng.hpp:38-40) x cnt, warp 0 only.
__device__ void draw_uniforms(uint64_t* mt, Ctl* ctl, double* out, int cnt) {
  const int lane = threadIdx.x & 31;
  int idx = ctl->mt_idx;
  int o = 0;
  while (o < cnt) {
    if (idx >= 312) {
      mt_twist_warp(mt);
      idx = 0;
    }
    const int k = min(cnt - o, 312 - idx);
    for (int j = lane; j < k; j += 32) out[o + j] = (double)(mt_temper(mt[idx + j]) >> 11) * 0x1.0p-53;
    idx += k;
    o += k;
  }
  __syncwarp();
  if (lane == 0) ctl->mt_idx = idx;
  __syncwarp();
}


__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

struct Win {
  int lo_dx, hi_dx, lo_dy, hi_dy, R, W;
  const double* surf;  // [W][W], entry (dy+R)*W + (dx+R): the warp's shared-memory copy
  __device__ __forceinline__ double val(int dx, int dy) const { return surf[(dy + R) * W + (dx + R)]; }
  __device__ __forceinline__ int pos(int dx, int dy) const { return (dy + R) * W + (dx + R); }
};

// evaluate_particle's probe set for a real position: round_clamp
// (integer_search.cpp:91-93) then star offsets clamped to the window (:205-225).
// Returns found; eff/c = star_best result (or the probe for plain PSO).
__device__ __forceinline__ bool star_eval(const Win& w, bool star, double x, double y, int& eff_dx, int& eff_dy,
                                          double& c) {
  const int dx = clampi((int)llround(x), w.lo_dx, w.hi_dx);
  const int dy = clampi((int)llround(y), w.lo_dy, w.hi_dy);
  eff_dx = dx;
  eff_dy = dy;
  if (!star) {
    c = w.val(dx, dy);
    return !isnan(c);
  }
  const int off[5][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  bool found = false;
  double best = -2.0;
#pragma unroll
  for (int o = 0; o < 5; ++o) {
    const int px = clampi(dx + off[o][0], w.lo_dx, w.hi_dx);
    const int py = clampi(dy + off[o][1], w.lo_dy, w.hi_dy);
    const double v = w.val(px, py);
    if (isnan(v)) continue;
    if (!found || improves(v, px, py, best, eff_dx, eff_dy)) {
      found = true;
      best = v;
      eff_dx = px;
      eff_dy = py;
    }
  }
  c = best;
  return found;
}

// Mark the committed particle's probes visited; returns how many were new
// (= the reference's memo misses for this evaluate_particle call).
__device__ __forceinline__ int commit_visits(const Win& w, bool star, double x, double y, uint32_t* visited) {
  const int dx = clampi((int)llround(x), w.lo_dx, w.hi_dx);
  const int dy = clampi((int)llround(y), w.lo_dy, w.hi_dy);
  const int np = star ? 5 : 1;
  const int off[5][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  int fresh = 0;
  for (int o = 0; o < np; ++o) {
    const int px = clampi(dx + off[o][0], w.lo_dx, w.hi_dx);
    const int py = clampi(dy + off[o][1], w.lo_dy, w.hi_dy);
    if (isnan(w.val(px, py))) continue;  // degenerate: "no result", not counted
    const int q = w.pos(px, py);
    const uint32_t bit = 1u << (q & 31);
    if (!(atomicOr(&visited[q >> 5], bit) & bit)) ++fresh;
  }
  return fresh;
}

__device__ void write_failure(dicb200_poi_record* rec, int cx, int cy, int status) {
  rec->x = cx;
  rec->y = cy;
  rec->u = 0.0;
  rec->v = 0.0;
  rec->zncc = __longlong_as_double(0x7ff8000000000000ULL);
  rec->converged = 0;
  rec->iterations = 0;
  rec->evaluations = 0;
  rec->update_evaluations = 0;
  rec->status = status;
  rec->integer_dx = 0;
  rec->integer_dy = 0;
  rec->pad = 0;
}

struct GBest {
  double c;
  int dx, dy, has;
};

template <int MINB>
__global__ void __launch_bounds__(32 * kWarpsPerCta, MINB) pso_walk_kernel(PsoParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerCta + warp;
  if (k >= p.n_records) return;
  // per-warp smem: mt[312] u64 | draws[4*P] double | visited[W*W/32] u32 | ctl | surface[W*W] double
  const int P = p.P;
  const int Wd = 2 * p.R + 1;
  const int nvis = (Wd * Wd + 31) / 32;
  const size_t head = ((312 * 8 + 4 * (size_t)(P > 0 ? P : 1) * 8 + (size_t)nvis * 4 + sizeof(Ctl)) + 15) & ~size_t(15);
  const size_t per_warp = head + (p.stage_surface ? (size_t)Wd * Wd * 8 : 0);
  unsigned char* base = smem_raw + per_warp * warp;
  uint64_t* mt = reinterpret_cast<uint64_t*>(base);
  double* draws = reinterpret_cast<double*>(base + 312 * 8);
  uint32_t* visited = reinterpret_cast<uint32_t*>(base + 312 * 8 + 4 * (size_t)(P > 0 ? P : 1) * 8);
  Ctl* ctl = reinterpret_cast<Ctl*>(base + 312 * 8 + 4 * (size_t)(P > 0 ? P : 1) * 8 + (size_t)nvis * 4);

  dicb200_poi_record* rec = p.rec + k;
  const int iy = p.row_begin + k / p.lat.nx, ix = k % p.lat.nx;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy);
  const uint64_t subset_index = (uint64_t)iy * p.lat.nx + ix;
  const int M = p.M;
  if (P < 1 || p.G < 1 || P > 32 * kMaxPC) {  // integer_search.cpp:110-111
    if (lane == 0) write_failure(rec, cx, cy, DICB200_POI_INVALID_SWARM);
    return;
  }
  Win w;
  w.R = p.R;
  w.W = Wd;
  w.lo_dx = max(-p.R, M - cx);  // feasible_window, integer_search.cpp:11-21
  w.hi_dx = min(p.R, p.tgt.width - 1 - M - cx);
  w.lo_dy = max(-p.R, M - cy);
  w.hi_dy = min(p.R, p.tgt.height - 1 - M - cy);
  if (w.lo_dx > w.hi_dx || w.lo_dy > w.hi_dy) {
    if (lane == 0) write_failure(rec, cx, cy, DICB200_POI_NO_VALID_POSITION);
    return;
  }
  w.surf = p.surface + (size_t)k * Wd * Wd;
  if (p.stage_surface) {  // the POI's ZNCC surface, staged once: every swarm probe then reads shared memory
    double* ss = reinterpret_cast<double*>(base + head);
    for (int i = lane; i < Wd * Wd; i += 32) ss[i] = __ldg(w.surf + i);
    w.surf = ss;
  }
  for (int i = lane; i < nvis; i += 32) visited[i] = 0u;
  if (lane == 0) {
    // std::mt19937_64 seeding (StreamRng(derive_stream_seed(...)), pipeline.cpp:84)
    uint64_t x = derive_stream_seed(p.seed, p.pair_index, subset_index);
    mt[0] = x;
    for (int i = 1; i < 312; ++i) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + (uint64_t)i;
      mt[i] = x;
    }
    ctl->mt_idx = 312;
  }
  __syncwarp();
  const int PC = (P + 31) / 32;
  const bool star = p.star;
  const double dlo_x = w.lo_dx, dhi_x = w.hi_dx, dlo_y = w.lo_dy, dhi_y = w.hi_dy;
  const double vspan = p.R / 2.0;

  // particle state: lane owns particles lane + 32*c
  double X[kMaxPC], Y[kMaxPC], VX[kMaxPC], VY[kMaxPC], BC[kMaxPC];
  int BDX[kMaxPC], BDY[kMaxPC], HB[kMaxPC];
  draw_uniforms(mt, ctl, draws, 4 * P);  // init: x, y, vx, vy per particle (integer_search.cpp:117-122)
#pragma unroll
  for (int c = 0; c < kMaxPC; ++c) {
    const int i = lane + 32 * c;
    X[c] = Y[c] = VX[c] = VY[c] = 0.0;
    BC[c] = -2.0;
    BDX[c] = BDY[c] = 0;
    HB[c] = 0;
    if (c < PC && i < P) {
      X[c] = __dadd_rn(dlo_x, __dmul_rn(__dsub_rn(dhi_x, dlo_x), draws[4 * i + 0]));
      Y[c] = __dadd_rn(dlo_y, __dmul_rn(__dsub_rn(dhi_y, dlo_y), draws[4 * i + 1]));
      VX[c] = __dadd_rn(-vspan, __dmul_rn(__dsub_rn(vspan, -vspan), draws[4 * i + 2]));
      VY[c] = __dadd_rn(-vspan, __dmul_rn(__dsub_rn(vspan, -vspan), draws[4 * i + 3]));
    }
  }
  // ---- init sweep: positions do not depend on g_best -> all particles commit ----
  GBest g = {-2.0, 0, 0, 0};
  long long misses = 0;
  {
    int fresh = 0;
#pragma unroll
    for (int c = 0; c < kMaxPC; ++c) {
      const int i = lane + 32 * c;
      if (c < PC && i < P) {
        int ex, ey;
        double cv;
        if (star_eval(w, star, X[c], Y[c], ex, ey, cv)) {
          fresh += commit_visits(w, star, X[c], Y[c], visited);
          if (star) {
            X[c] = ex;
            Y[c] = ey;
          }
          HB[c] = 1;
          BC[c] = cv;
          BDX[c] = ex;
          BDY[c] = ey;
        }
      }
    }
    // sequential offers == argmax in improves() order
#pragma unroll
    for (int c = 0; c < kMaxPC; ++c) {
      double bc = HB[c] ? BC[c] : -3.0;
      int bx = BDX[c], by = BDY[c], bh = HB[c];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const int ox = __shfl_xor_sync(0xffffffffu, bx, o), oy = __shfl_xor_sync(0xffffffffu, by, o),
                  oh = __shfl_xor_sync(0xffffffffu, bh, o);
        if (oh && (!bh || improves(oc, ox, oy, bc, bx, by))) {
          bc = oc;
          bx = ox;
          by = oy;
          bh = 1;
        }
      }
      if (bh && (!g.has || improves(bc, bx, by, g.c, g.dx, g.dy))) {
        g.c = bc;
        g.dx = bx;
        g.dy = by;
        g.has = 1;
      }
    }
    for (int o = 16; o; o >>= 1) fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
    misses += fresh;
  }
  if (!g.has) {  // integer_search.cpp:169
    if (lane == 0) write_failure(rec, cx, cy, DICB200_POI_ALL_DEGENERATE);
    return;
  }
  const long long init_misses = misses;

  if (g.c < p.stop) {
    for (int t = 0; t < p.G; ++t) {
      const double wgt = p.inertia_constant
                             ? p.w_const
                             : __dsub_rn(0.9, __ddiv_rn((double)t, __dmul_rn(2.0, (double)p.G)));  // :35-37
      draw_uniforms(mt, ctl, draws, 4 * P);  // r1x, r2x, r1y, r2y per particle (:180-181)
      int start = 0;
      while (start < P) {
        // speculate every particle >= start from the current g_best
        double nX[kMaxPC], nY[kMaxPC], nVX[kMaxPC], nVY[kMaxPC], rc[kMaxPC];
        int rx[kMaxPC], ry[kMaxPC], rok[kMaxPC];
        int first = P;  // first particle (>= start) whose result improves g_best
#pragma unroll
        for (int c = 0; c < kMaxPC; ++c) {
          const int i = lane + 32 * c;
          rok[c] = 0;
          nX[c] = X[c];
          nY[c] = Y[c];
          nVX[c] = VX[c];
          nVY[c] = VY[c];
          rc[c] = -2.0;
          rx[c] = ry[c] = 0;
          bool improving = false;
          if (c < PC && i < P && i >= start) {
            const double r1x = draws[4 * i], r2x = draws[4 * i + 1], r1y = draws[4 * i + 2], r2y = draws[4 * i + 3];
            // integer_search.cpp:182-187
            nVX[c] = __dadd_rn(__dadd_rn(__dmul_rn(wgt, VX[c]), __dmul_rn(__dmul_rn(p.c1, r1x), __dsub_rn((double)BDX[c], X[c]))),
                               __dmul_rn(__dmul_rn(p.c2, r2x), __dsub_rn((double)g.dx, X[c])));
            nVY[c] = __dadd_rn(__dadd_rn(__dmul_rn(wgt, VY[c]), __dmul_rn(__dmul_rn(p.c1, r1y), __dsub_rn((double)BDY[c], Y[c]))),
                               __dmul_rn(__dmul_rn(p.c2, r2y), __dsub_rn((double)g.dy, Y[c])));
            nX[c] = clampd(__dadd_rn(X[c], nVX[c]), dlo_x, dhi_x);
            nY[c] = clampd(__dadd_rn(Y[c], nVY[c]), dlo_y, dhi_y);
            int ex, ey;
            double cv;
            rok[c] = star_eval(w, star, nX[c], nY[c], ex, ey, cv);
            rc[c] = cv;
            rx[c] = ex;
            ry[c] = ey;
            improving = rok[c] && improves(cv, ex, ey, g.c, g.dx, g.dy);
          }
          const unsigned bal = __ballot_sync(0xffffffffu, improving);
          if (bal && first == P) first = 32 * c + (__ffs(bal) - 1);
        }
        const int last = first < P ? first : P - 1;  // commit [start, last]
        int fresh = 0;
#pragma unroll
        for (int c = 0; c < kMaxPC; ++c) {
          const int i = lane + 32 * c;
          if (c < PC && i >= start && i <= last) {
            X[c] = nX[c];
            Y[c] = nY[c];
            VX[c] = nVX[c];
            VY[c] = nVY[c];
            if (rok[c]) {
              fresh += commit_visits(w, star, X[c], Y[c], visited);
              if (star) {
                X[c] = rx[c];  // the descent step repositions the particle (:155-158)
                Y[c] = ry[c];
              }
              if (!HB[c] || improves(rc[c], rx[c], ry[c], BC[c], BDX[c], BDY[c])) {
                HB[c] = 1;
                BC[c] = rc[c];
                BDX[c] = rx[c];
                BDY[c] = ry[c];
              }
            }
          }
        }
        for (int o = 16; o; o >>= 1) fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
        misses += fresh;
        if (first < P) {  // adopt the improving particle's result as g_best
          const int src = first & 31, cc = first >> 5;
          double bc = 0.0;
          int bx = 0, by = 0;
#pragma unroll
          for (int c = 0; c < kMaxPC; ++c)
            if (c == cc) {
              bc = rc[c];
              bx = rx[c];
              by = ry[c];
            }
          g.c = __shfl_sync(0xffffffffu, bc, src);
          g.dx = __shfl_sync(0xffffffffu, bx, src);
          g.dy = __shfl_sync(0xffffffffu, by, src);
        }
        start = last + 1;
      }
      if (g.c >= p.stop) break;  // integer_search.cpp:191
    }
  }
  if (lane == 0) {
    rec->x = cx;
    rec->y = cy;
    rec->u = (double)g.dx;
    rec->v = (double)g.dy;
    rec->zncc = g.c;
    rec->converged = p.subpixel_none ? 1 : 0;
    rec->iterations = 0;
    rec->evaluations = misses;
    rec->update_evaluations = misses - init_misses;
    rec->status = DICB200_POI_OK;
    rec->integer_dx = g.dx;
    rec->integer_dy = g.dy;
    rec->pad = 0;
  }
}

}  // namespace

size_t pso_walk_smem(const PsoParams& p) {
  const int P = p.P > 0 ? p.P : 1;
  const int Wd = 2 * p.R + 1;
  const size_t head = ((312 * 8 + 4 * (size_t)P * 8 + (size_t)((Wd * Wd + 31) / 32) * 4 + sizeof(Ctl)) + 15) & ~size_t(15);
  return (head + (p.stage_surface ? (size_t)Wd * Wd * 8 : 0)) * kWarpsPerCta;
}

dicb200_status pso_walk_launch(PsoParams& p, cudaStream_t st) {
  if (p.n_records <= 0) return DICB200_OK;
  p.stage_surface = 1;  // the surfaces in shared memory when they fit, else read through L1/L2
  if (pso_walk_smem(p) > 200 * 1024) p.stage_surface = 0;
  const size_t smem = pso_walk_smem(p);
  if (smem > 200 * 1024) {
    set_error("particle_count / search window too large for the swarm walk kernel");
    return DICB200_ERR_INVALID;
  }
  cudaError_t e;
  auto go = [&](auto k) {
    e = set_dyn_smem(k, smem);
    if (e == cudaSuccess) {
      k<<<(p.n_records + kWarpsPerCta - 1) / kWarpsPerCta, 32 * kWarpsPerCta, smem, st>>>(p);
      e = cudaGetLastError();
    }
  };
  // 3 CTAs/SM (C3: <= 170 registers without spills, 3 x 67 KB of staged
  // surfaces). Measured and dropped: 128 registers for 4 CTAs/SM with the
  // surfaces read through L1/L2 (spills; no gain), and the row chunks' walks
  // and refinements forked onto a second stream (C3 7.43 -> 7.46 M subsets/s:
  // within noise, the per-chunk search setup eats the overlap)
  go(pso_walk_kernel<3>);
  count_launch();
  if (e != cudaSuccess) return cuda_fail(e, "pso_walk_kernel", __FILE__, __LINE__);
  return DICB200_OK;
}

}  // namespace dicb200
