// K2 — particle-swarm integer search: pso_search / mpso_search
// (swarm_search, integer_search.cpp:107-201; star_best :205-225) with the
// per-subset std::mt19937_64 stream keyed by derive_stream_seed(seed, pair,
// subset) (rng.hpp:20-55, pipeline.cpp:84).
//
// One CTA (4 warps) per POI. The feasible window's target region and the
// reference subset live in shared memory; a probe is one warp computing the
// exact integer moments (Sfg, Sg, Sgg) — u8 with __dp4a over byte-shifted
// words, u16 with IMAD — and the same fp64 ZNCC finalisation as K1, so every
// value equals the BFS kernel's bit-for-bit.
//
// The reference updates g_best asynchronously inside a generation
// (integer_search.cpp:128-137,165), so particle i depends on particles < i.
// Speculate-and-replay: all not-yet-replayed particles compute their velocity
// / position update in parallel from the CURRENT g_best (the RNG draws do not
// depend on it), their probes are evaluated in parallel into a value cache,
// then one thread replays particles in order, accepting each speculation whose
// g_best matches and re-speculating from the first that does not.
// `evaluations` counts only probes the reference itself would have made
// (a visited bit per window position, separate from the speculative cache);
// all particle arithmetic is fp64 with explicit _rn intrinsics (no FMA), and
// rounding is llround (half away from zero) as std::lround.
#include "common.cuh"
#include "pso.cuh"

namespace dicb200 {

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

struct Particle {
  double x, y, vx, vy, best_c;
  int best_dx, best_dy, has_best, pad;
};

struct Spec {
  double x, y, vx, vy;
  int gdx, gdy;
  int px[5], py[5];
};

struct Ctl {
  int mt_idx;
  int n_req;
  int start;
  int g_dx, g_dy, has_g;
  double g_c;
  long long misses;
  long long init_misses;
  int status;
  int lo_dx, hi_dx, lo_dy, hi_dy, wx, wy;
  long long sf;
  double sqrt_vf;
};

enum : uint32_t { F_CACHED = 1u, F_DEGEN = 2u, F_VISITED = 4u, F_REQ = 8u };

struct Layout {
  size_t ctl, mt, draws, parts, spec, req, flags, vals, F, region, total;
};

__host__ __device__ inline Layout pso_layout(int P, int wmax, int M, int u8, int region_pitch, int QP) {
  Layout L;
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = (off + 15) & ~size_t(15);
    off = o + b;
    return o;
  };
  const int side = 2 * M + 1;
  L.ctl = take(sizeof(Ctl));
  L.mt = take(312 * 8);
  L.draws = take((size_t)4 * P * 8);
  L.parts = take((size_t)P * sizeof(Particle));
  L.spec = take((size_t)P * sizeof(Spec));
  L.req = take((size_t)5 * P * 4);
  L.flags = take((size_t)wmax * wmax * 4);
  L.vals = take((size_t)wmax * wmax * 8);
  L.F = take(u8 ? (size_t)side * QP * 4 : (size_t)side * side * 2);
  L.region = take((size_t)(wmax + 2 * M) * region_pitch * (u8 ? 1 : 2));
  L.total = (off + 15) & ~size_t(15);
  return L;
}

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

// ------------------------------------------------------------ correlation

// Exact moments of one probe (warp-cooperative); returns zncc or flags degenerate.
template <bool kU8>
__device__ bool probe_zncc(const unsigned char* smem, const Layout& L, const Ctl* ctl, int M, int region_pitch,
                           int QP, int dx, int dy, double& c) {
  const int lane = threadIdx.x & 31;
  const int side = 2 * M + 1;
  const int ox = dx - ctl->lo_dx, oy = dy - ctl->lo_dy;
  uint64_t sfg = 0, sgg = 0;
  uint32_t sg = 0;
  if constexpr (kU8) {
    const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + L.F);
    const uint32_t* R32 = reinterpret_cast<const uint32_t*>(smem + L.region);
    const int rem = side - 4 * (QP - 1);  // valid bytes in the last word (1..4)
    const uint32_t lastmask = rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
    uint32_t a_fg = 0, a_g = 0, a_gg = 0;
    const int total = side * QP;
    int r = lane / QP, q = lane - (lane / QP) * QP;
    const int dr = 32 / QP, dq = 32 - dr * QP;
    for (int w = lane; w < total; w += 32) {
      const int off = (oy + r) * region_pitch + ox + 4 * q;
      const uint32_t lo = R32[off >> 2], hi = R32[(off >> 2) + 1];
      uint32_t gw = __byte_perm(lo, hi, 0x3210 + 0x1111 * (off & 3));
      if (q == QP - 1) gw &= lastmask;
      a_fg = __dp4a(F[w], gw, a_fg);
      a_g = __dp4a(gw, 0x01010101u, a_g);
      a_gg = __dp4a(gw, gw, a_gg);
      r += dr;
      q += dq;
      if (q >= QP) {
        q -= QP;
        ++r;
      }
    }
    sfg = a_fg;
    sg = a_g;
    sgg = a_gg;
  } else {
    const uint16_t* F = reinterpret_cast<const uint16_t*>(smem + L.F);
    const uint16_t* R16 = reinterpret_cast<const uint16_t*>(smem + L.region);
    const int total = side * side;
    int r = lane / side, cc = lane - (lane / side) * side;
    const int dr = 32 / side, dc = 32 - dr * side;
    for (int e = lane; e < total; e += 32) {
      const uint32_t f = F[e];
      const uint32_t g = R16[(oy + r) * region_pitch + ox + cc];
      sfg += (uint64_t)(f * g);
      sg += g;
      sgg += (uint64_t)(g * g);
      r += dr;
      cc += dc;
      if (cc >= side) {
        cc -= side;
        ++r;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sfg += __shfl_xor_sync(0xffffffffu, sfg, o);
    sg += __shfl_xor_sync(0xffffffffu, sg, o);
    sgg += __shfl_xor_sync(0xffffffffu, sgg, o);
  }
  const int64_t n = (int64_t)side * side;
  const int64_t vg = n * (int64_t)sgg - (int64_t)sg * (int64_t)sg;
  if (vg <= 0 || ctl->sqrt_vf <= 0.0) return false;
  c = zncc_from_moments(n, (int64_t)sfg, ctl->sf, (int64_t)sg, (int64_t)sgg, ctl->sqrt_vf);
  return true;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// positions probed by evaluate_particle for a (real) particle position
__device__ __forceinline__ void probe_positions(Spec& s, const Ctl* ctl, int star) {
  const int dx = clampi((int)llround(s.x), ctl->lo_dx, ctl->hi_dx);  // round_clamp, integer_search.cpp:91-93
  const int dy = clampi((int)llround(s.y), ctl->lo_dy, ctl->hi_dy);
  if (!star) {
    s.px[0] = dx;
    s.py[0] = dy;
    return;
  }
  const int off[5][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}};
#pragma unroll
  for (int o = 0; o < 5; ++o) {
    s.px[o] = clampi(dx + off[o][0], ctl->lo_dx, ctl->hi_dx);
    s.py[o] = clampi(dy + off[o][1], ctl->lo_dy, ctl->hi_dy);
  }
}

__device__ __forceinline__ void request(uint32_t* flags, int* req, Ctl* ctl, int pos) {
  if (flags[pos] & (F_CACHED | F_REQ)) return;
  const uint32_t old = atomicOr(&flags[pos], F_REQ);
  if (old & (F_CACHED | F_REQ)) return;
  const int i = atomicAdd(&ctl->n_req, 1);
  req[i] = pos;
}

// evaluate_particle (integer_search.cpp:139-166) against the value cache.
__device__ void apply_particle(Particle& P, const Spec& s, uint32_t* flags, const double* vals, Ctl* ctl, int star) {
  P.x = s.x;
  P.y = s.y;
  P.vx = s.vx;
  P.vy = s.vy;
  const int np = star ? 5 : 1;
  int eff_dx = s.px[0], eff_dy = s.py[0];
  double best_c = -2.0;
  bool found = false;
  for (int o = 0; o < np; ++o) {
    const int pos = (s.py[o] - ctl->lo_dy) * ctl->wx + (s.px[o] - ctl->lo_dx);
    const uint32_t f = flags[pos];
    if (f & F_DEGEN) continue;  // probe(): "no result", not counted
    if (!(f & F_VISITED)) {     // memo miss = one evaluation
      flags[pos] = f | F_VISITED;
      ctl->misses++;
    }
    const double c = vals[pos];
    if (!found || improves(c, s.px[o], s.py[o], best_c, eff_dx, eff_dy)) {
      found = true;
      best_c = c;
      eff_dx = s.px[o];
      eff_dy = s.py[o];
    }
  }
  if (!found) return;
  if (star) {
    P.x = eff_dx;
    P.y = eff_dy;
  }
  if (!P.has_best || improves(best_c, eff_dx, eff_dy, P.best_c, P.best_dx, P.best_dy)) {
    P.has_best = 1;
    P.best_c = best_c;
    P.best_dx = eff_dx;
    P.best_dy = eff_dy;
  }
  if (!ctl->has_g || improves(best_c, eff_dx, eff_dy, ctl->g_c, ctl->g_dx, ctl->g_dy)) {
    ctl->has_g = 1;
    ctl->g_c = best_c;
    ctl->g_dx = eff_dx;
    ctl->g_dy = eff_dy;
  }
}

template <bool kU8>
__device__ void evaluate_requests(unsigned char* smem, const Layout& L, Ctl* ctl, const PsoParams& p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* req = reinterpret_cast<const int*>(smem + L.req);
  uint32_t* flags = reinterpret_cast<uint32_t*>(smem + L.flags);
  double* vals = reinterpret_cast<double*>(smem + L.vals);
  const int nreq = ctl->n_req;
  for (int i = warp; i < nreq; i += kWarps) {
    const int pos = req[i];
    const int dy = pos / ctl->wx + ctl->lo_dy, dx = pos % ctl->wx + ctl->lo_dx;
    double c = 0.0;
    const bool ok = probe_zncc<kU8>(smem, L, ctl, p.M, p.region_pitch, p.QP, dx, dy, c);
    if (lane == 0) {
      vals[pos] = c;
      flags[pos] = (flags[pos] & ~F_REQ) | F_CACHED | (ok ? 0u : F_DEGEN);
    }
  }
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

template <bool kU8>
__global__ void __launch_bounds__(kThreads) pso_kernel(PsoParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int k = blockIdx.x;
  if (k >= p.n_records) return;
  dicb200_poi_record* rec = p.rec + k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int iy = p.row_begin + k / p.lat.nx, ix = k % p.lat.nx;
  const int cx = p.lat.cx(ix), cy = p.lat.cy(iy);
  const uint64_t subset_index = (uint64_t)iy * p.lat.nx + ix;
  const int M = p.M, side = 2 * M + 1;
  const int W = p.tgt.width, H = p.tgt.height;

  if (p.P < 1 || p.G < 1) {  // integer_search.cpp:110-111
    if (tid == 0) write_failure(rec, cx, cy, DICB200_POI_INVALID_SWARM);
    return;
  }
  const int lo_dx = max(-p.R, M - cx), hi_dx = min(p.R, W - 1 - M - cx);  // feasible_window
  const int lo_dy = max(-p.R, M - cy), hi_dy = min(p.R, H - 1 - M - cy);
  if (lo_dx > hi_dx || lo_dy > hi_dy) {
    if (tid == 0) write_failure(rec, cx, cy, DICB200_POI_NO_VALID_POSITION);
    return;
  }
  const Layout L = pso_layout(p.P, p.wmax, M, p.u8, p.region_pitch, p.QP);
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + L.ctl);
  uint64_t* mt = reinterpret_cast<uint64_t*>(smem + L.mt);
  double* draws = reinterpret_cast<double*>(smem + L.draws);
  Particle* parts = reinterpret_cast<Particle*>(smem + L.parts);
  Spec* spec = reinterpret_cast<Spec*>(smem + L.spec);
  int* req = reinterpret_cast<int*>(smem + L.req);
  uint32_t* flags = reinterpret_cast<uint32_t*>(smem + L.flags);
  double* vals = reinterpret_cast<double*>(smem + L.vals);
  const int wx = hi_dx - lo_dx + 1, wy = hi_dy - lo_dy + 1;

  // ---- stage reference subset, target region, flags ----
  if constexpr (kU8) {
    uint32_t* F = reinterpret_cast<uint32_t*>(smem + L.F);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.ref.data);
    for (int i = tid; i < side * p.QP; i += kThreads) {
      const int r = i / p.QP, q = i - r * p.QP;
      const uint8_t* row = src + (size_t)(cy - M + r) * p.ref.pitch + (cx - M);
      uint32_t w = 0;
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < side) w |= (uint32_t)row[4 * q + e] << (8 * e);
      F[i] = w;
    }
    uint8_t* Rg = smem + L.region;
    const uint8_t* tsrc = reinterpret_cast<const uint8_t*>(p.tgt.data);
    const int rows = wy + 2 * M, cols = wx + 2 * M;
    for (int i = tid; i < rows * p.region_pitch; i += kThreads) {
      const int r = i / p.region_pitch, c = i - r * p.region_pitch;
      Rg[i] = c < cols ? tsrc[(size_t)(cy + lo_dy - M + r) * p.tgt.pitch + (cx + lo_dx - M + c)] : 0;
    }
  } else {
    uint16_t* F = reinterpret_cast<uint16_t*>(smem + L.F);
    const uint16_t* src = reinterpret_cast<const uint16_t*>(p.ref.data);
    for (int i = tid; i < side * side; i += kThreads) {
      const int r = i / side, c = i - r * side;
      F[i] = src[(size_t)(cy - M + r) * p.ref.pitch + (cx - M + c)];
    }
    uint16_t* Rg = reinterpret_cast<uint16_t*>(smem + L.region);
    const uint16_t* tsrc = reinterpret_cast<const uint16_t*>(p.tgt.data);
    const int rows = wy + 2 * M, cols = wx + 2 * M;
    for (int i = tid; i < rows * p.region_pitch; i += kThreads) {
      const int r = i / p.region_pitch, c = i - r * p.region_pitch;
      Rg[i] = c < cols ? tsrc[(size_t)(cy + lo_dy - M + r) * p.tgt.pitch + (cx + lo_dx - M + c)] : 0;
    }
  }
  for (int i = tid; i < wx * wy; i += kThreads) flags[i] = 0u;
  if (tid == 0) {
    ctl->lo_dx = lo_dx;
    ctl->hi_dx = hi_dx;
    ctl->lo_dy = lo_dy;
    ctl->hi_dy = hi_dy;
    ctl->wx = wx;
    ctl->wy = wy;
    ctl->n_req = 0;
    ctl->start = 0;
    ctl->has_g = 0;
    ctl->g_c = -2.0;
    ctl->g_dx = ctl->g_dy = 0;
    ctl->misses = 0;
    ctl->status = DICB200_POI_OK;
    // std::mt19937_64 seeding (StreamRng(derive_stream_seed(...)), pipeline.cpp:84)
    uint64_t x = derive_stream_seed(p.seed, p.pair_index, subset_index);
    mt[0] = x;
    for (int i = 1; i < 312; ++i) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + (uint64_t)i;
      mt[i] = x;
    }
    ctl->mt_idx = 312;
  }
  __syncthreads();
  // reference moments (subset_stats): exact
  if (warp == 0) {
    uint64_t sf = 0, sff = 0;
    for (int e = lane; e < side * side; e += 32) {
      const int r = e / side, c = e - r * side;
      uint32_t f;
      if constexpr (kU8) {
        const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + L.F);
        f = (F[r * p.QP + (c >> 2)] >> (8 * (c & 3))) & 0xffu;
      } else {
        f = reinterpret_cast<const uint16_t*>(smem + L.F)[e];
      }
      sf += f;
      sff += (uint64_t)f * f;
    }
    for (int o = 16; o; o >>= 1) {
      sf += __shfl_xor_sync(0xffffffffu, sf, o);
      sff += __shfl_xor_sync(0xffffffffu, sff, o);
    }
    if (lane == 0) {
      const int64_t n = (int64_t)side * side;
      const int64_t vf = n * (int64_t)sff - (int64_t)sf * (int64_t)sf;
      ctl->sf = (long long)sf;
      ctl->sqrt_vf = vf > 0 ? sqrt((double)vf) : 0.0;
    }
    // init draws: x, y, vx, vy per particle (integer_search.cpp:117-122)
    draw_uniforms(mt, ctl, draws, 4 * p.P);
  }
  __syncthreads();

  const double vspan = p.R / 2.0;
  const double dlo_x = (double)lo_dx, dhi_x = (double)hi_dx, dlo_y = (double)lo_dy, dhi_y = (double)hi_dy;
  for (int i = tid; i < p.P; i += kThreads) {
    Particle& P = parts[i];
    P.x = __dadd_rn(dlo_x, __dmul_rn(__dsub_rn(dhi_x, dlo_x), draws[4 * i + 0]));
    P.y = __dadd_rn(dlo_y, __dmul_rn(__dsub_rn(dhi_y, dlo_y), draws[4 * i + 1]));
    P.vx = __dadd_rn(-vspan, __dmul_rn(__dsub_rn(vspan, -vspan), draws[4 * i + 2]));
    P.vy = __dadd_rn(-vspan, __dmul_rn(__dsub_rn(vspan, -vspan), draws[4 * i + 3]));
    P.best_c = -2.0;
    P.best_dx = P.best_dy = 0;
    P.has_best = 0;
    Spec& s = spec[i];
    s.x = P.x;
    s.y = P.y;
    s.vx = P.vx;
    s.vy = P.vy;
    s.gdx = s.gdy = 0;
    probe_positions(s, ctl, p.star);
    for (int o = 0; o < (p.star ? 5 : 1); ++o)
      request(flags, req, ctl, (s.py[o] - lo_dy) * wx + (s.px[o] - lo_dx));
  }
  __syncthreads();
  evaluate_requests<kU8>(smem, L, ctl, p);
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < p.P; ++i) apply_particle(parts[i], spec[i], flags, vals, ctl, p.star);
    ctl->init_misses = ctl->misses;
    ctl->n_req = 0;
  }
  __syncthreads();
  if (!ctl->has_g) {  // integer_search.cpp:169
    if (tid == 0) write_failure(rec, cx, cy, DICB200_POI_ALL_DEGENERATE);
    return;
  }

  if (ctl->g_c < p.stop) {
    for (int t = 0; t < p.G; ++t) {
      const double w = p.inertia_constant
                           ? p.w_const
                           : __dsub_rn(0.9, __ddiv_rn((double)t, __dmul_rn(2.0, (double)p.G)));  // :35-37
      if (warp == 0) draw_uniforms(mt, ctl, draws, 4 * p.P);  // r1x, r2x, r1y, r2y per particle
      if (tid == 0) ctl->start = 0;
      __syncthreads();
      while (true) {
        const int start = ctl->start;
        if (start >= p.P) break;
        const int gdx = ctl->g_dx, gdy = ctl->g_dy;
        for (int i = start + tid; i < p.P; i += kThreads) {
          const Particle& P = parts[i];
          const double r1x = draws[4 * i], r2x = draws[4 * i + 1], r1y = draws[4 * i + 2], r2y = draws[4 * i + 3];
          Spec& s = spec[i];
          // integer_search.cpp:182-187
          s.vx = __dadd_rn(__dadd_rn(__dmul_rn(w, P.vx), __dmul_rn(__dmul_rn(p.c1, r1x), __dsub_rn((double)P.best_dx, P.x))),
                           __dmul_rn(__dmul_rn(p.c2, r2x), __dsub_rn((double)gdx, P.x)));
          s.vy = __dadd_rn(__dadd_rn(__dmul_rn(w, P.vy), __dmul_rn(__dmul_rn(p.c1, r1y), __dsub_rn((double)P.best_dy, P.y))),
                           __dmul_rn(__dmul_rn(p.c2, r2y), __dsub_rn((double)gdy, P.y)));
          s.x = clampd(__dadd_rn(P.x, s.vx), dlo_x, dhi_x);
          s.y = clampd(__dadd_rn(P.y, s.vy), dlo_y, dhi_y);
          s.gdx = gdx;
          s.gdy = gdy;
          probe_positions(s, ctl, p.star);
          for (int o = 0; o < (p.star ? 5 : 1); ++o)
            request(flags, req, ctl, (s.py[o] - lo_dy) * wx + (s.px[o] - lo_dx));
        }
        __syncthreads();
        evaluate_requests<kU8>(smem, L, ctl, p);
        __syncthreads();
        if (tid == 0) {
          int i = start;
          for (; i < p.P; ++i) {
            if (spec[i].gdx != ctl->g_dx || spec[i].gdy != ctl->g_dy) break;  // speculation stale
            apply_particle(parts[i], spec[i], flags, vals, ctl, p.star);
          }
          ctl->start = i;
          ctl->n_req = 0;
        }
        __syncthreads();
      }
      if (ctl->g_c >= p.stop) break;  // integer_search.cpp:191
    }
  }
  if (tid == 0) {
    rec->x = cx;
    rec->y = cy;
    rec->u = (double)ctl->g_dx;
    rec->v = (double)ctl->g_dy;
    rec->zncc = ctl->g_c;
    rec->converged = p.subpixel_none ? 1 : 0;
    rec->iterations = 0;
    rec->evaluations = ctl->misses;
    rec->update_evaluations = ctl->misses - ctl->init_misses;
    rec->status = DICB200_POI_OK;
    rec->integer_dx = ctl->g_dx;
    rec->integer_dy = ctl->g_dy;
    rec->pad = 0;
  }
}

}  // namespace

dicb200_status pso_launch(PsoParams& p, cudaStream_t st) {
  if (p.n_records <= 0) return DICB200_OK;
  const int side = 2 * p.M + 1;
  const int P = p.P < 1 ? 1 : p.P;
  p.wmax = 2 * (p.R < 0 ? 0 : p.R) + 1;
  p.QP = (side + 3) / 4;
  if (p.u8)
    p.region_pitch = ((p.wmax + 2 * p.M + 8) + 3) & ~3;
  else
    p.region_pitch = ((p.wmax + 2 * p.M + 2) + 1) & ~1;
  const Layout L = pso_layout(P, p.wmax, p.M, p.u8, p.region_pitch, p.QP);
  p.smem = L.total;
  if (L.total > 200 * 1024) {
    set_error("search window too large for the PSO kernel's shared memory");
    return DICB200_ERR_INVALID;
  }
  cudaError_t e;
  if (p.u8) {
    e = cudaFuncSetAttribute(pso_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e == cudaSuccess) {
      pso_kernel<true><<<p.n_records, kThreads, L.total, st>>>(p);
      e = cudaGetLastError();
    }
  } else {
    e = cudaFuncSetAttribute(pso_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e == cudaSuccess) {
      pso_kernel<false><<<p.n_records, kThreads, L.total, st>>>(p);
      e = cudaGetLastError();
    }
  }
  count_launch();
  if (e != cudaSuccess) return cuda_fail(e, "pso_kernel", __FILE__, __LINE__);
  return DICB200_OK;
}

}  // namespace dicb200
