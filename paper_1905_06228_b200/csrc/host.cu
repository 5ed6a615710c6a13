// C-ABI of the dicb200 library (include/dicb200.h): pipeline orchestration
// (the role of dic::analyze_pair / analyze_sequence, pipeline.cpp:147-214),
// grid construction (image.cpp:140-158), device memory and streams.
//
// The product path is GPU-only: without a CUDA device every analysis entry
// point returns DICB200_ERR_NO_DEVICE; nothing falls back to the CPU.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "bfs.cuh"
#include "bfs_fp.cuh"
#include "common.cuh"
#include "pso.cuh"
#include "refine.cuh"

namespace dicb200 {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

struct StageEvent {
  int stage;
  cudaEvent_t a, b;
};
std::atomic<int> g_profile{0};
std::mutex g_profile_mu;
std::vector<StageEvent> g_events;
std::vector<cudaEvent_t> g_event_pool;  // recycled timing events (creation is slow on the hot path)

cudaEvent_t take_event() {
  {
    std::lock_guard<std::mutex> lk(g_profile_mu);
    if (!g_event_pool.empty()) {
      cudaEvent_t e = g_event_pool.back();
      g_event_pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

StageTimer::StageTimer(int s, cudaStream_t stream) : stage(s), st(stream) {
  if (!g_profile.load()) return;
  a = take_event();
  b = take_event();
  cudaEventRecord(a, st);
}

StageTimer::~StageTimer() {
  if (!a) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_profile_mu);
  g_events.push_back({stage, a, b});
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

void set_error(const char* msg) { g_last_error = msg ? msg : ""; }

cudaError_t set_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;  // (device, kernel) -> value set so far
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = limit[{dev, kernel}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

dicb200_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
                file, line, what);
  set_error(buf);
  return e == cudaErrorMemoryAllocation ? DICB200_ERR_NOMEM : DICB200_ERR_CUDA;
}

static dicb200_status invalid(const char* msg) {
  set_error(msg);
  return DICB200_ERR_INVALID;
}

// Lattice of grid_subsets (image.cpp:140-158) with effective_margin (pipeline.hpp:43-45).
static dicb200_status make_lattice(int w, int h, const dicb200_run_config* cfg, Lattice* lat) {
  const int m = cfg->half_width;
  if (m < 1) return invalid("half_width must be >= 1");
  if (cfg->spacing < 1) return invalid("spacing must be >= 1");
  const int margin = cfg->margin >= 0 ? cfg->margin : cfg->half_width + cfg->search_radius;
  if (margin < 0) return invalid("margin must be >= 0");
  auto axis = [&](int dim, int* first, int* count) {
    *first = 0;
    *count = 0;
    for (int c = margin; c <= dim - margin; c += cfg->spacing) {
      if (c >= m && c <= dim - 1 - m) {  // subset_fits, image.cpp:24-28 (separable)
        if (*count == 0) *first = c;
        ++*count;
      }
    }
  };
  axis(w, &lat->x0, &lat->nx);
  axis(h, &lat->y0, &lat->ny);
  lat->step = cfg->spacing;
  if (lat->nx == 0 || lat->ny == 0) return invalid("image too small to host any subset");
  return DICB200_OK;
}

// Keep stream-ordered allocations (PSO surfaces, per-call images/records) in
// the device pool across calls instead of returning them at every sync.
void host_trace(const char* what, long i) {
  static const bool on = std::getenv("DICB200_HOST_TRACE") != nullptr;
  if (!on) return;
  thread_local auto t_last = std::chrono::steady_clock::now();
  auto t = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(t - t_last).count();
  if (ms > 5.0) fprintf(stderr, "[dicb200 trace] %s %ld: %.1f ms\n", what, i, ms);
  t_last = t;
}

static void retain_pool_memory() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

static bool has_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (n > 0) retain_pool_memory();
  return n > 0;
}

static dicb200_status no_device() {
  set_error("no CUDA device visible: the dicb200 path runs only on the GPU (no CPU fallback)");
  return DICB200_ERR_NO_DEVICE;
}

static ImageView view(const dicb200_image* im) {
  return ImageView{im->data, im->width, im->height, im->pitch > 0 ? im->pitch : im->width};
}

static dicb200_status validate_pair(const dicb200_image* a, const dicb200_image* b, const dicb200_run_config* cfg) {
  if (!a || !b || !cfg || !a->data || !b->data) return invalid("null argument");
  if (a->width != b->width || a->height != b->height) return invalid("dimension mismatch");
  if (a->width < 1 || a->height < 1) return invalid("zero-dimension image");
  if (a->dtype != b->dtype || a->dtype < DICB200_U8 || a->dtype > DICB200_F64)
    return invalid("unsupported pixel type (u8, u16, f32 or f64, identical for both images)");
  if (cfg->integer_method < 0 || cfg->integer_method > 2) return invalid("unknown integer method");
  if (cfg->subpixel_method < 0 || cfg->subpixel_method > 2) return invalid("unknown subpixel method");
  if (cfg->interp != DICB200_INTERP_BILINEAR && cfg->interp != DICB200_INTERP_BICUBIC)
    return invalid("unknown interpolation");
  if (cfg->subpixel_method != DICB200_SUB_NONE) {
    int ppt, nt;
    if (!refine_plan(cfg->half_width, &ppt, &nt))
      return invalid("half_width too large for the device refiners (M <= 64)");
  }
  return DICB200_OK;
}

// Largest representable gray level of the pair (dicb200_image.bits, else the dtype's).
static double pixel_max(const dicb200_image* a, const dicb200_image* b) {
  const int bits = std::max(a->bits, b->bits);
  if (a->dtype == DICB200_U8 && b->dtype == DICB200_U8) return 255.0;
  return (bits > 0 && bits < 16) ? (double)((1 << bits) - 1) : 65535.0;
}

// ---- declared-width guard --------------------------------------------------
// dicb200_image.bits < the dtype's width selects exact u32 paths (block sums,
// u32 IMAD row sums) that would overflow silently on wider data. When a caller
// declares it, the frames are checked on the device (one read of each frame,
// 16 B per thread-load) and, on a violation, every record of the call is
// overwritten with DICB200_POI_BITS_EXCEEDED; the host entry points turn that
// into a pair-level DICB200_ERR_INVALID.
// (u8 data never takes a width-dependent path: pixel_max is 255 for it.)
static bool declares_bits(const dicb200_image* im) {
  return im->dtype == DICB200_U16 && im->bits > 0 && im->bits < 16;
}

template <typename Pix>
__global__ void __launch_bounds__(256) bits_check_kernel(const Pix* data, int pitch, int w, int h, uint32_t limit,
                                                         int* flag) {
  const int per = 16 / sizeof(Pix);
  const bool vec = ((uintptr_t)data % 16) == 0 && ((size_t)pitch * sizeof(Pix)) % 16 == 0;
  uint32_t mx = 0;
  const int chunks = (w + per - 1) / per;
#pragma unroll 4
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < (long)chunks * h; i += (long)gridDim.x * blockDim.x) {
    const int y = (int)(i / chunks), c = (int)(i - (long)y * chunks), x0 = c * per;
    const Pix* row = data + (size_t)y * pitch;
    if (vec && x0 + per <= w) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(row + x0));
      const uint32_t v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (sizeof(Pix) == 2)
          mx = max(mx, max(v[k] & 0xffffu, v[k] >> 16));
        else
          mx = max(mx, max(max(v[k] & 0xffu, (v[k] >> 8) & 0xffu), max((v[k] >> 16) & 0xffu, v[k] >> 24)));
      }
    } else {
      for (int x = x0; x < min(w, x0 + per); ++x) mx = max(mx, (uint32_t)row[x]);
    }
  }
  if (__any_sync(0xffffffffu, mx > limit) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void __launch_bounds__(256) bits_poison_kernel(const int* flag, dicb200_poi_record* rec, size_t n) {
  if (!(flag[0] | flag[1])) return;  // {reference, target}
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    dicb200_poi_record& r = rec[k];
    r.u = r.v = 0.0;
    r.zncc = __longlong_as_double(0x7ff8000000000000ll);
    r.converged = r.iterations = 0;
    r.evaluations = r.update_evaluations = 0;
    r.integer_dx = r.integer_dy = 0;
    r.status = DICB200_POI_BITS_EXCEEDED;
  }
}

// `cache` (the stream's reference-side cache, optional): the flags live there
// and the reference frame is checked once while it repeats along a sequence
// (fixed_first), not once per pair.
static dicb200_status enqueue_bits_guard(const dicb200_image* ref, const dicb200_image* tgt, dicb200_poi_record* rec,
                                         size_t n, cudaStream_t st, TcRefCache* cache, long ref_key) {
  if (!declares_bits(ref) && !declares_bits(tgt)) return DICB200_OK;
  int* flag = nullptr;
  bool ref_known = false;
  if (cache) {
    if (!cache->guard) {
      DICB200_CUDA_TRY(cudaMallocAsync((void**)&cache->guard, 2 * sizeof(int), st));
      cache->guard_key = -1;
    }
    flag = cache->guard;
    ref_known = ref_key >= 0 && cache->guard_key == ref_key && cache->guard_data == ref->data &&
                cache->guard_bits == (declares_bits(ref) ? (int)ref->bits : 0);
  } else {
    DICB200_CUDA_TRY(cudaMallocAsync((void**)&flag, 2 * sizeof(int), st));
  }
  DICB200_CUDA_TRY(cudaMemsetAsync(flag + (ref_known ? 1 : 0), 0, (ref_known ? 1 : 2) * sizeof(int), st));
  int slot = 0;
  for (const dicb200_image* im : {ref, tgt}) {
    const int s = slot++;
    if (!declares_bits(im) || (s == 0 && ref_known)) continue;
    const uint32_t limit = (1u << im->bits) - 1u;
    const int pitch = im->pitch > 0 ? im->pitch : im->width;
    if (im->dtype == DICB200_U8)
      bits_check_kernel<uint8_t><<<8 * 148, 256, 0, st>>>(static_cast<const uint8_t*>(im->data), pitch, im->width,
                                                           im->height, limit, flag + s);
    else
      bits_check_kernel<uint16_t><<<8 * 148, 256, 0, st>>>(static_cast<const uint16_t*>(im->data), pitch, im->width,
                                                            im->height, limit, flag + s);
    count_launch();
  }
  if (cache) {
    cache->guard_key = ref_key;
    cache->guard_data = ref->data;
    cache->guard_bits = declares_bits(ref) ? (int)ref->bits : 0;
  }
  bits_poison_kernel<<<148, 256, 0, st>>>(flag, rec, n);
  count_launch();
  DICB200_CUDA_TRY(cudaGetLastError());
  if (!cache) DICB200_CUDA_TRY(cudaFreeAsync(flag, st));
  return DICB200_OK;
}

static const char kBitsMsg[] = "pixel values exceed the declared dicb200_image.bits";

// Enqueue the whole per-pair chain for grid rows [rb, re) on `st`.
static dicb200_status enqueue_pair_impl(const dicb200_image* ref, const dicb200_image* tgt, const dicb200_run_config* cfg,
                                        uint64_t pair_index, const Lattice& lat, int rb, int re,
                                        dicb200_poi_record* out_dev, cudaStream_t st, TcRefCache* tcache,
                                        long ref_key, IcgnRefCache* icache) {
  const int rows = re - rb;
  if (rows <= 0) return DICB200_OK;
  const size_t nrec = (size_t)rows * lat.nx;
  const bool fp = ref->dtype == DICB200_F64;  // fractional gray levels: the exact fp64 path (bfs_fp.cu)
  auto fp_params = [&](int r0, dicb200_poi_record* rec, double* surface) {
    FpParams f{};
    f.ref = view(ref);
    f.tgt = view(tgt);
    f.lat = lat;
    f.row_begin = r0;
    f.M = cfg->half_width;
    f.R = cfg->search_radius;
    f.whole = surface ? 0 : cfg->bfs_domain == DICB200_BFS_WHOLE_IMAGE;
    f.subpixel_none = cfg->subpixel_method == DICB200_SUB_NONE;
    f.rec = rec;
    f.surface = surface;
    return f;
  };
  if (fp && cfg->integer_method == DICB200_INT_BFS) {
    if (cfg->bfs_domain != DICB200_BFS_WHOLE_IMAGE && cfg->search_radius < 0) return invalid("search radius must be >= 0");
    StageTimer tm(0, st);
    DICB200_CUDA_TRY(bfs_fp_launch(fp_params(rb, out_dev, nullptr), rows, st));
    goto refine;
  }
  if (cfg->integer_method == DICB200_INT_BFS) {
    BfsParams p{};
    p.ref = view(ref);
    p.tgt = view(tgt);
    p.lat = lat;
    p.row_begin = rb;
    p.M = cfg->half_width;
    p.R = cfg->search_radius;
    p.whole = cfg->bfs_domain == DICB200_BFS_WHOLE_IMAGE;
    p.u8 = ref->dtype == DICB200_U8;
    {
      const int bits = std::max(ref->bits, tgt->bits);
      const double maxv = (bits > 0 && bits < 16) ? (double)((1 << bits) - 1) : 65535.0;
      p.f64 = !p.u8 && (double)(2 * p.M + 1) * maxv * maxv >= 4294967296.0;
      if (std::getenv("DICB200_FORCE_F64")) p.f64 = !p.u8;  // experiment switch: all-DFMA path
    }
    p.subpixel_none = cfg->subpixel_method == DICB200_SUB_NONE;
    p.rec = out_dev;
    if (!p.whole && p.R < 0) return invalid("search radius must be >= 0");
    if (!p.whole) {  // tensor-core search when the window shape allows it
      TcParams t{};
      t.ref = p.ref;
      t.tgt = p.tgt;
      t.lat = lat;
      t.rb = rb;
      t.re = re;
      t.M = p.M;
      t.R = p.R;
      t.planes = p.u8 ? 1 : 2;
      t.subpixel_none = p.subpixel_none;
      t.maxv = pixel_max(ref, tgt);
      t.rec = out_dev;
      if (tc_plan(t)) {
        StageTimer tm(0, st);
        DICB200_CUDA_TRY(tc_launch(t, st, tcache, ref_key));
        goto refine;
      }
    }
    if (!bfs_plan(p, 72 * 1024) && !bfs_plan(p, 200 * 1024)) return invalid("subset too large for the BFS tile (shared memory)");
    BestPartial* partial = nullptr;
    if (p.n_chunks > 1) {
      DICB200_CUDA_TRY(cudaMallocAsync((void**)&partial, nrec * p.n_chunks * sizeof(BestPartial), st));
      p.partial = partial;
    }
    {
      StageTimer tm(0, st);
      DICB200_CUDA_TRY(bfs_launch(p, rows, st));
    }
    if (partial) DICB200_CUDA_TRY(cudaFreeAsync(partial, st));
  } else {
    // K2: exact ZNCC surface of every POI's +-R window (K1 kernel), then the
    // warp-per-POI swarm walk over it. Rows are processed in chunks so the
    // surface buffer stays bounded.
    const int W = 2 * cfg->search_radius + 1;
    if (cfg->search_radius < 0) return invalid("search radius must be >= 0");
    const size_t per_row = (size_t)lat.nx * W * W * sizeof(double);
    const int rows_per_chunk = std::max<int>(1, (int)std::min<size_t>((size_t)rows, ((size_t)1 << 30) / per_row));
    double* surface = nullptr;
    DICB200_CUDA_TRY(cudaMallocAsync((void**)&surface, per_row * rows_per_chunk, st));
    dicb200_status s = DICB200_OK;
    for (int r0 = rb; r0 < re && s == DICB200_OK; r0 += rows_per_chunk) {
      const int r1 = std::min(re, r0 + rows_per_chunk);
      dicb200_poi_record* out_chunk = out_dev + (size_t)(r0 - rb) * lat.nx;
      BfsParams b{};
      b.ref = view(ref);
      b.tgt = view(tgt);
      b.lat = lat;
      b.row_begin = r0;
      b.M = cfg->half_width;
      b.R = cfg->search_radius;
      b.whole = 0;  // the swarm always searches the feasible +-R window (integer_search.cpp:113-114)
      b.u8 = ref->dtype == DICB200_U8;
      {
        const int bits = std::max(ref->bits, tgt->bits);
        const double maxv = (bits > 0 && bits < 16) ? (double)((1 << bits) - 1) : 65535.0;
        b.f64 = !b.u8 && (double)(2 * b.M + 1) * maxv * maxv >= 4294967296.0;
      }
      b.subpixel_none = 1;
      b.rec = out_chunk;
      b.surface = surface;
      TcParams t{};
      t.ref = b.ref;
      t.tgt = b.tgt;
      t.lat = lat;
      t.rb = r0;
      t.re = r1;
      t.M = b.M;
      t.R = b.R;
      t.planes = b.u8 ? 1 : 2;
      t.subpixel_none = 1;
      t.maxv = pixel_max(ref, tgt);
      t.surface = surface;
      const bool use_tc = !fp && tc_plan(t);
      if (!fp && !use_tc && !bfs_plan(b, 72 * 1024) && !bfs_plan(b, 200 * 1024)) {
        s = invalid("subset too large for the BFS tile (shared memory)");
        break;
      }
      BestPartial* partial = nullptr;
      if (!fp && !use_tc && b.n_chunks > 1) {
        cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)(r1 - r0) * lat.nx * b.n_chunks * sizeof(BestPartial), st);
        if (e != cudaSuccess) {
          s = cuda_fail(e, "cudaMallocAsync(partial)", __FILE__, __LINE__);
          break;
        }
        b.partial = partial;
      }
      PsoParams p{};
      p.ref = view(ref);
      p.tgt = view(tgt);
      p.lat = lat;
      p.row_begin = r0;
      p.M = cfg->half_width;
      p.R = cfg->search_radius;
      p.u8 = ref->dtype == DICB200_U8;
      p.star = cfg->integer_method == DICB200_INT_MPSO;
      p.P = cfg->particle_count;
      p.G = cfg->max_generations;
      p.stop = cfg->stop_threshold;
      p.c1 = cfg->c1;
      p.c2 = cfg->c2;
      p.seed = cfg->rng_seed;
      p.pair_index = pair_index;
      p.inertia_constant = cfg->inertia_mode == DICB200_INERTIA_CONSTANT;
      p.w_const = cfg->inertia_constant;
      p.subpixel_none = cfg->subpixel_method == DICB200_SUB_NONE;
      p.rec = out_chunk;
      p.n_records = (r1 - r0) * lat.nx;
      p.surface = surface;
      {
        StageTimer tm(1, st);
        cudaError_t e = fp       ? bfs_fp_launch(fp_params(r0, out_chunk, surface), r1 - r0, st)
                        : use_tc ? tc_launch(t, st, tcache, ref_key)
                                 : bfs_launch(b, r1 - r0, st);
        if (e != cudaSuccess) s = cuda_fail(e, "bfs_launch(surface)", __FILE__, __LINE__);
        if (s == DICB200_OK) s = pso_walk_launch(p, st);
      }
      if (partial) cudaFreeAsync(partial, st);
    }
    cudaFreeAsync(surface, st);
    if (s != DICB200_OK) return s;
  }
refine:
  host_trace("search enqueued");
  if (cfg->subpixel_method != DICB200_SUB_NONE) {
    RefineParams r{};
    r.ref = view(ref);
    r.tgt = view(tgt);
    r.lat = lat;
    r.row_begin = rb;
    r.M = cfg->half_width;
    r.n_records = (int)nrec;
    r.method = cfg->subpixel_method == DICB200_SUB_NR ? 0 : 1;
    r.tol = cfg->tol;
    r.max_iter = cfg->max_iter;
    r.interp = cfg->interp;
    r.rec = out_dev;
    StageTimer tm(r.method == 0 ? 2 : 3, st);
    DICB200_CUDA_TRY(refine_launch(r, ref->dtype, st, icache, ref_key));
    host_trace("refine enqueued");
  }
  return enqueue_bits_guard(ref, tgt, out_dev, nrec, st, tcache, ref_key);
}

// Subsets below this half-width (under 17 x 17 px) hold so little texture that
// distinct candidates reach mathematically tied ZNCC values; the reference orders
// those by the rounding of its sequential fp64 sums, which the exact-integer
// kernels (they compare exact moments) cannot reproduce. Such grids run on the
// fp64 path instead, which evaluates zncc in the reference's own order (bit
// for bit): integer frames are widened for the call. The work per POI is tiny
// at these sizes; no BASELINE configuration is affected (M >= 10).
constexpr int kRefOrderBelowM = 8;

static dicb200_status enqueue_pair(const dicb200_image* ref, const dicb200_image* tgt, const dicb200_run_config* cfg,
                                   uint64_t pair_index, const Lattice& lat, int rb, int re,
                                   dicb200_poi_record* out_dev, cudaStream_t st, TcRefCache* tcache = nullptr,
                                   long ref_key = -1, IcgnRefCache* icache = nullptr) {
  const bool integer_frames = ref->dtype == DICB200_U8 || ref->dtype == DICB200_U16;
  // the A/B switches that force one of the exact-integer search kernels keep it (kernel-vs-kernel tests)
  const bool forced = std::getenv("DICB200_BFS_LEGACY") || std::getenv("DICB200_BFS_TC") || std::getenv("DICB200_BFS_BS");
  if (!integer_frames || cfg->half_width >= kRefOrderBelowM || re <= rb || forced)
    return enqueue_pair_impl(ref, tgt, cfg, pair_index, lat, rb, re, out_dev, st, tcache, ref_key, icache);
  double* buf[2] = {nullptr, nullptr};
  dicb200_image wide[2] = {*ref, *tgt};
  dicb200_status s = DICB200_OK;
  for (int k = 0; k < 2 && s == DICB200_OK; ++k) {
    const dicb200_image* im = k ? tgt : ref;
    const int pitch = im->pitch > 0 ? im->pitch : im->width;
    cudaError_t e = cudaMallocAsync((void**)&buf[k], (size_t)im->width * im->height * 8, st);
    if (e == cudaSuccess)
      e = widen_int_to_f64(im->data, im->dtype == DICB200_U8 ? 1 : 2, pitch, buf[k], im->width, im->height, st);
    if (e != cudaSuccess) s = cuda_fail(e, "widen integer frame", __FILE__, __LINE__);
    wide[k].dtype = DICB200_F64;
    wide[k].bits = 0;
    wide[k].pitch = im->width;
    wide[k].data = buf[k];
  }
  // the widened copies live for this call only: no reference-side caches
  if (s == DICB200_OK)
    s = enqueue_pair_impl(&wide[0], &wide[1], cfg, pair_index, lat, rb, re, out_dev, st, nullptr, -1, nullptr);
  for (double* b : buf)
    if (b) cudaFreeAsync(b, st);
  return s;
}

static size_t elem_size(int dtype) {
  return dtype == DICB200_U8 ? 1 : dtype == DICB200_U16 ? 2 : dtype == DICB200_F32 ? 4 : 8;
}
static bool is_float(int dtype) { return dtype == DICB200_F32 || dtype == DICB200_F64; }

// Fractional gray levels run on the exact fp64 path (bfs_fp.cu, the refiners'
// fp64 images): an F32 device image is widened (exactly) into `buf` for this
// call; F64 images are used as they are.
static dicb200_status widen_device(const dicb200_image* im, double** buf, dicb200_image* out, cudaStream_t st) {
  *out = *im;
  if (im->dtype == DICB200_F64) return DICB200_OK;
  const int pitch = im->pitch > 0 ? im->pitch : im->width;
  DICB200_CUDA_TRY(cudaMallocAsync((void**)buf, (size_t)im->width * im->height * 8, st));
  DICB200_CUDA_TRY(widen_f32_to_f64(static_cast<const float*>(im->data), pitch, *buf, im->width, im->height, st));
  out->dtype = DICB200_F64;
  out->bits = 0;
  out->pitch = im->width;
  out->data = *buf;
  return DICB200_OK;
}

// Host image (f32/f64) -> dense fp64 on the host; non-finite levels are an
// error (GrayImage's constructor rejects them, image.cpp:14-22).
static dicb200_status to_f64_host(const dicb200_image* im, std::vector<double>& v) {
  const int pitch = im->pitch > 0 ? im->pitch : im->width;
  v.resize((size_t)im->width * im->height);
  for (int y = 0; y < im->height; ++y)
    for (int x = 0; x < im->width; ++x) {
      const double g = im->dtype == DICB200_F32 ? (double)static_cast<const float*>(im->data)[(size_t)y * pitch + x]
                                                : static_cast<const double*>(im->data)[(size_t)y * pitch + x];
      if (!std::isfinite(g)) return invalid("non-finite gray level");
      v[(size_t)y * im->width + x] = g;
    }
  return DICB200_OK;
}

// ---- persistent per-device execution contexts ------------------------------
// Streams, events and grow-only device buffers are created once and reused by
// every analyze call. Contexts live in a pool so that concurrent callers (and
// the per-device workers of analyze_sequence) each own one while they run.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// Grow `b` to at least `bytes` in stream order on `st`.
static cudaError_t ensure(DevBuf& b, size_t bytes, cudaStream_t st) {
  if (b.cap >= bytes) return cudaSuccess;
  if (b.p) {
    cudaError_t e = cudaFreeAsync(b.p, st);
    if (e != cudaSuccess) return e;
    b.p = nullptr;
    b.cap = 0;
  }
  cudaError_t e = cudaMallocAsync(&b.p, bytes, st);
  if (e == cudaSuccess) b.cap = bytes;
  return e;
}

// A device-resident frame. `key` is the frame's index in the caller's image
// array for the duration of one analyze_sequence call (-1 = nothing cached).
struct FrameSlot {
  DevBuf buf;
  long key = -1, last_use = -1;
  cudaEvent_t ready = nullptr;  // upload finished (copy stream)
  cudaEvent_t idle = nullptr;   // last pair reading the frame finished (compute stream)
  cudaEvent_t idle2 = nullptr;  // the same on the second compute stream
  dicb200_image im{};
};

// Device records of one pair plus a pinned staging buffer for pageable outputs.
struct RecSlot {
  DevBuf dev;
  void* stage = nullptr;
  size_t stage_cap = 0;
  cudaEvent_t computed = nullptr;  // kernels of the pair finished (compute stream)
  cudaEvent_t done = nullptr;      // records are in host memory (read-back stream)
  long pair = -1;              // pair in flight (-1 = none)
  size_t n = 0;
  bool staged = false;
};

constexpr int kFrameSlots = 4;
constexpr int kSeqStreams = 2;  // concurrent pairs of analyze_sequence_device
constexpr int kRecSlots = 4;

struct DeviceContext {
  int dev = 0;
  cudaStream_t cs = nullptr;  // compute: kernels + record read-back
  cudaStream_t cs2 = nullptr;  // second compute stream: analyze_sequence keeps two pairs in flight
  cudaStream_t xs = nullptr;  // copy: frame uploads ahead of the compute stream
  cudaStream_t ds = nullptr;  // copy: record read-back behind the compute stream
  FrameSlot frames[kFrameSlots];
  RecSlot recs[kRecSlots];
  TcRefCache tcache;  // reference-side tensor-core inputs, reused while the reference frame repeats
  IcgnRefCache icache;  // reference-side IC-GN constants (Hessian inverse, sums), likewise
  TcRefCache tcache2;   // the second compute stream's own caches (no sharing between
  IcgnRefCache icache2;  // concurrently running pairs)
};

namespace {
std::mutex g_ctx_mu;
std::vector<DeviceContext*> g_ctx_idle;
}  // namespace

static void destroy_context(DeviceContext* c) {
  cudaSetDevice(c->dev);
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->cs2) cudaStreamSynchronize(c->cs2);
  if (c->xs) cudaStreamSynchronize(c->xs);
  if (c->ds) cudaStreamSynchronize(c->ds);
  for (auto& f : c->frames) {
    if (f.buf.p) cudaFree(f.buf.p);
    if (f.ready) cudaEventDestroy(f.ready);
    if (f.idle) cudaEventDestroy(f.idle);
    if (f.idle2) cudaEventDestroy(f.idle2);
  }
  for (auto& r : c->recs) {
    if (r.dev.p) cudaFree(r.dev.p);
    if (r.stage) cudaFreeHost(r.stage);
    if (r.done) cudaEventDestroy(r.done);
    if (r.computed) cudaEventDestroy(r.computed);
  }
  tc_cache_free(c->tcache);
  icgn_cache_free(c->icache);
  tc_cache_free(c->tcache2);
  icgn_cache_free(c->icache2);
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->cs2) cudaStreamDestroy(c->cs2);
  if (c->xs) cudaStreamDestroy(c->xs);
  if (c->ds) cudaStreamDestroy(c->ds);
  delete c;
}

// Take an idle context of the current device (or create one).
static DeviceContext* acquire_context(dicb200_status* st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *st = cuda_fail(e, "cudaGetDevice", __FILE__, __LINE__);
    return nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (size_t i = 0; i < g_ctx_idle.size(); ++i)
      if (g_ctx_idle[i]->dev == dev) {
        DeviceContext* c = g_ctx_idle[i];
        g_ctx_idle.erase(g_ctx_idle.begin() + (long)i);
        *st = DICB200_OK;
        return c;
      }
  }
  auto* c = new DeviceContext;
  c->dev = dev;
  e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cs2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->ds, cudaStreamNonBlocking);
  for (auto& f : c->frames) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.idle, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.idle2, cudaEventDisableTiming);
  }
  for (auto& r : c->recs) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.computed, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    *st = cuda_fail(e, "device context creation", __FILE__, __LINE__);
    destroy_context(c);
    return nullptr;
  }
  *st = DICB200_OK;
  return c;
}

// Return a context to the pool once both of its streams are drained.
static dicb200_status release_context(DeviceContext* c) {
  cudaError_t e1 = cudaStreamSynchronize(c->xs);
  cudaError_t e2 = cudaStreamSynchronize(c->cs);
  if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(c->cs2);
  cudaError_t e3 = cudaStreamSynchronize(c->ds);
  if (e2 == cudaSuccess) e2 = e3;
  for (auto& f : c->frames) f.key = f.last_use = -1;  // LRU state is per call
  c->tcache.reset();
  c->icache.reset();
  c->tcache2.reset();
  c->icache2.reset();
  for (auto& r : c->recs) r.pair = -1;
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_ctx_idle.push_back(c);
  if (e1 != cudaSuccess) return cuda_fail(e1, "cudaStreamSynchronize(copy)", __FILE__, __LINE__);
  if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamSynchronize(compute)", __FILE__, __LINE__);
  return DICB200_OK;
}

// H2D of a host image (any pitch) into `buf` on `st`; `dev` describes the copy.
static dicb200_status upload(const dicb200_image* host, DevBuf& buf, dicb200_image* dev, cudaStream_t st) {
  if (is_float(host->dtype)) {  // checked and widened on the host, uploaded as fp64
    std::vector<double> v;
    dicb200_status s = to_f64_host(host, v);
    if (s != DICB200_OK) return s;
    DICB200_CUDA_TRY(ensure(buf, v.size() * 8, st));
    DICB200_CUDA_TRY(cudaMemcpyAsync(buf.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, st));
    DICB200_CUDA_TRY(cudaStreamSynchronize(st));  // v is a temporary
    *dev = *host;
    dev->dtype = DICB200_F64;
    dev->bits = 0;
    dev->pitch = host->width;
    dev->data = buf.p;
    return DICB200_OK;
  }
  const size_t es = elem_size(host->dtype);
  const int pitch = host->pitch > 0 ? host->pitch : host->width;
  const size_t row = (size_t)host->width * es;
  DICB200_CUDA_TRY(ensure(buf, row * host->height, st));
  DICB200_CUDA_TRY(cudaMemcpy2DAsync(buf.p, row, host->data, pitch * es, row, host->height, cudaMemcpyHostToDevice, st));
  *dev = *host;
  dev->pitch = host->width;
  dev->data = buf.p;
  return DICB200_OK;
}

// Make frame `key` resident: reuse its slot, or upload it on the copy stream
// into the least recently used slot other than `pin` once that slot's last
// reader has finished.
static dicb200_status stage_frame(DeviceContext* c, const dicb200_image* host, long key, long use, int pin,
                                  int* slot) {
  for (int i = 0; i < kFrameSlots; ++i)
    if (c->frames[i].key == key) {
      c->frames[i].last_use = std::max(c->frames[i].last_use, use);
      *slot = i;
      return DICB200_OK;
    }
  int v = -1;
  for (int i = 0; i < kFrameSlots; ++i)
    if (i != pin && (v < 0 || c->frames[i].last_use < c->frames[v].last_use)) v = i;
  FrameSlot& f = c->frames[v];
  f.key = -1;
  DICB200_CUDA_TRY(cudaStreamWaitEvent(c->xs, f.idle, 0));
  DICB200_CUDA_TRY(cudaStreamWaitEvent(c->xs, f.idle2, 0));
  dicb200_status s = upload(host, f.buf, &f.im, c->xs);
  if (s != DICB200_OK) return s;
  DICB200_CUDA_TRY(cudaEventRecord(f.ready, c->xs));
  f.key = key;
  f.last_use = use;
  *slot = v;
  return DICB200_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Shape checks shared by the host-buffer entry points: lattice size and the
// caller's output capacity.
static dicb200_status precheck(const dicb200_image* ref, const dicb200_image* tgt, const dicb200_run_config* cfg,
                               size_t cap, Lattice* lat, size_t* n) {
  *n = 0;
  dicb200_status s = validate_pair(ref, tgt, cfg);
  if (s != DICB200_OK) return s;
  s = make_lattice(ref->width, ref->height, cfg, lat);
  if (s != DICB200_OK) return s;
  *n = (size_t)lat->nx * lat->ny;
  if (*n > cap) {
    set_error("output capacity smaller than the grid");
    return DICB200_ERR_CAPACITY;
  }
  return DICB200_OK;
}

}  // namespace dicb200

using namespace dicb200;

extern "C" {

int dicb200_abi_version(void) { return DICB200_ABI_VERSION; }

void dicb200_default_config(dicb200_run_config* c) {
  std::memset(c, 0, sizeof *c);
  c->integer_method = DICB200_INT_MPSO;
  c->subpixel_method = DICB200_SUB_NR;
  c->mode = DICB200_MODE_SERIAL;
  c->reference_policy = DICB200_POLICY_UPDATE;
  c->worker_count = 1;
  c->search_radius = 25;
  c->bfs_domain = DICB200_BFS_WHOLE_IMAGE;
  c->particle_count = 50;
  c->max_generations = 5;
  c->stop_threshold = 0.995;
  c->c1 = 2.0;
  c->c2 = 2.0;
  c->rng_seed = 0;
  c->tol = 0.01;
  c->max_iter = 20;
  c->half_width = 15;
  c->spacing = 10;
  c->margin = -1;
  c->inertia_mode = DICB200_INERTIA_REFERENCE;
  c->inertia_constant = 0.7;
}

const char* dicb200_last_error_message(void) { return g_last_error.c_str(); }

int dicb200_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

uint64_t dicb200_launch_count(void) { return g_launches.load(); }
void dicb200_reset_launch_count(void) { g_launches.store(0); }

dicb200_status dicb200_grid_size(int32_t width, int32_t height, const dicb200_run_config* cfg, size_t* count) {
  Lattice lat;
  dicb200_status s = make_lattice(width, height, cfg, &lat);
  if (s != DICB200_OK) return s;
  *count = (size_t)lat.nx * lat.ny;
  return DICB200_OK;
}

dicb200_status dicb200_grid(int32_t width, int32_t height, const dicb200_run_config* cfg, int32_t* xy, size_t cap,
                            size_t* count) {
  Lattice lat;
  dicb200_status s = make_lattice(width, height, cfg, &lat);
  if (s != DICB200_OK) return s;
  const size_t n = (size_t)lat.nx * lat.ny;
  *count = n;
  for (int iy = 0; iy < lat.ny; ++iy)
    for (int ix = 0; ix < lat.nx; ++ix) {
      const size_t k = (size_t)iy * lat.nx + ix;
      if (k < cap) {
        xy[2 * k] = lat.cx(ix);
        xy[2 * k + 1] = lat.cy(iy);
      }
    }
  return DICB200_OK;
}

dicb200_status dicb200_sequence_pairs(int32_t policy, int32_t image_count, int32_t* pairs) {
  if (image_count < 2) return invalid("insufficient images");
  for (int i = 1; i < image_count; ++i) {
    pairs[2 * (i - 1)] = policy == DICB200_POLICY_UPDATE ? i - 1 : 0;
    pairs[2 * (i - 1) + 1] = i;
  }
  return DICB200_OK;
}

dicb200_status dicb200_partition_ranges(size_t n, int32_t workers, size_t* ranges) {
  if (workers < 1) return invalid("worker count must be >= 1");
  const size_t k = (size_t)workers, base = n / k, extra = n % k;
  size_t begin = 0;
  for (size_t i = 0; i < k; ++i) {
    const size_t len = base + (i < extra ? 1 : 0);
    ranges[2 * i] = begin;
    ranges[2 * i + 1] = begin + len;
    begin += len;
  }
  return DICB200_OK;
}

dicb200_status dicb200_analyze_pair(const dicb200_image* ref, const dicb200_image* tgt, const dicb200_run_config* cfg,
                                    uint64_t pair_index, dicb200_poi_record* out, size_t out_cap, size_t* out_count) {
  if (!has_device()) return no_device();
  Lattice lat;
  size_t n = 0;
  dicb200_status s = precheck(ref, tgt, cfg, out_cap, &lat, &n);
  if (out_count) *out_count = n;
  if (s != DICB200_OK) return s;
  DeviceContext* c = acquire_context(&s);
  if (!c) return s;
  // one pair: everything in order on the compute stream, one sync at the end
  RecSlot& r = c->recs[0];
  s = upload(ref, c->frames[0].buf, &c->frames[0].im, c->cs);
  if (s == DICB200_OK) s = upload(tgt, c->frames[1].buf, &c->frames[1].im, c->cs);
  if (s == DICB200_OK) {
    cudaError_t e = ensure(r.dev, n * sizeof(dicb200_poi_record), c->cs);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMallocAsync(records)", __FILE__, __LINE__);
  }
  if (s == DICB200_OK)
    s = enqueue_pair(&c->frames[0].im, &c->frames[1].im, cfg, pair_index, lat, 0, lat.ny,
                     (dicb200_poi_record*)r.dev.p, c->cs);
  if (s == DICB200_OK) {
    cudaError_t e = cudaMemcpyAsync(out, r.dev.p, n * sizeof(dicb200_poi_record), cudaMemcpyDeviceToHost, c->cs);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(records)", __FILE__, __LINE__);
  }
  const dicb200_status rs = release_context(c);
  if (s == DICB200_OK && rs == DICB200_OK && n > 0 && out[0].status == DICB200_POI_BITS_EXCEEDED)
    return invalid(kBitsMsg);
  return s != DICB200_OK ? s : rs;
}

dicb200_status dicb200_analyze_pair_device(const dicb200_image* ref, const dicb200_image* tgt,
                                           const dicb200_run_config* cfg, uint64_t pair_index, int32_t row_begin,
                                           int32_t row_end, dicb200_poi_record* out_dev, size_t out_cap,
                                           size_t* out_count, void* stream) {
  if (!has_device()) return no_device();
  dicb200_status s = validate_pair(ref, tgt, cfg);
  if (s != DICB200_OK) return s;
  Lattice lat;
  s = make_lattice(ref->width, ref->height, cfg, &lat);
  if (s != DICB200_OK) return s;
  int rb = row_begin < 0 ? 0 : row_begin;
  int re = row_end < 0 ? lat.ny : std::min(row_end, lat.ny);
  if (re < rb) re = rb;
  const size_t n = (size_t)(re - rb) * lat.nx;
  if (out_count) *out_count = n;
  if (n > out_cap) {
    set_error("output capacity smaller than the grid rows");
    return DICB200_ERR_CAPACITY;
  }
  if (ref->dtype == DICB200_F32) {  // fractional levels: fp64 copies for this call
    const cudaStream_t st = (cudaStream_t)stream;
    double *ba = nullptr, *bb = nullptr;
    dicb200_image ra, rt;
    s = widen_device(ref, &ba, &ra, st);
    if (s == DICB200_OK) s = widen_device(tgt, &bb, &rt, st);
    if (s == DICB200_OK) s = enqueue_pair(&ra, &rt, cfg, pair_index, lat, rb, re, out_dev, st);
    if (ba) cudaFreeAsync(ba, st);
    if (bb) cudaFreeAsync(bb, st);
    return s;
  }
  return enqueue_pair(ref, tgt, cfg, pair_index, lat, rb, re, out_dev, (cudaStream_t)stream);
}

dicb200_status dicb200_analyze_sequence_device(const dicb200_image* images, size_t n_images,
                                               const dicb200_run_config* cfg, uint64_t first_pair_index,
                                               int32_t row_begin, int32_t row_end, dicb200_poi_record* out_dev,
                                               size_t pair_stride, size_t* per_pair_count, void* stream) {
  if (!has_device()) return no_device();
  if (!images || !cfg || !out_dev) return invalid("null argument");
  if (n_images < 2) return invalid("insufficient images");
  std::vector<int32_t> pairs(2 * (n_images - 1));
  dicb200_sequence_pairs(cfg->reference_policy, (int32_t)n_images, pairs.data());
  for (size_t i = 1; i < n_images; ++i) {
    if (images[i].width != images[0].width || images[i].height != images[0].height)
      return invalid("dimension mismatch");
    if (images[i].dtype != images[0].dtype) return invalid("unsupported pixel type (identical for every image)");
  }
  dicb200_status s = validate_pair(&images[0], &images[1], cfg);
  if (s != DICB200_OK) return s;
  Lattice lat;
  s = make_lattice(images[0].width, images[0].height, cfg, &lat);
  if (s != DICB200_OK) return s;
  const int rb = row_begin < 0 ? 0 : row_begin;
  const int re = std::max(rb, row_end < 0 ? lat.ny : std::min(row_end, lat.ny));
  const size_t n = (size_t)(re - rb) * lat.nx;
  if (per_pair_count) *per_pair_count = n;
  if (n > pair_stride) {
    set_error("pair stride smaller than the grid rows");
    return DICB200_ERR_CAPACITY;
  }
  // Reference-side inputs (tensor-core strips/moments, IC-GN constants) live for
  // this call only and are rebuilt whenever the pair's reference frame changes.
  const cudaStream_t st = (cudaStream_t)stream;
  std::vector<dicb200_image> conv;  // fractional f32 levels: fp64 copies for this call
  std::vector<double*> conv_buf;
  if (images[0].dtype == DICB200_F32) {
    conv.resize(n_images);
    conv_buf.assign(n_images, nullptr);
    for (size_t i = 0; i < n_images && s == DICB200_OK; ++i) s = widen_device(&images[i], &conv_buf[i], &conv[i], st);
    if (s == DICB200_OK) images = conv.data();
  }
  // Pairs alternate over kSeqStreams internal streams forked from (and joined
  // back into) the caller's stream, so one pair's kernels fill the tail waves
  // of the other's. Each stream owns its reference-side caches: nothing is
  // shared between concurrently running pairs.
  const bool fixed = cfg->reference_policy == DICB200_POLICY_FIXED_FIRST;
  auto mark = [](const char* what, long i) { host_trace(what, i); };
  host_trace("seq begin");
  const char* env = std::getenv("DICB200_SEQ_STREAMS");
  const int ns = std::max(1, std::min<int>(env ? std::atoi(env) : kSeqStreams, (int)(n_images - 1)));
  std::vector<cudaStream_t> ss(ns, st);
  std::vector<TcRefCache> tc(ns);
  std::vector<IcgnRefCache> ic(ns);
  cudaEvent_t fork = nullptr;
  if (s == DICB200_OK && ns > 1) {
    cudaError_t e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(fork, st);
    for (int k = 0; k < ns && e == cudaSuccess; ++k) {
      e = cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ss[k], fork, 0);
    }
    if (e != cudaSuccess) s = cuda_fail(e, "sequence stream fork", __FILE__, __LINE__);
  }
  mark("fork", 0);
  for (size_t i = 0; i + 1 < n_images && s == DICB200_OK; ++i) {
    const int k = (int)(i % ns);
    s = enqueue_pair(&images[pairs[2 * i]], &images[pairs[2 * i + 1]], cfg, first_pair_index + i, lat, rb, re,
                     out_dev + i * pair_stride, ss[k], &tc[k], (long)pairs[2 * i], fixed ? &ic[k] : nullptr);
    mark("pair", (long)i);
  }
  for (int k = 0; k < ns; ++k) {
    tc_cache_free(tc[k], ss[k], true);
    icgn_cache_free(ic[k], ss[k], true);
  }
  mark("free", 0);
  if (ns > 1) {  // join: the caller's stream waits for every internal stream
    for (int k = 0; k < ns; ++k) {
      if (ss[k] == st) continue;
      cudaEvent_t j = nullptr;
      if (cudaEventCreateWithFlags(&j, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(j, ss[k]);
        cudaStreamWaitEvent(st, j, 0);
        cudaEventDestroy(j);
      }
      cudaStreamDestroy(ss[k]);
    }
    if (fork) cudaEventDestroy(fork);
  }
  for (double* b : conv_buf)
    if (b) cudaFreeAsync(b, st);
  return s;
}

dicb200_status dicb200_analyze_sequence(const dicb200_image* images, size_t n_images, const dicb200_run_config* cfg,
                                        dicb200_field* fields, size_t n_fields) {
  return dicb200_analyze_sequence_cb(images, n_images, cfg, fields, n_fields, 0, nullptr, nullptr);
}

dicb200_status dicb200_analyze_sequence_cb(const dicb200_image* images, size_t n_images,
                                           const dicb200_run_config* cfg, dicb200_field* fields, size_t n_fields,
                                           uint64_t first_pair_index, dicb200_field_ready_fn field_ready,
                                           void* user) {
  if (!has_device()) return no_device();
  if (!images || !cfg || !fields) return invalid("null argument");
  if (n_images < 2) return invalid("insufficient images");
  if (n_fields != n_images - 1) return invalid("fields must hold one entry per pair");
  std::vector<int32_t> pairs(2 * (n_images - 1));
  dicb200_sequence_pairs(cfg->reference_policy, (int32_t)n_images, pairs.data());
  int ndev = dicb200_device_count();
  int workers = 1;
  if (cfg->mode == DICB200_MODE_IMAGE) {
    // the reference's worker threads (pipeline.cpp:201-209) become devices; each
    // worker already keeps two pairs in flight on its device.
    // DICB200_WORKERS_PER_DEVICE (default 1) lets several workers share a device
    // (worker w runs on device w % ndev).
    const char* wpd = std::getenv("DICB200_WORKERS_PER_DEVICE");
    const int slots = ndev * std::max(1, wpd ? std::atoi(wpd) : 1);
    workers = cfg->worker_count <= 0 ? slots : std::min(cfg->worker_count, slots);
  }
  workers = std::max(1, std::min<int>(workers, (int)n_fields));
  std::vector<size_t> ranges(2 * workers);
  dicb200_partition_ranges(n_fields, workers, ranges.data());
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<dicb200_status> result(workers, DICB200_OK);
  std::vector<std::string> errs(workers);

  // One worker per device over a contiguous range of pairs. Per pair: frames are
  // made resident on the copy stream (each frame uploaded once while it stays in
  // one of the LRU slots — the fixed_first reference, or the frame an
  // update_every_pair sequence shares between neighbouring pairs), the compute
  // stream waits for them, runs the pair and reads its records back. The next
  // pair's frames are uploaded while the current pair computes, and the host
  // finalises pair i-1 while the device runs pair i.
  auto run = [&](int wk) {
    const int dev = workers == 1 ? cur : wk % ndev;
    cudaSetDevice(dev);
    auto fail_field = [&](dicb200_field& f, dicb200_status s) {
      f.count = 0;
      f.status = s;
      std::strncpy(f.error, g_last_error.c_str(), sizeof f.error - 1);
      f.error[sizeof f.error - 1] = 0;
      if (s != DICB200_ERR_INVALID) {  // a pair-level dic::Error does not fail the call (pipeline.cpp:191-198)
        result[wk] = s;
        errs[wk] = g_last_error;
      }
      if (field_ready) field_ready(user, (size_t)(&f - fields));
    };
    const size_t lo = ranges[2 * wk], hi = ranges[2 * wk + 1];
    std::vector<Lattice> lat(hi - lo);
    std::vector<size_t> cnt(hi - lo, 0);
    std::vector<dicb200_status> pre(hi - lo);
    for (size_t i = lo; i < hi; ++i) {
      dicb200_field& f = fields[i];
      f.pair_index = (int32_t)(first_pair_index + i);
      f.ref_id = images[pairs[2 * i]].id;
      f.tgt_id = images[pairs[2 * i + 1]].id;
      f.count = 0;
      f.status = DICB200_OK;
      f.error[0] = 0;
      pre[i - lo] = precheck(&images[pairs[2 * i]], &images[pairs[2 * i + 1]], cfg, f.capacity, &lat[i - lo],
                             &cnt[i - lo]);
      if (pre[i - lo] != DICB200_OK) fail_field(f, pre[i - lo]);
    }
    dicb200_status cs_ = DICB200_OK;
    DeviceContext* c = acquire_context(&cs_);
    if (!c) {
      for (size_t i = lo; i < hi; ++i)
        if (pre[i - lo] == DICB200_OK) fail_field(fields[i], cs_);
      return;
    }
    auto stage_pair = [&](size_t i, int* sa, int* sb) -> dicb200_status {
      dicb200_status s = stage_frame(c, &images[pairs[2 * i]], pairs[2 * i], (long)i, -1, sa);
      if (s != DICB200_OK) return s;
      return stage_frame(c, &images[pairs[2 * i + 1]], pairs[2 * i + 1], (long)i, *sa, sb);
    };
    auto finalize = [&](RecSlot& r) {
      if (r.pair < 0) return;
      dicb200_field& f = fields[r.pair];
      r.pair = -1;
      cudaError_t e = cudaEventSynchronize(r.done);
      if (e != cudaSuccess) {
        fail_field(f, cuda_fail(e, "pair execution", __FILE__, __LINE__));
        return;
      }
      if (r.staged) std::memcpy(f.records, r.stage, r.n * sizeof(dicb200_poi_record));
      if (r.n > 0 && f.records[0].status == DICB200_POI_BITS_EXCEEDED) {
        fail_field(f, invalid(kBitsMsg));
        return;
      }
      f.count = r.n;
      f.status = DICB200_OK;
      if (field_ready) field_ready(user, (size_t)(&f - fields));
    };
    auto next_valid = [&](size_t i) {
      while (i < hi && pre[i - lo] != DICB200_OK) ++i;
      return i;
    };
    // valid pairs alternate over the two compute streams (two pairs in flight)
    size_t q = 0;
    for (size_t i = next_valid(lo); i < hi; i = next_valid(i + 1), ++q) {
      dicb200_field& f = fields[i];
      const size_t n = cnt[i - lo];
      const size_t bytes = n * sizeof(dicb200_poi_record);
      const int k = (int)(q & 1);
      const cudaStream_t cst = k ? c->cs2 : c->cs;
      RecSlot& r = c->recs[q % kRecSlots];
      finalize(r);
      int sa = 0, sb = 0;
      dicb200_status s = stage_pair(i, &sa, &sb);
      cudaError_t e = cudaSuccess;
      if (s == DICB200_OK) {
        e = ensure(r.dev, bytes, cst);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cst, c->frames[sa].ready, 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cst, c->frames[sb].ready, 0);
        if (e != cudaSuccess) s = cuda_fail(e, "compute stream setup", __FILE__, __LINE__);
      }
      const bool staged_ok = s == DICB200_OK;
      if (s == DICB200_OK)
        s = enqueue_pair(&c->frames[sa].im, &c->frames[sb].im, cfg, first_pair_index + i, lat[i - lo], 0,
                         lat[i - lo].ny,
                         (dicb200_poi_record*)r.dev.p, cst, k ? &c->tcache2 : &c->tcache, (long)pairs[2 * i],
                         cfg->reference_policy == DICB200_POLICY_FIXED_FIRST ? (k ? &c->icache2 : &c->icache)
                                                                             : nullptr);
      if (staged_ok) {
        // the frames' last reader is this stream, also when enqueue_pair failed
        // after queueing some kernels: a later upload into either slot waits for them
        e = cudaEventRecord(k ? c->frames[sa].idle2 : c->frames[sa].idle, cst);
        if (e == cudaSuccess) e = cudaEventRecord(k ? c->frames[sb].idle2 : c->frames[sb].idle, cst);
        if (e != cudaSuccess && s == DICB200_OK) s = cuda_fail(e, "frame idle event", __FILE__, __LINE__);
      }
      if (s == DICB200_OK) {
        r.staged = !is_pinned(f.records);
        void* dst = f.records;
        if (e == cudaSuccess && r.staged) {
          if (r.stage_cap < bytes) {
            if (r.stage) cudaFreeHost(r.stage);
            r.stage = nullptr;
            r.stage_cap = 0;
            e = cudaMallocHost(&r.stage, bytes);
            if (e == cudaSuccess) r.stage_cap = bytes;
          }
          dst = r.stage;
        }
        // read-back on its own stream so the next pair's kernels start at once;
        // r.dev is rewritten only after finalize(r) has seen r.done
        if (e == cudaSuccess) e = cudaEventRecord(r.computed, cst);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->ds, r.computed, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, r.dev.p, bytes, cudaMemcpyDeviceToHost, c->ds);
        if (e == cudaSuccess) e = cudaEventRecord(r.done, c->ds);
        if (e != cudaSuccess) s = cuda_fail(e, "record read-back", __FILE__, __LINE__);
      }
      if (s != DICB200_OK) {
        fail_field(f, s);
        continue;
      }
      r.pair = (long)i;
      r.n = n;
      // prefetch the next pair's frames, then retire the pair two back (the one
      // before is still running beside this one)
      const size_t j = next_valid(i + 1);
      if (j < hi) {
        int ja = 0, jb = 0;
        stage_pair(j, &ja, &jb);  // an upload error resurfaces when pair j stages again
      }
      finalize(c->recs[(q + kRecSlots - 2) % kRecSlots]);
    }
    for (auto& r : c->recs) finalize(r);
    const dicb200_status rs = release_context(c);
    if (rs != DICB200_OK && result[wk] == DICB200_OK) {
      result[wk] = rs;
      errs[wk] = g_last_error;
    }
  };
  if (workers == 1) {
    run(0);
  } else {
    std::vector<std::thread> pool;
    for (int wk = 0; wk < workers; ++wk) pool.emplace_back(run, wk);
    for (auto& t : pool) t.join();
    cudaSetDevice(cur);
  }
  for (int wk = 0; wk < workers; ++wk)
    if (result[wk] != DICB200_OK) {
      set_error(errs[wk].c_str());
      return result[wk];
    }
  return DICB200_OK;
}

void dicb200_profile_enable(int on) { g_profile.store(on ? 1 : 0); }

int dicb200_profile_read(double* ms, uint64_t* launches) {
  for (int i = 0; i < DICB200_N_STAGES; ++i) {
    ms[i] = 0.0;
    launches[i] = 0;
  }
  std::vector<StageEvent> ev;
  {
    std::lock_guard<std::mutex> lk(g_profile_mu);
    ev.swap(g_events);
  }
  int rc = 0;
  for (auto& e : ev) {
    float t = 0.f;
    if (cudaEventSynchronize(e.b) != cudaSuccess || cudaEventElapsedTime(&t, e.a, e.b) != cudaSuccess) rc = 1;
    ms[e.stage] += t;
    launches[e.stage] += 1;
  }
  {
    std::lock_guard<std::mutex> lk(g_profile_mu);
    for (auto& e : ev) {
      g_event_pool.push_back(e.a);
      g_event_pool.push_back(e.b);
    }
  }
  return rc;
}

void dicb200_shutdown(void) {
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<DeviceContext*> idle;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    idle.swap(g_ctx_idle);
  }
  for (DeviceContext* c : idle) destroy_context(c);
  int n = dicb200_device_count();
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  if (n > 0) cudaSetDevice(cur);
}

}  // extern "C"
