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
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bfs.cuh"
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

struct StageTimer {
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  StageTimer(int s, cudaStream_t stream) : stage(s), st(stream) {
    if (!g_profile.load()) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~StageTimer() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> lk(g_profile_mu);
    g_events.push_back({stage, a, b});
  }
};
}  // namespace

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

void set_error(const char* msg) { g_last_error = msg ? msg : ""; }

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
  if (a->dtype != b->dtype || (a->dtype != DICB200_U8 && a->dtype != DICB200_U16))
    return invalid("unsupported pixel type (u8 or u16, identical for both images)");
  if (cfg->integer_method < 0 || cfg->integer_method > 2) return invalid("unknown integer method");
  if (cfg->subpixel_method < 0 || cfg->subpixel_method > 2) return invalid("unknown subpixel method");
  if (cfg->subpixel_method != DICB200_SUB_NONE) {
    int ppt, nt;
    if (!refine_plan(cfg->half_width, &ppt, &nt))
      return invalid("half_width too large for the device refiners (M <= 64)");
  }
  return DICB200_OK;
}

// Enqueue the whole per-pair chain for grid rows [rb, re) on `st`.
static dicb200_status enqueue_pair(const dicb200_image* ref, const dicb200_image* tgt, const dicb200_run_config* cfg,
                                   uint64_t pair_index, const Lattice& lat, int rb, int re,
                                   dicb200_poi_record* out_dev, cudaStream_t st) {
  const int rows = re - rb;
  if (rows <= 0) return DICB200_OK;
  const size_t nrec = (size_t)rows * lat.nx;
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
      if (!bfs_plan(b, 72 * 1024) && !bfs_plan(b, 200 * 1024)) {
        s = invalid("subset too large for the BFS tile (shared memory)");
        break;
      }
      BestPartial* partial = nullptr;
      if (b.n_chunks > 1) {
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
        cudaError_t e = bfs_launch(b, r1 - r0, st);
        if (e != cudaSuccess) s = cuda_fail(e, "bfs_launch(surface)", __FILE__, __LINE__);
        if (s == DICB200_OK) s = pso_walk_launch(p, st);
      }
      if (partial) cudaFreeAsync(partial, st);
    }
    cudaFreeAsync(surface, st);
    if (s != DICB200_OK) return s;
  }
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
    r.rec = out_dev;
    StageTimer tm(r.method == 0 ? 2 : 3, st);
    DICB200_CUDA_TRY(refine_launch(r, ref->dtype == DICB200_U8, st));
  }
  return DICB200_OK;
}

static size_t elem_size(int dtype) { return dtype == DICB200_U8 ? 1 : 2; }

// Upload a host image (tight pitch) on `st`.
static dicb200_status upload(const dicb200_image* host, dicb200_image* dev, void** buf, cudaStream_t st) {
  const size_t es = elem_size(host->dtype);
  const int pitch = host->pitch > 0 ? host->pitch : host->width;
  const size_t bytes = (size_t)host->width * host->height * es;
  DICB200_CUDA_TRY(cudaMallocAsync(buf, bytes, st));
  DICB200_CUDA_TRY(cudaMemcpy2DAsync(*buf, host->width * es, host->data, pitch * es, host->width * es, host->height,
                                     cudaMemcpyHostToDevice, st));
  *dev = *host;
  dev->pitch = host->width;
  dev->data = *buf;
  return DICB200_OK;
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  ~StreamGuard() {
    if (s) cudaStreamDestroy(s);
  }
};

static dicb200_status analyze_pair_on_stream(const dicb200_image* ref, const dicb200_image* tgt,
                                             const dicb200_run_config* cfg, uint64_t pair_index,
                                             dicb200_poi_record* out, size_t out_cap, size_t* out_count,
                                             cudaStream_t st, const dicb200_image* ref_dev_cached) {
  dicb200_status s = validate_pair(ref, tgt, cfg);
  if (s != DICB200_OK) return s;
  Lattice lat;
  s = make_lattice(ref->width, ref->height, cfg, &lat);
  if (s != DICB200_OK) return s;
  const size_t n = (size_t)lat.nx * lat.ny;
  if (out_count) *out_count = n;
  if (n > out_cap) {
    set_error("output capacity smaller than the grid");
    return DICB200_ERR_CAPACITY;
  }
  dicb200_image dref, dtgt;
  void *bref = nullptr, *btgt = nullptr, *brec = nullptr;
  if (ref_dev_cached) {
    dref = *ref_dev_cached;
  } else {
    s = upload(ref, &dref, &bref, st);
    if (s != DICB200_OK) return s;
  }
  s = upload(tgt, &dtgt, &btgt, st);
  if (s == DICB200_OK) {
    cudaError_t e = cudaMallocAsync(&brec, n * sizeof(dicb200_poi_record), st);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMallocAsync(records)", __FILE__, __LINE__);
  }
  if (s == DICB200_OK)
    s = enqueue_pair(&dref, &dtgt, cfg, pair_index, lat, 0, lat.ny, (dicb200_poi_record*)brec, st);
  if (s == DICB200_OK) {
    cudaError_t e = cudaMemcpyAsync(out, brec, n * sizeof(dicb200_poi_record), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(records)", __FILE__, __LINE__);
  }
  if (brec) cudaFreeAsync(brec, st);
  if (btgt) cudaFreeAsync(btgt, st);
  if (bref) cudaFreeAsync(bref, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (s == DICB200_OK && e != cudaSuccess) s = cuda_fail(e, "cudaStreamSynchronize", __FILE__, __LINE__);
  return s;
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
  StreamGuard g;
  DICB200_CUDA_TRY(cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking));
  return analyze_pair_on_stream(ref, tgt, cfg, pair_index, out, out_cap, out_count, g.s, nullptr);
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
  return enqueue_pair(ref, tgt, cfg, pair_index, lat, rb, re, out_dev, (cudaStream_t)stream);
}

dicb200_status dicb200_analyze_sequence(const dicb200_image* images, size_t n_images, const dicb200_run_config* cfg,
                                        dicb200_field* fields, size_t n_fields) {
  if (!has_device()) return no_device();
  if (n_images < 2) return invalid("insufficient images");
  if (n_fields != n_images - 1) return invalid("fields must hold one entry per pair");
  std::vector<int32_t> pairs(2 * (n_images - 1));
  dicb200_sequence_pairs(cfg->reference_policy, (int32_t)n_images, pairs.data());
  int ndev = dicb200_device_count();
  int workers = 1;
  if (cfg->mode == DICB200_MODE_IMAGE) workers = cfg->worker_count <= 0 ? ndev : std::min(cfg->worker_count, ndev);
  workers = std::max(1, std::min<int>(workers, (int)n_fields));
  std::vector<size_t> ranges(2 * workers);
  dicb200_partition_ranges(n_fields, workers, ranges.data());
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<dicb200_status> result(workers, DICB200_OK);
  std::vector<std::string> errs(workers);
  auto run = [&](int wk) {
    const int dev = workers == 1 ? cur : wk;
    cudaSetDevice(dev);
    StreamGuard g;
    if (cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking) != cudaSuccess) {
      result[wk] = DICB200_ERR_CUDA;
      errs[wk] = "stream creation failed";
      return;
    }
    // fixed_first: keep frame 0 resident on this device for all its pairs
    dicb200_image ref0{};
    void* ref0_buf = nullptr;
    const bool fixed = cfg->reference_policy == DICB200_POLICY_FIXED_FIRST;
    for (size_t i = ranges[2 * wk]; i < ranges[2 * wk + 1]; ++i) {
      const dicb200_image* a = &images[pairs[2 * i]];
      const dicb200_image* b = &images[pairs[2 * i + 1]];
      dicb200_field& f = fields[i];
      f.pair_index = (int32_t)i;
      f.ref_id = a->id;
      f.tgt_id = b->id;
      f.count = 0;
      f.error[0] = 0;
      const dicb200_image* cached = nullptr;
      if (fixed && validate_pair(a, b, cfg) == DICB200_OK) {
        if (!ref0_buf && upload(a, &ref0, &ref0_buf, g.s) != DICB200_OK) ref0_buf = nullptr;
        if (ref0_buf) cached = &ref0;
      }
      size_t cnt = 0;
      const dicb200_status s = analyze_pair_on_stream(a, b, cfg, i, f.records, f.capacity, &cnt, g.s, cached);
      f.count = s == DICB200_OK ? cnt : 0;
      f.status = s;
      if (s == DICB200_ERR_INVALID) {
        std::strncpy(f.error, g_last_error.c_str(), sizeof f.error - 1);
        f.error[sizeof f.error - 1] = 0;
      } else if (s != DICB200_OK) {
        result[wk] = s;
        errs[wk] = g_last_error;
        std::strncpy(f.error, g_last_error.c_str(), sizeof f.error - 1);
        f.error[sizeof f.error - 1] = 0;
      }
    }
    if (ref0_buf) {
      cudaFreeAsync(ref0_buf, g.s);
      cudaStreamSynchronize(g.s);
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
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  return rc;
}

void dicb200_shutdown(void) {
  int n = dicb200_device_count();
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  if (n > 0) cudaSetDevice(cur);
}

}  // extern "C"
