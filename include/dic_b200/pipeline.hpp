// Drop-in C++ shim: the reference's dic::analyze_pair / dic::analyze_sequence
// signatures (/root/reference/proj/core/include/dic/pipeline.hpp:76-80) served
// by the B200 library through the C-ABI (include/dicb200.h).
//
// Header-only; include it inside the reference build (it needs the reference's
// dic/pipeline.hpp) and link libdicb200.so:
//
//   #include "dic_b200/pipeline.hpp"
//   dic::DisplacementField f = dic::b200::analyze_pair(ref, tgt, cfg, pair_index);
//
// Semantics: identical records to dic::analyze_pair (same grid order, same
// per-POI failure semantics). Pair-level failures throw dic::Error with the
// reference's message. Integer GrayImage levels in [0, 65535] (every 8/16-bit
// camera frame) travel as u8/u16 to the exact-integer kernels; any other levels
// (e.g. the reference's fractional synthetic frames) are passed as the
// GrayImage's own doubles to the exact fp64 path (see detail::Frames).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <future>
#include <memory>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "dic/error.hpp"
#include "dic/pipeline.hpp"
#include "dicb200.h"

namespace dic {
namespace b200 {

namespace detail {

inline dicb200_run_config to_c(const RunConfig& c) {
  dicb200_run_config r;
  dicb200_default_config(&r);
  r.integer_method = static_cast<int32_t>(c.integer_method);
  r.subpixel_method = static_cast<int32_t>(c.subpixel_method);
  r.mode = static_cast<int32_t>(c.mode);
  r.reference_policy = static_cast<int32_t>(c.reference_policy);
  r.worker_count = c.worker_count;
  r.search_radius = c.search.search_radius;
  r.bfs_domain = static_cast<int32_t>(c.search.bfs_domain);
  r.particle_count = c.search.particle_count;
  r.max_generations = c.search.max_generations;
  r.stop_threshold = c.search.stop_threshold;
  r.c1 = c.search.c1;
  r.c2 = c.search.c2;
  r.rng_seed = c.search.rng_seed;
  r.tol = c.refine.tol;
  r.max_iter = c.refine.max_iter;
  r.half_width = c.grid.half_width;
  r.spacing = c.grid.spacing;
  r.margin = c.grid.margin;
  return r;
}

// Pinned host blocks reused across calls (cudaMallocHost is slow; frames are
// uploaded asynchronously from pinned memory). Grow-only, process lifetime.
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool pool;
    return pool;
  }
  // `count` blocks of at least `bytes` each, held until release()
  std::vector<void*> take(size_t count, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<void*> out;
    for (auto it = free_.begin(); it != free_.end() && out.size() < count;) {
      if (it->second >= bytes) {
        out.push_back(it->first);
        cap_[it->first] = it->second;
        it = free_.erase(it);
      } else {
        ++it;
      }
    }
    while (out.size() < count) {
      void* p = dicb200_host_alloc(bytes);
      if (!p) {
        for (void* q : out) free_.emplace_back(q, cap_[q]);
        throw std::runtime_error("dicb200: pinned host allocation failed");
      }
      cap_[p] = bytes;
      out.push_back(p);
    }
    return out;
  }
  void release(const std::vector<void*>& blocks) {
    std::lock_guard<std::mutex> lk(mu_);
    for (void* p : blocks) free_.emplace_back(p, cap_[p]);
  }

 private:
  std::mutex mu_;
  std::vector<std::pair<void*, size_t>> free_;
  std::map<void*, size_t> cap_;
};

// GrayImages (doubles) -> device gray levels, one multithreaded pass per frame
// (dicb200_pack_gray). Integer levels in [0, 65535] map losslessly; when every
// level of every frame is <= 255 they travel as u8 (narrowed in place). When a
// frame has any other level (non-integral, e.g. the reference's synth_speckle /
// synth_warped_pair frames, or outside [0, 65535]) every frame of the call is
// handed over as its GrayImage's doubles (DICB200_F64): the integer search then
// evaluates the reference's zncc in its own order (bit-identical values) and
// the refiners gather fp32 samples of the fp64 images.
class Frames {
 public:
  explicit Frames(const std::vector<const GrayImage*>& images) : pool_(PinnedPool::get()) {
    const size_t n = images.size();
    size_t px = 0;
    for (const GrayImage* g : images) px = std::max(px, static_cast<size_t>(g->width()) * g->height());
    blocks_ = pool_.take(n, std::max<size_t>(px * 2, 16));
    imgs_.resize(n);
    int maxv = 0;
    bool fp = false;  // some frame is not integral in [0, 65535]: all frames as doubles
    bool same = true;  // frames of one size pack in one batched call
    for (const GrayImage* g : images)
      same = same && g->width() == images[0]->width() && g->height() == images[0]->height();
    std::vector<int32_t> frac(n, 0), mx(n, 0);
    if (same && n > 0) {
      std::vector<const double*> src(n);
      std::vector<uint16_t*> dst(n);
      for (size_t i = 0; i < n; ++i) {
        src[i] = images[i]->pixels().data();
        dst[i] = static_cast<uint16_t*>(blocks_[i]);
      }
      const dicb200_status st = dicb200_pack_gray_batch(src.data(), static_cast<int32_t>(n), images[0]->width(),
                                                        images[0]->height(), images[0]->width(), dst.data(),
                                                        frac.data(), mx.data(), 0);
      fp = st != DICB200_OK;
    } else {
      for (size_t i = 0; i < n && !fp; ++i) {
        const GrayImage& g = *images[i];
        fp = dicb200_pack_gray(g.pixels().data(), g.width(), g.height(), g.width(), 1,
                               static_cast<uint16_t*>(blocks_[i]), &frac[i], &mx[i], 0) != DICB200_OK;
      }
    }
    for (size_t i = 0; i < n && !fp; ++i) {
      if (frac[i]) {
        fp = true;
        break;
      }
      const GrayImage& g = *images[i];
      dicb200_image& im = imgs_[i];
      im.width = g.width();
      im.height = g.height();
      im.pitch = g.width();
      im.id = g.id();
      im.dtype = DICB200_U16;
      im.data = blocks_[i];
      im.bits = 1;
      while (im.bits < 16 && (1 << im.bits) - 1 < mx[i]) ++im.bits;
      maxv = std::max(maxv, (int)mx[i]);
    }
    if (fp) {  // the GrayImages' own doubles (read-only for the call); non-finite levels fail the pair
      for (size_t i = 0; i < n; ++i) {
        const GrayImage& g = *images[i];
        dicb200_image& im = imgs_[i];
        im.width = g.width();
        im.height = g.height();
        im.pitch = g.width();
        im.id = g.id();
        im.dtype = DICB200_F64;
        im.bits = 0;
        im.data = g.pixels().data();
      }
    } else if (maxv <= 255) {  // every frame 8-bit: u8 (one byte plane on the device)
      auto narrow = [this](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i) {
          dicb200_image& im = imgs_[i];
          const uint16_t* s16 = static_cast<const uint16_t*>(im.data);
          uint8_t* d8 = static_cast<uint8_t*>(const_cast<void*>(im.data));
          const size_t m = static_cast<size_t>(im.width) * im.height;
          for (size_t k = 0; k < m; ++k) d8[k] = static_cast<uint8_t>(s16[k]);  // in place, front to back
          im.dtype = DICB200_U8;
          im.bits = 8;
        }
      };
      const size_t nt = std::min<size_t>(n, std::max(1u, std::thread::hardware_concurrency()));
      if (nt <= 1 || px < (size_t(1) << 18)) {
        narrow(0, n);
      } else {  // whole frames per thread
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nt; ++t) pool.emplace_back(narrow, n * t / nt, n * (t + 1) / nt);
        for (auto& th : pool) th.join();
      }
    } else {  // one dtype for all frames (the C-ABI's rule); bits = the widest frame's
      int bits = 1;
      for (const dicb200_image& im : imgs_) bits = std::max(bits, static_cast<int>(im.bits));
      for (dicb200_image& im : imgs_) im.bits = bits;
    }
  }
  ~Frames() { pool_.release(blocks_); }
  Frames(const Frames&) = delete;
  Frames& operator=(const Frames&) = delete;
  const dicb200_image* data() const { return imgs_.data(); }
  const dicb200_image& operator[](size_t i) const { return imgs_[i]; }

 private:
  PinnedPool& pool_;
  std::vector<void*> blocks_;
  std::vector<dicb200_image> imgs_;
};

inline PoiRecord to_record(const dicb200_poi_record& r) {
  PoiRecord o;
  o.x = r.x;
  o.y = r.y;
  o.u = r.u;
  o.v = r.v;
  o.zncc = r.zncc;
  o.converged = r.converged != 0;
  o.iterations = r.iterations;
  o.evaluations = static_cast<long>(r.evaluations);
  o.update_evaluations = static_cast<long>(r.update_evaluations);
  return o;
}

[[noreturn]] inline void raise(dicb200_status st) {
  if (st == DICB200_ERR_INVALID) throw Error(dicb200_last_error_message());
  throw std::runtime_error(dicb200_last_error_message());
}

}  // namespace detail

inline DisplacementField analyze_pair(const GrayImage& reference, const GrayImage& target,
                                      const RunConfig& cfg, std::uint64_t pair_index = 0) {
  if (reference.width() != target.width() || reference.height() != target.height())
    throw Error("dimension mismatch");
  const dicb200_run_config c = detail::to_c(cfg);
  size_t n = 0;
  dicb200_status st = dicb200_grid_size(reference.width(), reference.height(), &c, &n);
  if (st != DICB200_OK) detail::raise(st);
  const detail::Frames fr({&reference, &target});
  std::vector<dicb200_poi_record> recs(n);
  st = dicb200_analyze_pair(&fr[0], &fr[1], &c, pair_index, recs.data(), recs.size(), &n);
  if (st != DICB200_OK) detail::raise(st);
  DisplacementField f;
  f.pair_index = static_cast<int>(pair_index);
  f.ref_id = reference.id();
  f.tgt_id = target.id();
  f.records.reserve(n);
  for (size_t i = 0; i < n; ++i) f.records.push_back(detail::to_record(recs[i]));
  return f;
}

// pipeline.cpp:182-214 semantics: pairs from sequence_pairs(cfg.reference_policy),
// fields in pair order, per-pair dic::Error -> field.error. The sequence goes
// to dicb200_analyze_sequence_cb (pipelined uploads / compute / read-back;
// cfg.mode == image_parallel shards contiguous pair chunks over
// min(worker_count, devices) devices, as the reference shards them over worker
// threads) in chunks of pairs: while the device works on one chunk, the host
// packs the next chunk's GrayImage doubles (all cores), so for long sequences
// of large frames only the first chunk's packing is exposed; up to two chunk
// calls are in flight, so the device does not drain between them. Each chunk
// call carries its first pair index, so RNG keys and results are those of one call.
// DICB200_SHIM_CHUNK=<pairs> overrides the chunk length (0 = one call).
inline std::vector<DisplacementField> analyze_sequence(const std::vector<GrayImage>& images,
                                                       const RunConfig& cfg) {
  const auto pairs = sequence_pairs(cfg.reference_policy, static_cast<int>(images.size()));
  const dicb200_run_config c = detail::to_c(cfg);
  const bool trace = std::getenv("DICB200_SHIM_TRACE") != nullptr;  // phase times on stderr
  const size_t np = pairs.size();
  // chunking pays when packing a chunk takes long enough to be worth hiding
  size_t px = 0;
  for (const GrayImage& g : images) px = std::max(px, static_cast<size_t>(g.width()) * g.height());
  size_t chunk = (np >= 16 && px >= (size_t(1) << 20)) ? 8 : np;  // measured on C5: 8 and 16 within 2 %
  if (const char* e = std::getenv("DICB200_SHIM_CHUNK")) chunk = std::atoi(e) > 0 ? std::atoi(e) : np;
  chunk = std::max<size_t>(1, std::min(chunk, std::max<size_t>(np, 1)));

  struct Ctx {
    const std::vector<GrayImage>* images;
    const std::vector<std::pair<int, int>>* pairs;
    size_t first;  // global index of the chunk's first pair
    std::vector<dicb200_field> cf;
    std::vector<DisplacementField>* fields;
  };
  std::vector<DisplacementField> fields(np);
  size_t cap = 0;
  std::vector<size_t> counts(np, 0);
  for (size_t i = 0; i < np; ++i) {
    const GrayImage& a = images[pairs[i].first];
    if (dicb200_grid_size(a.width(), a.height(), &c, &counts[i]) != DICB200_OK) counts[i] = 0;
    cap = std::max(cap, counts[i]);
  }
  // records are read back straight into pinned blocks (no staging copy, no
  // zero fill) and each field is converted as soon as it is final, on the
  // library's worker thread, while the device runs the following pairs
  // two chunk calls may be in flight (the second ramps up while the first
  // drains): two sets of record blocks, alternating
  const size_t nchunks = (np + chunk - 1) / chunk;
  detail::PinnedPool& pool = detail::PinnedPool::get();
  const std::vector<void*> blocks =
      pool.take(nchunks > 1 ? 2 * chunk : chunk, std::max<size_t>(cap, 1) * sizeof(dicb200_poi_record));
  struct Release {
    detail::PinnedPool& pool;
    const std::vector<void*>& blocks;
    ~Release() { pool.release(blocks); }
  } release{pool, blocks};
  auto ready = [](void* user, size_t i) {
    Ctx& x = *static_cast<Ctx*>(user);
    const size_t gi = x.first + i;
    DisplacementField& f = (*x.fields)[gi];
    const dicb200_field& cf = x.cf[i];
    f.pair_index = static_cast<int>(gi);
    f.ref_id = (*x.images)[(*x.pairs)[gi].first].id();
    f.tgt_id = (*x.images)[(*x.pairs)[gi].second].id();
    if (cf.status != DICB200_OK) {
      f.error = cf.error;
      return;
    }
    f.records.reserve(cf.count);
    for (size_t k = 0; k < cf.count; ++k) f.records.push_back(detail::to_record(cf.records[k]));
  };
  // frames of pairs [a, b): the library derives the same pairs from them
  // (fixed_first: frame 0 then the targets; update_every_pair: frames a .. b)
  auto frames_of = [&](size_t a, size_t b) {
    std::vector<const GrayImage*> ptrs;
    ptrs.push_back(&images[pairs[a].first]);
    for (size_t i = a; i < b; ++i) ptrs.push_back(&images[pairs[i].second]);
    return std::shared_ptr<detail::Frames>(new detail::Frames(ptrs));
  };
  // one chunk call; a failure of the call itself (not of a pair) is returned with its message
  struct CallResult {
    dicb200_status st = DICB200_OK;
    std::string msg;
  };
  auto call = [&](size_t k, std::shared_ptr<detail::Frames> fr) {
    const size_t a = k * chunk, b = std::min(np, a + chunk);
    Ctx ctx;
    ctx.images = &images;
    ctx.pairs = &pairs;
    ctx.first = a;
    ctx.fields = &fields;
    ctx.cf.resize(b - a);
    for (size_t i = a; i < b; ++i) {
      ctx.cf[i - a] = dicb200_field{};
      ctx.cf[i - a].records = static_cast<dicb200_poi_record*>(blocks[(k & 1) * chunk + (i - a)]);
      ctx.cf[i - a].capacity = counts[i];
    }
    CallResult r;
    r.st = dicb200_analyze_sequence_cb(fr->data(), b - a + 1, &c, ctx.cf.data(), ctx.cf.size(),
                                       static_cast<uint64_t>(a), ready, &ctx);
    if (r.st != DICB200_OK) r.msg = dicb200_last_error_message();
    return r;
  };
  double pack_ms = 0.0, wait_ms = 0.0;
  auto ms_since = [](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
  };
  const auto t_begin = std::chrono::steady_clock::now();
  std::shared_ptr<detail::Frames> cur = frames_of(0, std::min(np, chunk));
  pack_ms = ms_since(t_begin);
  CallResult bad;
  if (nchunks == 1) {
    bad = call(0, cur);
  } else {
    std::vector<std::future<CallResult>> runs(nchunks);
    auto settle = [&](size_t k) {
      if (!runs[k].valid()) return;
      const CallResult r = runs[k].get();
      if (r.st != DICB200_OK && bad.st == DICB200_OK) bad = r;
    };
    for (size_t k = 0; k < nchunks && bad.st == DICB200_OK; ++k) {
      if (k >= 2) settle(k - 2);  // its record blocks are reused by call k
      if (bad.st != DICB200_OK) break;
      runs[k] = std::async(std::launch::async, call, k, cur);
      if (k + 1 < nchunks) {
        const auto t2 = std::chrono::steady_clock::now();
        cur = frames_of((k + 1) * chunk, std::min(np, (k + 2) * chunk));  // packed while calls k - 1, k run
        wait_ms += ms_since(t2);
      }
    }
    for (size_t k = 0; k < nchunks; ++k) settle(k);
  }
  const double total_ms = ms_since(t_begin);
  if (bad.st != DICB200_OK) {
    if (bad.st == DICB200_ERR_INVALID) throw Error(bad.msg);
    throw std::runtime_error(bad.msg);
  }
  if (trace)
    std::fprintf(stderr,
                 "[dicb200 shim] %zu pairs in %zu call(s), two in flight: first chunk packed in %.1f ms, later "
                 "chunks packed in %.1f ms beside the device work, total %.1f ms\n",
                 np, nchunks, pack_ms, wait_ms, total_ms);
  return fields;
}

}  // namespace b200
}  // namespace dic
