// TEST INFRASTRUCTURE ONLY (oracle/_ref): extern "C" entry points over the
// UNMODIFIED reference library (/root/reference/proj/core/src/*.cpp, compiled
// by oracle/Makefile into oracle/_ref/libdicref.so). Used by tests/ to pin the
// C restatement (oracle/dic_oracle.c) and to generate tests/golden/, and by
// bench.py --impl reference / cpu_baseline as the reference's own CPU path.
// Never linked into the product.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <random>
#include <string>
#include <vector>

#include "dic/correlation.hpp"
#include "dic/error.hpp"
#include "dic/image.hpp"
#include "dic/integer_search.hpp"
#include "dic/pipeline.hpp"
#include "dic/rng.hpp"
#include "dic/subpixel.hpp"
#include "dicb200.h"

namespace {

dic::RunConfig to_run_config(const dicb200_run_config& c) {
  // the reference has bilinear interpolation only (subpixel.cpp:59-128)
  if (c.interp != DICB200_INTERP_BILINEAR) throw std::runtime_error("reference build: bilinear interpolation only");
  dic::RunConfig r;
  r.integer_method = static_cast<dic::IntegerMethod>(c.integer_method);
  r.subpixel_method = static_cast<dic::SubpixelMethod>(c.subpixel_method);
  r.mode = static_cast<dic::ExecMode>(c.mode);
  r.reference_policy = static_cast<dic::ReferencePolicy>(c.reference_policy);
  r.worker_count = c.worker_count;
  r.search.search_radius = c.search_radius;
  r.search.bfs_domain = static_cast<dic::BfsDomain>(c.bfs_domain);
  r.search.particle_count = c.particle_count;
  r.search.max_generations = c.max_generations;
  r.search.stop_threshold = c.stop_threshold;
  r.search.c1 = c.c1;
  r.search.c2 = c.c2;
  r.search.rng_seed = c.rng_seed;
  r.refine.tol = c.tol;
  r.refine.max_iter = c.max_iter;
  r.grid.half_width = c.half_width;
  r.grid.spacing = c.spacing;
  r.grid.margin = c.margin;
  return r;
}

void copy_err(const char* what, char* err, size_t cap) {
  if (!err || cap == 0) return;
  std::strncpy(err, what, cap - 1);
  err[cap - 1] = 0;
}

void to_record(const dic::PoiRecord& r, dicb200_poi_record& o) {
  std::memset(&o, 0, sizeof o);
  o.x = r.x;
  o.y = r.y;
  o.u = r.u;
  o.v = r.v;
  o.zncc = r.zncc;
  o.converged = r.converged ? 1 : 0;
  o.iterations = r.iterations;
  o.evaluations = r.evaluations;
  o.update_evaluations = r.update_evaluations;
  o.status = -1;  // the reference does not expose which error aborted a POI
}

dic::GrayImage make_image(const double* px, int w, int h, int id = 0) {
  return dic::GrayImage(w, h, std::vector<double>(px, px + static_cast<size_t>(w) * h), id);
}

}  // namespace

extern "C" {

int dicref_analyze_pair(const double* ref, const double* tgt, int w, int h,
                        const dicb200_run_config* cfg, uint64_t pair_index,
                        dicb200_poi_record* out, size_t cap, size_t* count, char* err,
                        size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h, 0), b = make_image(tgt, w, h, 1);
    const dic::DisplacementField f = dic::analyze_pair(a, b, to_run_config(*cfg), pair_index);
    *count = f.records.size();
    if (f.records.size() > cap) return 4;
    for (size_t i = 0; i < f.records.size(); ++i) to_record(f.records[i], out[i]);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

// Timed variant for the CPU baseline: images are wrapped once; only
// analyze_pair runs between the two steady_clock reads (bench.cpp:36-48 style).
// `out` (optional, capacity `cap`) receives the last repeat's records, so the
// bench can check its own device records against the timed reference run.
int dicref_analyze_pair_timed(const double* ref, const double* tgt, int w, int h,
                              const dicb200_run_config* cfg, uint64_t pair_index, int repeats,
                              double* seconds_out, size_t* count, dicb200_poi_record* out, size_t cap,
                              char* err, size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h, 0), b = make_image(tgt, w, h, 1);
    const dic::RunConfig rc = to_run_config(*cfg);
    double best = 1e300;
    for (int r = 0; r < repeats; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const dic::DisplacementField f = dic::analyze_pair(a, b, rc, pair_index);
      const auto t1 = std::chrono::steady_clock::now();
      *count = f.records.size();
      const double s = std::chrono::duration<double>(t1 - t0).count();
      if (s < best) best = s;
      if (out && r == repeats - 1)
        for (size_t i = 0; i < f.records.size() && i < cap; ++i) to_record(f.records[i], out[i]);
    }
    *seconds_out = best;
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

int dicref_analyze_sequence(const double* const* images, size_t n, int w, int h,
                            const dicb200_run_config* cfg, dicb200_field* fields, size_t n_fields,
                            double* seconds_out) {
  std::vector<dic::GrayImage> imgs;
  imgs.reserve(n);
  for (size_t i = 0; i < n; ++i) imgs.push_back(make_image(images[i], w, h, static_cast<int>(i)));
  const auto t0 = std::chrono::steady_clock::now();
  const auto out = dic::analyze_sequence(imgs, to_run_config(*cfg));
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
  if (out.size() != n_fields) return 4;
  for (size_t i = 0; i < out.size(); ++i) {
    dicb200_field& f = fields[i];
    f.pair_index = out[i].pair_index;
    f.ref_id = out[i].ref_id;
    f.tgt_id = out[i].tgt_id;
    f.status = out[i].failed() ? 1 : 0;
    std::memset(f.error, 0, sizeof f.error);
    copy_err(out[i].error.c_str(), f.error, sizeof f.error);
    f.count = out[i].records.size();
    for (size_t k = 0; k < out[i].records.size() && k < f.capacity; ++k)
      to_record(out[i].records[k], f.records[k]);
  }
  return 0;
}

// --- per-subset operators (unit-level pins) ------------------------------

// Returns 0 and the coefficient, or 1 with the error message.
int dicref_zncc(const double* ref, const double* tgt, int w, int h, int cx, int cy, int m,
                int dx, int dy, double* out, char* err, size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h), b = make_image(tgt, w, h);
    const dic::SubsetSpec spec{cx, cy, m};
    *out = dic::zncc(dic::subset_stats(a, spec), b, spec, dx, dy);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

// method: 0 bfs, 1 pso, 2 mpso. result: dx, dy, generations_used; zncc; evals.
int dicref_integer_search(const double* ref, const double* tgt, int w, int h, int cx, int cy,
                          int m, const dicb200_run_config* cfg, uint64_t stream_seed,
                          int32_t* ires /*3*/, double* zncc, int64_t* evals /*2*/, char* err,
                          size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h), b = make_image(tgt, w, h);
    const dic::SubsetSpec spec{cx, cy, m};
    const dic::RunConfig rc = to_run_config(*cfg);
    const auto stats = dic::subset_stats(a, spec);
    dic::IntegerResult r;
    dic::CorrelationMemo memo;
    dic::StreamRng rng(stream_seed);
    if (cfg->integer_method == 0)
      r = dic::bfs_search(stats, b, spec, rc.search);
    else if (cfg->integer_method == 1)
      r = dic::pso_search(stats, b, spec, rc.search, memo, rng);
    else
      r = dic::mpso_search(stats, b, spec, rc.search, memo, rng);
    ires[0] = r.dx;
    ires[1] = r.dy;
    ires[2] = r.generations_used;
    *zncc = r.zncc;
    evals[0] = r.evaluations;
    evals[1] = r.update_evaluations;
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

// method: 0 nr, 1 icgn. out: u, v, zncc, ux, uy, vx, vy; iters_conv: iterations, converged.
int dicref_refine(const double* ref, const double* tgt, int w, int h, int cx, int cy, int m,
                  int init_dx, int init_dy, int method, double tol, int max_iter, double* out,
                  int32_t* iters_conv, char* err, size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h), b = make_image(tgt, w, h);
    const dic::SubsetSpec spec{cx, cy, m};
    dic::RefineConfig rc;
    rc.tol = tol;
    rc.max_iter = max_iter;
    dic::SubpixelResult r;
    if (method == 0) {
      r = dic::refine_nr(dic::subset_stats(a, spec), b, spec, {init_dx, init_dy}, rc);
    } else {
      const auto st = dic::icgn_precompute(a, spec);
      r = dic::refine_icgn(st, b, spec, {init_dx, init_dy}, rc);
    }
    out[0] = r.u;
    out[1] = r.v;
    out[2] = r.zncc;
    out[3] = r.warp.ux;
    out[4] = r.warp.uy;
    out[5] = r.warp.vx;
    out[6] = r.warp.vy;
    iters_conv[0] = r.iterations;
    iters_conv[1] = r.converged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

// IC-GN precompute pin: Hessian (36, row-major) and condition number.
int dicref_icgn_hessian(const double* ref, int w, int h, int cx, int cy, int m, double* hess,
                        double* condition, char* err, size_t errcap) {
  try {
    const dic::GrayImage a = make_image(ref, w, h);
    const auto st = dic::icgn_precompute(a, dic::SubsetSpec{cx, cy, m});
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) hess[i * 6 + j] = st.hessian(i, j);
    *condition = st.condition;
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

double dicref_interp_bilinear(const double* img, int w, int h, double x, double y, int* ok) {
  try {
    *ok = 1;
    return dic::interp_bilinear(make_image(img, w, h), x, y);
  } catch (const std::exception&) {
    *ok = 0;
    return 0.0;
  }
}

uint64_t dicref_derive_stream_seed(uint64_t seed, uint64_t pair, uint64_t subset) {
  return dic::derive_stream_seed(seed, pair, subset);
}

// n raw mt19937_64 outputs (std::mt19937_64 via StreamRng::next_bits).
void dicref_mt64(uint64_t seed, size_t n, uint64_t* out) {
  dic::StreamRng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.next_bits();
}

void dicref_uniform01(uint64_t seed, size_t n, double* out) {
  dic::StreamRng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.uniform01();
}

int dicref_grid(int w, int h, int half_width, int spacing, int margin, int32_t* xy, size_t cap,
                size_t* count, char* err, size_t errcap) {
  try {
    const dic::GrayImage img(w, h, std::vector<double>(static_cast<size_t>(w) * h, 0.0));
    const auto g = dic::grid_subsets(img, half_width, spacing, margin);
    *count = g.size();
    for (size_t i = 0; i < g.size() && i < cap; ++i) {
      xy[2 * i] = g[i].center_x;
      xy[2 * i + 1] = g[i].center_y;
    }
    return 0;
  } catch (const std::exception& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

unsigned dicref_hardware_threads(void) { return std::thread::hardware_concurrency(); }

// dic::load_image / dic::load_sequence (image.cpp:60-138) for the ingestion
// parity tests: 0 = ok, 1 = dic::Error (message copied to err).
int dicref_load_image(const char* path, double* out, size_t cap, int* w, int* h, char* err, size_t errcap) {
  try {
    const dic::GrayImage img = dic::load_image(path);
    *w = img.width();
    *h = img.height();
    if (out && cap >= img.pixels().size()) std::copy(img.pixels().begin(), img.pixels().end(), out);
    return 0;
  } catch (const dic::Error& e) {
    std::snprintf(err, errcap, "%s", e.what());
    return 1;
  }
}

int dicref_load_sequence(const char* dir, const char* pattern, double* out, size_t cap, int* n, int* w, int* h,
                         int* ids, size_t ids_cap, char* err, size_t errcap) {
  try {
    const auto seq = dic::load_sequence(dir, pattern);
    *n = (int)seq.size();
    *w = seq.front().width();
    *h = seq.front().height();
    const size_t per = seq.front().pixels().size();
    for (size_t i = 0; i < seq.size(); ++i) {
      if (i < ids_cap) ids[i] = seq[i].id();
      if (out && cap >= per * (i + 1)) std::copy(seq[i].pixels().begin(), seq[i].pixels().end(), out + per * i);
    }
    return 0;
  } catch (const dic::Error& e) {
    std::snprintf(err, errcap, "%s", e.what());
    return 1;
  }
}

}  // extern "C"

// ---- f-4: the reference's generators and accuracy sweep (synth.cpp, accuracy.cpp) ----
#include "dic/accuracy.hpp"
#include "dic/synth.hpp"

namespace {
dic::SpeckleParams to_speckle(const dicb200_speckle_params& p) {
  dic::SpeckleParams s;
  s.blob_count = p.blob_count;
  s.sigma_min = p.sigma_min;
  s.sigma_max = p.sigma_max;
  s.amp_min = p.amp_min;
  s.amp_max = p.amp_max;
  s.background = p.background;
  s.variance_floor = p.variance_floor;
  s.texture_window = p.texture_window;
  return s;
}
dic::WarpSpec to_warp(const dicb200_warp_spec& w) {
  dic::WarpSpec s;
  s.u = w.u;
  s.v = w.v;
  s.ux = w.ux;
  s.uy = w.uy;
  s.vx = w.vx;
  s.vy = w.vy;
  return s;
}
}  // namespace

extern "C" {

int dicref_synth_speckle(int w, int h, uint64_t seed, const dicb200_speckle_params* p, double* out, char* err,
                         size_t errcap) {
  try {
    const dic::GrayImage img = dic::synth_speckle(w, h, seed, to_speckle(*p));
    std::copy(img.pixels().begin(), img.pixels().end(), out);
    return 0;
  } catch (const dic::Error& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

int dicref_synth_warped_pair(const double* ref, int w, int h, const dicb200_warp_spec* warp, double* target,
                             uint8_t* mask, char* err, size_t errcap) {
  try {
    const auto [tgt, truth] = dic::synth_warped_pair(make_image(ref, w, h), to_warp(*warp));
    std::copy(tgt.pixels().begin(), tgt.pixels().end(), target);
    if (mask)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) mask[(size_t)y * w + x] = truth.valid(x, y) ? 1 : 0;
    return 0;
  } catch (const dic::Error& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

// dic::run_accuracy_sweep on the reference's own (unquantized) frames.
int dicref_accuracy_sweep(const int32_t* combos, size_t n, const dicb200_sweep_config* c, dicb200_combo_accuracy* out,
                          int* warp_count, int* poi_count, double* elapsed, char* err, size_t errcap) {
  try {
    dic::SweepConfig s;
    s.width = c->width;
    s.height = c->height;
    s.seed = c->seed;
    s.speckle = to_speckle(c->speckle);
    s.base = to_run_config(c->base);
    s.fractions.assign(c->fractions, c->fractions + c->n_fractions);
    s.offsets.assign(c->offsets, c->offsets + c->n_offsets);
    std::vector<std::pair<dic::IntegerMethod, dic::SubpixelMethod>> cs;
    for (size_t i = 0; i < n; ++i)
      cs.emplace_back(static_cast<dic::IntegerMethod>(combos[2 * i]), static_cast<dic::SubpixelMethod>(combos[2 * i + 1]));
    const dic::SweepReport r = dic::run_accuracy_sweep(cs, s);
    for (size_t i = 0; i < n; ++i) {
      const auto& a = r.combos[i];
      out[i].integer_method = static_cast<int32_t>(a.integer_method);
      out[i].subpixel_method = static_cast<int32_t>(a.subpixel_method);
      out[i].max_err = a.max_err;
      out[i].mean_err = a.mean_err;
      out[i].measurements = a.measurements;
      out[i].unconverged = a.unconverged;
      out[i].pass = a.pass ? 1 : 0;
      out[i].mean_flagged = a.mean_flagged ? 1 : 0;
    }
    *warp_count = r.warp_count;
    *poi_count = r.poi_count;
    *elapsed = r.elapsed_s;
    return 0;
  } catch (const dic::Error& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

}  // extern "C"

// ---- f-3 / f-4: field CSV and the bench matrix (pipeline.cpp:216-238, bench.cpp) ----
#include "dic/bench.hpp"

namespace {
dic::BenchRecord to_bench(const dicb200_bench_record& r) {
  dic::BenchRecord b;
  b.cell.integer_method = static_cast<dic::IntegerMethod>(r.cell.integer_method);
  b.cell.subpixel_method = static_cast<dic::SubpixelMethod>(r.cell.subpixel_method);
  b.cell.mode = static_cast<dic::ExecMode>(r.cell.mode);
  b.dataset_id = r.dataset_id;
  b.repeats = r.repeats;
  b.pair_count = r.pair_count;
  b.mean_s = r.mean_s;
  b.stddev_s = r.stddev_s;
  b.per_pair_s = r.per_pair_s;
  b.frame_rate_hz = r.frame_rate_hz;
  b.total_evaluations = r.total_evaluations;
  b.failed = r.failed != 0;
  b.error = r.error;
  return b;
}
dic::BenchReport to_report(const dicb200_bench_record* recs, size_t n, const char* dataset_id) {
  dic::BenchReport rep;
  rep.dataset_id = dataset_id;
  for (size_t i = 0; i < n; ++i) rep.records.push_back(to_bench(recs[i]));
  return rep;
}
}  // namespace

extern "C" {

int dicref_field_csv(const dicb200_poi_record* recs, size_t n, char* out, size_t cap, size_t* needed) {
  dic::DisplacementField f;
  for (size_t i = 0; i < n; ++i) {
    dic::PoiRecord r;
    r.x = recs[i].x;
    r.y = recs[i].y;
    r.u = recs[i].u;
    r.v = recs[i].v;
    r.zncc = recs[i].zncc;
    r.converged = recs[i].converged != 0;
    r.iterations = recs[i].iterations;
    r.evaluations = recs[i].evaluations;
    f.records.push_back(r);
  }
  const std::string s = dic::field_csv_string(f);
  *needed = s.size() + 1;
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

int dicref_bench_csvs(const dicb200_bench_record* recs, size_t n, const char* dataset_id, const char* times,
                      const char* records, const char* ratios, char* err, size_t errcap) {
  try {
    const dic::BenchReport rep = to_report(recs, n, dataset_id);
    dic::write_times_csv(rep, times);
    dic::write_records_csv(rep, records);
    dic::write_ratios_csv(dic::derive_ratios(rep), ratios);
    return 0;
  } catch (const dic::Error& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

int dicref_auto_repeats(double s) { return dic::auto_repeats(s); }

// dic::run_bench on the CPU (tiny datasets only: tests).
int dicref_run_bench(const dicb200_bench_cell* cells, size_t n, const char* dir, const char* pattern,
                     const dicb200_run_config* base, int auto_bands, int fixed, const char* scratch,
                     dicb200_bench_record* out, char* err, size_t errcap) {
  try {
    std::vector<dic::BenchCell> cs;
    for (size_t i = 0; i < n; ++i) {
      dic::BenchCell c;
      c.integer_method = static_cast<dic::IntegerMethod>(cells[i].integer_method);
      c.subpixel_method = static_cast<dic::SubpixelMethod>(cells[i].subpixel_method);
      c.mode = static_cast<dic::ExecMode>(cells[i].mode);
      cs.push_back(c);
    }
    dic::RepeatsPolicy rp;
    rp.auto_bands = auto_bands != 0;
    rp.fixed = fixed;
    const dic::BenchReport rep = dic::run_bench(cs, dir, pattern, to_run_config(*base), rp, scratch);
    for (size_t i = 0; i < n; ++i) {
      const dic::BenchRecord& r = rep.records[i];
      std::memset(&out[i], 0, sizeof out[i]);
      out[i].cell = cells[i];
      out[i].repeats = r.repeats;
      out[i].pair_count = r.pair_count;
      out[i].failed = r.failed ? 1 : 0;
      out[i].mean_s = r.mean_s;
      out[i].stddev_s = r.stddev_s;
      out[i].per_pair_s = r.per_pair_s;
      out[i].frame_rate_hz = r.frame_rate_hz;
      out[i].total_evaluations = r.total_evaluations;
      std::snprintf(out[i].dataset_id, sizeof out[i].dataset_id, "%s", r.dataset_id.c_str());
      std::snprintf(out[i].error, sizeof out[i].error, "%s", r.error.c_str());
    }
    return 0;
  } catch (const dic::Error& e) {
    copy_err(e.what(), err, errcap);
    return 1;
  }
}

}  // extern "C"
