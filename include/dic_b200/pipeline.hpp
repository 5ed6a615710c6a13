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
// reference's message. GrayImage values must be integers in [0, 65535]
// (every 8/16-bit camera frame is) or fractional levels in [0, 255], which are
// carried as 8.8 fixed point (see detail::pack); anything else throws dic::Error.
#pragma once

#include <cmath>
#include <cstdint>
#include <string>
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

// GrayImage (doubles) -> packed u8/u16 + descriptor. Integer gray levels in
// [0, 65535] map losslessly. Non-integer levels in [0, 255] (e.g. the
// reference's synth_speckle / synth_warped_pair frames) are carried with 8
// fractional bits: u16 = round(256 v). ZNCC, the IC-GN / NR steps and every
// decision derived from them are invariant to a positive gray-level scale, so
// only the 2^-9 quantisation of each sample separates the result from the
// reference's doubles. Anything else (negative, > 65535, fractional above
// 255, non-finite) throws dic::Error.
struct Packed {
  std::vector<uint8_t> u8;
  std::vector<uint16_t> u16;
  dicb200_image img{};
};

inline bool is_integral(const GrayImage& g) {
  for (double v : g.pixels())
    if (v != std::floor(v)) return false;
  return true;
}

inline void pack(const GrayImage& g, Packed& out, bool force16) {
  const auto& px = g.pixels();
  const bool frac = !is_integral(g);
  double mx = 0.0;
  for (double v : px) {
    if (!(v >= 0.0) || v > (frac ? 255.0 : 65535.0))
      throw Error(frac ? "dicb200: fractional gray levels must lie in [0, 255]"
                       : "dicb200: gray levels must be integers in [0, 65535]");
    mx = v > mx ? v : mx;
  }
  out.img.width = g.width();
  out.img.height = g.height();
  out.img.pitch = g.width();
  out.img.id = g.id();
  if (frac) {
    out.u16.resize(px.size());
    for (size_t i = 0; i < px.size(); ++i) out.u16[i] = static_cast<uint16_t>(std::lround(px[i] * 256.0));
    out.img.dtype = DICB200_U16;
    out.img.bits = 16;
    out.img.data = out.u16.data();
  } else if (mx <= 255.0 && !force16) {
    out.u8.assign(px.begin(), px.end());
    out.img.dtype = DICB200_U8;
    out.img.bits = 8;
    out.img.data = out.u8.data();
  } else {
    out.u16.assign(px.begin(), px.end());
    out.img.dtype = DICB200_U16;
    int bits = 1;
    while (bits < 16 && (1 << bits) - 1 < mx) ++bits;
    out.img.bits = bits;
    out.img.data = out.u16.data();
  }
}

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

inline bool max_is_u8(const GrayImage& g) {
  for (double v : g.pixels())
    if (v > 255.0) return false;
  return is_integral(g);  // fractional frames travel as 8.8 fixed point (u16)
}

}  // namespace detail

inline DisplacementField analyze_pair(const GrayImage& reference, const GrayImage& target,
                                      const RunConfig& cfg, std::uint64_t pair_index = 0) {
  if (reference.width() != target.width() || reference.height() != target.height())
    throw Error("dimension mismatch");
  const bool wide = !detail::max_is_u8(reference) || !detail::max_is_u8(target);
  detail::Packed a, b;
  detail::pack(reference, a, wide);
  detail::pack(target, b, wide);
  a.img.bits = b.img.bits = std::max(a.img.bits, b.img.bits);
  const dicb200_run_config c = detail::to_c(cfg);
  size_t n = 0;
  dicb200_status st = dicb200_grid_size(reference.width(), reference.height(), &c, &n);
  if (st != DICB200_OK) throw Error(dicb200_last_error_message());
  std::vector<dicb200_poi_record> recs(n);
  st = dicb200_analyze_pair(&a.img, &b.img, &c, pair_index, recs.data(), recs.size(), &n);
  if (st == DICB200_ERR_INVALID) throw Error(dicb200_last_error_message());
  if (st != DICB200_OK) throw std::runtime_error(dicb200_last_error_message());
  DisplacementField f;
  f.pair_index = static_cast<int>(pair_index);
  f.ref_id = reference.id();
  f.tgt_id = target.id();
  f.records.reserve(n);
  for (size_t i = 0; i < n; ++i) f.records.push_back(detail::to_record(recs[i]));
  return f;
}

// pipeline.cpp:182-214 semantics: per-pair dic::Error -> field.error, fields in pair order.
inline std::vector<DisplacementField> analyze_sequence(const std::vector<GrayImage>& images,
                                                       const RunConfig& cfg) {
  const auto pairs = sequence_pairs(cfg.reference_policy, static_cast<int>(images.size()));
  std::vector<DisplacementField> fields(pairs.size());
  for (size_t i = 0; i < pairs.size(); ++i) {
    const auto& [a, b] = pairs[i];
    try {
      fields[i] = b200::analyze_pair(images[a], images[b], cfg, i);
    } catch (const Error& e) {
      fields[i].pair_index = static_cast<int>(i);
      fields[i].ref_id = images[a].id();
      fields[i].tgt_id = images[b].id();
      fields[i].error = e.what();
    }
  }
  return fields;
}

}  // namespace b200
}  // namespace dic
