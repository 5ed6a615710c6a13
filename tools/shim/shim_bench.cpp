// e2e through the C++ drop-in shim (include/dic_b200/pipeline.hpp), the way a
// reference application calls it: dic::GrayImage doubles in, dic::b200::
// analyze_sequence (or analyze_pair for a 2-frame file), DisplacementFields out.
// The timed region is the shim call only: packing the doubles, H2D, the GPU
// pipeline, D2H and building the DisplacementField records.
//
//   shim_bench <frames.raw> <config.bin> <warmup> <steps>
//
// frames.raw: int32 {width, height, count, bytes_per_px} + count frames of
// u8/u16 pixels (bench.py writes the device-rendered frames). config.bin: one
// dicb200_run_config (the bench's RunConfig). Prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "dic/pipeline.hpp"
#include "dic_b200/pipeline.hpp"

static dic::RunConfig from_c(const dicb200_run_config& r) {
  dic::RunConfig c;
  c.integer_method = static_cast<dic::IntegerMethod>(r.integer_method);
  c.subpixel_method = static_cast<dic::SubpixelMethod>(r.subpixel_method);
  c.mode = static_cast<dic::ExecMode>(r.mode);
  c.reference_policy = static_cast<dic::ReferencePolicy>(r.reference_policy);
  c.worker_count = r.worker_count;
  c.search.search_radius = r.search_radius;
  c.search.bfs_domain = static_cast<dic::BfsDomain>(r.bfs_domain);
  c.search.particle_count = r.particle_count;
  c.search.max_generations = r.max_generations;
  c.search.stop_threshold = r.stop_threshold;
  c.search.c1 = r.c1;
  c.search.c2 = r.c2;
  c.search.rng_seed = r.rng_seed;
  c.refine.tol = r.tol;
  c.refine.max_iter = r.max_iter;
  c.grid.half_width = r.half_width;
  c.grid.spacing = r.spacing;
  c.grid.margin = r.margin;
  return c;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: shim_bench frames.raw config.bin warmup steps\n");
    return 2;
  }
  FILE* f = std::fopen(argv[1], "rb");
  int32_t hdr[4];
  if (!f || std::fread(hdr, sizeof hdr, 1, f) != 1) return 3;
  const int W = hdr[0], H = hdr[1], N = hdr[2], B = hdr[3];
  std::vector<dic::GrayImage> frames;
  std::vector<uint8_t> raw((size_t)W * H * B);
  for (int k = 0; k < N; ++k) {
    if (std::fread(raw.data(), raw.size(), 1, f) != 1) return 3;
    std::vector<double> px((size_t)W * H);
    for (size_t i = 0; i < px.size(); ++i)
      px[i] = B == 1 ? raw[i] : (double)reinterpret_cast<const uint16_t*>(raw.data())[i];
    frames.emplace_back(W, H, std::move(px), k);
  }
  std::fclose(f);
  dicb200_run_config rc;
  FILE* g = std::fopen(argv[2], "rb");
  if (!g || std::fread(&rc, sizeof rc, 1, g) != 1) return 3;
  std::fclose(g);
  const dic::RunConfig cfg = from_c(rc);
  const int warmup = std::atoi(argv[3]), steps = std::atoi(argv[4]);
  size_t pois = 0;
  auto once = [&]() {
    pois = 0;
    if (N == 2) {
      pois = dic::b200::analyze_pair(frames[0], frames[1], cfg, 0).records.size();
    } else {
      for (const auto& fld : dic::b200::analyze_sequence(frames, cfg)) {
        if (!fld.error.empty()) throw std::runtime_error(fld.error);
        pois += fld.records.size();
      }
    }
  };
  for (int i = 0; i < warmup; ++i) once();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) once();
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"value\": %.6g, \"unit\": \"subsets/s\", \"pois_per_step\": %zu, \"steps\": %d, \"seconds\": %.6g, "
              "\"path\": \"dic::b200::%s (C++ shim, GrayImage doubles in, DisplacementField out)\", "
              "\"mode\": %d, \"worker_count\": %d}\n",
              (double)pois * steps / s, pois, steps, s, N == 2 ? "analyze_pair" : "analyze_sequence", rc.mode,
              rc.worker_count);
  return 0;
}
