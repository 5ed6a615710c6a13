// TEST INFRASTRUCTURE ONLY: builds the C++ drop-in shim (include/dic_b200/pipeline.hpp)
// INSIDE the reference build and compares dic::b200::analyze_pair with the
// reference's own dic::analyze_pair on a synthetic pair (run on the GPU box by
// tests/test_gpu_shim.py). Output: one line per check, exit code 0 on parity.
#include <cmath>
#include <cstdio>
#include <vector>

#include "dic/pipeline.hpp"
#include "dic/synth.hpp"
#include "dic_b200/pipeline.hpp"
#include "dicb200_synth.h"

int main() {
  const int W = 192, H = 160;
  dicb200_synth_spec sp{};
  sp.width = W;
  sp.height = H;
  sp.dtype = DICB200_U8;
  sp.max_value = 255;
  sp.seed = 11;
  sp.blob_count = W * H / 60;
  sp.field = DICB200_FIELD_NONE;
  sp.sigma_min = 2.0;
  sp.sigma_max = 4.0;
  sp.peak_min = 60.0;
  sp.peak_max = 200.0;
  std::vector<uint8_t> a(W * H), b(W * H);
  dicb200_synth_render(&sp, a.data(), W, 1);
  sp.field = DICB200_FIELD_AFFINE;
  sp.a[0] = 2.3;
  sp.a[3] = -1.4;
  dicb200_synth_render(&sp, b.data(), W, 1);
  dic::GrayImage ga(W, H, std::vector<double>(a.begin(), a.end()), 0);
  dic::GrayImage gb(W, H, std::vector<double>(b.begin(), b.end()), 1);
  int bad = 0;
  for (int method = 0; method < 3; ++method) {
    dic::RunConfig cfg;
    cfg.integer_method = static_cast<dic::IntegerMethod>(method);
    cfg.subpixel_method = method == 1 ? dic::SubpixelMethod::icgn : dic::SubpixelMethod::nr;
    cfg.search.bfs_domain = dic::BfsDomain::window;
    cfg.search.search_radius = 8;
    cfg.grid.half_width = 10;
    cfg.grid.spacing = 12;
    cfg.refine.tol = 1e-4;
    const auto ref = dic::analyze_pair(ga, gb, cfg, 3);
    const auto got = dic::b200::analyze_pair(ga, gb, cfg, 3);
    int mism = 0;
    double du = 0.0;
    for (size_t i = 0; i < ref.records.size(); ++i) {
      const auto &r = ref.records[i], &g = got.records[i];
      if (r.x != g.x || r.y != g.y || r.evaluations != g.evaluations || r.converged != g.converged) ++mism;
      if (r.converged) du = std::fmax(du, std::fmax(std::fabs(r.u - g.u), std::fabs(r.v - g.v)));
    }
    const bool ok = ref.records.size() == got.records.size() && mism == 0 && du < 1e-3;
    std::printf("method %d: %zu POIs, integer mismatches %d, max |du|,|dv| %.3g -> %s\n", method,
                ref.records.size(), mism, du, ok ? "ok" : "FAIL");
    bad += !ok;
  }
  // fractional gray levels (the reference's own synthetic frames): the shim
  // hands the doubles to the fp64 path, whose integer stage evaluates the
  // reference's zncc bit for bit: evaluations and convergence must match
  {
    dic::SpeckleParams spk;
    spk.blob_count = dic::default_blob_count(W, H);
    const dic::GrayImage fa = dic::synth_speckle(W, H, 5, spk);
    dic::WarpSpec wsp;
    wsp.u = 1.35;
    wsp.v = -2.6;
    wsp.ux = 0.004;
    wsp.vy = -0.003;
    const auto [fb, truth] = dic::synth_warped_pair(fa, wsp);
    for (int method = 0; method < 3; ++method) {
      dic::RunConfig cfg;
      cfg.integer_method = static_cast<dic::IntegerMethod>(method);
      cfg.subpixel_method = method == 1 ? dic::SubpixelMethod::icgn : dic::SubpixelMethod::nr;
      cfg.search.bfs_domain = dic::BfsDomain::window;
      cfg.search.search_radius = 8;
      cfg.grid.half_width = 10;
      cfg.grid.spacing = 12;
      cfg.refine.tol = 1e-4;
      const auto ref = dic::analyze_pair(fa, fb, cfg, 3);
      const auto got = dic::b200::analyze_pair(fa, fb, cfg, 3);
      int conv_mism = 0, n_both = 0, eval_mism = 0;
      double du = 0.0;
      for (size_t i = 0; i < ref.records.size(); ++i) {
        const auto &r = ref.records[i], &g = got.records[i];
        if (r.converged != g.converged) ++conv_mism;
        if (r.evaluations != g.evaluations || r.update_evaluations != g.update_evaluations) ++eval_mism;
        if (r.converged && g.converged) {
          ++n_both;
          du = std::fmax(du, std::fmax(std::fabs(r.u - g.u), std::fabs(r.v - g.v)));
        }
      }
      const bool ok = ref.records.size() == got.records.size() && conv_mism == 0 && eval_mism == 0 && du < 1e-3 &&
                      n_both > 0;
      std::printf("fractional method %d: %zu POIs, converged mismatches %d, evaluation mismatches %d, max |du|,|dv| "
                  "%.3g -> %s\n",
                  method, ref.records.size(), conv_mism, eval_mism, du, ok ? "ok" : "FAIL");
      bad += !ok;
    }
  }
  // sequences: both reference policies, serial and image-parallel modes, one
  // frame of the wrong size (its pairs fail with the reference's message, the
  // sequence continues: pipeline.cpp:182-214)
  {
    std::vector<dic::GrayImage> seq;
    for (int k = 0; k < 5; ++k) {
      std::vector<uint8_t> px(W * H);
      sp.field = k == 0 ? DICB200_FIELD_NONE : DICB200_FIELD_AFFINE;
      sp.a[0] = 0.7 * k;
      sp.a[3] = -0.45 * k;
      sp.a[1] = 0.001 * k;
      dicb200_synth_render(&sp, px.data(), W, 1);
      seq.emplace_back(W, H, std::vector<double>(px.begin(), px.end()), k);
    }
    seq[3] = dic::GrayImage(W - 8, H, std::vector<double>((W - 8) * H, 7.0), 3);
    // mode 2: serial again with the swarm search (mPSO + NR), whose RNG streams
    // are keyed by the pair index: with DICB200_SHIM_CHUNK set, the shim hands
    // the sequence over in several calls and the keys must still be the global ones
    for (int policy = 0; policy < 2; ++policy)
      for (int mode = 0; mode < 3; ++mode) {
        dic::RunConfig cfg;
        cfg.integer_method = mode == 2 ? dic::IntegerMethod::mpso : dic::IntegerMethod::bfs;
        cfg.subpixel_method = mode == 2 ? dic::SubpixelMethod::nr : dic::SubpixelMethod::icgn;
        cfg.search.bfs_domain = dic::BfsDomain::window;
        cfg.search.search_radius = 8;
        cfg.grid.half_width = 10;
        cfg.grid.spacing = 12;
        cfg.refine.tol = 1e-4;
        cfg.reference_policy = policy ? dic::ReferencePolicy::update_every_pair : dic::ReferencePolicy::fixed_first;
        cfg.mode = mode == 1 ? dic::ExecMode::image_parallel : dic::ExecMode::serial;
        cfg.worker_count = mode == 1 ? 2 : 1;
        const auto ref = dic::analyze_sequence(seq, cfg);
        const auto got = dic::b200::analyze_sequence(seq, cfg);
        int mism = 0, errs = 0;
        double du = 0.0;
        bool ok = ref.size() == got.size();
        for (size_t i = 0; ok && i < ref.size(); ++i) {
          const auto &rf = ref[i], &gf = got[i];
          ok = ok && rf.pair_index == gf.pair_index && rf.ref_id == gf.ref_id && rf.tgt_id == gf.tgt_id &&
               rf.error == gf.error && rf.records.size() == gf.records.size();
          errs += !rf.error.empty();
          for (size_t k = 0; ok && k < rf.records.size(); ++k) {
            const auto &r = rf.records[k], &g = gf.records[k];
            if (r.x != g.x || r.y != g.y || r.evaluations != g.evaluations || r.converged != g.converged) ++mism;
            if (r.converged) du = std::fmax(du, std::fmax(std::fabs(r.u - g.u), std::fabs(r.v - g.v)));
          }
        }
        ok = ok && mism == 0 && du < 1e-3 && errs > 0;
        std::printf("sequence policy %d mode %d: %zu fields (%d pair errors), integer mismatches %d, "
                    "max |du|,|dv| %.3g -> %s\n", policy, mode, ref.size(), errs, mism, du, ok ? "ok" : "FAIL");
        bad += !ok;
      }
  }
  try {
    dic::GrayImage small(W, H - 1, std::vector<double>(W * (H - 1), 0.0));
    dic::b200::analyze_pair(ga, small, dic::RunConfig{});
    ++bad;
  } catch (const dic::Error& e) {
    std::printf("pair error rethrown as dic::Error: %s\n", e.what());
  }
  return bad;
}
