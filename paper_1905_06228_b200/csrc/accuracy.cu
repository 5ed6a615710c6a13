// f-4 accuracy sweep: dic::run_accuracy_sweep (accuracy.cpp:10-78)
// with the analysis on the GPU, plus the two generators it needs, restated on
// the host from synth.cpp so the frames are the reference's doubles bit for bit:
//
//   synth_speckle      synth.cpp:55-93   Gaussian blobs on a mid-gray background
//   check_texture      synth.cpp:22-50   summed-area variance floor
//   synth_warped_pair  synth.cpp:127-172 inverse-mapped bilinear target + mask
//   interp_bilinear    subpixel.cpp:59-101
//
// The generators are data preparation, not the measured path: they run once per
// sweep on 160x160 frames. The device sees integer gray levels (the C-ABI's
// image type), so the doubles are quantized round(v * gray_scale) — scale 1 is
// what the reference's own save_pgm/load_image round trip would feed it, scale
// 256 keeps 8 fractional bits in u16. Each combo's warps then run as ONE
// pipelined fixed-first sequence (reference frame resident, its tensor-core
// inputs cached, pair p = warp p so PSO streams match accuracy.cpp:49-50).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"

using namespace dicb200;

namespace {

dicb200_status fail(const std::string& msg) {
  set_error(msg.c_str());
  return DICB200_ERR_INVALID;
}

// splitmix64 finalizer (rng.hpp:11-16): seeds the blob stream.
uint64_t finalize64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// StreamRng's mappings (rng.hpp:33-44) over the standard mt19937_64.
struct BlobStream {
  std::mt19937_64 gen;
  explicit BlobStream(uint64_t seed) : gen(seed) {}
  double unit() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double between(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

// Every win x win window must have variance >= the floor (synth.cpp:22-50).
// Same prefix-sum recurrence and operation order, so the decision is identical.
bool texture_ok(const std::vector<double>& img, int w, int h, const dicb200_speckle_params& p) {
  const int win = std::min(std::min(p.texture_window, w), h);
  const size_t W1 = (size_t)w + 1;
  std::vector<double> a((size_t)(h + 1) * W1, 0.0), b((size_t)(h + 1) * W1, 0.0);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double v = img[(size_t)y * w + x];
      const size_t k = (size_t)(y + 1) * W1 + (x + 1);
      a[k] = v + a[k - 1] + a[k - W1] - a[k - W1 - 1];
      b[k] = v * v + b[k - 1] + b[k - W1] - b[k - W1 - 1];
    }
  const double n = (double)win * win;
  for (int y = 0; y + win <= h; ++y)
    for (int x = 0; x + win <= w; ++x) {
      const size_t tl = (size_t)y * W1 + x, tr = tl + win, bl = (size_t)(y + win) * W1 + x, br = bl + win;
      const double s = a[br] - a[tr] - a[bl] + a[tl];
      const double ss = b[br] - b[tr] - b[bl] + b[tl];
      const double mean = s / n;
      if (std::max(0.0, ss / n - mean * mean) < p.variance_floor) return false;
    }
  return true;
}

// subpixel.cpp:59-101 for in-domain coordinates (the caller checks the domain).
double bilinear(const double* img, int w, int h, double x, double y) {
  int x0 = 0, y0 = 0;
  double fx = 0.0, fy = 0.0;
  if (w > 1) {
    x0 = std::min((int)std::floor(x), w - 2);
    fx = x - x0;
  }
  if (h > 1) {
    y0 = std::min((int)std::floor(y), h - 2);
    fy = y - y0;
  }
  const int x1 = std::min(x0 + 1, w - 1), y1 = std::min(y0 + 1, h - 1);
  const double p00 = img[(size_t)y0 * w + x0], p10 = img[(size_t)y0 * w + x1];
  const double p01 = img[(size_t)y1 * w + x0], p11 = img[(size_t)y1 * w + x1];
  if (fy == 0.0) {  // integer coordinates return the stored sample exactly
    if (fx == 0.0) return p00;
    if (fx == 1.0) return p10;
  } else if (fy == 1.0) {
    if (fx == 0.0) return p01;
    if (fx == 1.0) return p11;
  }
  const double cx = p10 - p00, cy = p01 - p00, cxy = p00 + p11 - p10 - p01;
  const double g = p00 + cx * fx + cy * fy + cxy * fx * fy;
  const double lo = std::min(std::min(p00, p10), std::min(p01, p11));
  const double hi = std::max(std::max(p00, p10), std::max(p01, p11));
  return std::min(std::max(g, lo), hi);
}

struct Truth {  // GroundTruth::displacement_at (synth.cpp:117-121)
  dicb200_warp_spec w;
  double ox, oy;
  void at(double x, double y, double* u, double* v) const {
    const double rx = x - ox, ry = y - oy;
    *u = w.u + w.ux * rx + w.uy * ry;
    *v = w.v + w.vx * rx + w.vy * ry;
  }
};

template <typename T>
void quantize(const std::vector<double>& src, int scale, std::vector<uint8_t>& dst) {
  dst.resize(src.size() * sizeof(T));
  T* o = reinterpret_cast<T*>(dst.data());
  const double top = 255.0 * scale;
  for (size_t i = 0; i < src.size(); ++i) o[i] = (T)std::min(std::max(std::round(src[i] * scale), 0.0), top);
}

const double kFractions[5] = {0.1, 0.25, 0.5, 0.75, 0.9};
const int32_t kOffsets[3] = {-3, 0, 4};

}  // namespace

extern "C" {

void dicb200_default_speckle(dicb200_speckle_params* p) {
  if (!p) return;
  p->blob_count = 0;
  p->texture_window = 31;
  p->sigma_min = 1.0;
  p->sigma_max = 2.5;
  p->amp_min = 40.0;
  p->amp_max = 140.0;
  p->background = 128.0;
  p->variance_floor = 25.0;
}

int32_t dicb200_default_blob_count(int32_t width, int32_t height) { return std::max(1, width * height / 50); }

void dicb200_default_sweep(dicb200_sweep_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->width = 160;
  c->height = 160;
  c->seed = 7;
  dicb200_default_speckle(&c->speckle);
  dicb200_default_config(&c->base);
  c->fractions = kFractions;
  c->n_fractions = 5;
  c->offsets = kOffsets;
  c->n_offsets = 3;
  c->gray_scale = 256;
}

dicb200_status dicb200_synth_speckle(int32_t width, int32_t height, uint64_t seed, const dicb200_speckle_params* prm,
                                     double* out) {
  if (!prm || !out) return fail("null argument");
  if (width < 1 || height < 1) return fail("zero-dimension image");
  const dicb200_speckle_params& p = *prm;
  if (p.sigma_min <= 0 || p.sigma_max < p.sigma_min) return fail("invalid blob radius range");
  std::vector<double> img((size_t)width * height, p.background);
  BlobStream rng(finalize64(seed));
  const double ls0 = std::log(p.sigma_min), ls1 = std::log(p.sigma_max);
  for (int k = 0; k < p.blob_count; ++k) {
    // draw order: centre x, centre y, log-radius, amplitude, sign
    const double bx = rng.between(0.0, width - 1.0);
    const double by = rng.between(0.0, height - 1.0);
    const double sigma = std::exp(rng.between(ls0, ls1));
    double amp = rng.between(p.amp_min, p.amp_max) * std::pow(p.sigma_min / sigma, 0.8);
    if (rng.unit() < 0.5) amp = -amp;
    const int r = (int)std::ceil(3.0 * sigma);
    const int xa = std::max(0, (int)std::floor(bx) - r), xb = std::min(width - 1, (int)std::ceil(bx) + r);
    const int ya = std::max(0, (int)std::floor(by) - r), yb = std::min(height - 1, (int)std::ceil(by) + r);
    const double k2 = 1.0 / (2.0 * sigma * sigma);
    for (int y = ya; y <= yb; ++y) {
      double* row = img.data() + (size_t)y * width;
      const double ey = y - by;
      for (int x = xa; x <= xb; ++x) {
        const double ex = x - bx;
        row[x] += amp * std::exp(-(ex * ex + ey * ey) * k2);
      }
    }
  }
  for (double& v : img) v = std::min(std::max(v, 0.0), 255.0);
  if (!texture_ok(img, width, height, p)) return fail("textureless pattern");
  std::memcpy(out, img.data(), img.size() * sizeof(double));
  return DICB200_OK;
}

dicb200_status dicb200_synth_warped_pair(const double* ref, int32_t w, int32_t h, const dicb200_warp_spec* warp,
                                         double* target, uint8_t* mask) {
  if (!ref || !warp || !target) return fail("null argument");
  if (w < 1 || h < 1) return fail("zero-dimension image");
  const dicb200_warp_spec& s = *warp;
  const double ox = (w - 1) / 2.0, oy = (h - 1) / 2.0;
  // Forward map x -> x + d(x), d affine about the centre; the target samples
  // the reference at the preimage s = o + A^-1 (x - o - t).
  const double m00 = 1.0 + s.ux, m01 = s.uy, m10 = s.vx, m11 = 1.0 + s.vy;
  const double det = m00 * m11 - m01 * m10;
  if (std::abs(det) < 1e-8) return fail("warp not invertible");
  const double n00 = m11 / det, n01 = -m01 / det, n10 = -m10 / det, n11 = m00 / det;
  const bool shift_only = s.ux == 0 && s.uy == 0 && s.vx == 0 && s.vy == 0;
  size_t valid = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double sx, sy;
      if (shift_only) {
        sx = x - s.u;
        sy = y - s.v;
      } else {
        const double qx = x - ox - s.u, qy = y - oy - s.v;
        sx = ox + n00 * qx + n01 * qy;
        sy = oy + n10 * qx + n11 * qy;
      }
      const size_t i = (size_t)y * w + x;
      const bool in = sx >= 0.0 && sx <= w - 1.0 && sy >= 0.0 && sy <= h - 1.0;
      target[i] = in ? bilinear(ref, w, h, sx, sy) : 0.0;
      if (mask) mask[i] = in ? 1 : 0;
      valid += in;
    }
  if (valid == 0) return fail("warp out of bounds");
  return DICB200_OK;
}

dicb200_status dicb200_accuracy_sweep(const int32_t* combos, size_t n_combos, const dicb200_sweep_config* cfg,
                                      dicb200_combo_accuracy* out, int32_t* warp_count, int32_t* poi_count,
                                      double* elapsed_s) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!cfg || (n_combos && (!combos || !out))) return fail("null argument");
  if ((cfg->n_fractions && !cfg->fractions) || (cfg->n_offsets && !cfg->offsets)) return fail("null argument");
  const int scale = cfg->gray_scale <= 0 ? 256 : cfg->gray_scale;
  if (scale > 257) return fail("gray_scale must be in [1, 257] (255 * scale must fit 16 bits)");
  const int W = cfg->width, H = cfg->height;
  dicb200_speckle_params sp = cfg->speckle;
  if (sp.blob_count <= 0) sp.blob_count = dicb200_default_blob_count(W, H);

  // frames: reference, then one target per (offset, fraction) — accuracy.cpp:38-45
  std::vector<std::vector<double>> frames(1, std::vector<double>((size_t)std::max(W, 0) * std::max(H, 0)));
  dicb200_status st = dicb200_synth_speckle(W, H, cfg->seed, &sp, frames[0].data());
  if (st) return st;
  size_t npoi = 0;
  st = dicb200_grid_size(W, H, &cfg->base, &npoi);
  if (st) return st;
  std::vector<Truth> truths;
  for (int a = 0; a < cfg->n_offsets; ++a)
    for (int b = 0; b < cfg->n_fractions; ++b) {
      Truth t;
      std::memset(&t.w, 0, sizeof t.w);
      t.w.u = cfg->offsets[a] + cfg->fractions[b];
      t.w.v = -(cfg->offsets[a] + cfg->fractions[b]);
      t.ox = (W - 1) / 2.0;
      t.oy = (H - 1) / 2.0;
      frames.emplace_back(frames[0].size());
      st = dicb200_synth_warped_pair(frames[0].data(), W, H, &t.w, frames.back().data(), nullptr);
      if (st) return st;
      truths.push_back(t);
    }
  const int nwarp = (int)truths.size();
  if (warp_count) *warp_count = nwarp;
  if (poi_count) *poi_count = (int32_t)npoi;

  // integer gray levels for the device
  const bool wide = scale > 1;
  std::vector<std::vector<uint8_t>> q(frames.size());
  std::vector<dicb200_image> imgs(frames.size());
  for (size_t i = 0; i < frames.size(); ++i) {
    if (wide)
      quantize<uint16_t>(frames[i], scale, q[i]);
    else
      quantize<uint8_t>(frames[i], scale, q[i]);
    dicb200_image& im = imgs[i];
    std::memset(&im, 0, sizeof im);
    im.width = W;
    im.height = H;
    im.pitch = W;
    im.dtype = wide ? DICB200_U16 : DICB200_U8;
    im.id = i == 0 ? 0 : 1;  // synth_warped_pair: target id = reference id + 1
    im.data = q[i].data();
  }

  std::vector<dicb200_poi_record> recs((size_t)nwarp * npoi);
  std::vector<dicb200_field> fields(nwarp);
  for (size_t c = 0; c < n_combos; ++c) {
    dicb200_combo_accuracy& acc = out[c];
    std::memset(&acc, 0, sizeof acc);
    acc.integer_method = combos[2 * c];
    acc.subpixel_method = combos[2 * c + 1];
    if (nwarp == 0) continue;
    dicb200_run_config run = cfg->base;
    run.integer_method = acc.integer_method;
    run.subpixel_method = acc.subpixel_method;
    run.reference_policy = DICB200_POLICY_FIXED_FIRST;  // pair p = (reference, warp p), pair_index p
    run.mode = DICB200_MODE_SERIAL;
    for (int k = 0; k < nwarp; ++k) {
      std::memset(&fields[k], 0, sizeof fields[k]);
      fields[k].records = recs.data() + (size_t)k * npoi;
      fields[k].capacity = npoi;
    }
    st = dicb200_analyze_sequence(imgs.data(), imgs.size(), &run, fields.data(), fields.size());
    if (st) return st;
    double err_sum = 0.0;
    for (int k = 0; k < nwarp; ++k) {
      const dicb200_field& f = fields[k];
      if (f.status != DICB200_OK) return fail(f.error);  // analyze_pair would have thrown
      for (size_t i = 0; i < f.count; ++i) {
        const dicb200_poi_record& r = f.records[i];
        double tu, tv;
        truths[k].at(r.x, r.y, &tu, &tv);
        const double eu = std::abs(r.u - tu), ev = std::abs(r.v - tv);
        acc.max_err = std::max({acc.max_err, eu, ev});
        err_sum += eu + ev;
        acc.measurements += 2;
        if (!r.converged) ++acc.unconverged;
      }
    }
    // accuracy.cpp:64-72
    acc.mean_err = acc.measurements > 0 ? err_sum / acc.measurements : 0.0;
    const bool integer_only = acc.subpixel_method == DICB200_SUB_NONE;
    const bool within = integer_only ? acc.max_err <= 0.5 + 1e-9 : acc.max_err < 0.1;
    acc.pass = acc.unconverged == 0 && acc.measurements > 0 && within;
    acc.mean_flagged = acc.mean_err >= 0.05;
  }
  if (elapsed_s) *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return DICB200_OK;
}

}  // extern "C"
