// f-2 image ingestion: portable graymaps and frame sequences,
// restating image.cpp:40-138 of the reference (load_image, save_pgm,
// load_sequence) in native host code, plus pinned host buffers so loaded
// frames reach analyze_sequence's asynchronous uploads directly.
//
// 8-bit P5/P2 behaves exactly as the reference (byte n -> gray level n, the same
// error conditions and message prefixes). DICB200_PGM_16BIT additionally accepts
// maxval 256..65535 (P5: two big-endian bytes per sample, the Netpbm layout),
// which the reference rejects as "unsupported format (only 8-bit graymaps)".
#include <dirent.h>
#include <fnmatch.h>
#include <sys/stat.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "common.cuh"

using namespace dicb200;

extern "C" void dicb200_pack_span(const double* s, size_t n, uint16_t* d, int* frac, int* bad, int* mx);  // csrc/pack.c

namespace {

dicb200_status io_error(const std::string& msg) {
  set_error(msg.c_str());
  return DICB200_ERR_INVALID;
}

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// Header fields may be separated by whitespace and '#' comment lines
// (image.cpp:44-57); false = unreadable header.
bool next_header_int(FILE* f, int* value) {
  int c;
  while ((c = std::fgetc(f)) != EOF) {
    if (c == '#') {
      while ((c = std::fgetc(f)) != EOF && c != '\n') {
      }
    } else if (!std::isspace(c)) {
      std::ungetc(c, f);
      break;
    }
  }
  return std::fscanf(f, "%d", value) == 1;
}

// ASCII sample, as `in >> value` (skips whitespace; no comments in the raster).
bool next_ascii_int(FILE* f, long* value) { return std::fscanf(f, "%ld", value) == 1; }

}  // namespace

extern "C" {

dicb200_status dicb200_load_pgm(const char* path, int32_t flags, int32_t* width, int32_t* height, int32_t* dtype,
                                int32_t* maxval_out, void* pixels, size_t cap) {
  if (!path) return io_error("null argument");
  const std::string p(path);
  File in(path, "rb");
  if (!in.f) return io_error("unreadable file: " + p);
  char magic[2] = {0, 0};
  if (std::fread(magic, 1, 2, in.f) != 2 || magic[0] != 'P' || (magic[1] != '5' && magic[1] != '2'))
    return io_error("unsupported format (want P5 or P2 graymap): " + p);
  const bool binary = magic[1] == '5';
  int w, h, maxval;
  if (!next_header_int(in.f, &w) || !next_header_int(in.f, &h) || !next_header_int(in.f, &maxval))
    return io_error("unreadable portable graymap header");
  if (w < 1 || h < 1) return io_error("zero-dimension image: " + p);
  const bool wide_ok = (flags & DICB200_PGM_16BIT) != 0;
  if (maxval < 1 || maxval > (wide_ok ? 65535 : 255))
    return io_error("unsupported format (only 8-bit graymaps): " + p);
  const int dt = maxval <= 255 ? DICB200_U8 : DICB200_U16;
  if (width) *width = w;
  if (height) *height = h;
  if (dtype) *dtype = dt;
  if (maxval_out) *maxval_out = maxval;
  if (!pixels) return DICB200_OK;  // header query
  const size_t n = (size_t)w * (size_t)h;
  if (cap < n) {
    set_error("pixel buffer smaller than width * height");
    return DICB200_ERR_CAPACITY;
  }
  if (binary) {
    std::fgetc(in.f);  // the single whitespace byte after maxval
    if (dt == DICB200_U8) {
      if (std::fread(pixels, 1, n, in.f) != n) return io_error("unreadable file (truncated pixel data): " + p);
    } else {
      std::vector<unsigned char> raw(2 * n);
      if (std::fread(raw.data(), 1, raw.size(), in.f) != raw.size())
        return io_error("unreadable file (truncated pixel data): " + p);
      uint16_t* out = static_cast<uint16_t*>(pixels);
      for (size_t i = 0; i < n; ++i) {
        const uint16_t v = (uint16_t)((raw[2 * i] << 8) | raw[2 * i + 1]);
        if (v > maxval) return io_error("unreadable file (sample out of range): " + p);
        out[i] = v;
      }
    }
  } else {
    for (size_t i = 0; i < n; ++i) {
      long v;
      if (!next_ascii_int(in.f, &v)) return io_error("unreadable file (truncated pixel data): " + p);
      if (v < 0 || v > maxval) return io_error("unreadable file (sample out of range): " + p);
      if (dt == DICB200_U8)
        static_cast<uint8_t*>(pixels)[i] = (uint8_t)v;
      else
        static_cast<uint16_t*>(pixels)[i] = (uint16_t)v;
    }
  }
  return DICB200_OK;
}

dicb200_status dicb200_save_pgm(const char* path, const dicb200_image* img) {
  if (!path || !img || !img->data) return io_error("null argument");
  File out(path, "wb");
  if (!out.f) return io_error(std::string("cannot open for writing: ") + path);
  std::fprintf(out.f, "P5\n%d %d\n255\n", img->width, img->height);
  const int pitch = img->pitch > 0 ? img->pitch : img->width;
  std::vector<unsigned char> row((size_t)img->width);
  for (int y = 0; y < img->height; ++y) {
    for (int x = 0; x < img->width; ++x) {
      // save_pgm (image.cpp:98-104): round, clamp to [0, 255]
      const size_t i = (size_t)y * pitch + x;
      double v;
      switch (img->dtype) {
        case DICB200_U8: v = static_cast<const uint8_t*>(img->data)[i]; break;
        case DICB200_U16: v = static_cast<const uint16_t*>(img->data)[i]; break;
        case DICB200_F32: v = static_cast<const float*>(img->data)[i]; break;
        default: v = static_cast<const double*>(img->data)[i]; break;
      }
      row[x] = (unsigned char)std::min(std::max(std::round(v), 0.0), 255.0);
    }
    if (std::fwrite(row.data(), 1, row.size(), out.f) != row.size())
      return io_error(std::string("write failed: ") + path);
  }
  return DICB200_OK;
}

dicb200_status dicb200_sequence_files(const char* dir, const char* pattern, char* buf, size_t cap, size_t* needed,
                                      size_t* count) {
  if (!dir || !pattern) return io_error("null argument");
  struct stat sb;
  if (stat(dir, &sb) != 0 || !S_ISDIR(sb.st_mode)) return io_error(std::string("not a directory: ") + dir);
  DIR* d = opendir(dir);
  if (!d) return io_error(std::string("not a directory: ") + dir);
  std::vector<std::string> names;
  while (dirent* e = readdir(d)) {
    const std::string full = std::string(dir) + "/" + e->d_name;
    struct stat fs;
    if (stat(full.c_str(), &fs) != 0 || !S_ISREG(fs.st_mode)) continue;  // regular files only
    if (fnmatch(pattern, e->d_name, 0) == 0) names.push_back(e->d_name);
  }
  closedir(d);
  std::sort(names.begin(), names.end());  // lexicographic by filename (image.cpp:121-123)
  if (names.size() < 2)
    return io_error(std::string("insufficient images (need at least 2 matching '") + pattern + "')");
  size_t total = 0;
  for (const auto& s : names) total += s.size() + 1;
  if (needed) *needed = total;
  if (count) *count = names.size();
  if (!buf) return DICB200_OK;
  if (cap < total) {
    set_error("name buffer too small");
    return DICB200_ERR_CAPACITY;
  }
  for (const auto& s : names) {
    std::memcpy(buf, s.c_str(), s.size() + 1);
    buf += s.size() + 1;
  }
  return DICB200_OK;
}

// GrayImage doubles -> device gray levels (the C++ shim's one pass per frame).
dicb200_status dicb200_pack_gray(const double* src, int32_t width, int32_t height, int32_t src_pitch,
                                 int32_t scale, uint16_t* dst, int32_t* fractional, int32_t* max_level,
                                 int32_t threads) {
  if (!src || !dst || width < 1 || height < 1) return io_error("null argument");
  if (scale != 1 && scale != 256) return io_error("pack scale must be 1 or 256");
  const int pitch = src_pitch > 0 ? src_pitch : width;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  // below ~256 K pixels per thread the spawn costs more than the scan
  threads = std::max(1, std::min<int>(threads, (int)(((size_t)width * height) >> 18)));
  threads = std::min(threads, height);
  struct Part {
    int frac = 0, bad = 0, mx = 0;
  };
  std::vector<Part> part(threads);
  const double lim = scale == 1 ? 65535.0 : 255.0;
  auto work = [&](int t) {
    Part& r = part[t];
    const int y0 = (int)((long)height * t / threads), y1 = (int)((long)height * (t + 1) / threads);
    int mx = 0, frac = 0, bad = 0;
    for (int y = y0; y < y1; ++y) {
      const double* s = src + (size_t)y * pitch;
      uint16_t* d = dst + (size_t)y * width;
      if (scale == 1) {
        dicb200_pack_span(s, (size_t)width, d, &frac, &bad, &mx);  // csrc/pack.c (AVX2 when present)
        continue;
      }
      for (int x = 0; x < width; ++x) {
        const double v = s[x];
        const bool b = !(v >= 0.0 && v <= lim);  // also catches NaN
        bad |= b;
        const uint16_t q = (uint16_t)(b ? 0 : std::lround(v * 256.0));  // 8.8 fixed point
        d[x] = q;
        mx = q > mx ? q : mx;
      }
    }
    r.mx = mx;
    r.frac = frac;
    r.bad = bad;
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int mx = 0, frac = 0, bad = 0;
  for (const Part& r : part) {
    mx = std::max(mx, r.mx);
    frac |= r.frac;
    bad |= r.bad;
  }
  if (fractional) *fractional = frac;
  if (max_level) *max_level = mx;
  if (bad)
    return io_error(scale == 1 ? "dicb200: gray levels must be integers in [0, 65535]"
                               : "dicb200: fractional gray levels must lie in [0, 255]");
  return DICB200_OK;
}

// Every frame of a sequence in one call: row bands of all frames are dealt to
// one set of threads (no per-frame thread start-up), per-frame flags out.
dicb200_status dicb200_pack_gray_batch(const double* const* src, int32_t count, int32_t width, int32_t height,
                                       int32_t src_pitch, uint16_t* const* dst, int32_t* fractional,
                                       int32_t* max_level, int32_t threads) {
  if (!src || !dst || count < 1 || width < 1 || height < 1) return io_error("null argument");
  for (int k = 0; k < count; ++k)
    if (!src[k] || !dst[k]) return io_error("null argument");
  const int pitch = src_pitch > 0 ? src_pitch : width;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int band = std::max(1, std::min(height, (1 << 17) / std::max(1, width)));  // ~128 K pixels per task
  const int bands = (height + band - 1) / band;
  const long tasks = (long)count * bands;
  threads = (int)std::max<long>(1, std::min<long>(threads, tasks / 2));
  struct Flags {
    std::atomic<int> frac{0}, bad{0}, mx{0};
  };
  std::vector<Flags> fl(count);
  std::atomic<long> next{0};
  auto work = [&]() {
    for (long t = next.fetch_add(1); t < tasks; t = next.fetch_add(1)) {
      const int k = (int)(t / bands), y0 = (int)(t % bands) * band, y1 = std::min(height, y0 + band);
      int frac = 0, bad = 0, mx = 0;
      if (pitch == width) {
        dicb200_pack_span(src[k] + (size_t)y0 * width, (size_t)(y1 - y0) * width, dst[k] + (size_t)y0 * width, &frac,
                          &bad, &mx);
      } else {
        for (int y = y0; y < y1; ++y)
          dicb200_pack_span(src[k] + (size_t)y * pitch, (size_t)width, dst[k] + (size_t)y * width, &frac, &bad, &mx);
      }
      if (frac) fl[k].frac.store(1, std::memory_order_relaxed);
      if (bad) fl[k].bad.store(1, std::memory_order_relaxed);
      int cur = fl[k].mx.load(std::memory_order_relaxed);
      while (mx > cur && !fl[k].mx.compare_exchange_weak(cur, mx, std::memory_order_relaxed)) {
      }
    }
  };
  if (threads == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  int any_bad = 0;
  for (int k = 0; k < count; ++k) {
    if (fractional) fractional[k] = fl[k].frac.load();
    if (max_level) max_level[k] = fl[k].mx.load();
    any_bad |= fl[k].bad.load();
  }
  if (any_bad) return io_error("dicb200: gray levels must be integers in [0, 65535]");
  return DICB200_OK;
}

void* dicb200_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dicb200_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
