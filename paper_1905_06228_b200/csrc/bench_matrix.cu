// f-3 field CSV output (pipeline.cpp:216-238) and the f-4 bench matrix
// (bench.hpp:12-90, bench.cpp:14-293): the reference's end-to-end harness —
// load a frame sequence, analyse it, write every field CSV, per cell and
// repeat — with the analysis on the GPU and the same record / ratio / CSV
// layouts, so the reference's relative-ranking tables (BFS vs PSO, parallel
// speed-ups) can be regenerated on B200 and diffed against the reference's.
//
// Timing boundary as the reference (bench.hpp:40-41): per repeat, from just
// before image loading to after the last field CSV is written (host wall
// clock — this is the harness's end-to-end number, not a kernel time).
#include <sys/stat.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"

using namespace dicb200;

namespace {

dicb200_status bad(const std::string& msg) {
  set_error(msg.c_str());
  return DICB200_ERR_INVALID;
}

const char* int_name(int m) { return m == 0 ? "bfs" : m == 1 ? "pso" : m == 2 ? "mpso" : "?"; }
const char* sub_name(int m) { return m == 0 ? "nr" : m == 1 ? "icgn" : m == 2 ? "none" : "?"; }
const char* mode_name(int m) { return m == 0 ? "serial" : m == 1 ? "subimage" : m == 2 ? "image" : "?"; }

void put(char* dst, size_t cap, const std::string& s) {
  std::snprintf(dst, cap, "%s", s.c_str());
}

std::string csv_text(const dicb200_field& f) {
  std::string out = "x,y,u,v,zncc,converged,iterations,evaluations\n";
  char line[192];
  for (size_t i = 0; i < f.count; ++i) {
    const dicb200_poi_record& r = f.records[i];
    std::snprintf(line, sizeof line, "%d,%d,%.17g,%.17g,%.17g,%d,%d,%ld\n", r.x, r.y, r.u, r.v, r.zncc,
                  r.converged ? 1 : 0, r.iterations, (long)r.evaluations);
    out += line;
  }
  return out;
}

bool write_text(const std::string& path, const std::string& text, std::string* err) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) {
    *err = "cannot open for writing: " + path;
    return false;
  }
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  if (std::fclose(f) != 0 || !ok) {
    *err = "write failed: " + path;
    return false;
  }
  return true;
}

bool make_dirs(const std::string& path) {  // mkdir -p
  std::string cur;
  for (size_t i = 0; i <= path.size(); ++i) {
    if (i == path.size() || path[i] == '/') {
      if (!cur.empty()) {
        struct stat sb;
        if (stat(cur.c_str(), &sb) != 0 && mkdir(cur.c_str(), 0755) != 0) return false;
      }
    }
    if (i < path.size()) cur += path[i];
  }
  return true;
}

std::string filename_of(const std::string& dir) {  // std::filesystem::path::filename
  const size_t k = dir.find_last_of('/');
  return k == std::string::npos ? dir : dir.substr(k + 1);
}

// One repetition: load, analyse, serialise (bench.cpp:34-52).
struct Rep {
  double seconds = 0;
  int pairs = 0;
  long long evaluations = 0;
  bool failed = false;
  std::string error;
};

Rep run_once(const std::string& dir, const char* pattern, const dicb200_run_config& cfg, const std::string& out_dir,
             int32_t load_flags) {
  Rep rep;
  const auto t0 = std::chrono::steady_clock::now();
  // --- load_sequence (image.cpp:112-138) into one pinned block
  size_t need = 0, count = 0;
  if (dicb200_sequence_files(dir.c_str(), pattern, nullptr, 0, &need, &count) != DICB200_OK) {
    rep.failed = true;
    rep.error = dicb200_last_error_message();
    return rep;
  }
  std::vector<char> names(need);
  dicb200_sequence_files(dir.c_str(), pattern, names.data(), need, &need, &count);
  std::vector<std::string> paths;
  for (const char* p = names.data(); paths.size() < count; p += std::strlen(p) + 1) paths.push_back(dir + "/" + p);
  std::vector<dicb200_image> imgs(count);
  std::vector<size_t> offs(count + 1, 0);
  for (size_t i = 0; i < count; ++i) {
    int32_t w, h, dt, mv;
    if (dicb200_load_pgm(paths[i].c_str(), load_flags, &w, &h, &dt, &mv, nullptr, 0) != DICB200_OK) {
      rep.failed = true;
      rep.error = dicb200_last_error_message();
      return rep;
    }
    if (i && (w != imgs[0].width || h != imgs[0].height)) {
      rep.failed = true;
      rep.error = "dimension mismatch in sequence: " + paths[i];
      return rep;
    }
    std::memset(&imgs[i], 0, sizeof imgs[i]);
    imgs[i].width = w;
    imgs[i].height = h;
    imgs[i].pitch = w;
    imgs[i].dtype = dt;
    imgs[i].id = (int32_t)i;
    offs[i + 1] = offs[i] + (((size_t)w * h * (dt == DICB200_U8 ? 1 : 2) + 255) & ~(size_t)255);
  }
  uint8_t* block = static_cast<uint8_t*>(dicb200_host_alloc(std::max<size_t>(offs[count], 1)));
  std::vector<uint8_t> fallback;
  if (!block) {  // pinned memory exhausted: pageable copies still work
    fallback.resize(std::max<size_t>(offs[count], 1));
    block = fallback.data();
  }
  bool ok = true;
  for (size_t i = 0; i < count && ok; ++i) {
    int32_t w, h, dt, mv;
    imgs[i].data = block + offs[i];
    ok = dicb200_load_pgm(paths[i].c_str(), load_flags, &w, &h, &dt, &mv, block + offs[i],
                          (size_t)imgs[i].width * imgs[i].height) == DICB200_OK;
  }
  if (ok) {
    // --- analyze_sequence
    size_t npoi = 0;
    dicb200_grid_size(imgs[0].width, imgs[0].height, &cfg, &npoi);
    std::vector<dicb200_poi_record> recs((count - 1) * npoi);
    std::vector<dicb200_field> fields(count - 1);
    for (size_t k = 0; k + 1 < count; ++k) {
      std::memset(&fields[k], 0, sizeof fields[k]);
      fields[k].records = recs.data() + k * npoi;
      fields[k].capacity = npoi;
    }
    ok = dicb200_analyze_sequence(imgs.data(), count, &cfg, fields.data(), fields.size()) == DICB200_OK;
    if (!ok) {
      rep.error = dicb200_last_error_message();
    } else {
      // --- write_field_csv per field
      for (const auto& f : fields) {
        char name[32];
        dicb200_field_filename(f.pair_index, name, sizeof name);
        std::string err;
        if (!write_text(out_dir + "/" + name, csv_text(f), &err)) {
          ok = false;
          rep.error = err;
          break;
        }
        if (f.status != DICB200_OK && !rep.failed) {
          rep.failed = true;
          rep.error = f.error;
        }
        for (size_t i = 0; i < f.count; ++i) rep.evaluations += f.records[i].evaluations;
      }
      rep.pairs = (int)fields.size();
    }
  } else {
    rep.error = dicb200_last_error_message();
  }
  if (block != fallback.data()) dicb200_host_free(block);
  if (!ok) rep.failed = true;
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

const dicb200_bench_record* find_cell(const dicb200_bench_record* r, size_t n, int im, int sm, int mode) {
  for (size_t i = 0; i < n; ++i)
    if (!r[i].failed && r[i].cell.integer_method == im && r[i].cell.subpixel_method == sm && r[i].cell.mode == mode &&
        r[i].mean_s > 0)
      return &r[i];
  return nullptr;
}

}  // namespace

extern "C" {

dicb200_status dicb200_field_csv(const dicb200_field* field, char* buf, size_t cap, size_t* needed) {
  if (!field) return bad("null argument");
  const std::string s = csv_text(*field);
  if (needed) *needed = s.size() + 1;
  if (!buf) return DICB200_OK;
  if (cap < s.size() + 1) {
    set_error("csv buffer too small");
    return DICB200_ERR_CAPACITY;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return DICB200_OK;
}

dicb200_status dicb200_write_field_csv(const dicb200_field* field, const char* path) {
  if (!field || !path) return bad("null argument");
  std::string err;
  return write_text(path, csv_text(*field), &err) ? DICB200_OK : bad(err);
}

dicb200_status dicb200_field_filename(int32_t pair_index, char* buf, size_t cap) {
  if (!buf || cap < 16) return bad("name buffer too small");
  std::snprintf(buf, cap, "field_%04d.csv", pair_index);
  return DICB200_OK;
}

int32_t dicb200_auto_repeats(double s) {
  if (s > 60.0) return 25;
  if (s >= 10.0) return 100;
  if (s >= 1.0) return 250;
  return 1000;
}

dicb200_status dicb200_run_bench(const dicb200_bench_cell* cells, size_t n_cells, const char* dataset_dir,
                                 const char* pattern, const dicb200_run_config* base, int32_t auto_bands,
                                 int32_t fixed_repeats, const char* scratch_dir, int32_t load_flags,
                                 dicb200_bench_record* out) {
  if (!dataset_dir || !pattern || !base || !scratch_dir || (n_cells && (!cells || !out)))
    return bad("null argument");
  if (n_cells == 0) return bad("empty benchmark matrix");
  if (!auto_bands && fixed_repeats < 1) return bad("repeats must be >= 1");
  std::string dir(dataset_dir);
  std::string id = filename_of(dir);
  if (id.empty()) id = dir;
  for (size_t c = 0; c < n_cells; ++c) {
    dicb200_bench_record& rec = out[c];
    std::memset(&rec, 0, sizeof rec);
    rec.cell = cells[c];
    put(rec.dataset_id, sizeof rec.dataset_id, id);
    dicb200_run_config cfg = *base;
    cfg.integer_method = cells[c].integer_method;
    cfg.subpixel_method = cells[c].subpixel_method;
    cfg.mode = cells[c].mode;
    const std::string out_dir = std::string(scratch_dir) + "/cell-" + int_name(cfg.integer_method) + "-" +
                                sub_name(cfg.subpixel_method) + "-" + mode_name(cfg.mode);
    std::string error;
    if (!make_dirs(out_dir)) {
      error = "cannot create directory: " + out_dir;
    } else {
      const Rep warm = run_once(dir, pattern, cfg, out_dir, load_flags);
      if (warm.failed) {
        error = warm.error;
      } else {
        rec.repeats = auto_bands ? dicb200_auto_repeats(warm.seconds) : fixed_repeats;
        rec.pair_count = warm.pairs;
        rec.total_evaluations = warm.evaluations;
        double sum = 0, sumsq = 0;
        for (int r = 0; r < rec.repeats && error.empty(); ++r) {
          const Rep run = run_once(dir, pattern, cfg, out_dir, load_flags);
          if (run.failed)
            error = run.error;
          else if (run.evaluations != rec.total_evaluations)
            error = "evaluation counts differ between repeats";
          sum += run.seconds;
          sumsq += run.seconds * run.seconds;
        }
        if (error.empty()) {
          rec.mean_s = sum / rec.repeats;
          const double var =
              rec.repeats > 1 ? std::max(0.0, (sumsq - sum * sum / rec.repeats) / (rec.repeats - 1)) : 0.0;
          rec.stddev_s = std::sqrt(var);
          rec.per_pair_s = rec.pair_count > 0 ? rec.mean_s / rec.pair_count : 0.0;
          rec.frame_rate_hz = rec.mean_s > 0 ? rec.pair_count / rec.mean_s : 0.0;
        }
      }
    }
    if (!error.empty()) {  // the reference's catch (bench.cpp:113-116): fields filled so far stay
      rec.failed = 1;
      put(rec.error, sizeof rec.error, error);
    }
  }
  return DICB200_OK;
}

dicb200_status dicb200_derive_ratios(const dicb200_bench_record* R, size_t n, const char* dataset_id,
                                     dicb200_ratio_row* rows, size_t cap, size_t* count) {
  if ((n && !R) || !dataset_id || !count) return bad("null argument");
  std::vector<dicb200_ratio_row> out;
  auto any = [&](auto pred) {
    for (size_t i = 0; i < n; ++i)
      if (pred(R[i].cell)) return true;
    return false;
  };
  auto add = [&](const char* kind, const std::string& detail, const dicb200_bench_record* num,
                 const dicb200_bench_record* den) {
    dicb200_ratio_row row;
    std::memset(&row, 0, sizeof row);
    put(row.kind, sizeof row.kind, kind);
    put(row.detail, sizeof row.detail, detail);
    if (num && den) {
      row.value = num->mean_s / den->mean_s;
    } else {
      row.value = std::numeric_limits<double>::quiet_NaN();
      put(row.note, sizeof row.note, "missing cell");
    }
    out.push_back(row);
  };
  const std::string ds = dataset_id;
  // bfs_vs_pso per (subpixel, mode) that any record asks for (bench.cpp:150-176)
  if (any([](const dicb200_bench_cell& c) { return c.integer_method == DICB200_INT_BFS; }) &&
      any([](const dicb200_bench_cell& c) { return c.integer_method == DICB200_INT_PSO; }))
    for (int sm : {DICB200_SUB_NR, DICB200_SUB_ICGN, DICB200_SUB_NONE})
      for (int mode : {DICB200_MODE_SERIAL, DICB200_MODE_SUBIMAGE, DICB200_MODE_IMAGE}) {
        if (!any([&](const dicb200_bench_cell& c) { return c.subpixel_method == sm && c.mode == mode; })) continue;
        add("bfs_vs_pso", std::string("sub=") + sub_name(sm) + ",mode=" + mode_name(mode) + ",dataset=" + ds,
            find_cell(R, n, DICB200_INT_BFS, sm, mode), find_cell(R, n, DICB200_INT_PSO, sm, mode));
      }
  // parallel speed-ups over serial per (integer, subpixel) (bench.cpp:178-207)
  for (int im : {DICB200_INT_BFS, DICB200_INT_PSO, DICB200_INT_MPSO})
    for (int sm : {DICB200_SUB_NR, DICB200_SUB_ICGN, DICB200_SUB_NONE}) {
      if (!any([&](const dicb200_bench_cell& c) { return c.integer_method == im && c.subpixel_method == sm; }))
        continue;
      const dicb200_bench_record* serial = find_cell(R, n, im, sm, DICB200_MODE_SERIAL);
      const struct {
        const char* kind;
        int mode;
      } targets[] = {{"image_speedup_vs_serial", DICB200_MODE_IMAGE},
                     {"subimage_speedup_vs_serial", DICB200_MODE_SUBIMAGE}};
      for (const auto& t : targets) {
        if (!any([&](const dicb200_bench_cell& c) {
              return c.integer_method == im && c.subpixel_method == sm && c.mode == t.mode;
            }))
          continue;
        add(t.kind, std::string("int=") + int_name(im) + ",sub=" + sub_name(sm) + ",dataset=" + ds, serial,
            find_cell(R, n, im, sm, t.mode));
      }
    }
  *count = out.size();
  if (!rows) return DICB200_OK;
  if (cap < out.size()) {
    set_error("ratio buffer too small");
    return DICB200_ERR_CAPACITY;
  }
  std::copy(out.begin(), out.end(), rows);
  return DICB200_OK;
}

dicb200_status dicb200_write_times_csv(const dicb200_bench_record* R, size_t n, const char* dataset_id,
                                       const char* path) {
  if ((n && !R) || !dataset_id || !path) return bad("null argument");
  std::vector<int> modes;  // modes present, in enum order (bench.cpp:214-220)
  for (int mode : {DICB200_MODE_SERIAL, DICB200_MODE_SUBIMAGE, DICB200_MODE_IMAGE})
    for (size_t i = 0; i < n; ++i)
      if (R[i].cell.mode == mode) {
        modes.push_back(mode);
        break;
      }
  std::string s = "integer_method,subpixel_method";
  for (int mode : modes) s += std::string(",") + dataset_id + "_" + mode_name(mode) + "_mean_s";
  s += "\n";
  char buf[64];
  for (int im : {DICB200_INT_BFS, DICB200_INT_PSO, DICB200_INT_MPSO})
    for (int sm : {DICB200_SUB_NR, DICB200_SUB_ICGN, DICB200_SUB_NONE}) {
      bool present = false;
      for (size_t i = 0; i < n; ++i) present |= R[i].cell.integer_method == im && R[i].cell.subpixel_method == sm;
      if (!present) continue;
      s += std::string(int_name(im)) + "," + sub_name(sm);
      for (int mode : modes) {
        const dicb200_bench_record* rec = nullptr;  // the last matching record wins
        for (size_t i = 0; i < n; ++i)
          if (R[i].cell.integer_method == im && R[i].cell.subpixel_method == sm && R[i].cell.mode == mode) rec = &R[i];
        if (!rec || rec->failed) {
          s += ",";
        } else {
          std::snprintf(buf, sizeof buf, ",%.6f", rec->mean_s);
          s += buf;
        }
      }
      s += "\n";
    }
  std::string err;
  return write_text(path, s, &err) ? DICB200_OK : bad(err);
}

dicb200_status dicb200_write_records_csv(const dicb200_bench_record* R, size_t n, const char* path) {
  if ((n && !R) || !path) return bad("null argument");
  std::string s =
      "integer_method,subpixel_method,mode,dataset,repeats,pairs,mean_s,stddev_s,"
      "per_pair_s,frame_rate_hz,total_evaluations,failed,error\n";
  char buf[256];
  for (size_t i = 0; i < n; ++i) {
    const dicb200_bench_record& r = R[i];
    std::snprintf(buf, sizeof buf, "%s,%s,%s,%s,%d,%d,%.6f,%.6f,%.6f,%.4f,%lld,%d,", int_name(r.cell.integer_method),
                  sub_name(r.cell.subpixel_method), mode_name(r.cell.mode), r.dataset_id, r.repeats, r.pair_count,
                  r.mean_s, r.stddev_s, r.per_pair_s, r.frame_rate_hz, (long long)r.total_evaluations,
                  r.failed ? 1 : 0);
    s += buf;
    s += r.error;
    s += "\n";
  }
  std::string err;
  return write_text(path, s, &err) ? DICB200_OK : bad(err);
}

dicb200_status dicb200_write_ratios_csv(const dicb200_ratio_row* rows, size_t n, const char* path) {
  if ((n && !rows) || !path) return bad("null argument");
  std::string s = "kind,detail,value,note\n";
  char buf[64];
  for (size_t i = 0; i < n; ++i) {
    std::snprintf(buf, sizeof buf, "%.4f", rows[i].value);
    s += std::string(rows[i].kind) + "," + rows[i].detail + "," + (std::isnan(rows[i].value) ? "" : buf) + "," +
         rows[i].note + "\n";
  }
  std::string err;
  return write_text(path, s, &err) ? DICB200_OK : bad(err);
}

}  // extern "C"
