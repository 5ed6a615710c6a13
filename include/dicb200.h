/*
 * dicb200 — C-ABI of the B200-native DIC correlation path (integer search +
 * sub-pixel refinement) of arXiv 1905.06228 / the reference `dicbench` library.
 *
 * The reference has no FFI layer; its operator surface is the C++ namespace
 * `dic`. The drop-in granularity is the batched pipeline entry point
 * (SURVEY.md §8b):
 *
 *   dicb200_analyze_pair      replaces dic::analyze_pair
 *                             (/root/reference/proj/core/include/dic/pipeline.hpp:76-77,
 *                              proj/core/src/pipeline.cpp:147-180)
 *   dicb200_analyze_sequence  replaces dic::analyze_sequence
 *                             (pipeline.hpp:79-80, pipeline.cpp:182-214)
 *   dicb200_grid_size /       replaces dic::grid_subsets + RunConfig::effective_margin
 *   dicb200_grid                (image.hpp:58-61, image.cpp:140-158; pipeline.hpp:43-45)
 *   dicb200_sequence_pairs    replaces dic::sequence_pairs (pipeline.hpp:71, pipeline.cpp:43-54)
 *   dicb200_partition_ranges  replaces dic::partition_ranges (pipeline.hpp:74, pipeline.cpp:56-69)
 *
 * Every per-subset stage of dic::process_subset (pipeline.cpp:76-135) —
 * subset_stats, bfs_search / pso_search / mpso_search, refine_nr,
 * icgn_precompute + refine_icgn — runs inside these calls as sm_100a kernels.
 *
 * Plain pointers and sizes only. Images are 8- or 16-bit unsigned gray levels
 * (the reference stores doubles; integer gray levels map losslessly, which is
 * what every BASELINE configuration uses) or f32/f64 levels (the exact fp64
 * path for fractional frames). Errors: pair-level failures that the
 * reference raises as dic::Error return DICB200_ERR_INVALID with the reference's
 * message in dicb200_last_error_message(); per-POI failures never fail the call
 * — they are reported in dicb200_poi_record.status with the reference's
 * partial-fill semantics (pipeline.cpp:82-133).
 *
 * Thread safety: every entry point is reentrant (per-call stream, device pools
 * guarded by a mutex), matching the reference's concurrent analyze_pair calls
 * from image-parallel workers (pipeline.cpp:201-209).
 */
#ifndef DICB200_H
#define DICB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DICB200_ABI_VERSION 1

typedef enum {
  DICB200_OK = 0,
  DICB200_ERR_INVALID = 1,  /* a dic::Error at pair level (message set)      */
  DICB200_ERR_CUDA = 2,     /* CUDA runtime failure (message set)            */
  DICB200_ERR_NOMEM = 3,
  DICB200_ERR_CAPACITY = 4, /* out_cap smaller than the grid                 */
  DICB200_ERR_NO_DEVICE = 5 /* no CUDA device: the product path never falls back to the CPU */
} dicb200_status;

/* Pixel storage. U8/U16: integer gray levels, used as they are (exact
 * integer search kernels). F32/F64: any finite gray levels (e.g. the
 * reference's fractional synthetic frames) on the fp64 path: F32 is widened
 * exactly, the integer search evaluates the reference's zncc in its own order
 * (bit-identical correlation values and decisions), the refiners gather fp32
 * samples of the fp64 image. Host entry points reject non-finite levels. */
enum { DICB200_U8 = 0, DICB200_U16 = 1, DICB200_F32 = 2, DICB200_F64 = 3 };

/* Enum values follow the declaration order of the reference enums. */
enum { DICB200_INT_BFS = 0, DICB200_INT_PSO = 1, DICB200_INT_MPSO = 2 };   /* IntegerMethod, pipeline.hpp:17 */
enum { DICB200_SUB_NR = 0, DICB200_SUB_ICGN = 1, DICB200_SUB_NONE = 2 };   /* SubpixelMethod, pipeline.hpp:18 */
enum { DICB200_MODE_SERIAL = 0, DICB200_MODE_SUBIMAGE = 1, DICB200_MODE_IMAGE = 2 }; /* ExecMode, pipeline.hpp:19 */
enum { DICB200_POLICY_UPDATE = 0, DICB200_POLICY_FIXED_FIRST = 1 };        /* ReferencePolicy, pipeline.hpp:20 */
enum { DICB200_BFS_WINDOW = 0, DICB200_BFS_WHOLE_IMAGE = 1 };              /* BfsDomain, integer_search.hpp:12 */
/* B200 extension (BASELINE.json asks for a constant 0.7 inertia; the reference
 * hard-codes w(t) = 0.9 - t/(2G), integer_search.cpp:35-37). */
enum { DICB200_INERTIA_REFERENCE = 0, DICB200_INERTIA_CONSTANT = 1 };

/* Image descriptor: host pointer for the host entry points, device pointer for
 * the *_device entry points. pitch is in elements (>= width). */
typedef struct {
  int32_t width;
  int32_t height;
  int32_t pitch;
  int32_t dtype;  /* DICB200_U8 | DICB200_U16 | DICB200_F32 | DICB200_F64 */
  int32_t id;     /* GrayImage::id(), copied into field ref_id/tgt_id */
  int32_t bits;     /* significant bits per pixel (0 = full dtype width); lets u16
                    * data of <= 12 bits use the exact u32 IMAD path */
  const void* data;
} dicb200_image;

/* POD mirror of RunConfig + SearchConfig + RefineConfig + GridParams
 * (pipeline.hpp:27-49, integer_search.hpp:14-23, subpixel.hpp:41-44).
 * dicb200_default_config() fills the reference defaults. */
typedef struct {
  int32_t integer_method;   /* default mpso */
  int32_t subpixel_method;  /* default nr */
  int32_t mode;             /* default serial; controls multi-device use in analyze_sequence */
  int32_t reference_policy; /* default update_every_pair */
  int32_t worker_count;     /* default 1; for image mode = number of devices to use (0 = all) */
  /* SearchConfig */
  int32_t search_radius;    /* 25 */
  int32_t bfs_domain;       /* whole_image */
  int32_t particle_count;   /* 50 */
  int32_t max_generations;  /* 5 */
  int32_t pad0;
  double stop_threshold;    /* 0.995 */
  double c1;                /* 2.0 */
  double c2;                /* 2.0 */
  uint64_t rng_seed;        /* 0 */
  /* RefineConfig */
  double tol;               /* 0.01 px on max(|du|,|dv|) */
  int32_t max_iter;         /* 20 */
  /* GridParams */
  int32_t half_width;       /* 15 */
  int32_t spacing;          /* 10 */
  int32_t margin;           /* -1: auto = half_width + search_radius */
  /* B200 extensions */
  int32_t inertia_mode;     /* DICB200_INERTIA_REFERENCE */
  int32_t interp;           /* DICB200_INTERP_BILINEAR (reference, default) | DICB200_INTERP_BICUBIC */
  double inertia_constant;  /* used when inertia_mode == CONSTANT */
} dicb200_run_config;

/* Sub-pixel interpolation of the refiners. BILINEAR = the reference's
 * interp_bilinear / grad_bilinear (subpixel.cpp:59-128), the parity default.
 * BICUBIC = BASELINE.json's "bicubic interpolation": Keys cubic convolution
 * (a = -0.5) over 4 x 4 taps with replicated borders and its analytic
 * gradient — a B200 extension the reference does not have, so
 * its parity is pinned only to the builder's CPU restatement
 * (oracle/dic_oracle.c, "parity unpinned"). */
enum { DICB200_INTERP_BILINEAR = 0, DICB200_INTERP_BICUBIC = 1 };

/* Per-POI status: 0 = no dic::Error was raised; otherwise which reference
 * error aborted the chain (the reference swallows the message, pipeline.cpp:131-133,
 * keeping the fields already filled). */
enum {
  DICB200_POI_OK = 0,
  DICB200_POI_SUBSET_OUT_OF_BOUNDS = 1,   /* "subset out of image bounds"          correlation.cpp:10-11 */
  DICB200_POI_NO_VALID_POSITION = 2,      /* "no valid search position"            integer_search.cpp:19,31 */
  DICB200_POI_ALL_DEGENERATE = 3,         /* "all positions degenerate"            integer_search.cpp:77,169 */
  DICB200_POI_INVALID_SWARM = 4,          /* "invalid swarm configuration"         integer_search.cpp:110-111 */
  DICB200_POI_DEGENERATE_SUBSET = 5,      /* "degenerate subset"                   subpixel.cpp:227,269,271 */
  DICB200_POI_DRIFTED = 6,                /* "drifted out of bounds"               subpixel.cpp:140,171 */
  DICB200_POI_DEGENERATE_TARGET = 7,      /* "degenerate target subset"            subpixel.cpp:239,289,318,349 */
  DICB200_POI_BORDER_GRADIENTS = 8,       /* "subset too close to border for gradients" subpixel.cpp:193-195 */
  DICB200_POI_DEGENERATE_TEXTURE = 9,     /* "degenerate texture"                  subpixel.cpp:200,219,335 */
  DICB200_POI_WARP_NOT_INVERTIBLE = 10,   /* "warp not invertible"                 subpixel.cpp:279,339 */
  DICB200_POI_INCREMENT_NOT_INVERTIBLE = 11, /* "non-invertible warp increment"    subpixel.cpp:30 */
  /* B200 extension: a frame holds a pixel above its declared dicb200_image.bits
   * (the exact u32 paths chosen from it would overflow); every record of the
   * call carries it and the host entry points fail the pair with
   * DICB200_ERR_INVALID. No reference counterpart (GrayImage has no width). */
  DICB200_POI_BITS_EXCEEDED = 12
};

/* PoiRecord (pipeline.hpp:51-59) + status. */
typedef struct {
  int32_t x, y;
  double u, v;
  double zncc;              /* NaN when the integer stage failed */
  int32_t converged;
  int32_t iterations;
  int64_t evaluations;
  int64_t update_evaluations;
  int32_t status;
  int32_t integer_dx, integer_dy; /* integer-stage displacement (diagnostic) */
  int32_t pad;
} dicb200_poi_record;

/* DisplacementField (pipeline.hpp:61-67); records are caller-owned. */
typedef struct {
  int32_t pair_index;
  int32_t ref_id;
  int32_t tgt_id;
  int32_t status;           /* DICB200_OK or the pair-level error */
  dicb200_poi_record* records;
  size_t capacity;
  size_t count;
  char error[160];          /* reference's dic::Error message when status != OK */
} dicb200_field;

int dicb200_abi_version(void);
void dicb200_default_config(dicb200_run_config* cfg);
const char* dicb200_last_error_message(void);
int dicb200_device_count(void);

/* Grid (no GPU needed). */
dicb200_status dicb200_grid_size(int32_t width, int32_t height, const dicb200_run_config* cfg,
                                 size_t* count);
dicb200_status dicb200_grid(int32_t width, int32_t height, const dicb200_run_config* cfg,
                            int32_t* xy_out /* 2*count */, size_t cap, size_t* count);
dicb200_status dicb200_sequence_pairs(int32_t policy, int32_t image_count, int32_t* pairs_out /* 2*(n-1) */);
dicb200_status dicb200_partition_ranges(size_t n, int32_t workers, size_t* ranges_out /* 2*workers */);

/* Host-buffer entry points (synchronous). Runs on device `device` (-1 = current). */
dicb200_status dicb200_analyze_pair(const dicb200_image* reference, const dicb200_image* target,
                                    const dicb200_run_config* cfg, uint64_t pair_index,
                                    dicb200_poi_record* out, size_t out_cap, size_t* out_count);

/* Sequence: pairs from dicb200_sequence_pairs(cfg->reference_policy, n).
 * fields[i] must have records/capacity set. Pair-level failures land in
 * fields[i].status/error (pipeline.cpp:191-198); the call still returns OK.
 * mode == IMAGE shards contiguous pair chunks over worker_count devices
 * (0 = all visible) with partition_ranges semantics. */
dicb200_status dicb200_analyze_sequence(const dicb200_image* images, size_t n_images,
                                        const dicb200_run_config* cfg, dicb200_field* fields,
                                        size_t n_fields);
/* The same for a contiguous part of a longer sequence, with a completion hook:
 * pair i of this call uses pair index first_pair_index + i (the RNG key of
 * derive_stream_seed, rng.hpp:20-55, and fields[i].pair_index), so a caller can
 * hand a long sequence over in chunks — packing / loading the next chunk's
 * frames while this one runs — and get the records of one whole call.
 * field_ready(user, i) is called on the host as soon as fields[i] is final
 * (records read back, or its pair-level error stored), while the device runs
 * the following pairs: the caller converts / consumes field i there instead of
 * after the whole call (the C++ shim builds the reference's DisplacementField
 * records in it). Called once per field, from the worker thread of the field's
 * device (concurrently for mode == IMAGE over several devices); it must not
 * call back into the library. NULL = none. */
typedef void (*dicb200_field_ready_fn)(void* user, size_t field_index);
dicb200_status dicb200_analyze_sequence_cb(const dicb200_image* images, size_t n_images,
                                           const dicb200_run_config* cfg, dicb200_field* fields,
                                           size_t n_fields, uint64_t first_pair_index,
                                           dicb200_field_ready_fn field_ready, void* user);

/* Device-resident entry point: images hold device pointers, records are
 * written to device memory `out_dev`, everything is enqueued on `stream`
 * (a cudaStream_t; NULL = legacy default) without host synchronisation.
 * grid rows [row_begin,row_end) only (subset-parallel sharding; -1 = all).
 * Subset indices (RNG keys) stay global. */
dicb200_status dicb200_analyze_pair_device(const dicb200_image* reference, const dicb200_image* target,
                                           const dicb200_run_config* cfg, uint64_t pair_index,
                                           int32_t row_begin, int32_t row_end,
                                           dicb200_poi_record* out_dev, size_t out_cap,
                                           size_t* out_count, void* stream);

/* Device-resident sequence: images hold device pointers; the pairs of
 * dicb200_sequence_pairs(cfg->reference_policy, n_images) are enqueued on
 * `stream` in order, pair i writing out_dev + i * pair_stride and using pair
 * index first_pair_index + i (RNG keys; lets image-parallel ranks pass a
 * contiguous sub-sequence). Like analyze_sequence, reference-side inputs are
 * built once per reference frame and reused by the following pairs on it. */
dicb200_status dicb200_analyze_sequence_device(const dicb200_image* images, size_t n_images,
                                               const dicb200_run_config* cfg, uint64_t first_pair_index,
                                               int32_t row_begin, int32_t row_end, dicb200_poi_record* out_dev,
                                               size_t pair_stride, size_t* per_pair_count, void* stream);

/* Kernel launches issued by this thread since the last reset (evidence for
 * bench.py "gpu_launches"). */
uint64_t dicb200_launch_count(void);
void dicb200_reset_launch_count(void);

/* Stage timing (bench evidence): while enabled, every enqueued stage kernel
 * is bracketed by CUDA events on the stream it runs on. dicb200_profile_read
 * waits for them and returns per-stage totals (ms) and launch counts, then
 * clears. Stages: 0 BFS-ZNCC, 1 PSO/mPSO, 2 NR, 3 IC-GN (whole stages);
 * inside stage 0 or 1 when the window search runs on the cross-term path:
 * 4 the tensor-core cross-term kernel, 5 the ZNCC argmax/surface kernel,
 * 6 the block-sum cross-term kernel (whichever of 4 / 6 the plan picked). */
#define DICB200_N_STAGES 7
void dicb200_profile_enable(int on);
int dicb200_profile_read(double* ms_out, uint64_t* launches_out);

/* ---- f-2 image ingestion (image.cpp:40-138): portable graymaps --------------
 * dicb200_load_pgm: P5 (binary) / P2 (ASCII) graymap. 8-bit exactly as
 * dic::load_image (byte n -> gray level n; same errors, DICB200_ERR_INVALID with
 * the reference's message). DICB200_PGM_16BIT also accepts maxval 256..65535
 * (P5: big-endian 2-byte samples), which the reference rejects. Call with
 * pixels == NULL to read the header; then with width*height elements (u8 for
 * maxval <= 255, else u16) — e.g. dicb200_host_alloc'ed pinned memory, which
 * analyze_sequence uploads asynchronously.
 * dicb200_save_pgm: 8-bit P5 like dic::save_pgm (values clamped to 255).
 * dicb200_sequence_files: regular files of `dir` matching the glob `pattern`,
 * lexicographic by filename, as NUL-separated names (dic::load_sequence's file
 * list; >= 2 required). Call with buf == NULL for the size. */
#define DICB200_PGM_16BIT 1
dicb200_status dicb200_load_pgm(const char* path, int32_t flags, int32_t* width, int32_t* height, int32_t* dtype,
                                int32_t* maxval, void* pixels, size_t cap);
dicb200_status dicb200_save_pgm(const char* path, const dicb200_image* img);
dicb200_status dicb200_sequence_files(const char* dir, const char* pattern, char* buf, size_t cap, size_t* needed,
                                      size_t* count);
/* GrayImage (row-major doubles, src_pitch elements per row; 0 = width) ->
 * the device path's gray levels in dst (width*height u16, packed rows), one
 * multithreaded pass (threads <= 0: all cores). Replaces the reference's
 * image storage (image.hpp:14-31) at the drop-in boundary, used by the C++
 * shim include/dic_b200/pipeline.hpp.
 *   scale 1:   integral levels in [0, 65535], stored losslessly. A
 *              non-integral level sets *fractional (dst is then not usable:
 *              pack again with scale 256).
 *   scale 256: levels in [0, 255] as 8.8 fixed point, lround(256 v).
 * *max_level = largest stored value. Out-of-range or non-finite levels:
 * DICB200_ERR_INVALID with the shim's dic::Error message. */
dicb200_status dicb200_pack_gray(const double* src, int32_t width, int32_t height, int32_t src_pitch,
                                 int32_t scale, uint16_t* dst, int32_t* fractional, int32_t* max_level,
                                 int32_t threads);
/* The same for every frame of a sequence in one call (scale 1): the row bands
 * of all frames are dealt to one set of threads; fractional[k] / max_level[k]
 * per frame. */
dicb200_status dicb200_pack_gray_batch(const double* const* src, int32_t count, int32_t width, int32_t height,
                                       int32_t src_pitch, uint16_t* const* dst, int32_t* fractional,
                                       int32_t* max_level, int32_t threads);
void* dicb200_host_alloc(size_t bytes); /* pinned host memory (NULL on failure) */
void dicb200_host_free(void* p);

/* ---- f-4 accuracy sweep (accuracy.hpp:15-50, accuracy.cpp:10-78; synth.hpp:14-66) ----
 * dicb200_synth_speckle / dicb200_synth_warped_pair restate dic::synth_speckle
 * (synth.cpp:55-93) and dic::synth_warped_pair (synth.cpp:127-172) on the host,
 * bit-identical doubles (same mt19937_64 stream, same libm calls, same
 * evaluation order); errors as the reference ("textureless pattern", "zero-dimension
 * image", "invalid blob radius range", "warp not invertible", "warp out of bounds").
 * dicb200_accuracy_sweep replaces dic::run_accuracy_sweep: the frames are
 * synthesized as above, quantized to integer gray levels (round(value * gray_scale):
 * gray_scale 1 = the reference's own 8-bit PGM round trip, 256 = 16-bit, keeping
 * 8 fractional bits of the reference's doubles), and every (offset, fraction)
 * warp of every combo is analysed on the GPU — one pipelined fixed-first
 * sequence per combo, so pair_index == warp index as in accuracy.cpp:49-50.
 * Pass / flag rules are the reference's (accuracy.cpp:64-72). */
typedef struct {  /* SpeckleParams, synth.hpp:14-23 */
  int32_t blob_count;      /* <= 0 in a sweep: scale by area (default_blob_count) */
  int32_t texture_window;  /* 31 */
  double sigma_min;        /* 1.0 */
  double sigma_max;        /* 2.5 */
  double amp_min;          /* 40 */
  double amp_max;          /* 140 */
  double background;       /* 128 */
  double variance_floor;   /* 25 */
} dicb200_speckle_params;

typedef struct {  /* WarpSpec, synth.hpp:30-35 */
  double u, v, ux, uy, vx, vy;
} dicb200_warp_spec;

typedef struct {  /* SweepConfig, accuracy.hpp:15-23 */
  int32_t width;                 /* 160 */
  int32_t height;                /* 160 */
  uint64_t seed;                 /* 7 */
  dicb200_speckle_params speckle;
  dicb200_run_config base;       /* methods overridden per combo */
  const double* fractions;       /* {0.1, 0.25, 0.5, 0.75, 0.9} */
  int32_t n_fractions;
  int32_t n_offsets;
  const int32_t* offsets;        /* {-3, 0, 4} */
  int32_t gray_scale;            /* B200: 1 (u8) or 256 (u16, default) */
  int32_t pad;
} dicb200_sweep_config;

typedef struct {  /* ComboAccuracy, accuracy.hpp:25-34 */
  int32_t integer_method;
  int32_t subpixel_method;
  double max_err;
  double mean_err;
  int32_t measurements;
  int32_t unconverged;
  int32_t pass;
  int32_t mean_flagged;
} dicb200_combo_accuracy;

void dicb200_default_speckle(dicb200_speckle_params* p);
int32_t dicb200_default_blob_count(int32_t width, int32_t height); /* synth.cpp:14-16 */
/* fractions/offsets point at static default arrays. */
void dicb200_default_sweep(dicb200_sweep_config* cfg);
dicb200_status dicb200_synth_speckle(int32_t width, int32_t height, uint64_t seed,
                                     const dicb200_speckle_params* params, double* out /* w*h */);
dicb200_status dicb200_synth_warped_pair(const double* reference, int32_t width, int32_t height,
                                         const dicb200_warp_spec* warp, double* target /* w*h */,
                                         uint8_t* valid_mask /* w*h, may be NULL */);
/* combos: n pairs (integer_method, subpixel_method). */
dicb200_status dicb200_accuracy_sweep(const int32_t* combos, size_t n_combos, const dicb200_sweep_config* cfg,
                                      dicb200_combo_accuracy* out, int32_t* warp_count, int32_t* poi_count,
                                      double* elapsed_s);

/* ---- f-3 output format (pipeline.cpp:216-238) ----
 * dicb200_field_csv: dic::field_csv_string (header + "%d,%d,%.17g,%.17g,%.17g,%d,%d,%ld"
 * rows); buf == NULL returns the size (incl. NUL) in *needed.
 * dicb200_write_field_csv: dic::write_field_csv. dicb200_field_filename:
 * "field_%04d.csv" (dic::field_filename). */
dicb200_status dicb200_field_csv(const dicb200_field* field, char* buf, size_t cap, size_t* needed);
dicb200_status dicb200_write_field_csv(const dicb200_field* field, const char* path);
dicb200_status dicb200_field_filename(int32_t pair_index, char* buf, size_t cap);

/* ---- f-4 bench matrix (bench.hpp:12-90, bench.cpp:14-293) ----
 * dicb200_run_bench replaces dic::run_bench: every cell strictly in order; per
 * cell one untimed warm-up repetition, then `repeats` timed repetitions
 * (auto_repeats bands from the warm-up unless auto_bands == 0), each = load the
 * sequence from disk (native PGM loader, pinned frames), analyze_sequence on
 * the GPU, write every field CSV under scratch_dir/cell-<int>-<sub>-<mode>/.
 * Cell failures (a failed pair, changing evaluation counts) are recorded in the
 * record, as the reference does; the call itself fails only on bad arguments.
 * dicb200_derive_ratios / dicb200_write_*_csv: dic::derive_ratios and the
 * reference's three CSV layouts, byte-identical formatting. */
typedef struct {  /* BenchCell, bench.hpp:12-16 */
  int32_t integer_method;
  int32_t subpixel_method;
  int32_t mode;
} dicb200_bench_cell;

typedef struct {  /* BenchRecord, bench.hpp:18-31 */
  dicb200_bench_cell cell;
  int32_t repeats;
  int32_t pair_count;
  int32_t failed;
  double mean_s;
  double stddev_s;
  double per_pair_s;
  double frame_rate_hz;  /* pair_count / mean_s */
  int64_t total_evaluations;
  char dataset_id[128];
  char error[160];
} dicb200_bench_record;

typedef struct {  /* RatioRow, bench.hpp:56-61 */
  char kind[32];     /* bfs_vs_pso | image_speedup_vs_serial | subimage_speedup_vs_serial */
  char detail[160];
  double value;      /* NaN when a needed cell is missing / failed */
  char note[32];
} dicb200_ratio_row;

int32_t dicb200_auto_repeats(double warmup_seconds); /* bench.cpp:14-19 */
dicb200_status dicb200_run_bench(const dicb200_bench_cell* cells, size_t n_cells, const char* dataset_dir,
                                 const char* pattern, const dicb200_run_config* base, int32_t auto_bands,
                                 int32_t fixed_repeats, const char* scratch_dir, int32_t load_flags,
                                 dicb200_bench_record* out);
/* rows: at most 3*3 + 3*3*2 = 27. */
dicb200_status dicb200_derive_ratios(const dicb200_bench_record* records, size_t n, const char* dataset_id,
                                     dicb200_ratio_row* rows, size_t cap, size_t* count);
dicb200_status dicb200_write_times_csv(const dicb200_bench_record* records, size_t n, const char* dataset_id,
                                       const char* path);
dicb200_status dicb200_write_records_csv(const dicb200_bench_record* records, size_t n, const char* path);
dicb200_status dicb200_write_ratios_csv(const dicb200_ratio_row* rows, size_t n, const char* path);

/* Release pooled device memory on all devices. */
void dicb200_shutdown(void);

#ifdef __cplusplus
}
#endif

#endif /* DICB200_H */
