/*
 * ltci_cuda.h -- C-ABI of the B200 dual-scale cascade (DS-GRFT / DS-KT-MFP).
 *
 * This is the drop-in boundary under the reference's C++ detector API.  Every
 * signature uses plain pointers, sizes and POD structs; no C++ or torch types.
 * A caller holding the reference types (`ltci::FreqPulseCube`,
 * `ltci::DualScaleSpace`, `ltci::DetectorOptions`, `ltci::DetectionMap`) fills
 * the POD mirrors below field by field; `paper_2403_06788_b200/csrc/dropin.cpp`
 * is that caller for C++ and `paper_2403_06788_b200/_lib.py` for Python.
 *
 * Reference interfaces replaced (paths relative to the reference repo root):
 *   ltci_cuda_ds_grft      -> ltci::ds_grft    proj/include/ltci/detectors.hpp:42-43
 *                                               proj/src/detectors.cpp:414-449
 *   ltci_cuda_ds_kt_mfp    -> ltci::ds_kt_mfp  proj/include/ltci/detectors.hpp:47-48
 *                                               proj/src/detectors.cpp:451-481
 *   ltci_cuda_keystone     -> ltci::keystone   proj/include/ltci/transforms.hpp:40
 *   ltci_cuda_mgift        -> ltci::mgift      proj/include/ltci/transforms.hpp:52-53
 *   ltci_cuda_td_grft      -> ltci::td_grft    proj/include/ltci/detectors.hpp:29-31
 *   ltci_cuda_kt_mfp       -> ltci::kt_mfp     proj/include/ltci/detectors.hpp:33-37
 *   ltci_cuda_gft          -> ltci::gft        proj/include/ltci/transforms.hpp:74-75
 *   ltci_cuda_detection_threshold -> ltci::detection_threshold
 *                                               proj/include/ltci/detectors.hpp:55
 * POD mirrors:
 *   ltci_radar        <- RadarParams     proj/include/ltci/radar_params.hpp:15-54
 *   ltci_grid         <- Grid            proj/include/ltci/search_space.hpp:12-22
 *   ltci_dual_space   <- DualScaleSpace  proj/include/ltci/search_space.hpp:68-77
 *                        (+ StepSizes :38-45, RangeRoi :30-36)
 *   ltci_ambiguity    <- AmbiguitySpace  proj/include/ltci/search_space.hpp:84-90
 *   ltci_options      <- DetectorOptions proj/include/ltci/detectors.hpp:14-20
 *   ltci_detection_map<- DetectionMap    proj/include/ltci/detection.hpp:47-73
 *
 * Cubes cross the boundary as interleaved (re, im) float64 arrays in the
 * reference's column-major layout, sample (k, m) at element k + K*m
 * (proj/include/ltci/cube.hpp:10-11).  Status codes map onto the reference's
 * exception types (see LTCI_* below); the message is in ltci_cuda_last_error().
 */
#ifndef LTCI_CUDA_H_
#define LTCI_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTCI_MAX_ORDER 4
#define LTCI_MAX_AXES 12  /* DS-GRFT has 2P + 1 axes: 9 at P = 4 */

/* status codes: the C++ shim rethrows the matching exception type */
enum {
    LTCI_OK = 0,
    LTCI_INVALID_ARGUMENT = 1, /* std::invalid_argument            */
    LTCI_CONDITION_VIOLATED = 2, /* ltci::ConditionViolated        */
    LTCI_RUNTIME_ERROR = 3,    /* std::runtime_error (CUDA failure) */
    LTCI_BAD_ALLOC = 4,        /* std::bad_alloc (result too large) */
    LTCI_NO_DEVICE = 5,        /* no CUDA device / extension missing */
    LTCI_IO_ERROR = 6,         /* ltci::IoError (cube file container) */
    LTCI_OUT_OF_RANGE = 7      /* std::out_of_range (td_grft, TrajectoryPolicy::Error) */
};

/* detector kinds, same order as ltci::DetectorKind (detection.hpp:12) */
enum { LTCI_FD_GRFT = 0, LTCI_TD_GRFT = 1, LTCI_KT_MFP = 2, LTCI_DS_GRFT = 3, LTCI_DS_KT_MFP = 4 };

/* axis roles, same order as ltci::AxisDesc::Role (detection.hpp:37) */
enum {
    LTCI_AXIS_RANGE = 0,
    LTCI_AXIS_VELOCITY = 1,
    LTCI_AXIS_HIGHER = 2,
    LTCI_AXIS_DOPPLER = 3,
    LTCI_AXIS_COARSE = 4,
    LTCI_AXIS_FINE = 5,
    LTCI_AXIS_FOLDING = 6
};

/* compensation variants, ltci::DetectorVariant (transforms.hpp:11) */
enum { LTCI_VARIANT_GRFT = 0, LTCI_VARIANT_KTMFP = 1 };

/* fine-stage formulations (both compute the same sums) */
enum {
    LTCI_FINE_AUTO = 0,
    LTCI_FINE_FFT_CUDA_CORE = 1, /* chirp recurrence + register/smem FFT, FP32   */
    LTCI_FINE_TC_DENSE = 2,      /* tcgen05 dense complex contraction, 3-term fp16 split (FP32 class) */
    LTCI_FINE_TC_FAST = 3        /* tcgen05, single fp16 term (~3e-4 of the row max; opt-in) */
};

typedef struct {
    double fc, fs, Br, delta_f, PRF;
    int32_t M, K, K_valid;
} ltci_radar;

typedef struct {
    double start, step;
    int32_t count;
} ltci_grid;

typedef struct {
    ltci_radar radar;
    int32_t order; /* P */
    ltci_grid coarse[LTCI_MAX_ORDER]; /* index p-1 for p = 1..P */
    ltci_grid fine[LTCI_MAX_ORDER];   /* index p-1, centred on 0, unscaled */
    double rm_step[LTCI_MAX_ORDER];   /* StepSizes::rm  */
    double dfm_step[LTCI_MAX_ORDER];  /* StepSizes::dfm */
    double alpha[LTCI_MAX_ORDER];     /* StepSizes::alpha */
    double kappa;
    int32_t roi_first, roi_last;      /* RangeRoi, inclusive */
} ltci_dual_space;

typedef struct {
    int32_t q_min, q_max;
} ltci_ambiguity;

/* SingleScaleSpace (proj/include/ltci/search_space.hpp:50-58): per-order grids
 * at the DFM step, c[p-1] for order p = 1..P, and the range ROI.  Built by
 * build_single_scale (proj/src/search_space.cpp:69-79). */
typedef struct {
    ltci_radar radar;
    int32_t order;                    /* P */
    ltci_grid c[LTCI_MAX_ORDER];      /* index p-1 */
    double rm_step[LTCI_MAX_ORDER];
    double dfm_step[LTCI_MAX_ORDER];
    double alpha[LTCI_MAX_ORDER];
    int32_t roi_first, roi_last;      /* RangeRoi, inclusive */
} ltci_single_space;

typedef struct {
    double retain_threshold; /* keep cells with |Y| > this (strict) */
    int32_t keep_dense;
    int32_t threads;         /* CPU threads in the reference; ignored (results never depend on it) */
    int32_t keystone_taps;
    int32_t trajectory;      /* ignored by the dual-scale detectors */
    int32_t fine_path;       /* LTCI_FINE_* (extension; AUTO picks per shape) */
    int32_t device;          /* CUDA device ordinal (extension) */
} ltci_options;

typedef struct {
    int32_t role, order, size;
} ltci_axis;

/* Result of one detector run.  All arrays are owned by the map and released
 * with ltci_cuda_free_map().  Candidate and dense values are complex
 * interleaved float64 (re, im), as ltci::DetectionMap stores them. */
typedef struct {
    int32_t kind;
    int32_t n_axes;
    ltci_axis axes[LTCI_MAX_AXES]; /* slowest first */
    uint64_t counters[4];          /* kt, mf, ifft, fft */
    double retain_threshold;
    int32_t doppler_first;

    uint64_t argmax;
    double argmax_value[2];

    uint64_t n_candidates;
    uint64_t *cand_index;  /* sorted ascending */
    double *cand_value;    /* 2 * n_candidates */

    int32_t dense_stored;
    uint64_t dense_count;
    double *dense;         /* 2 * dense_count */

    /* extension (no reference counterpart): per ROI range cell, the strongest
     * hypothesis over all coarse/fine/Doppler cells, ties to the lowest flat
     * index -- the per-cell peak map gathered across GPUs. */
    int32_t n_rows;
    uint64_t *peak_index;  /* n_rows */
    double *peak_value;    /* 2 * n_rows */
} ltci_detection_map;

/* ---- drop-in detectors (host buffers) ---------------------------------- */
int ltci_cuda_ds_grft(const double *cube, const ltci_radar *cube_params,
                      const ltci_dual_space *space, const ltci_options *opt,
                      ltci_detection_map **out);
int ltci_cuda_ds_kt_mfp(const double *cube, const ltci_radar *cube_params,
                        const ltci_ambiguity *amb, const ltci_dual_space *space,
                        const ltci_options *opt, ltci_detection_map **out);
void ltci_cuda_free_map(ltci_detection_map *map);

/* ---- kernel-level secondary boundary (host buffers, float64 complex) ---- */
/* ltci::fd_grft (proj/include/ltci/detectors.hpp:25-26, proj/src/detectors.cpp:105-197):
 * the single-scale frequency-domain GRFT, SURVEY.md §8(f) rank 2.  Same map
 * contract as the reference (axes c_P..c_2, c_1, range; flat index
 * cell * R + r; counters mf += K and ifft += 1 per motion cell; candidates
 * |v| > retain sorted by index; argmax over every cell, ties to the lowest
 * index).  Extension: an ROI outside [0, K) is LTCI_INVALID_ARGUMENT. */
int ltci_cuda_fd_grft(const double *cube, const ltci_radar *cube_params, const ltci_single_space *space,
                      const ltci_options *opt, ltci_detection_map **out);
/* ltci::td_grft (proj/include/ltci/detectors.hpp:29-31, proj/src/detectors.cpp:199-264):
 * the single-scale time-domain GRFT over a RANGE-pulse cube (data[n + K*m]):
 * per motion cell and ROI row the sum over pulses of the nearest-bin sample
 * along the trajectory, n(m) = lround(n0 + (2 fs / c) S(t_m)), times
 * exp(j 4 pi S(t_m) / lambda).  opt->trajectory is the reference's
 * TrajectoryPolicy for bins outside [0, K): 0 contribute zero, 1 wrap modulo
 * K, 2 raise (LTCI_OUT_OF_RANGE = std::out_of_range, same message).  Map
 * contract as fd_grft's (kind LTCI_TD_GRFT; counter mf += 1 per (cell, row)). */
int ltci_cuda_td_grft(const double *range_cube, const ltci_radar *cube_params, const ltci_single_space *space,
                      const ltci_options *opt, ltci_detection_map **out);
/* ltci::kt_mfp (proj/include/ltci/detectors.hpp:33-37, proj/src/detectors.cpp:266-326):
 * keystone once, then per (folding number q, acceleration c2) cell the
 * matched filter over the full Doppler axis.  `space` must have order 2 (its
 * velocity grid is unused).  Axes [Folding, Higher 2, Range, Doppler], flat
 * index ((iq * n2 + i2) * R + r) * M + j, counters kt = 1, mf += K, ifft += M,
 * fft += R per cell.  Runs the dual-scale keystone cascade with one fine cell. */
int ltci_cuda_kt_mfp(const double *cube, const ltci_radar *cube_params, const ltci_ambiguity *amb,
                     const ltci_single_space *space, const ltci_options *opt, ltci_detection_map **out);
int ltci_cuda_keystone(const double *cube, const ltci_radar *p, int taps, double *out);
/* keystone on device complex64 cubes (K*M float2, column-major), asynchronous
 * on the given cudaStream_t: the K4 kernel ds_kt_mfp runs, for timing it over
 * back-to-back calls and for device-resident pipelines */
int ltci_cuda_keystone_device(const void *d_in, void *d_out, const ltci_radar *p, int taps, void *stream);
/* range_fft -> ltci::range_fft  proj/include/ltci/signal_model.hpp:37
 * (proj/src/signal_model.cpp:97-107): per pulse the unnormalised forward
 * K-point DFT of a range-pulse cube (K*M complex, column-major k + K m),
 * giving the freq-pulse cube the detectors take; range_fft(range_ifft(x)) ==
 * K x.  K a power of two in [16, 8192].  Values out are complex64-exact. */
int ltci_cuda_range_fft(const double *range_cube, const ltci_radar *p, double *out);
int ltci_cuda_range_fft_device(const void *d_in, void *d_out, const ltci_radar *p, void *stream);
int ltci_cuda_mgift(const double *cube, const ltci_radar *p, const double *ctilde, int n_ctilde,
                    int variant, double *out /* K*M complex */);
int ltci_cuda_gft(const double *rows, const ltci_radar *p, const double *fine_higher, int n_fine,
                  int roi_first, int roi_last, double *out /* R*M complex, (r,j) at r+R*j */);
double ltci_cuda_detection_threshold(const ltci_radar *p, double sigma2, double pfa, int bins,
                                     int *status);

/* ---- detection extraction (host C++, over the returned candidates) ------ */
/* One detection: motion estimate c[0..n_coef-1] (c0 = range, c1 = velocity,
 * c_p = order-p coefficient), statistic |Y|, flat cell index, and for
 * DS-KT-MFP the folding factor and baseband velocity.
 * Replaces Detection (proj/include/ltci/detection.hpp:76-82). */
typedef struct {
    double statistic;
    double c[LTCI_MAX_ORDER + 1];
    int32_t n_coef;
    int32_t has_q;
    int32_t q;
    double baseband_velocity;
    uint64_t flat_index;
} ltci_detection;

/* extract_detections (proj/src/detection.cpp:158-244): local maxima over the
 * range / Doppler / order-2 axes among candidates above gamma, recomposed with
 * detection_from_cell (:124-153), near-duplicates merged along the ridge,
 * strongest first.  Writes min(n, max_out) detections, returns n in *n_out.
 * amb may be NULL for DS-GRFT maps. */
int ltci_cuda_extract_detections(const ltci_detection_map *map, const ltci_dual_space *space,
                                 const ltci_ambiguity *amb, double gamma, ltci_detection *out,
                                 int max_out, int *n_out);
/* extract_detections for single-scale (FD-GRFT) maps: detection_from_cell
 * proj/src/detection.cpp:101-111, cell sizes :59-63 */
int ltci_cuda_extract_detections_single(const ltci_detection_map *map, const ltci_single_space *space,
                                        double gamma, ltci_detection *out, int max_out, int *n_out);

/* ---- engine: device-resident plan for streaming / benchmarking ---------- */
typedef struct ltci_engine ltci_engine;

/* variant: LTCI_VARIANT_GRFT (ds_grft) or LTCI_VARIANT_KTMFP (ds_kt_mfp; amb required).
 * row_begin/row_end select a contiguous slice [row_begin, row_end) of the ROI
 * rows (0 .. roi.count()) for range-cell sharding; pass 0, -1 for all rows. */
int ltci_engine_create(const ltci_radar *p, const ltci_dual_space *space, const ltci_ambiguity *amb,
                       int variant, const ltci_options *opt, int row_begin, int row_end,
                       ltci_engine **out);
void ltci_engine_destroy(ltci_engine *e);
/* Run on a device-resident complex64 cube (K*M float2, column-major) on the
 * given cudaStream_t (NULL = legacy default).  Asynchronous.  The engine keeps
 * a private copy of the cube (queued on the stream behind the run), so the
 * caller may overwrite its buffer once the stream has passed this run, even
 * before ltci_engine_result(). */
int ltci_engine_run_device(ltci_engine *e, const void *d_cube_c64, void *stream);
/* Same from a host float64 cube: H2D, run, D2H of the reduced results. */
int ltci_engine_run_host(ltci_engine *e, const double *cube, void *stream);
/* configs[3] front end: the input is a RANGE-pulse cube (range-compressed
 * fast-time samples, K*M column-major); K0 (ltci::range_fft,
 * proj/src/signal_model.cpp:97-107) turns it into the freq-pulse cube on the
 * device, then the cascade runs.  Device complex64 or host float64 input. */
int ltci_engine_run_range_device(ltci_engine *e, const void *d_range_c64, void *stream);
int ltci_engine_run_range_host(ltci_engine *e, const double *range_cube, void *stream);
/* Copy the reduced results of the last run to the host and build a map
 * (synchronises the stream).  Candidates overflowing the device buffer make
 * the engine re-run with a larger buffer, or fail with LTCI_BAD_ALLOC. */
int ltci_engine_result(ltci_engine *e, void *stream, ltci_detection_map **out);
/* Device pointer to the per-row peak records of the last run:
 * n_rows records of {float re, float im, uint64 flat_index} (16 B each). */
int ltci_engine_peaks_device(ltci_engine *e, void **d_ptr, int32_t *n_rows);
/* Instrumentation: number of kernel launches issued by the last run, and the
 * device time (ms) of the fine and coarse stages when timing is enabled. */
int ltci_engine_stats(ltci_engine *e, int64_t *launches, double *fine_ms, double *coarse_ms,
                      double *keystone_ms);
int ltci_engine_set_timing(ltci_engine *e, int enable);
/* Fine-stage formulation this engine runs (LTCI_FINE_FFT_CUDA_CORE or
 * LTCI_FINE_TC_DENSE / LTCI_FINE_TC_FAST) and its fp16 split terms (0 for FFT). */
int ltci_engine_fine_path(ltci_engine *e, int32_t *path, int32_t *terms);
/* Coarse-stage (mgift, proj/src/transforms.cpp:134-173) formulation this engine
 * runs: LTCI_COARSE_TRANSFORM = one K-point transform per (coarse cell, pulse),
 * LTCI_COARSE_GATHER = interpolation of 2x-oversampled range profiles tabulated
 * once per pulse (the default before the FP32 fine path; LTCI_COARSE=transform
 * or =gather in the environment forces one). */
enum { LTCI_COARSE_TRANSFORM = 0, LTCI_COARSE_GATHER = 1 };
int ltci_engine_coarse_path(ltci_engine *e, int32_t *path);
/* hypotheses (cells) and integrations covered by this engine's row slice */
int ltci_engine_work(ltci_engine *e, uint64_t *hypotheses, uint64_t *integrations);
/* extension: restrict the engine to coarse cells [c_begin, c_end) of the plan
 * (coarse-cell sharding: each GPU searches its coarse cells over every ROI row,
 * nothing is replicated; flat indices stay global; c_end = UINT64_MAX means
 * the last coarse cell).  Per-row peaks of the
 * shards combine with ltci_cuda_merge_peaks, candidates by concatenation. */
int ltci_engine_set_coarse_slice(ltci_engine *e, uint64_t c_begin, uint64_t c_end);
/* per-row best of n_maps device peak-slot arrays ({f32 re, f32 im, u64 flat},
 * n_maps x n_rows, map-major) with the kernels' own magnitude and tie-break */
int ltci_cuda_merge_peaks(const void *d_slots, int n_maps, int n_rows, void *d_out, void *stream);

/* ---- cube file container ------------------------
 * The reference's "LTCI" little-endian container (proj/include/ltci/cube_io.hpp:
 * 9-14): magic, version u32 = 1, domain u8 (0 freq-pulse, 1 range-pulse),
 * K, M, K_valid u32, fc, fs, Br, PRF, sigma2 f64 (61-byte header), then K*M
 * complex samples as (re, im) f64 pairs, pulse-major.  Errors mirror
 * ltci::IoError (LTCI_IO_ERROR) with the reference's messages. */
typedef struct {
    int32_t domain;     /* 0 = freq-pulse, 1 = range-pulse */
    ltci_radar radar;   /* rebuilt with RadarParams::create semantics */
    double sigma2;
} ltci_cube_header;

/* header only (read_cube_file's checks on the first 61 bytes and the
 * payload length / trailing bytes; proj/src/cube_io.cpp:121-170) */
int ltci_cuda_cube_file_info(const char *path, ltci_cube_header *out);
/* read_cube_file (proj/src/cube_io.cpp:121-179): payload into a host buffer of
 * 2*K*M doubles (capacity checked) */
int ltci_cuda_cube_file_read(const char *path, ltci_cube_header *hdr, double *out, uint64_t capacity_doubles);
/* write_cube_file (proj/src/cube_io.cpp:66-119): temp file + rename */
int ltci_cuda_cube_file_write(const char *path, const ltci_cube_header *hdr, const double *data);
/* The wire path: stream a freq-pulse cube file through pinned staging buffers
 * straight into the engine's device echo (chunked fread overlapped with async
 * H2D, f64 -> c64 on the device), then run.  Replaces read_cube_file +
 * CubeFile::to_freq_cube + ds_grft/ds_kt_mfp (proj/tools/ltci_main.cpp:67-137).
 * The file's radar must equal the engine's (reference: radar mismatch ->
 * invalid_argument); a range-pulse file is ConditionViolated as in
 * CubeFile::to_freq_cube (proj/src/cube_io.cpp:48-52). */
int ltci_engine_run_file(ltci_engine *e, const char *path, void *stream);

/* ---- batched Monte-Carlo Pd ----------------------
 * Target / Scenario / PdPoint of proj/include/ltci/{signal_model,bench}.hpp. */
#define LTCI_MAX_TARGETS 8
#define LTCI_MAX_SNR 64
typedef struct {
    double amp[2];                      /* complex amplitude (unit scale in a Scenario) */
    int32_t order;                      /* motion order: c[0..order] used */
    double c[LTCI_MAX_ORDER + 1];       /* slant range c0 + c1 t + c2 t^2 + ... (MotionParams) */
} ltci_target;

typedef struct {
    ltci_radar radar;
    int32_t n_targets;
    ltci_target targets[LTCI_MAX_TARGETS];  /* targets[0] is the truth */
    int32_t n_snr;
    double snr_db[LTCI_MAX_SNR];
    int32_t trials;
    double pfa, sigma2;
    uint64_t seed;
    int32_t n_detectors;
    int32_t detectors[5];               /* LTCI_FD_GRFT, LTCI_DS_GRFT, LTCI_DS_KT_MFP (GPU-built kinds) */
    int32_t P;
    double bound_lo[LTCI_MAX_ORDER], bound_hi[LTCI_MAX_ORDER], alpha[LTCI_MAX_ORDER];
    int32_t roi_first, roi_last;
    int32_t keystone_taps;
    int32_t device;
} ltci_scenario;

typedef struct {
    double snr_db, pd;
    int32_t trials;
    double ci_lo, ci_hi;                /* 95 % Wilson interval (bench.cpp:60-68) */
} ltci_pd_point;

/* synthesize_cube (proj/src/signal_model.cpp:32-51) evaluated on the device in
 * FP64; out = 2*K*M doubles, data[k + K*m] */
int ltci_cuda_synthesize(const ltci_radar *p, int n_targets, const ltci_target *targets, double *out);
/* add_noise (proj/src/signal_model.cpp:53-60): the splitmix64 / Box-Muller
 * stream of GaussianRng (proj/src/rng.cpp:8-43) generated per element on the
 * device (element i uses draws 2i+1, 2i+2 of the counter-based stream) */
int ltci_cuda_add_noise(const double *cube, const ltci_radar *p, double sigma2, uint64_t seed, double *out);
/* run_pd (proj/src/bench.cpp:72-124): every trial's noisy cube is generated on
 * the device and searched there; out[d * n_snr + s] for detector d, SNR s */
int ltci_cuda_run_pd(const ltci_scenario *sc, ltci_pd_point *out);

/* Idle one-shot engines (ltci_cuda_ds_grft / ds_kt_mfp) and fd_grft
 * workspaces pooled for a device.  Both pools are process-wide and keep at
 * most LTCI_POOL_IDLE (default 2) idle objects per device, however many host
 * threads call in parallel (the reference's callers fan detector calls out
 * over threads, proj/src/bench.cpp:94-110). */
int ltci_cuda_pool_idle(int device, int64_t *engines, int64_t *fd_workspaces);

/* Roofline denominator for the CUDA-core fine path: dense FP32 FFMA issue
 * rate of this device, measured with a register-resident FMA chain kernel
 * over all SMs (TFLOP/s, 2 flop per FFMA). */
int ltci_cuda_measure_fp32_peak(int device, double *tflops);

const char *ltci_cuda_last_error(void);
int ltci_cuda_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LTCI_CUDA_H_ */
