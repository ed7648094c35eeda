/*
 * frir.h -- C ABI of the B200-native FRAM-RIR generator (libfrir.so).
 *
 * The reference (arxiv 2304.08052, /root/reference/pkg) has no native FFI: its
 * drop-in boundary is the pure-Python call
 *     framrir.simulate_rir(params, scene, include_early=True)   core.py:268-316
 * and the dataloader veneer
 *     framrir_binding.py_simulate_rir(config, include_early)    binding/.../__init__.py:66-94
 * Both are mirrored in Python by paper_2304_08052_b200 (same names, arguments,
 * defaults and ValueError texts) on top of the entry points declared here.
 * Each entry point below names the reference function(s) whose arithmetic it
 * replaces.  Plain C types only: no torch, no C++ across the boundary.
 *
 * Conventions
 *   - Every function returns FRIR_OK (0) or a negative status; the message of
 *     the last failure on the calling thread is in frir_last_error().
 *   - Device pointers are allocated by the caller (the library never allocates
 *     on the hot path); `stream` is a cudaStream_t passed as void*.
 *   - frir_simulate is asynchronous on `stream` and re-entrant across streams
 *     (the plan is read-only after creation).
 */
#ifndef FRIR_H_
#define FRIR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRIR_ABI_VERSION 3

enum {
  FRIR_OK = 0,
  FRIR_EINVAL = -1, /* invalid argument (reference ValueError) */
  FRIR_ECUDA = -2,  /* CUDA runtime / launch failure */
  FRIR_ERANGE = -3, /* size outside what the kernels support */
  FRIR_ENOMEM = -4  /* workspace too small */
};

/* Table ids for frir_design_table (host-only test hooks). */
enum {
  FRIR_TAB_H1 = 0,        /* stage-1 Kaiser taps, resample.py:74-78 (firwin, unscaled) */
  FRIR_TAB_H2 = 1,        /* stage-2 Kaiser taps */
  FRIR_TAB_SOS = 2,       /* 80 Hz Butterworth HP section [b0 b1 b2 1 a1 a2], resample.py:109 */
  FRIR_TAB_COMP_D = 3,    /* composite decimation table, t in [t0, t0 + r_h*sup) */
  FRIR_TAB_COMP_W = 4,    /* composite low-pass-branch table, same t range */
  FRIR_TAB_KAPPA = 5,     /* tail-correction state gains, [half2][2] */
  FRIR_TAB_U = 6,         /* tail-correction input response (h2 * HP impulse), [half2] */
  FRIR_TAB_ZPHASE = 7,    /* per-phase modal tap sums, [down][2] (re, im) */
  FRIR_TAB_PPOW = 8,      /* p^m, m < horizon, [horizon][2] (re, im) */
  FRIR_TAB_LPCOEF = 9,    /* [c1, c2, v0 (4 doubles: re0 im0 re1 im1)] */
  FRIR_TAB_GW = 10        /* low-pass-branch filter h2 * N * B' (head correction) */
};

typedef struct frir_plan frir_plan;

/* Per-sample-rate constants (resample.py:59-71 rate_factors, :74-78, :107-113). */
typedef struct {
  int32_t sample_rate;
  int32_t r_h, r_l;          /* rate factors: r_h = 10^6 // fs, r_l = isqrt(r_h) */
  int32_t up, down;          /* stage-1 ratio reduced by gcd (scipy resample_poly) */
  int32_t half1, len1;       /* stage-1 taps: 2*half1 + 1 */
  int32_t half2, len2;       /* stage-2 taps */
  int32_t t0, sup;           /* composite support: t in [t0, t0 + r_h*sup) */
  int32_t nb;                /* look-back windows for the 32-sample gather */
  int32_t horizon;           /* mid-rate samples of HP memory kept by the tail fix */
  int32_t lt_max;            /* max stage-1 taps past n1 */
  int32_t pad_;
  double sos[6];             /* [b0 b1 b2 1 a1 a2] */
  double c1, c2;             /* output-rate LP recursion */
} frir_plan_desc;

/*
 * One RIR job = one (room, source).  Inputs mirror SimParams (params.py:38-47)
 * and Scene (params.py:77-80).  Layout/derived fields are filled by
 * frir_jobs_prepare() on the host.  Keep in sync with
 * paper_2304_08052_b200/_abi.py (numpy structured dtype).
 */
typedef struct {
  /* ---- inputs ---- */
  double room[3];            /* room_dims (m) */
  double center[3];          /* array reference point in the mic frame (params.py:149-153) */
  double d0, az, el;         /* source (distance, azimuth, elevation) rel. to center */
  double t60;                /* SimParams.t60 */
  double c0;                 /* SimParams.sound_speed */
  double alpha, beta;        /* distance-ratio support */
  double perturb_lo, perturb_hi;
  double tau;
  uint64_t seed;             /* SimParams.seed (0 <= seed < 2^64) */
  int32_t source_index;      /* k: Philox stream (seed, k, stage), core.py:86-91 */
  int32_t n_images;          /* I (SimParams.num_images), per job */
  int32_t mic_off;           /* first mic row in frir_batch.mics */
  int32_t n_mics;            /* M */
  /* ---- extensions (defaults reproduce the reference) ---- */
  int32_t n_images_hi;       /* > n_images: I ~ U{n_images..n_images_hi} from stream (seed, k, 2) */
  int32_t normalize;         /* 0: reference scaling; 1: direct path of every channel = 1/1 m (x D_0m) */
  int32_t kind;              /* FRIR_KIND_FRAM (0) or FRIR_KIND_ISM (1), see below */
  int32_t lattice;           /* ISM: 1 + max_order to generate the image lattice on the device (0: images as batch draws) */
  double early_lo_ms;        /* early window [-lo, +hi] ms around the direct path; 0/0 means 6/50 */
  double early_hi_ms;
  double duration;           /* ISM: train length in s (0: t60), ism.py:39-60 */
  double reflection;         /* ISM: reflection coefficient override (0: Eyring from room, t60) */
  /* ---- layout (frir_jobs_prepare) ---- */
  int64_t img_off;           /* first image row (row 0 = direct path) */
  int64_t item_off;          /* first (image, mic) item */
  int64_t out_off;           /* first output sample (floats) */
  int32_t chan_off;          /* first channel */
  int32_t out_stride;        /* floats between channel rows */
  int32_t L;                 /* high-rate train length ceil(t60 * r_h * fs) */
  int32_t n1, n2;            /* mid / output lengths */
  int32_t pad_;
  /* ---- derived (frir_jobs_prepare) ---- */
  double r;                  /* reflection coefficient, core.py:113-128 */
  double rr_max;             /* max_reflections, core.py:186-192 (0 when I == 0) */
  double alpha3, b3a3;       /* alpha**3 and beta**3 - alpha**3 (core.py:100) */
  double log2r;              /* log2(r): gains r**g are evaluated as exp2(g log2 r) in FP32 */
  int32_t e_lo, e_hi;        /* early window in high-rate samples (core.py:257-258) */
  uint64_t key[4];          /* Philox keys of streams (seed, k, 0) and (seed, k, 1) */
} frir_job;

/* Job kinds.  FRIR_KIND_ISM runs the shoebox image-source reference
   (ism.py:81-147, ism_rir) through the same chain.  Row 0 is the source
   itself at `center` (d0 = 0); the images are either generated on the device
   (`lattice` = K + 1: the (2K + 1)^3 - 1 lattice points of enumerate_images,
   ism.py:80-104, in its order without the origin; frir_jobs_prepare sets
   n_images) or given as batch draws (draw_dist, draw_az, draw_el = ABSOLUTE
   x, y, z of image i, draw_refl = its integer reflection count g).  Gains are
   r^g / D with r = exp(-0.0805 V/S/t60) (ism.py:63-78) unless `reflection`
   > 0, and arrivals past the train end are dropped instead of clamped
   (ism.py:131-133).  Full variant only. */
/* FRIR_KIND_TRAIN: an explicit high-rate train (downsample_highpass_downsample
   on a HighRateTrain or (M, L) array, resample.py:81-136) rendered by
   frir_simulate_train; `duration` holds its length L in samples and
   n_images + 1 the item slots per channel (frir_train_nonzeros). */
enum { FRIR_KIND_FRAM = 0, FRIR_KIND_ISM = 1, FRIR_KIND_TRAIN = 2 };

typedef struct {
  const frir_job* jobs;      /* device, n_jobs entries */
  int32_t n_jobs;
  int32_t total_channels;    /* sum of n_mics */
  const int32_t* chan_job;   /* device, job index of every channel */
  const int32_t* chan_order; /* device, processing order of channels (longest first) or NULL */
  const double* mics;        /* device, mic rows (x, y, z) */
  /* Oracle mode: the reference's own draws (ImageSet fields, core.py:43-62),
     indexed img_off + i for i in [1, I]; all NULL in native mode. */
  const double* draw_dist;   /* ImageSet.distances   */
  const double* draw_az;     /* ImageSet.azimuths    */
  const double* draw_el;     /* ImageSet.elevations  */
  const double* draw_refl;   /* ImageSet.reflections */
  int64_t total_images;      /* sum (I + 1) */
  int64_t total_items;       /* sum M (I + 1) */
  int64_t total_out;         /* floats per output buffer */
  int32_t max_rows;          /* max (I + 1) */
  int32_t max_windows;       /* max ceil((n2 + 10) / 32) */
} frir_batch;

/* ---- plans ---------------------------------------------------------------- */

/* Host filter design (firwin/kaiser/butter restated, composite tables) and upload
   to the current CUDA device.  Replaces resample.py:74-78,107-113 setup. */
int frir_plan_create(int32_t sample_rate, frir_plan** out);
int frir_plan_describe(const frir_plan* plan, frir_plan_desc* out);
int frir_plan_destroy(frir_plan* plan);

/* Host-only (no GPU): design tables for tests.  Writes up to `cap` doubles. */
int frir_design_describe(int32_t sample_rate, frir_plan_desc* out);
int frir_design_table(int32_t sample_rate, int32_t which, double* out, int64_t cap,
                      int64_t* n_out);

/* Host-only (no GPU): uniform doubles of numpy's
   Generator(Philox(SeedSequence((seed, k, stage)))).random(), words
   [first, first + n).  Restates core.py:86-91 + numpy 2.x Philox4x64-10. */
int frir_philox_doubles(uint64_t seed, uint64_t source_index, uint64_t stage,
                        uint64_t first_word, int64_t n, double* out);

/* ---- batches -------------------------------------------------------------- */

/* Host (no GPU): validate jobs (reference ValueError rules, core.py:113-128,140-148,186-192,
   209-210) and fill layout + derived fields.  `padded` != 0 lays the outputs out
   as [job][mic][max_n2]; otherwise packed.  Fills the totals of `batch` (pointers
   untouched).  chan_job / chan_order (nullable, sum(n_mics) entries each)
   receive the job of every channel and a longest-first processing order. */
int frir_jobs_prepare(int32_t sample_rate, frir_job* jobs_host, int32_t n_jobs,
                      int32_t padded, frir_batch* batch, int32_t* chan_job,
                      int32_t* chan_order);

/* Bytes of device workspace frir_simulate needs for `batch`. */
size_t frir_workspace_size(const frir_plan* plan, const frir_batch* batch);

/* Render every job of the batch: full (and, if out_early != NULL, early) RIRs.
   `workspace` must be 256-byte aligned and the outputs 16-byte aligned (any
   cudaMalloc'd buffer is); otherwise FRIR_EINVAL.
   Replaces core.py:131-265 (sampling, delays, train, early window) and
   resample.py:81-136 (both decimation stages and the HP).  direct_index gets
   RirFilter.direct_path_sample per channel (resample.py:115-119).  Draws come
   from device Philox streams unless the batch carries oracle draws. */
int frir_simulate(const frir_plan* plan, const frir_batch* batch, void* workspace,
                  size_t workspace_bytes, float* out_full, float* out_early,
                  int32_t* direct_index, void* stream);

/* frir_simulate split into its stages (bit 0: sampling/geometry K1, bit 1:
   delays + per-channel sort K2 and tail corrections K2b, bit 2: render K3 and,
   for batches with long channels, the segment seams K4); stages must run in order on
   one stream with the same workspace.  Lets callers time the render kernel. */
#define FRIR_STAGE_GEOM 1
#define FRIR_STAGE_DELAY 2
#define FRIR_STAGE_RENDER 4
#define FRIR_STAGE_ALL 7
int frir_simulate_stages(const frir_plan* plan, const frir_batch* batch, void* workspace,
                         size_t workspace_bytes, float* out_full, float* out_early,
                         int32_t* direct_index, void* stream, int32_t stages);

/* Kernel launches frir_simulate issues for `batch` (for launch accounting). */
int32_t frir_launch_count(const frir_plan* plan, const frir_batch* batch, int32_t early);

/* ---- spatialise-and-mix consumer (mixture.py:216-332) ----
   All pointers are device pointers. */

/* Hand-written FFT convolution of every filter row with its source (the
   fftconvolve of mixture.py:216-218): uniformly partitioned overlap-save with
   8192-point shared-memory FFTs (csrc/frir_fftconv.cu).  Sources: speaker k
   of item b is dry[b*dry_stride_b + k*dry_stride_k + 0 .. lengths[b][k]),
   placed at offsets[b][k] (mixture.py:274-287); the point noise
   noise[b*noise_stride ..] tiled to dry_len[b] samples (noise_len[b] long,
   mixture.py:307-312).  Filters: item b's [S+1][M][R] full rows at
   rir_full + b*full_stride_b and [>= S][M][R] early rows at rir_early +
   b*early_stride_b (full when rir_early is NULL), rir_len[b] valid taps.
   Output y[b][j][y_stride] with rows j as for
   frir_mix_combine, valid for t < T.  frir_mix_convolve_scratch returns the
   scratch bytes (spectra) and the minimum y_stride. */
int64_t frir_mix_convolve_scratch(int32_t B, int32_t S, int32_t M, int64_t R, int64_t T, int64_t* y_stride);
int frir_mix_convolve(const float* dry, int64_t dry_stride_b, int64_t dry_stride_k, const float* noise,
                      int64_t noise_stride, const int32_t* offsets, const int32_t* lengths, const int32_t* noise_len,
                      const int32_t* dry_len, const float* rir_full, int64_t full_stride_b, const float* rir_early,
                      int64_t early_stride_b, const int32_t* rir_len, int32_t B, int32_t S, int32_t M, int64_t R,
                      int64_t T, void* scratch, int64_t scratch_bytes, float* y, int64_t y_stride, void* stream);
/* _power (mixture.py:221-222): out[r] = mean(y[req_row[r]][req_lo[r]:req_hi[r]]^2),
   FP64, fixed-order sums; scratch holds FRIR_MIX_POWER_CHUNKS doubles per request. */
#define FRIR_MIX_POWER_CHUNKS 32
int frir_mix_powers(const float* y, int64_t F, const int64_t* req_row, const int32_t* req_lo,
                    const int32_t* req_hi, int32_t n_req, double* scratch, double* out, void* stream);
/* SIR / SNR gains (mixture.py:285-311): powers[b] = {p_ref, (p_int_k, p_tgt_k)
   for k = 1..S-1, p_noise}; gains[b] = {1, g_1 .. g_{S-1}, g_noise};
   sir_db is [B][max(S-1, 1)], snr_db [B]. */
int frir_mix_gains(const double* powers, const double* sir_db, const double* snr_db, int32_t B,
                   int32_t S, double* gains, void* stream);
/* Scaled references and the mixture (mixture.py:293-313) from the convolved
   rows y[b][j][F] (j = kM+m full of speaker k, (S+k)M+m early, 2SM+m noise):
   outputs [B][S][M][T] (sources, early), [B][M][T] (noise, mixture); samples
   at t >= total[b] are zero. */
int frir_mix_combine(const float* y, const double* gains, const int32_t* total, int32_t B, int32_t S,
                     int32_t M, int64_t F, int64_t T, float* mixture, float* sources, float* early,
                     float* noise, void* stream);

/* ---- on-device scene sampler (mixture.py:171-213) ----
   Items first_index .. first_index + count - 1 of sample_scene's stream
   Philox(SeedSequence((seed, index))): room, T60, then n_sources placements
   (distance, azimuth, elevation) and the simulation seed, bit-identical to
   numpy's draws; written as n_sources render jobs per item (SimParams
   defaults for the other knobs, the reference's validation rules) with a
   fixed row stride, plus chan_job, and a per-item status (0 ok; 1 aperture
   not below the smallest room dimension; 2 c0*t60 not above a source
   distance; 3 reflection / rr_max rule; 4 T60 longer than out_stride allows).
   Jobs are ready for frir_simulate with batch totals computed by the caller
   from the fixed sizes. */
typedef struct {
  double room_length[2], room_width[2], room_height[2];  /* uniform ranges */
  double t60[2];             /* spec.t60_range or the curriculum bounds */
  double distance[2];        /* spec.speaker_distance */
  double elevation[2];       /* spec.elevation_range */
  double center[3];          /* array reference point (mic centroid) */
  double aperture;           /* largest mic-to-mic distance */
  double c0;                 /* sound speed */
  double alpha3, b3a3;       /* alpha**3, beta**3 - alpha**3 of the SimParams defaults (host pow) */
  int32_t n_sources;         /* speakers + point noise */
  int32_t n_mics;
  int32_t num_images;
  int32_t out_stride;        /* floats per channel row: >= max n2, multiple of 4 */
} frir_scene_spec;
int frir_sample_scene_jobs(const frir_plan* plan, const frir_scene_spec* spec, uint64_t seed, int64_t first_index,
                           int32_t count, frir_job* jobs, int32_t* chan_job, int32_t* status, void* stream);

/* ---- batched decay measurement (decay.py:8-49) ----
   Rows h[c][0:len[c]] (float32, row stride ld floats).  frir_edc writes the
   unnormalised energy decay curve edc[c][i] = sum_{j>=i} h[c][j]^2 in FP64,
   summed sequentially from the end exactly like numpy's cumsum of the
   reversed squares (bit-identical), zeros for len[c] <= i < ld_out, and
   amax[c] = max |h[c]|. */
int frir_edc(const float* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
             double* amax, void* stream);
/* measure_t60 (decay.py:20-49) per row from frir_edc's outputs: NaN when the
   row has no energy or less than min_drop dB of usable range. */
int frir_t60(const float* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
             const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
             double* t60, void* stream);
/* The same two entry points on float64 rows (the reference works in FP64,
   decay.py:11-17): squares and sums in FP64 from the FP64 samples, so the
   curve is bit-identical to numpy's for any input the reference accepts. */
int frir_edc_f64(const double* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
                 double* amax, void* stream);
int frir_t60_f64(const double* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
                 const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
                 double* t60, void* stream);

/* ---- stage API (reference framrir/__init__.py:15-28) ---------------------
   Device forms of the reference's public stage functions, for callers that
   use them one by one; the batched hot path above never materialises these
   intermediates.  All buffers are device memory, FP64 in numpy's operation
   order, asynchronous on `stream`. */

/* Elementwise stage arithmetic.  params[0..3] per op:
   FRIR_STAGE_RATIO_SAMPLE  quadratic_ratio_sample (core.py:94-100) from the
                            uniform draws x0: {alpha**3, beta**3, -, -}
   FRIR_STAGE_RESCALE       rescale_distance_ratio (core.py:103-110) of x0:
                            {alpha, beta, max_ratio, -}
   FRIR_STAGE_REFLECTIONS   sample_reflection_counts (core.py:213-220): x0 = D,
                            x1 = DR, x2 = perturbation p: {c0*t60, rr_max, tau, -} */
#define FRIR_STAGE_RATIO_SAMPLE 0
#define FRIR_STAGE_RESCALE 1
#define FRIR_STAGE_REFLECTIONS 2
int frir_stage_eval(int32_t op, const double* x0, const double* x1, const double* x2, int64_t n,
                    const double* params /* host, 4 */, double* out, void* stream);
/* Generator(Philox(SeedSequence((seed, k, stage)))).uniform(lo, hi) words
   [first_word, first_word + n) on the device (core.py:86-91, :215). */
int frir_philox_uniform(uint64_t seed, uint64_t source_index, uint64_t stage, int64_t first_word, int64_t n,
                        double lo, double hi, double* out, void* stream);
/* sample_image_geometry (core.py:131-183) for every (native-draw) job of the
   batch: ImageSet rows at img_off + i (i = 0 the direct path), per-mic
   distances row-major at item_off + i * n_mics + m; reflection counts from
   the stage-1 stream when with_reflections, else NaN (rows >= 1) as the
   reference leaves them. */
int frir_image_set(const frir_plan* plan, const frir_batch* batch, double* distances, double* azimuths,
                   double* elevations, double* distance_ratios, double* reflections, double* mic_distances,
                   int32_t with_reflections, void* stream);
/* build_impulse_train (core.py:228-251): q = min(ceil(D / c0 * rate), L - 1)
   (int32, rows x n_mics) and the dense (n_mics, L) FP64 train, colliding
   arrivals summed in row order like np.add.at.  scratch: device bytes >=
   frir_impulse_train_scratch(). */
int64_t frir_impulse_train_scratch(int32_t rows, int32_t n_mics, int32_t length);
int frir_impulse_train(const double* mic_distances, const double* reflections, int32_t rows, int32_t n_mics,
                       double r, double sound_speed, int64_t rate, int32_t length, double* train, int32_t* q,
                       void* scratch, int64_t scratch_bytes, void* stream);
/* early_reverb_train (core.py:254-265): out = train where
   -lo <= n - q0[m] <= hi, else 0. */
int frir_early_window(const double* train, int32_t n_mics, int64_t length, const int32_t* q0, int64_t lo,
                      int64_t hi, double* out, void* stream);
/* downsample_highpass_downsample (resample.py:81-136) of explicit trains:
   frir_train_nonzeros counts the samples with sign * x > 0 per row (the item
   slots a FRIR_KIND_TRAIN job needs); frir_simulate_train renders the full
   variant of every job's rows (channel c = row c of `train`, stride ld) from
   those samples through the same sort / tail / render kernels as
   frir_simulate.  A train with negative samples is rendered as sign +1 minus
   sign -1. */
int frir_train_nonzeros(const double* train, int64_t ld, int32_t rows, int32_t length, int32_t sign,
                        int32_t* counts, void* stream);
int frir_simulate_train(const frir_plan* plan, const frir_batch* batch, void* workspace, size_t workspace_bytes,
                        const double* train, int64_t ld, int32_t sign, float* out_full, int32_t* direct_scratch,
                        void* stream);

const char* frir_last_error(void);
int32_t frir_abi_version(void);
/* Debug builds (-DFRIR_DEBUG): source line of the first failed in-kernel
   bounds check since load, 0 if none (always 0 in release builds). */
int32_t frir_debug_status(void);
/* sizeof of frir_job (0), frir_batch (1), frir_plan_desc (2): lets bindings
   verify their struct mirrors. */
int64_t frir_struct_size(int32_t which);

#ifdef __cplusplus
}
#endif
#endif /* FRIR_H_ */
