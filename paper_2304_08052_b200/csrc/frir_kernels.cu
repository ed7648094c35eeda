// sm_100a kernels of the FRAM-RIR hot path.
//
//   K1 geom_kernel    per (job, 4 images): Philox draws (or oracle draws) ->
//                     FP64 image position, r^g, then per mic the exact integer
//                     delay q, FP32 gain and output-rate start/phase items
//                                                             core.py:131-251
//   K2 sort_kernel    per channel: early flags, stable two-pass counting sort
//                     of the items by 32-sample output window core.py:254-265
//   K2b tail_kernel   per channel: the exact corrections of the reference's
//                     truncation of the mid-rate signal    resample.py:107-113
//   K3 render_kernel  persistent warps, one channel at a time: gather the
//                     composite decimation/low-pass tables into 32-sample
//                     windows (FP32), FP64 output-rate LP scan, exact tail
//                     correction, coalesced full (+ early) stores; for
//                     batches of >= 1,024 channels the early variant is a
//                     second pass over the early buckets only (K3e)
//                                                             resample.py:81-136
// No atomics touch sample values, so outputs are bit-reproducible.
#include <cstdlib>

#include "frir_internal.h"
#include "frir_philox.cuh"

// Debug builds (-DFRIR_DEBUG, build.py --debug) trap on any out-of-range
// table/item/output index; compute-sanitizer is not available on the pool.
__device__ int g_frir_check_line = 0;  // first failed FRIR_CHECK (debug builds)
#ifdef FRIR_DEBUG
#define FRIR_CHECK(cond)                                 \
  do {                                                   \
    if (!(cond)) g_frir_check_line = __LINE__;           \
  } while (0)
#else
#define FRIR_CHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace frir {
namespace {

constexpr double kTwoPi = 6.283185307179586;       // 2.0 * np.pi
constexpr double kHalfPi = 1.5707963267948966;     // np.pi / 2.0
constexpr double kPi = 3.141592653589793;          // np.pi/2 - (-np.pi/2)

struct Workspace {
  int2* items;      // per channel, sorted by output window (K2 -> K3)
  int2* items_raw;  // per channel, image order (K1 -> K2)
  int* chan_q0;
  int* chan_rows;   // items per channel before the dropped-arrival bucket (K2 -> K2b, K3)
  int* chan_tail;   // first item of the HP-horizon suffix per channel (K2 -> K2b)
  int2* chan_erange; // items [x, y): the buckets that hold the channel's early items (K2 -> K3 early pass)
  float* chan_scale;
  double* corr;     // per channel [F, E][32]: tail corrections of outputs n_c + i (K2 -> K3)
  longlong2* chan_row;  // per channel {first item, rows} (K1 -> K2: the row's TMA load issues after one load)
  int* counter;
};

// Segments of long channels (see seg_count); null when the batch has none.
struct SegWs {
  int* seg;           // per channel [kSegInts]: segment windows / item ranges (K2 -> K3, K4)
  double* state;      // per channel [kMaxSeg][F0, F1, E0, E1]: zero-start end states (K3 -> K4)
  int* units;         // segments >= 1 of long channels as c * kMaxSeg + k (K2 -> K3 work queue)
  int* nextra;        // entries of units
};

// Long channels (more than kSegRows items) are rendered as up to kMaxSeg
// segments of whole tiles by different warps, each from a zero LP state; the
// seam kernel K4 adds the free response of the true start state afterwards
// (the LP recursion is linear).  The count depends only on the channel, so a
// channel renders the same bits in any batch.
constexpr int kSegRows = 16384, kMaxSeg = 16;
constexpr int kSegInts = 64;  // [0, S]: first window of each segment; 17 + k: item lo; 33 + k: item hi
__host__ __device__ inline int seg_count(int rows, int n2) {
  const int nwin = (n2 + kExt + kWin - 1) / kWin;
  int s = (rows + kSegRows - 1) / kSegRows;
  s = s < kMaxSeg ? s : kMaxSeg;
  const int by_len = nwin / 16 > 1 ? nwin / 16 : 1;  // at least 4 tiles per segment
  s = s < by_len ? s : by_len;
  return s > 1 ? s : 1;
}
inline int batch_seg_max(const frir_batch* b) {  // upper bound over the batch's channels
  return seg_count(b->max_rows, b->max_windows * kWin - kExt);
}


__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// The raw region holds K1's unsorted item list.
inline size_t raw_bytes(const frir_batch* b) { return align_up((size_t)b->total_items * 8); }

Workspace carve(void* base, const frir_batch* b) {
  char* p = (char*)base;
  Workspace w;
  w.items = (int2*)p; p += align_up((size_t)b->total_items * 8);
  w.items_raw = (int2*)p; p += raw_bytes(b);
  w.chan_q0 = (int*)p; p += align_up((size_t)b->total_channels * 4);
  w.chan_rows = (int*)p; p += align_up((size_t)b->total_channels * 4);
  w.chan_tail = (int*)p; p += align_up((size_t)b->total_channels * 4);
  w.chan_erange = (int2*)p; p += align_up((size_t)b->total_channels * 8);
  w.chan_scale = (float*)p; p += align_up((size_t)b->total_channels * 4);
  w.corr = (double*)p; p += align_up((size_t)b->total_channels * 64 * 8);
  w.chan_row = (longlong2*)p; p += align_up((size_t)b->total_channels * 16);
  w.counter = (int*)p;
  return w;
}

// The segment tables follow the base workspace (workspace_bytes).
SegWs carve_seg(void* base, const frir_batch* b) {
  SegWs g{nullptr, nullptr, nullptr, nullptr};
  if (batch_seg_max(b) <= 1) return g;
  char* p = (char*)base + align_up((size_t)b->total_items * 8) + raw_bytes(b) +
            4 * align_up((size_t)b->total_channels * 4) + align_up((size_t)b->total_channels * 8) +
            align_up((size_t)b->total_channels * 64 * 8) + align_up((size_t)b->total_channels * 16) + 256;
  g.seg = (int*)p; p += align_up((size_t)b->total_channels * kSegInts * 4);
  g.state = (double*)p; p += align_up((size_t)b->total_channels * kMaxSeg * 4 * 8);
  g.units = (int*)p; p += align_up((size_t)b->total_channels * kMaxSeg * 4);
  g.nextra = (int*)p;
  return g;
}

// ---------------------------------------------------------------- K1 geometry + delays
// numpy operation order is kept with explicit _rn intrinsics (no FMA
// contraction): positions/distances feed the exact integer delays.
__device__ __forceinline__ void image_position(const frir_job& J, double dist, double az,
                                               double el, double* x, double* y, double* z) {
  // params.py:138-146 sph_to_cart; params.py:149-159 center + offset
  double ce, se, ca, sa;  // sincos == (sin, cos) bit for bit (tools/checks/sincos_identity.cu)
  sincos(el, &se, &ce);
  sincos(az, &sa, &ca);
  double dce = __dmul_rn(dist, ce);
  *x = __dadd_rn(J.center[0], __dmul_rn(dce, ca));
  *y = __dadd_rn(J.center[1], __dmul_rn(dce, sa));
  *z = __dadd_rn(J.center[2], __dmul_rn(dist, se));
}

// Words o .. o + 3 of the 8-word concatenation a|b (o in [0, 4)), with static
// register indices only (a runtime-indexed array would live in local memory).
__device__ __forceinline__ u64x4 words4(const u64x4& a, const u64x4& b, int o) {
  u64x4 r;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t c0 = a.v[k];
    const uint64_t c1 = k + 1 < 4 ? a.v[(k + 1) & 3] : b.v[(k + 1) & 3];
    const uint64_t c2 = k + 2 < 4 ? a.v[(k + 2) & 3] : b.v[(k + 2) & 3];
    const uint64_t c3 = k + 3 < 4 ? a.v[(k + 3) & 3] : b.v[(k + 3) & 3];
    r.v[k] = o == 0 ? c0 : (o == 1 ? c1 : (o == 2 ? c2 : c3));
  }
  return r;
}

struct GeomArgs {
  const frir_job* jobs;
  const double* mics;
  const double* draw_dist;
  const double* draw_az;
  const double* draw_el;
  const double* draw_refl;
  Workspace ws;
  int32_t* direct_index;
  int r_h, t0;
  unsigned rh_magic;  // ceil(2^32 / r_h): exact floor division for n < 2^32 / r_h
  double rate;        // r_h * fs
};

// Integer high-rate delay of core.py:242-243, q = min(ceil((D / c0) * rate), L - 1),
// with D = sqrt(dx^2 + dy^2 + dz^2) summed x, y, z (params.py:170-171).  The
// product D * (rate / c0) is within 3 ulp of the reference's (D / c0) * rate, so
// unless it lies within 1e-14 (relative) of an integer the ceiling is the
// same; the exact division runs only in that (practically never) case.
__device__ __forceinline__ int delay_of(double px, double py, double pz, const double* mic,
                                        double c0, double rate, double rate_c0, int L, double* D) {
  const double dx = __dsub_rn(px, mic[0]), dy = __dsub_rn(py, mic[1]), dz = __dsub_rn(pz, mic[2]);
  const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  *D = d;
  double x = __dmul_rn(d, rate_c0);
  double k = ceil(x);
  const double eps = 1e-14 * x;
  if (k - x < eps || x - (k - 1.0) < eps) k = ceil(__dmul_rn(__ddiv_rn(d, c0), rate));
  return k >= (double)(L - 1) ? L - 1 : (int)k;
}

// 1/sqrt(x) for normal x > 0: the hardware approximation (relative error
// <= 2^-20) refined by one Newton step (<= 1.4e-12).
__device__ __forceinline__ double rsqrt_nr1(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double r = fma(-(x * y), y, 1.0);  // 1 - x y^2
  return fma(0.5 * y, r, y);
}

// Item of the (image, mic) pair: biased output-rate start s' + 64 (20 bits) and
// the phase phi (10 bits) of the composite tables, gain in the second word.
__device__ __forceinline__ int2 make_item(int q, float a, int r_h, int t0, unsigned magic) {
  // s = ceil((q + t0) / r_h); n = q + t0 + 64 r_h >= 0 (q >= 0, -t0 < 64 r_h)
  const unsigned n = (unsigned)(q + t0 + 64 * r_h + r_h - 1);
  const int s = (int)__umulhi(n, magic) - 64;
  const unsigned spb = (unsigned)(s + kExt + kSpBias);
  const unsigned phi = (unsigned)(r_h * s - q - t0);
  return make_int2((int)(spb | (phi << 20)), __float_as_int(a));
}

// Per-image part of K1 for images 4g + 1 .. 4g + 4 of job J: absolute image
// positions (FP64, numpy's operation order) and the FP32 gains r^g.  Shared by
// geom_kernel and image_kernel.
// The sampled ImageSet fields of the 4 images (core.py:43-62), for image_set_kernel.
struct ImageDraws {
  double dist[4], az[4], el[4], ratio[4], refl[4];
};

__device__ __forceinline__ void image_group(const GeomArgs& A, const frir_job& J, int g, double (&px)[4],
                                            double (&py)[4], double (&pz)[4], float (&lg)[4],
                                            ImageDraws* draws = nullptr) {
  const int I = J.n_images;
  const int ism = J.kind == FRIR_KIND_ISM;
  const double c_max = __dmul_rn(J.c0, J.t60);
  double th[4], ph[4], dist[4], refl[4];
  if (ism && J.lattice > 0) {
    // enumerate_images (ism.py:80-104) on the device: image row i is lattice
    // point i - 1 of the (2K+1)^3 grid in meshgrid 'ij' order, skipping the
    // origin (the source, row 0); per axis m L + s (m even) or m L + (L - s)
    const int K = J.lattice - 1, n = 2 * K + 1, origin = (K * n + K) * n + K;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = min(4 * g + k + 1, I);
      const int li = (i - 1) < origin ? i - 1 : i;
      const int m3[3] = {li / (n * n) - K, (li / n) % n - K, li % n - K};
      double p3[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double L = J.room[a], s = J.center[a], mL = __dmul_rn((double)m3[a], L);
        p3[a] = (m3[a] & 1) ? __dadd_rn(mL, __dsub_rn(L, s)) : __dadd_rn(mL, s);
      }
      dist[k] = p3[0]; th[k] = p3[1]; ph[k] = p3[2];
      refl[k] = (double)(abs(m3[0]) + abs(m3[1]) + abs(m3[2]));
    }
  } else if (A.draw_dist != nullptr) {  // oracle mode: the reference's own ImageSet rows
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int i = 4 * g + k + 1;
      size_t o = (size_t)J.img_off + (i <= I ? i : 0);
      dist[k] = A.draw_dist[o]; th[k] = A.draw_az[o]; ph[k] = A.draw_el[o]; refl[k] = A.draw_refl[o];
    }
  } else {
    // stage-0 stream: theta words [0, I), phi words [I, 2I), u words [2I, 3I);
    // stage-1 stream: perturbation words [0, I).  One Philox block serves 4 images.
    const uint64_t w0 = 4ull * g;
    u64x4 bt = philox4x64_10((uint64_t)g + 1, 0, 0, 0, J.key[0], J.key[1]);
    uint64_t wp = (uint64_t)I + w0, wu = 2ull * I + w0;
    u64x4 bp0 = philox4x64_10(wp / 4 + 1, 0, 0, 0, J.key[0], J.key[1]);
    u64x4 bp1 = bp0;
    if (wp & 3) bp1 = philox4x64_10(wp / 4 + 2, 0, 0, 0, J.key[0], J.key[1]);
    u64x4 bu0 = philox4x64_10(wu / 4 + 1, 0, 0, 0, J.key[0], J.key[1]);
    u64x4 bu1 = bu0;
    if (wu & 3) bu1 = philox4x64_10(wu / 4 + 2, 0, 0, 0, J.key[0], J.key[1]);
    u64x4 bq = philox4x64_10((uint64_t)g + 1, 0, 0, 0, J.key[2], J.key[3]);
    const double alpha = J.alpha, beta = J.beta;
    const double kres = __ddiv_rn(alpha, __dsub_rn(beta, alpha));
    const double mr1 = __dsub_rn(__ddiv_rn(c_max, J.d0), 1.0);
    const double rrm1 = __dsub_rn(J.rr_max, 1.0);
    const double prange = __dsub_rn(J.perturb_hi, J.perturb_lo);
    const u64x4 bp = words4(bp0, bp1, (int)(wp & 3)), bu = words4(bu0, bu1, (int)(wu & 3));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t wpk = bp.v[k], wuk = bu.v[k];
      th[k] = __dmul_rn(kTwoPi, u64_to_unit(bt.v[k]));                // uniform(0, 2pi), core.py:154
      ph[k] = __dadd_rn(-kHalfPi, __dmul_rn(kPi, u64_to_unit(wpk)));  // uniform(-pi/2, pi/2), :155
      // core.py:94-100 quadratic_ratio_sample
      double u = u64_to_unit(wuk);
      double drh = cbrt(__dadd_rn(J.alpha3, __dmul_rn(__dsub_rn(1.0, u), J.b3a3)));
      // core.py:103-110 rescale_distance_ratio, max_ratio = c_max / d0
      double dr = __dadd_rn(1.0, __dmul_rn(__dmul_rn(kres, __dsub_rn(__ddiv_rn(drh, alpha), 1.0)), mr1));
      double dd = __dmul_rn(J.d0, dr);
      // core.py:215-220 reflection counts (stage-1 stream)
      double pr = __dadd_rn(J.perturb_lo, __dmul_rn(prange, u64_to_unit(bq.v[k])));
      double qq = __ddiv_rn(dd, c_max);
      // dr**tau in FP64 (core.py:219): two correctly rounded square roots for
      // the default tau = 0.25 (<= 1 ulp from numpy's pow), pow otherwise
      const double drt = J.tau == 0.25 ? __dsqrt_rn(__dsqrt_rn(dr)) : pow(dr, J.tau);
      double gg = __dadd_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(qq, qq), rrm1)), __dmul_rn(pr, drt));
      gg = fmin(fmax(gg, 1.0), J.rr_max);
      dist[k] = dd;
      refl[k] = gg;
      if (draws) draws->ratio[k] = dr;
    }
  }
  if (draws) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      draws->dist[k] = dist[k]; draws->az[k] = th[k]; draws->el[k] = ph[k]; draws->refl[k] = refl[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (J.kind == FRIR_KIND_ISM) {  // lattice images arrive as absolute positions
      px[k] = dist[k]; py[k] = th[k]; pz[k] = ph[k];
    } else {
      image_position(J, dist[k], th[k], ph[k], &px[k], &py[k], &pz[k]);
    }
    // core.py:246 r ** g; the gain is an FP32 quantity (exp2 of an FP64 exponent)
    const double x = refl[k] * J.log2r, xi = floor(x);
    lg[k] = ldexpf(exp2f((float)(x - xi)), (int)xi);
  }
}

#ifndef FRIR_GEOM_MINB
#define FRIR_GEOM_MINB 6  // 85 registers: fewer spills in the FP64 + Philox code than at 8 (measured)
#endif
// geom_kernel's per-warp transpose rows: 36 entries of 8 bytes keep both the
// row writes and the column reads free of bank conflicts
constexpr int kTrStride = 36;
// Buckets of a channel's items (32-sample output windows, biased) and the
// extra bucket after them that holds ISM arrivals past the train end
// (ism.py:131-133 drops them): the sort puts them last and K2b / K3 stop
// before them.
__host__ __device__ inline int legit_buckets(int n2) { return ((n2 + kExt + kSpBias) >> 5) + 2; }
__device__ __forceinline__ int2 dropped_item(int n2) { return make_int2(legit_buckets(n2) << 5, 0); }

__global__ void __launch_bounds__(128, FRIR_GEOM_MINB) geom_kernel(GeomArgs A) {
  const int j = blockIdx.x;
  const frir_job& J = A.jobs[j];
  const int I = J.n_images, rows = I + 1, M = J.n_mics;
  const int g = blockIdx.y * blockDim.x + threadIdx.x;  // group of 4 images
  const int ngroups = (I + 3) / 4;
  const double* mics = A.mics + 3 * (size_t)J.mic_off;
  const double rate_c0 = __ddiv_rn(A.rate, J.c0);
  int2* items = A.ws.items_raw + J.item_off;
  const int ism = J.kind == FRIR_KIND_ISM;  // 1: arrivals past L - 1 are dropped, not clamped
  if (g == 0) {  // row 0: direct path (core.py:169, params.py:156-159), r**0 = 1
    double x, y, z;
    image_position(J, J.d0, J.az, J.el, &x, &y, &z);
    for (int m = 0; m < M; ++m) {
      double D;
      int q = delay_of(x, y, z, mics + 3 * m, J.c0, A.rate, rate_c0, J.L + ism, &D);
      // ISM drops arrivals past the train end (ism.py:131-133): they go to the
      // dropped-arrival bucket; the direct index still clamps (:134-136)
      const bool drop = q > J.L - 1;
      q = min(q, J.L - 1);
      items[(size_t)m * rows] = drop ? dropped_item(J.n2) : make_item(q, (float)__drcp_rn(D), A.r_h, A.t0, A.rh_magic);
      A.ws.chan_q0[J.chan_off + m] = q;
      A.ws.chan_row[J.chan_off + m] = make_longlong2((long long)J.item_off + (long long)m * rows, rows);
      A.ws.chan_scale[J.chan_off + m] = J.normalize ? (float)D : 1.0f;  // direct path -> 1/(1 m)
      // resample.py:115-119: clip(round(q0 / r_h), 0, n2 - 1), half-even
      int di = (int)rint(__ddiv_rn((double)q, (double)A.r_h));
      A.direct_index[J.chan_off + m] = di < 0 ? 0 : (di > J.n2 - 1 ? J.n2 - 1 : di);
    }
  }
  // Lanes own 4 consecutive rows; per mic the warp's 128 items go through a
  // padded shared-memory transpose so each store writes 32 consecutive rows
  // (coalesced 256-byte stores instead of 8-byte writes at a 32-byte stride).
  const int lane = threadIdx.x & 31;
  const bool live = g < ngroups;
  if (!__any_sync(0xffffffffu, live)) return;
  __shared__ int2 s_tr[128 / 32][4 * kTrStride];
  int2* tr = s_tr[threadIdx.x >> 5];
  double px[4], py[4], pz[4];
  float lg[4];
  if (live) {
    image_group(A, J, g, px, py, pz, lg);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) { px[k] = py[k] = pz[k] = 1.0; lg[k] = 0.f; }
  }
  const int nk = live ? min(4, I - 4 * g) : 0;
  const int wrow = 4 * (g - lane) + 1;  // first row of the warp
  // per-job constants in registers: the item stores may alias the job table
  // for the compiler, which would reload these fields for every item
  const int q_hi = J.L + ism - 1;  // last representable arrival (ISM: one past the train = dropped)
  const int q_keep = J.L - 1;      // arrivals after this are dropped (ISM only)
  const int2 drop = dropped_item(J.n2);
  const double c0 = J.c0;
  const double half_band = 0.5 - 2e-12 * (double)(J.L + ism);
  for (int m = 0; m < M; ++m) {
    int2* out = items + (size_t)m * rows + wrow;
    const double mx = __ldg(mics + 3 * m), my = __ldg(mics + 3 * m + 1), mz = __ldg(mics + 3 * m + 2);
    // Hot-loop form of delay_of for the image rows: the distance comes from
    // the FP64 reciprocal square root with ONE Newton step (D = d2 * rsqrt(d2);
    // relative error <= 1.4e-12: 1.5 e0^2 for the hardware approximation's
    // e0 <= 2^-20, measured by tools/checks/rsqrt_err.cu) instead of the
    // correctly rounded sqrt, so x = D * rate / c0 lies within ~1.5e-12 x of
    // the reference's value; outside a 2e-12 L guard band around the integers
    // the ceiling is identical (x >= L clamps to L - 1 either way), and 1/D (the
    // gain's denominator) comes for free.  Branch-free for all 4 rows (rows
    // past I are computed on valid data and never stored); the exact reference
    // arithmetic (sqrt_rn, div_rn) runs only for rows in the band (~1e-6 of
    // them; warp-uniform test).
    double d2[4], kc[4];
    float inv_d[4];
    unsigned gm = 0;  // rows in the guard band
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double dx = __dsub_rn(px[k], mx), dy = __dsub_rn(py[k], my), dz = __dsub_rn(pz[k], mz);
      d2[k] = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      const double y = rsqrt_nr1(d2[k]);  // no branches
      inv_d[k] = (float)y;
      const double x = __dmul_rn(__dmul_rn(d2[k], y), rate_c0);
      kc[k] = ceil(x);
      if (k < nk && fabs(__dsub_rn(kc[k], x) - 0.5) > half_band) gm |= 1u << k;  // |frac - 1/2| > 1/2 - band
    }
    if (__any_sync(0xffffffffu, gm != 0u)) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((gm >> k) & 1u) kc[k] = ceil(__dmul_rn(__ddiv_rn(__dsqrt_rn(d2[k]), c0), A.rate));
    }
    int2 it[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = min(__double2int_rz(kc[k]), q_hi);  // (kc >= 0; the conversion saturates)
      FRIR_CHECK(k >= nk || (q >= 0 && q < J.L + ism && 4 * g + 1 + k < rows));
      it[k] = q > q_keep ? drop  // ISM only: dropped arrival
                         : make_item(q, lg[k] * inv_d[k], A.r_h, A.t0, A.rh_magic);  // r^g / D
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) tr[k * kTrStride + lane] = it[k];  // item 4 lane + k
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // rows 32 kk + lane of the warp
      const int row = 32 * kk + lane;
      if (wrow + row <= I) out[row] = tr[(lane & 3) * kTrStride + 8 * kk + (lane >> 2)];
    }
  }
}

// ---------------------------------------------------------------- K2 bucket sort
// Stable counting sort of one channel's items by 32-sample output window, in
// place.  Early flags (core.py:259-264) are set here from the channel's q0.
// Per-warp 16-bit histograms make the placement stable (row order within a
// bucket) without atomics deciding the order, so outputs are bit-reproducible.
struct Cplx {
  double re, im;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) {  // (this file builds with -fmad=false: fused explicitly)
  return {fma(a.re, b.re, -(a.im * b.im)), fma(a.re, b.im, a.im * b.re)};
}

// First output whose value needs the truncation correction (outputs whose
// stage-2 window reaches past the stage-1 length n1, resample.py:107-113).
__host__ __device__ inline int first_corrected(const frir_plan_desc& d, int n1) {
  return n1 - d.half2 > 0 ? (n1 - d.half2 + d.r_l - 1) / d.r_l : 0;
}

// Lanes of the warp holding the same key b (b < 2^kbits; distinct keys for
// idle lanes): one ballot per key bit (MATCH.ANY measured slower on B200).
__device__ __forceinline__ unsigned peers_of(int b, int kbits) {
  unsigned peers = 0xffffffffu;
  for (int k = 0; k < kbits; ++k) {
    const bool bit = (b >> k) & 1;
    const unsigned ones = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? ones : ~ones;
  }
  return peers;
}

struct SortArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  Workspace ws;
  SegWs sw;
  DevPlan plan;
  int r_h, t0;
  int atom_ranks;  // 1: ranks from shared-memory atomics (see sort_kernel pass 2)
  int stage_off;   // > 0: byte offset of a max_rows-item shared-memory buffer the
                   // scatter writes first (then copied out coalesced); 0: scatter to HBM
};


// Two passes over the channel's raw items (K1's output, read twice; the second
// read hits L2): per-warp 16-bit bucket histograms over contiguous row chunks,
// one exclusive scan in (bucket, warp) order, then a stable scatter into the
// sorted buffer.  Only the counters live in smem, so long channels keep the
// SM occupied.
// Counter type CT: 16-bit (packed pairs) while rows <= 65535, else 32-bit.
// One-shot TMA bulk copy global -> shared completing on an mbarrier (sm_90+
// PTX; the row is staged without passing through registers).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

// Counter of (bucket b, warp w): the lanes of one warp instruction hit
// different buckets of the same warp, so consecutive buckets of a warp sit in
// consecutive 32-bit words (distinct banks); the two 16-bit halves of a word
// belong to warps 2k and 2k + 1, never to lanes of one instruction.
template <typename CT>
__device__ __forceinline__ int cnt_idx(int b, int w, int nbk) {
  if constexpr (sizeof(CT) == 2)
    return (((w >> 1) * nbk + b) << 1) | (w & 1);
  else
    return w * nbk + b;
}

template <typename CT>
__device__ __forceinline__ void count_add(CT* cnt, int idx) {
  if constexpr (sizeof(CT) == 2)
    atomicAdd(reinterpret_cast<unsigned*>(cnt) + (idx >> 1), 1u << (16 * (idx & 1)));
  else
    atomicAdd(reinterpret_cast<unsigned*>(cnt) + idx, 1u);
}

// K > 0 (rows <= NW * 32 * K, atomic ranks, no segment tables): the channel's
// raw row is read ONCE, by a TMA bulk copy into the shared-memory buffer at
// stage_off; both passes read it there (pass 2 takes each thread's K items
// into registers first), the scatter rewrites the buffer in sorted order and
// the sorted row leaves in coalesced stores.
template <typename CT, int NW, bool SEG, int K = 0>  // NW warps per channel (more for long rows); SEG: segment tables
__global__ void __launch_bounds__(NW * 32, (K > 0 ? 1024 : 2048) / (NW * 32)) sort_kernel(SortArgs A) {
  constexpr int kSortWarps = NW, kSortThreads = NW * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_wsum[kSortWarps];
  const int c = blockIdx.x;
  __shared__ __align__(8) unsigned long long s_bar;
  if constexpr (K > 0) {
    // K > 0: the raw row lands in the staging buffer by one TMA bulk copy of
    // its 16-byte-aligned cover (lead = 0 or 1 item before the row; the cover
    // ends at most 8 bytes past it, inside the 256-byte-aligned workspace),
    // issued from K1's per-channel row descriptor before the job is read
    if (threadIdx.x == 0) {
      const longlong2 cr = A.ws.chan_row[c];
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.ws.items_raw + cr.x);
      const uintptr_t g0 = a0 & ~(uintptr_t)15, g1 = (a0 + 8 * (uintptr_t)cr.y + 15) & ~(uintptr_t)15;
      const unsigned bar = smem_u32(&s_bar);
      mbar_init_expect(bar, (unsigned)(g1 - g0));
      bulk_g2s(smem_u32(smem + A.stage_off), reinterpret_cast<const void*>(g0), (unsigned)(g1 - g0), bar);
    }
  }
  const int j = A.chan_job[c];
  const frir_job& J = A.jobs[j];
  const int m = c - J.chan_off;
  const int rows = J.n_images + 1;
  const int nbk = legit_buckets(J.n2) + 1;  // buckets 0 .. nbk-1, the last one for dropped arrivals
  const size_t base = J.item_off + (size_t)m * rows;
  const int2* src = A.ws.items_raw + base;
  int2* dst = A.ws.items + base;
  CT* s_cnt = reinterpret_cast<CT*>(smem);  // (bucket, warp) counters at cnt_idx<CT>
  int2* s_sorted = A.stage_off ? reinterpret_cast<int2*>(smem + A.stage_off) : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = nbk * kSortWarps;
  const int nwords = (int)((n * sizeof(CT) + 3) / 4);
  // pass 1: per-warp histograms over a contiguous row chunk per warp (K > 0:
  // whole 32-row groups per warp, the row held in registers)
  const int chunk = K > 0 ? (rows + kSortThreads - 1) / kSortThreads * 32 : (rows + kSortWarps - 1) / kSortWarps;
  const int r_lo = warp * chunk, r_hi = min(rows, r_lo + chunk);
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
  const int lead = (int)((sa >> 3) & 1);
  const int2* s_raw = K > 0 ? s_sorted + lead : nullptr;
  for (int i = tid; i < nwords; i += kSortThreads) reinterpret_cast<unsigned*>(s_cnt)[i] = 0u;
  // Buckets whose starts the later kernels need, found by thread 0 while the
  // row loads (the scan writes the starts): K2b's HP-horizon suffix begins at
  // the first bucket whose items can feed the state at n1 (k_hi >= n1 -
  // horizon; bucket b bounds q by qmax(b)); the render's early pass reads the
  // buckets of the early items (q in [q0 - e_lo, q0 + e_hi], core.py:257-264).
  __shared__ int s_mark[3];  // [suffix start, first early bucket, one past the last] (<= nbk - 1)
  if (tid == 0) {
    const frir_plan_desc& d = A.plan.d;
    const long long kthr = (long long)J.n1 - d.horizon;
    int lo = 0, hi = nbk - 1;  // smallest b not below the horizon (nbk - 1: none)
    while (kthr > 0 && lo < hi) {
      const int mid = (lo + hi) >> 1;
      const long long qmax = (long long)d.r_h * ((mid << 5) + 31 - kSpBias - kExt) - d.t0;
      if ((long long)d.up * qmax + d.half1 < kthr * d.down) lo = mid + 1; else hi = mid;
    }
    auto bucket_of = [&](int q) {  // as make_item computes it
      const int sq = (q + d.t0 + 64 * d.r_h + d.r_h - 1) / d.r_h - 64;  // ceil((q + t0) / r_h), q >= 0
      return (sq + kExt + kSpBias) >> 5;
    };
    const int q0 = A.ws.chan_q0[c];
    s_mark[0] = lo;
    s_mark[1] = min(bucket_of(max(q0 - J.e_lo, 0)), nbk - 1);
    s_mark[2] = min(bucket_of(min(q0 + J.e_hi, J.L - 1)) + 1, nbk - 1);
  }
  __syncthreads();
  if constexpr (K > 0) {
    mbar_wait(smem_u32(&s_bar), 0);
    for (int r = r_lo + lane; r < r_hi; r += 32)
      count_add(s_cnt, cnt_idx<CT>((s_raw[r].x & 0xFFFFF) >> 5, warp, nbk));
  } else {
#pragma unroll 4
    for (int r = r_lo + lane; r < r_hi; r += 32) {
      const int b = (__ldg(&src[r].x) & 0xFFFFF) >> 5;
      count_add(s_cnt, cnt_idx<CT>(b, warp, nbk));
    }
  }
  __syncthreads();
  // exclusive scan over (bucket, warp) in bucket-major order: thread t takes
  // buckets t, t + T, ..., sums its bucket's NW counters in registers, the
  // bucket totals are scanned across the CTA (shuffles, one smem round), and
  // the NW positions are written back (one word per warp pair)
  unsigned* s_w = reinterpret_cast<unsigned*>(s_cnt);
  int carry = 0;
  for (int b0 = 0; b0 < nbk; b0 += kSortThreads) {
    const int b = b0 + tid;
    constexpr int kWords = sizeof(CT) == 2 ? NW / 2 : NW;  // counter words of one bucket
    int tot = 0;
    if (b < nbk) {
#pragma unroll
      for (int k = 0; k < kWords; ++k) {
        const unsigned wv = s_w[k * nbk + b];
        tot += sizeof(CT) == 2 ? (int)((wv & 0xFFFFu) + (wv >> 16)) : (int)wv;
      }
    }
    int inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    const int ws = lane < kSortWarps ? s_wsum[lane] : 0;  // warp totals scanned by lanes
    int wi = ws;
#pragma unroll
    for (int o = 1; o < kSortWarps; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    int run = carry + inc - tot + __shfl_sync(0xffffffffu, wi - ws, warp);
    if (b == s_mark[0]) A.ws.chan_tail[c] = run;  // (bucket b starts at item `run`)
    if (b == s_mark[1]) A.ws.chan_erange[c].x = run;
    if (b == s_mark[2]) A.ws.chan_erange[c].y = run;
    const int all = __shfl_sync(0xffffffffu, wi, kSortWarps - 1);
    if (b < nbk) {
#pragma unroll
      for (int k = 0; k < kWords; ++k) {  // (the words are read again: fewer live registers)
        const unsigned wv = s_w[k * nbk + b];
        if constexpr (sizeof(CT) == 2) {
          const unsigned lo16 = wv & 0xFFFFu;
          s_w[k * nbk + b] = (unsigned)run | ((unsigned)(run + lo16) << 16);
          run += (int)(lo16 + (wv >> 16));
        } else {
          s_w[k * nbk + b] = (unsigned)run;
          run += (int)wv;
        }
      }
    }
    carry += all;
    __syncthreads();
  }
  const int nvalid = (int)s_cnt[cnt_idx<CT>(nbk - 1, 0, nbk)];  // items before the dropped-arrival bucket
  if (tid == 0) A.ws.chan_rows[c] = nvalid;
  const int S = SEG ? seg_count(nvalid, J.n2) : 1;
  if (SEG && tid == 0) A.sw.seg[(size_t)c * kSegInts + 63] = S;  // read by K3 / K4
  if (S > 1) {
    // segment boundaries of a long channel: whole tiles, about rows / S items
    // each, every segment at least one tile.  s_cnt at (b, 0) is now the number
    // of items in buckets < b.  Bucket b feeds windows b - 2 .. b - 2 + tbk
    // (tbk = 32-tap table blocks), so segment k renders windows [W_k, W_k+1)
    // from the items of buckets [W_k + 2 - tbk, W_k+1 + 1].
    if (tid == 0) {
      const int nwin = (J.n2 + kExt + kWin - 1) / kWin;
      const int top = (nwin / kTileWin) * kTileWin;  // last segment start <= top - kTileWin
      const int tbk = (A.plan.d.sup + 31) / 32;
      auto start = [&](int b) { return (int)s_cnt[cnt_idx<CT>(b, 0, nbk)]; };
      int* seg = A.sw.seg + (size_t)c * kSegInts;
      int wprev = 0;
      seg[0] = 0;
      for (int k = 1; k < S; ++k) {
        const long long t = (long long)k * nvalid / S;
        int lo = 0, hi = nbk - 1;  // smallest b with start(b) >= t
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (start(mid) >= t) hi = mid; else lo = mid + 1;
        }
        int wk = ((lo > 1 ? lo - 1 : 0) / kTileWin) * kTileWin;
        wk = max(wk, wprev + kTileWin);
        wk = min(wk, top - kTileWin * (S - k));
        seg[k] = wk;
        seg[17 + k] = start(wk + 2 - tbk);
        seg[33 + k - 1] = start(wk + 2);
        wprev = wk;
      }
      seg[S] = nwin;
      seg[17] = 0;
      seg[33 + S - 1] = nvalid;
      const int at = atomicAdd(A.sw.nextra, S - 1);  // queue order only: outputs do not depend on it
      for (int k = 1; k < S; ++k) A.sw.units[at + k - 1] = c * kMaxSeg + k;
    }
    __syncthreads();  // the scatter below advances s_cnt
  }
  // pass 2: stable scatter, warp w walks its chunk in row order; early flags
  // (core.py:259-264) from the channel's direct arrival q0
  const int q0 = A.ws.chan_q0[c];
  if constexpr (K > 0) {
    int2 reg[K];  // the warp's rows leave the buffer before the scatter rewrites it
    // this warp's 32-row groups (warp-uniform: the loops below stop there)
    const int ngrp = __shfl_sync(0xffffffffu, r_hi > r_lo ? (r_hi - r_lo + 31) >> 5 : 0, 0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k >= ngrp) break;
      const int r = r_lo + 32 * k + lane;
      reg[k] = r < r_hi ? s_raw[r] : make_int2(0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k >= ngrp) break;
      if (r_lo + 32 * k + lane < r_hi) {
        int2 it = reg[k];
        const int sp = (it.x & 0xFFFFF) - kSpBias - kExt;
        const int phi = ((unsigned)it.x >> 20) & 0x3FF;
        const int rel = A.r_h * sp - A.t0 - phi - q0;  // q - q0
        if (rel >= -J.e_lo && rel <= J.e_hi) it.y ^= 0x80000000;  // early: negative gain
        const int idx = cnt_idx<CT>((it.x & 0xFFFFF) >> 5, warp, nbk);
        const unsigned sh = 16u * (idx & 1);
        const int pos = (int)((atomicAdd(reinterpret_cast<unsigned*>(s_cnt) + (idx >> 1), 1u << sh) >> sh) & 0xFFFFu);
        FRIR_CHECK(pos >= 0 && pos < rows);
        s_sorted[lead + pos] = it;  // the sorted row keeps dst's alignment mod 16
      }
    }
    // the sorted row leaves by one TMA bulk store of its 16-byte-aligned
    // interior (the async proxy reads smem written by st.shared: fence first);
    // the <= 1 item before and after it go by plain stores
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const int i0 = lead, n_int = (rows - i0) & ~1;  // dst + i0 is 16-byte aligned (same offset as src)
      if (lead) dst[0] = s_sorted[1];
      if (i0 + n_int < rows) dst[rows - 1] = s_sorted[lead + rows - 1];
      if (n_int > 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + i0),
                     "r"(smem_u32(s_sorted + lead + i0)), "r"((unsigned)n_int * 8u)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read before the CTA exits
      }
    }
    return;
  }
  int2 v = r_lo + lane < r_hi ? src[r_lo + lane] : make_int2(0, 0);
  if (A.atom_ranks) {
    // ranks from the shared-memory atomics: each item takes its bucket's
    // next slot (row order within a warp instruction follows the hardware's
    // lane-ascending service of conflicting atomics; tests compare this path
    // bit for bit with the ballot path below)
    for (int rb = r_lo; rb < r_hi; rb += 32) {
      const int r = rb + lane;
      const int2 cur = v;
      if (r + 32 < r_hi) v = src[r + 32];  // prefetch the next row group
      if (r < r_hi) {
        int2 it = cur;
        const int sp = (it.x & 0xFFFFF) - kSpBias - kExt;
        const int phi = ((unsigned)it.x >> 20) & 0x3FF;
        const int rel = A.r_h * sp - A.t0 - phi - q0;  // q - q0
        if (rel >= -J.e_lo && rel <= J.e_hi) it.y ^= 0x80000000;  // early: negative gain
        const int idx = cnt_idx<CT>((it.x & 0xFFFFF) >> 5, warp, nbk);
        int pos;
        if constexpr (sizeof(CT) == 2) {
          const unsigned sh = 16u * (idx & 1);
          pos = (int)((atomicAdd(reinterpret_cast<unsigned*>(s_cnt) + (idx >> 1), 1u << sh) >> sh) & 0xFFFFu);
        } else {
          pos = (int)atomicAdd(reinterpret_cast<unsigned*>(s_cnt) + idx, 1u);
        }
        FRIR_CHECK(pos >= 0 && pos < rows);
        if (s_sorted) s_sorted[pos] = it;
        else dst[pos] = it;
      }
    }
    if (s_sorted) {  // the sorted row leaves shared memory in coalesced stores
      __syncthreads();
      for (int i = tid; i < rows; i += kSortThreads) dst[i] = s_sorted[i];
    }
    return;
  }
  const int kbits = 32 - __clz(nbk + 31);  // bits of every key below nbk + 32
  for (int rb = r_lo; rb < r_hi; rb += 32) {
    const int r = rb + lane;
    const bool ok = r < r_hi;
    const int2 cur = v;
    if (r + 32 < r_hi) v = src[r + 32];  // prefetch the next row group
    int2 it = cur;
    const int sp = (it.x & 0xFFFFF) - kSpBias - kExt;
    const int phi = ((unsigned)it.x >> 20) & 0x3FF;
    const int rel = A.r_h * sp - A.t0 - phi - q0;  // q - q0
    if (rel >= -J.e_lo && rel <= J.e_hi) it.y ^= 0x80000000;  // early: negative gain
    const int b = ok ? (it.x & 0xFFFFF) >> 5 : nbk + lane;  // distinct for idle lanes
    const unsigned peers = peers_of(b, kbits);  // lanes with the same bucket
    const int rank = __popc(peers & ((1u << lane) - 1u));
    CT* slot = s_cnt + (ok ? cnt_idx<CT>(b, warp, nbk) : 0);
    const int pos = ok ? *slot + rank : 0;
    FRIR_CHECK(!ok || (pos >= 0 && pos < rows && b < nbk));
    __syncwarp();
    if (ok) {
      dst[pos] = it;
      if (rank == 0) *slot = (CT)(*slot + __popc(peers));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- K2b tail corrections
// The reference truncates the stage-1 output at its length n1 before the HP
// filter and stage 2 (resample.py:107-113); the render's untruncated chain
// differs from it only in outputs n >= n_c, by a correction that depends on
// the HP state at n1 (a modal sum over the items within the HP horizon, a
// suffix of the sorted row) and on the stage-1 taps the items put past n1.
// One warp per channel; the small power tables live in smem.  Every sum runs
// in a fixed order, so the corrections are bit-reproducible.  Segmented
// (long) channels are left to the SPLIT instance, where the CTA's warps take
// contiguous parts of the suffix and warp 0 adds their sums in warp order.
struct TailArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  Workspace ws;
  SegWs sw;
  DevPlan plan;
  int total_channels;
};

constexpr int kTailThreads = 128;
constexpr int kTailWarps = kTailThreads / 32;
#ifndef FRIR_TAIL_CHUNK
#define FRIR_TAIL_CHUNK 256
#endif
constexpr int kTailChunk = FRIR_TAIL_CHUNK;  // items per TMA chunk of the suffix (2 chunks in flight per warp)

template <bool SPLIT>
__global__ void __launch_bounds__(kTailThreads) tail_kernel(const __grid_constant__ TailArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& P = A.plan;
  const frir_plan_desc& d = P.d;
  const int nphi = d.horizon / 128 + 1;
  const int ltc = lt_cap(d);
  double2* s_plo = reinterpret_cast<double2*>(smem);  // p^i, i < 128
  double2* s_zph = s_plo + 128;                      // Z[rho], rho < down
  double2* s_phi = s_zph + d.down;                   // p^(128 j)
  double* s_xt = reinterpret_cast<double*>(s_phi + nphi);  // [warp][F, E][ltc], then the chunk buffers
  __shared__ __align__(8) unsigned long long s_bar[kTailWarps][2];
  if ((threadIdx.x & 31) < 2) mbar_init(smem_u32(&s_bar[threadIdx.x >> 5][threadIdx.x & 1]));
  for (int i = threadIdx.x; i < 128; i += blockDim.x) s_plo[i] = make_double2(P.ppow_lo[2 * i], P.ppow_lo[2 * i + 1]);
  for (int i = threadIdx.x; i < d.down; i += blockDim.x) s_zph[i] = make_double2(P.zphase[2 * i], P.zphase[2 * i + 1]);
  for (int i = threadIdx.x; i < nphi; i += blockDim.x) s_phi[i] = make_double2(P.ppow_hi[2 * i], P.ppow_hi[2 * i + 1]);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = SPLIT ? blockIdx.x : blockIdx.x * kTailWarps + warp;
  if (c >= A.total_channels) return;
  const bool long_chan = A.sw.seg != nullptr && A.sw.seg[(size_t)c * kSegInts + 63] > 1;
  if (long_chan != SPLIT) return;  // (CTA-uniform when SPLIT)
  const int j = A.chan_job[c];
  const frir_job& J = A.jobs[j];
  const int2* items = A.ws.items + A.ws.chan_row[c].x;  // (K1's row descriptor: no wait for the job)
  const int rows = A.ws.chan_rows[c];  // sorted items before the dropped-arrival bucket
  const int n1 = J.n1, n2 = J.n2;
  const int up = d.up, down = d.down, half1 = d.half1, r_h = d.r_h;
  const unsigned down_magic = (unsigned)((0x100000000ull + down - 1) / down);  // exact for e < 2^32 / down
  const int kthr = n1 - d.horizon;  // items with k_hi >= kthr feed the state
  double* xt_s = s_xt + 2 * ltc * warp;
  for (int i = lane; i < 2 * ltc; i += 32) xt_s[i] = 0.0;
  __syncwarp();

  int p_t = A.ws.chan_tail[c];  // HP-horizon suffix start (K2)
  int p_hi = rows;  // this warp's part of the suffix [p_t, p_hi)
  if (SPLIT) {
    const int chunk = ((rows - p_t + 32 * kTailWarps - 1) / (32 * kTailWarps)) * 32;
    p_t = min(rows, p_t + warp * chunk);
    p_hi = min(rows, p_t + chunk);
  }
  double4 z = make_double4(0.0, 0.0, 0.0, 0.0);  // this lane's partial modal sums (F, E)
  // One straddler (taps on both sides of n1) or head item at high-rate delay qs
  // with full / early amplitudes aF / aE, processed by the whole warp.
  auto straddle = [&](int qs, double aF, double aE) {
    const int khs = (int)__umulhi((unsigned)(up * qs + half1), down_magic);
    const int xs = up * qs - half1 + 1024 * down;  // >= 0 (half1 = 10 r_h <= 1024 down)
    const int klo = max(0, (int)__umulhi((unsigned)xs, down_magic) - 1024 + (xs % down != 0));
    const int kend = min(khs + 1, n1);
    for (int k = klo + lane; k < kend; k += 32) {  // taps 0 <= k < n1 feed the state
      const int mm = n1 - 1 - k;
      if (mm >= d.horizon) continue;
      FRIR_CHECK(down * k + half1 - up * qs >= 0 && down * k + half1 - up * qs < d.len1);
      const double h = P.h1up[down * k + half1 - up * qs];
      const double2 lo = s_plo[mm & 127], hi = s_phi[mm >> 7];
      const Cplx pm = cmul({hi.x, hi.y}, {lo.x, lo.y});
      const double cF = aF * h, cE = aE * h;
      z.x = fma(cF, pm.re, z.x);
      z.y = fma(cF, pm.im, z.y);
      z.z = fma(cE, pm.re, z.z);
      z.w = fma(cE, pm.im, z.w);
    }
    for (int l = lane; l < d.lt_max; l += 32) {  // taps k >= n1: input past the truncation point
      const int k = n1 + l;
      if (k <= khs) {
        const int idx = down * k + half1 - up * qs;
        if (idx >= 0 && idx < d.len1) {
          const double h = P.h1up[idx];
          xt_s[l] += aF * h;
          xt_s[ltc + l] += aE * h;
        }
      }
    }
  };
  // Arrivals clamped to the last train sample (core.py:242-243, q = L - 1) are
  // straddlers with identical taps: their amplitudes are summed (fixed order:
  // per batch a shuffle tree, batches in row order) and they are processed once.
  const int q_last = J.L - 1;
  double clampF = 0.0, clampE = 0.0;
  // The suffix streams through a per-warp double buffer in shared memory:
  // lane 0 issues TMA bulk copies of kTailChunk items (their 16-byte-aligned
  // cover) one chunk ahead, so the loads are in flight while the warp works
  // through the current chunk's batches.
  int2* stage = reinterpret_cast<int2*>(s_xt + 2 * ltc * kTailWarps) + warp * 2 * (kTailChunk + 2);
  const unsigned bar0 = smem_u32(&s_bar[warp][0]);
  const int nchunk = p_hi > p_t ? (p_hi - p_t + kTailChunk - 1) / kTailChunk : 0;
  auto issue = [&](int ci) {  // (lane 0)
    const int lo = p_t + ci * kTailChunk, hi = min(p_hi, lo + kTailChunk);
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(items + lo) & ~(uintptr_t)15;
    const uintptr_t g1 = (reinterpret_cast<uintptr_t>(items + hi) + 15) & ~(uintptr_t)15;
    const unsigned bar = bar0 + 8u * (ci & 1);
    mbar_arrive_expect(bar, (unsigned)(g1 - g0));
    bulk_g2s(smem_u32(stage + (ci & 1) * (kTailChunk + 2)), reinterpret_cast<const void*>(g0), (unsigned)(g1 - g0), bar);
  };
  if (lane == 0 && nchunk > 0) issue(0);
  for (int ci = 0; ci < nchunk; ++ci) {
    __syncwarp();  // every lane is done with chunk ci - 1 (its buffer is refilled next)
    if (lane == 0 && ci + 1 < nchunk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(ci + 1);
    }
    mbar_wait(bar0 + 8u * (ci & 1), (ci >> 1) & 1);
    const int c_lo = p_t + ci * kTailChunk, c_hi = min(p_hi, c_lo + kTailChunk);
    const int2* buf = stage + (ci & 1) * (kTailChunk + 2) + (int)((reinterpret_cast<uintptr_t>(items + c_lo) >> 3) & 1);
  for (int p = c_lo; p < c_hi; p += 32) {
    const int cnt = min(32, c_hi - p);
    const int2 it = lane < cnt ? buf[p - c_lo + lane] : make_int2(0xFFFFF, 0);
    {
    const int spb = it.x & 0xFFFFF;
    const int qm = r_h * (spb - kSpBias - kExt) - d.t0 - (((unsigned)it.x >> 20) & 0x3FF);
    const int e = up * qm + half1;  // >= 0
    const int khi = (int)__umulhi((unsigned)e, down_magic);
    const bool valid = lane < cnt && khi >= kthr;
    if (!__any_sync(0xffffffffu, valid)) continue;  // (next batch of the group)
    const float ae = __int_as_float(it.y);
    const bool early = ae < 0.f;
    const double a = fabs((double)ae);
    const bool head_item = e < 2 * half1;  // some stage-1 taps at k < 0
    if (valid && khi < n1 && !head_item) {
      const int rho = e - down * khi;
      const int mm = n1 - 1 - khi;
      FRIR_CHECK(mm >= 0 && (mm >> 7) < nphi && rho >= 0 && rho < down);
      const double2 lo = s_plo[mm & 127], hi = s_phi[mm >> 7], zr = s_zph[rho];
      const Cplx t = cmul(cmul({hi.x, hi.y}, {lo.x, lo.y}), {zr.x, zr.y});
      z.x = fma(a, t.re, z.x);
      z.y = fma(a, t.im, z.y);
      if (early) {
        z.z = fma(a, t.re, z.z);
        z.w = fma(a, t.im, z.w);
      }
    }
    const bool strad_lane = valid && (khi >= n1 || head_item);
    const bool clamped = strad_lane && qm == q_last && !head_item;
    if (__any_sync(0xffffffffu, clamped)) {
      double sF = clamped ? a : 0.0, sE = clamped && early ? a : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sF += __shfl_xor_sync(0xffffffffu, sF, o);
        sE += __shfl_xor_sync(0xffffffffu, sE, o);
      }
      clampF += sF;
      clampE += sE;
    }
    // other straddlers and head items: one at a time
    unsigned strad = __ballot_sync(0xffffffffu, strad_lane && !clamped);
    while (strad) {
      const int src = __ffs(strad) - 1;
      strad &= strad - 1;
      const int qs = __shfl_sync(0xffffffffu, qm, src);
      const float aes = __int_as_float(__shfl_sync(0xffffffffu, it.y, src));
      const double as = fabs((double)aes);
      straddle(qs, as, aes < 0.f ? as : 0.0);
    }
    }
  }
  }  // chunks
  if (clampF != 0.0 || clampE != 0.0) straddle(q_last, clampF, clampE);  // (warp-uniform)
  // boundary state s = 2 Re(v0 zeta) and the corrections of outputs n_c + lane
  Cplx zF = {z.x, z.y}, zE = {z.z, z.w};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zF.re += __shfl_xor_sync(0xffffffffu, zF.re, o);
    zF.im += __shfl_xor_sync(0xffffffffu, zF.im, o);
    zE.re += __shfl_xor_sync(0xffffffffu, zE.re, o);
    zE.im += __shfl_xor_sync(0xffffffffu, zE.im, o);
  }
  __syncwarp();
  if (SPLIT) {  // warp 0 adds the warps' sums and xt rows in warp order
    __shared__ double s_z[kTailWarps][4];
    if (lane == 0) {
      s_z[warp][0] = zF.re; s_z[warp][1] = zF.im; s_z[warp][2] = zE.re; s_z[warp][3] = zE.im;
    }
    __syncthreads();
    if (warp != 0) return;
    for (int w2 = 1; w2 < kTailWarps; ++w2) {
      zF.re += s_z[w2][0]; zF.im += s_z[w2][1]; zE.re += s_z[w2][2]; zE.im += s_z[w2][3];
      for (int i = lane; i < 2 * ltc; i += 32) xt_s[i] += s_xt[2 * ltc * w2 + i];
    }
    __syncwarp();
  }
  const Cplx v0a = {P.lp[2], P.lp[3]}, v0b = {P.lp[4], P.lp[5]};
  const Cplx ta = cmul(v0a, zF), tb = cmul(v0b, zF), ea = cmul(v0a, zE), eb = cmul(v0b, zE);
  const double s0 = 2.0 * ta.re, s1 = 2.0 * tb.re, se0 = 2.0 * ea.re, se1 = 2.0 * eb.re;
  double corrF = 0.0, corrE = 0.0;
  const int n = first_corrected(d, n1) + lane;
  const int ee = d.r_l * n + d.half2 - n1;
  if (n < n2 && ee >= 0 && ee < d.half2) {
    corrF = P.kappa[2 * ee] * s0 + P.kappa[2 * ee + 1] * s1;
    corrE = P.kappa[2 * ee] * se0 + P.kappa[2 * ee + 1] * se1;
    for (int l = 0; l < d.lt_max && l <= ee; ++l) {
      const double uu = P.u[ee - l];
      corrF += xt_s[l] * uu;
      corrE += xt_s[ltc + l] * uu;
    }
  }
  A.ws.corr[64 * (size_t)c + lane] = corrF;
  A.ws.corr[64 * (size_t)c + 32 + lane] = corrE;
}

static size_t tail_smem(const frir_plan_desc& d) {
  return (size_t)(128 + d.down + d.horizon / 128 + 1) * 16 + (size_t)kTailWarps * 2 * lt_cap(d) * 8 +
         (size_t)kTailWarps * 2 * (kTailChunk + 2) * 8;
}

// ---------------------------------------------------------------- K3 render
struct RenderArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  const int32_t* chan_order;
  int total_channels;
  Workspace ws;
  SegWs sw;
  DevPlan plan;
  float* out_full;
  float* out_early;
  int seg_max;  // upper bound of seg_count over the batch (work units = seg_max x channels)
};

__device__ __forceinline__ void sts_f32(unsigned addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
constexpr int kTileRow = kTile + 2 * kWin;  // tile buffer row: 2 scratch windows + the tile
constexpr int kRenderThreads = 256;  // 8 warps x 3 CTAs per SM
constexpr int kWarps = kRenderThreads / 32;
__device__ __forceinline__ int ceil_div_i(int a, int b) {  // b > 0, any sign of a
  return a >= 0 ? (a + b - 1) / b : -((-a) / b);
}


__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }

// One variant's LP recursion over a tile: lane L owns outputs [C L, C L + C)
// of the tile (C = kChunk).  W comes from the FP32 tile buffer; the chunk runs
// serially in FP64 from zero state, the tile's start state s enters as lane 0's
// carry (chunk 0 ends at M^C s + e0), chunks are combined with a Kogge-Stone
// scan of the affine maps s -> M^C s + e, and every output is corrected by the
// free response of its chunk's true start state.  The matrices are kernel
// parameters (constant-bank operands).  On return lp[] holds LP[C L + k] and
// (s0, s1) = (LP[last], LP[last - 1]) of the tile.
__device__ __forceinline__ void lp_scan_tile(const float* wbuf, const DevPlan& P, double c1,
                                             double c2, double& s0, double& s1, int lane,
                                             double (&lp)[kChunk]) {
  const float4* w4 = reinterpret_cast<const float4*>(wbuf + kChunk * lane);
  float wv[kChunk];
#pragma unroll
  for (int k = 0; k < kChunk / 4; ++k) {
    float4 v = w4[k];
    wv[4 * k] = v.x; wv[4 * k + 1] = v.y; wv[4 * k + 2] = v.z; wv[4 * k + 3] = v.w;
  }
#pragma unroll
  for (int k = 0; k < kChunk; ++k) {
    double p1 = k >= 1 ? lp[k - 1] : 0.0, p2 = k >= 2 ? lp[k - 2] : 0.0;
    lp[k] = fma(c1, p1, fma(c2, p2, (double)wv[k]));
  }
  double e0 = lp[kChunk - 1], e1 = lp[kChunk - 2];
  if (lane == 0) {
    e0 = fma(P.mc[0], s0, fma(P.mc[1], s1, e0));
    e1 = fma(P.mc[2], s0, fma(P.mc[3], s1, e1));
  }
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int dd = 1 << s;
    double u0 = shfl_up_d(e0, dd), u1 = shfl_up_d(e1, dd);
    if (lane >= dd) {
      e0 = fma(P.ks[4 * s], u0, fma(P.ks[4 * s + 1], u1, e0));
      e1 = fma(P.ks[4 * s + 2], u0, fma(P.ks[4 * s + 3], u1, e1));
    }
  }
  double x0 = shfl_up_d(e0, 1), x1 = shfl_up_d(e1, 1);
  if (lane == 0) { x0 = s0; x1 = s1; }
#pragma unroll
  for (int k = 0; k < kChunk; ++k) lp[k] += fma(P.fr0[2 * k], x0, P.fr0[2 * k + 1] * x1);
  s0 = shfl_d(lp[kChunk - 1], 31);
  s1 = shfl_d(lp[kChunk - 2], 31);
}

// Write the tile's outputs of one variant: y = D - LP - tail correction for
// outputs n in [n_base + C lane, +C) that lie in [0, n2); float4 stores when
// the whole chunk is inside (rows are 16-byte aligned, n_base % 32 == 0).
template <bool HAS_D = true>
__device__ __forceinline__ void store_chunk(float* out, int n_base, int n2, int nrow, int n_c,
                                            const float* dbuf, const double* s_corr, int lane,
                                            const double (&lp)[kChunk], double scale) {
  const int n0 = n_base + kChunk * lane;
  const float4* d4 = reinterpret_cast<const float4*>(dbuf + kChunk * lane);
  float y[kChunk];
#pragma unroll
  for (int k = 0; k < kChunk / 4; ++k) {
    const float4 v = HAS_D ? d4[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    y[4 * k] = (float)(((double)v.x - lp[4 * k]) * scale);  // scale == 1 unless normalising
    y[4 * k + 1] = (float)(((double)v.y - lp[4 * k + 1]) * scale);
    y[4 * k + 2] = (float)(((double)v.z - lp[4 * k + 2]) * scale);
    y[4 * k + 3] = (float)(((double)v.w - lp[4 * k + 3]) * scale);
  }
  if (n0 + kChunk > n_c) {  // tail outputs: subtract the exact truncation correction
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const int n = n0 + k;
      if (n >= n_c && n < n2)
        y[k] = (float)(((HAS_D ? (double)dbuf[kChunk * lane + k] : 0.0) - lp[k] - s_corr[n - n_c]) * scale);
    }
  }
  if (n0 >= 0 && n0 + kChunk <= n2) {
    float4* o4 = reinterpret_cast<float4*>(out + n0);
#pragma unroll
    for (int k = 0; k < kChunk / 4; ++k) o4[k] = make_float4(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {  // row tail; the alignment padding gets zeros
      const int n = n0 + k;
      if (n >= 0 && n < nrow) out[n] = n < n2 ? y[k] : 0.f;
    }
  }
}

// One warp renders one channel (full + optional early variant) in a single
// ordered sweep over its bucket-sorted items.  Items of bucket b start in
// output window b - 2 (n' = s' + k, biased by kSpBias = 64); each is visited
// ONCE: lane L takes tap k = (L - delta) mod 32 (+32 j) of its phase row and
// adds it to the window it lands in (accumulators a0, a1[, a2] for the current
// and next windows).  When the sweep passes a bucket, the current window is
// final and is emitted to the per-warp tile buffer; every kTileWin windows the
// FP64 LP scan runs and y = D - LP is stored with coalesced writes.
template <bool EARLY, int NBK>
struct Channel {
  // accumulators of windows w, w+1, w+2: D and W, full and early
  float dF[NBK + 1], wF[NBK + 1], dE[NBK + 1], wE[NBK + 1];

  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i <= NBK; ++i) { dF[i] = 0.f; wF[i] = 0.f; dE[i] = 0.f; wE[i] = 0.f; }
  }
  __device__ __forceinline__ void shift() {
#pragma unroll
    for (int i = 0; i < NBK; ++i) { dF[i] = dF[i + 1]; wF[i] = wF[i + 1]; dE[i] = dE[i + 1]; wE[i] = wE[i + 1]; }
    dF[NBK] = 0.f; wF[NBK] = 0.f; dE[NBK] = 0.f; wE[NBK] = 0.f;
  }
  // One staged item: dec = byte offset of (phase row, 32 - start mod 32) in the
  // doubled table (every 64-entry block holds its 32 taps twice), ae = +-gain
  // (sign = early flag).  Lane L reads entry L + 32 - delta: tap (L - delta)
  // mod 32 (+32 j), which lands in window j if L >= delta (bit 8 of the byte
  // offset set) else in window j + 1.  Predicated FMAs keep the warp converged
  // with no selects; only the early test branches, and it is warp-uniform.
  template <bool EW>
  __device__ __forceinline__ void add(unsigned dec, float ae, unsigned lane8, unsigned comp_sh) {
    const unsigned addr = dec + lane8;
    const unsigned lo = addr & 256u;
    const float a = fabsf(ae);
#pragma unroll
    for (int j = 0; j < NBK; ++j) {
      float tx, ty;
      asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(tx), "=f"(ty) : "r"(comp_sh + addr + 512u * j));
      asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
          "@p fma.rn.f32 %0, %5, %6, %0;\n\t@p fma.rn.f32 %1, %5, %7, %1;\n\t"
          "@!p fma.rn.f32 %2, %5, %6, %2;\n\t@!p fma.rn.f32 %3, %5, %7, %3;\n\t}"
          : "+f"(dF[j]), "+f"(wF[j]), "+f"(dF[j + 1]), "+f"(wF[j + 1])
          : "r"(lo), "f"(a), "f"(tx), "f"(ty));
      if (EW && ae < 0.f) {
        asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
            "@p fma.rn.f32 %0, %5, %6, %0;\n\t@p fma.rn.f32 %1, %5, %7, %1;\n\t"
            "@!p fma.rn.f32 %2, %5, %6, %2;\n\t@!p fma.rn.f32 %3, %5, %7, %3;\n\t}"
            : "+f"(dE[j]), "+f"(wE[j]), "+f"(dE[j + 1]), "+f"(wE[j + 1])
            : "r"(lo), "f"(a), "f"(tx), "f"(ty));
      }
    }
  }
};

// SEG: the batch may hold segmented channels.  EONLY (with EARLY = false,
// SEG = false): the early pass -- the early variant alone, from the items of
// the buckets K2 marked (chan_erange), with the full variant's machinery: the
// same sums in the same order as a full + early sweep (identical bits), while
// the full pass (EARLY = false) carries no early work in its item loop.
template <bool EARLY, int NBK, bool SEG, bool EONLY = false>
__global__ void __launch_bounds__(kRenderThreads, 3) render_kernel(const __grid_constant__ RenderArgs A) {
  static_assert(!EONLY || (!EARLY && !SEG), "the early pass: unsegmented channels, one variant");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_stidx[kWarps];
  const frir_plan_desc& d = A.plan.d;
  constexpr int kRow = 64 * NBK;  // doubled rows (see Channel::add)
  constexpr int V = EARLY ? 2 : 1;
  const int ncomp = d.r_h * kRow;
  float2* s_comp = reinterpret_cast<float2*>(smem);
  double* s_corr_all = reinterpret_cast<double*>(smem + (size_t)ncomp * 8);  // [warp][V][32]
  // [warp][V][D, W][2 scratch windows + kTile]: emits of windows -2, -1 land
  // in the scratch windows, so the per-window store needs no branch
  float* s_tile = reinterpret_cast<float*>(s_corr_all + kWarps * V * 32);
  int2* s_items = reinterpret_cast<int2*>(s_tile + (size_t)kWarps * V * 2 * kTileRow);
  float* s_head = reinterpret_cast<float*>(s_items + 32 * kWarps);          // [warp][V][D, W][64]
  for (int i = threadIdx.x; i < ncomp; i += blockDim.x) s_comp[i] = A.plan.comp[i];
  if (!EARLY && !EONLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the early pass may start
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned comp_sh = (unsigned)__cvta_generic_to_shared(s_comp);
  const unsigned lane8 = 8u * lane;
  float* dF_t = s_tile + (size_t)warp * V * 2 * kTileRow + 2 * kWin;  // window 0 of the tile
  float* wF_t = dF_t + kTileRow;
  float* dE_t = wF_t + kTileRow;
  float* wE_t = dE_t + kTileRow;
  const unsigned t_sh = (unsigned)__cvta_generic_to_shared(dF_t) + 4u * lane;  // emit stores: slot * 128 B
  double* corrF_s = s_corr_all + warp * V * 32;
  double* corrE_s = corrF_s + 32;
  int2* s_it = s_items + 32 * warp;
  float* head_s = s_head + warp * V * 2 * 64;
  const double c1 = A.plan.lp[0], c2 = A.plan.lp[1];
  const int sup = d.sup, r_h = d.r_h, up = d.up, down = d.down, half1 = d.half1;
  const unsigned down_magic = (unsigned)((0x100000000ull + down - 1) / down);  // exact for e < 2^32 / down

  for (;;) {
    // work unit v: first the later segments of long channels (K2's list, the
    // longest work), then the first segment of every channel, longest first
    int v = 0;
    if (lane == 0) v = atomicAdd(A.ws.counter + (EONLY ? 1 : 0), 1);
    v = __shfl_sync(0xffffffffu, v, 0);
    const int nextra = SEG ? *A.sw.nextra : 0;
    int c, sg = 0;
    constexpr bool eonly = EONLY;
    if (v < nextra) {
      const int u = A.sw.units[v];
      c = u / kMaxSeg;
      sg = u - c * kMaxSeg;
    } else {
      const int ci = v - nextra;
      if (ci >= A.total_channels) break;
      c = A.chan_order ? A.chan_order[ci] : ci;
    }
    const int j = A.chan_job[c];
    const frir_job& J = A.jobs[j];
    const int m = c - J.chan_off;
    const int rows = J.n_images + 1;
    const int n1 = J.n1, n2 = J.n2;
    const int nseg = SEG ? A.sw.seg[(size_t)c * kSegInts + 63] : 1;  // K2's seg_count
    if (SEG && lane == 0) s_stidx[warp] = nseg > 1 ? c * kMaxSeg + sg : -1;  // end-state slot (flush of the last tile)
    const int nrow = min(J.out_stride, (n2 + 3) & ~3);  // row incl. alignment padding
    const double scale = (double)A.ws.chan_scale[c];
    const int2* items = A.ws.items + J.item_off + (size_t)m * rows;
    const int nvalid = A.ws.chan_rows[c];  // sorted items before the dropped-arrival bucket
    float* outF = (eonly ? A.out_early : A.out_full) + J.out_off + (size_t)m * J.out_stride;  // (eonly: early)
    float* outE = EARLY ? A.out_early + J.out_off + (size_t)m * J.out_stride : nullptr;

    const int n_c = first_corrected(d, n1);  // outputs n >= n_c get K2's tail corrections
    // windows touched by early items (q in [q0 - lo, q0 + hi], core.py:257-264)
    int ew_lo = 0, ew_hi = -1;
    if (EARLY || EONLY) {
      const int q0 = A.ws.chan_q0[c];
      ew_lo = (ceil_div_i(q0 - J.e_lo + d.t0, r_h) + kExt) >> 5;
      ew_hi = (ceil_div_i(q0 + J.e_hi + d.t0, r_h) + kExt + sup - 1) >> 5;
    }
    __syncwarp();

    // ---- head pre-pass: items whose stage-1 taps reach mid index < 0 (a
    // prefix of the bucket-sorted list; only sources within a few cm of a mic)
    bool head_on = false;  // head corrections pending in head_s
    for (int p = 0; sg == 0 && p < nvalid; p += 32) {
      const int2 mine = p + lane < nvalid ? items[p + lane] : make_int2(0xFFFFF, 0);
      const int cnt = min(32, nvalid - p);
      const int qm = r_h * ((mine.x & 0xFFFFF) - kSpBias - kExt) - d.t0 - (((unsigned)mine.x >> 20) & 0x3FF);
      unsigned hm = __ballot_sync(0xffffffffu, lane < cnt && up * qm < half1);
      if (hm) {
        if (!head_on) {
          for (int i = lane; i < V * 2 * 64; i += 32) head_s[i] = 0.f;
          head_on = true;
        }
        while (hm) {
          const int src = __ffs(hm) - 1;
          hm &= hm - 1;
          const int qs = __shfl_sync(0xffffffffu, qm, src);
          const float aes = __int_as_float(__shfl_sync(0xffffffffu, mine.y, src));
          const double as = fabs((double)aes);
          const int xs = up * qs - half1 + 1024 * down;
          const int klo = (int)__umulhi((unsigned)xs, down_magic) - 1024 + (xs % down != 0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int np = lane + 32 * h;  // n'' in [0, 64)
            const int n = np - kExt;
            double cd = 0.0, cw = 0.0;
            for (int k = klo; k < 0; ++k) {
              FRIR_CHECK(down * k + half1 - up * qs >= 0 && down * k + half1 - up * qs < d.len1);
              const double cc = as * A.plan.h1up[down * k + half1 - up * qs];
              const int idx = d.r_l * n + d.half2 - k;
              if (idx >= 0 && idx < d.len2) cd += cc * A.plan.h2[idx];
              if (idx >= 0 && idx < d.len2 + 2 * d.r_l) cw += cc * A.plan.gw[idx];
            }
            if (!eonly || aes < 0.f) {  // (the early pass: early head items only)
              head_s[np] -= (float)cd;
              head_s[64 + np] -= (float)cw;
            }
            if (EARLY && aes < 0.f) {
              head_s[128 + np] -= (float)cd;
              head_s[192 + np] -= (float)cw;
            }
          }
        }
        __syncwarp();
      }
      // later items have bucket >= this batch's last: stop once none can be a head item
      const int bk_last = __shfl_sync(0xffffffffu, (mine.x & 0xFFFFF) >> 5, cnt - 1);
      const long long qmin = (long long)r_h * ((bk_last << 5) - kSpBias - kExt) - d.t0 - (r_h - 1);
      if ((long long)up * qmin >= half1) break;
    }

    // ---- tail corrections of outputs n >= n_c (computed by K2)
    corrF_s[lane] = A.ws.corr[64 * (size_t)c + (eonly ? 32 : 0) + lane];
    if (EARLY) corrE_s[lane] = A.ws.corr[64 * (size_t)c + 32 + lane];
    __syncwarp();

    // ---- ordered sweep: windows w = -2 .. nwin-1 over n'' = n + kExt
    // this segment: windows [w_lo, nwin), items [i_lo, i_hi) of the sorted row
    int w_lo = 0, nwin = (n2 + kExt + kWin - 1) / kWin, i_lo = 0, i_hi = nvalid;  // this segment
    if (SEG && nseg > 1) {
      const int* seg = A.sw.seg + (size_t)c * kSegInts;
      w_lo = seg[sg]; nwin = seg[sg + 1]; i_lo = seg[17 + sg]; i_hi = seg[33 + sg];
    }
    if (eonly) {  // the early pass: the buckets of the early items; the tiles before them are zeros
      const int2 er = A.ws.chan_erange[c];
      i_lo = er.x;
      i_hi = er.y;
      if (i_lo < i_hi && !head_on) {  // (q0 itself is early, so the range is never empty)
        const int b_first = (items[i_lo].x & 0xFFFFF) >> 5;  // feeds windows b_first - 2 ..
        w_lo = max(0, (b_first - 2) & ~(kTileWin - 1));
      }
      const int pre = min(nrow, w_lo * kWin - kExt);  // (a multiple of 4)
      for (int n = 4 * lane; n < pre; n += 128) *reinterpret_cast<float4*>(outF + n) = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    Channel<EARLY, NBK> ch;
    ch.clear();
    double sF0 = 0.0, sF1 = 0.0, sE0 = 0.0, sE1 = 0.0;
    bool e_dead = false;  // early ring-down negligible: outputs are zeros
    double e_ref = 0.0;   // largest early LP state seen while early items fed tiles
    int w = w_lo - 2;     // window held by the front accumulators
    int slot = -2;        // next tile slot (negative: scratch windows)
    bool est = true;      // the current tile is not quiet: early windows are stored
    auto flush = [&]() {
      const int w0 = w - slot + 1;  // first window of the tile
      const int n_base = w0 * kWin - kExt;
      for (int s2 = slot; s2 < kTileWin; ++s2) {  // pad a partial last tile
        wF_t[s2 * kWin + lane] = 0.f;
        dF_t[s2 * kWin + lane] = 0.f;
        if (EARLY) { wE_t[s2 * kWin + lane] = 0.f; dE_t[s2 * kWin + lane] = 0.f; }
      }
      if (head_on && w0 == 0) {  // head corrections of windows 0 and 1 (warp-uniform, once)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          dF_t[s2 * kWin + lane] += head_s[32 * s2 + lane];
          wF_t[s2 * kWin + lane] += head_s[64 + 32 * s2 + lane];
          if (EARLY) {
            dE_t[s2 * kWin + lane] += head_s[128 + 32 * s2 + lane];
            wE_t[s2 * kWin + lane] += head_s[192 + 32 * s2 + lane];
          }
        }
      }
      __syncwarp();
      double lp[kChunk];
      // the early variant's tile: scanned while early items feed it, then the
      // closed-form decay of its LP state, then zeros
      auto early_tile = [&](float* out, const float* d_t, const float* w_t, const double* corr_s, double& s0,
                            double& s1) {
        const bool quiet = w0 > ew_hi;  // no early item feeds this tile: pure decay
        if (!quiet) {
          lp_scan_tile(w_t, A.plan, c1, c2, s0, s1, lane, lp);
          store_chunk(out, n_base, n2, nrow, n_c, d_t, corr_s, lane, lp, scale);
          e_ref = fmax(e_ref, fabs(s0) + fabs(s1));
        } else if (!e_dead) {
          // LP[k] = row0(M^(k+1)) . s for the whole tile; y = -LP (D = W = 0)
          const double* fr = A.plan.scan + kScanFree + 2 * kChunk * lane;  // global (L1)
#pragma unroll
          for (int k = 0; k < kChunk; ++k) lp[k] = fma(fr[2 * k], s0, fr[2 * k + 1] * s1);
          const double* Mt = A.plan.mt;
          const double n0v = fma(Mt[0], s0, Mt[1] * s1), n1v = fma(Mt[2], s0, Mt[3] * s1);
          s0 = n0v;
          s1 = n1v;
          store_chunk<false>(out, n_base, n2, nrow, n_c, d_t, corr_s, lane, lp, scale);
          // the ring-down after the early window decays by ~0.06 per tile at
          // 16 kHz; once |s| < 2^-44 of its early-window maximum, the rest
          // (|LP| <= ~400 |s|) is below 1e-10 of the channel's level
          e_dead = fabs(s0) + fabs(s1) < fmax(1e-50, 0x1p-44 * e_ref);
        } else {
          const int n0 = n_base + kChunk * lane;
          if (n0 >= 0 && n0 + kChunk <= nrow) {  // (rows are 16-byte aligned, n_base % 4 == 0)
            *reinterpret_cast<float4*>(out + n0) = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
#pragma unroll
            for (int k = 0; k < kChunk; ++k)
              if (n0 + k >= 0 && n0 + k < nrow) out[n0 + k] = 0.f;
          }
        }
      };
      if (eonly) {
        early_tile(outF, dF_t, wF_t, corrF_s, sF0, sF1);
      } else {
        lp_scan_tile(wF_t, A.plan, c1, c2, sF0, sF1, lane, lp);
        store_chunk(outF, n_base, n2, nrow, n_c, dF_t, corrF_s, lane, lp, scale);
        if (EARLY) early_tile(outE, dE_t, wE_t, corrE_s, sE0, sE1);
      }
      if (SEG && w == nwin - 1 && lane == 0) {  // last tile of the sweep: zero-start end state of a segment (K4)
        const int si = s_stidx[warp];
        if (si >= 0) {
          double* st = A.sw.state + (size_t)si * 4;
          st[0] = sF0; st[1] = sF1; st[2] = sE0; st[3] = sE1;
        }
      }
      __syncwarp();
      slot = 0;
      est = w + 1 <= ew_hi;  // the next tile starts at window w + 1
    };
    auto emit = [&]() {
      const unsigned a = t_sh + (unsigned)(slot * (kWin * 4));
      sts_f32(a, ch.dF[0]);
      sts_f32(a + kTileRow * 4, ch.wF[0]);
      if (EARLY && est) {  // tile not quiet: its early slots are read
        sts_f32(a + 2 * kTileRow * 4, ch.dE[0]);
        sts_f32(a + 3 * kTileRow * 4, ch.wE[0]);
      }
      ++slot;
      if (slot == kTileWin || w == nwin - 1) flush();
      ch.shift();
      ++w;
    };
    const int2* sitems = items + i_lo;  // the segment's items
    const int srows = i_hi - i_lo;
    int2 nxt = lane < srows ? sitems[lane] : make_int2(0xFFFFF, 0);  // sentinel: last bucket
    for (int p = 0; p < srows; p += 32) {
      const int2 mine = nxt;
      const int pn = p + 32 + lane;
      nxt = pn < srows ? sitems[pn] : make_int2(0xFFFFF, 0);  // prefetch the next batch
      const int bk = (mine.x & 0xFFFFF) >> 5;
      const unsigned dec = (((unsigned)mine.x >> 20) & 0x3FFu) * (512u * NBK) + 8u * (32u - (mine.x & 31));
      FRIR_CHECK(p + lane >= srows || (((unsigned)mine.x >> 20) & 0x3FFu) < (unsigned)r_h);
      __syncwarp();
      s_it[lane] = make_int2((int)dec, eonly && mine.y >= 0 ? 0 : mine.y);  // (early pass: late items add +0)
      __syncwarp();
      const int cnt = min(32, srows - p);
      const unsigned emask = EARLY ? __ballot_sync(0xffffffffu, lane < cnt && mine.y < 0) : 0u;
      int jj = 0;
      while (jj < cnt) {  // runs of equal bucket (items are bucket-sorted)
        const int b = __shfl_sync(0xffffffffu, bk, jj);
        while (b > w + 2) emit();
        const unsigned same = __ballot_sync(0xffffffffu, bk == b && lane < cnt);
        const int end = 32 - __clz(same);
        if (EARLY && (same & emask)) {
#pragma unroll 2
          for (; jj < end; ++jj) {
            const int2 it = s_it[jj];
            ch.template add<true>((unsigned)it.x, __int_as_float(it.y), lane8, comp_sh);
          }
        } else {
#pragma unroll 4
          for (; jj < end; ++jj) {
            const int2 it = s_it[jj];
            ch.template add<false>((unsigned)it.x, __int_as_float(it.y), lane8, comp_sh);
          }
        }
      }
    }
    if (eonly) {
      // the tiles early items feed go through the sweep; the quiet ones after
      // them need no windows: the closed-form decay of the LP state tile by
      // tile (as early_tile does), then zeros to the end of the row
      while (w < nwin && !(slot == 0 && w > ew_hi)) emit();
      for (; w < nwin && !e_dead; w += kTileWin) {
        const int n_base = w * kWin - kExt;
        double lp[kChunk];
        const double* fr = A.plan.scan + kScanFree + 2 * kChunk * lane;  // global (L1)
#pragma unroll
        for (int k = 0; k < kChunk; ++k) lp[k] = fma(fr[2 * k], sF0, fr[2 * k + 1] * sF1);
        const double* Mt = A.plan.mt;
        const double n0v = fma(Mt[0], sF0, Mt[1] * sF1), n1v = fma(Mt[2], sF0, Mt[3] * sF1);
        sF0 = n0v;
        sF1 = n1v;
        store_chunk<false>(outF, n_base, n2, nrow, n_c, dF_t, corrF_s, lane, lp, scale);
        e_dead = fabs(sF0) + fabs(sF1) < fmax(1e-50, 0x1p-44 * e_ref);
      }
      const int n_from = max(0, w * kWin - kExt);  // first output of tile w
      if (w < nwin)
        for (int n = n_from + 4 * lane; n < nrow; n += 128) *reinterpret_cast<float4*>(outF + n) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      while (w < nwin) emit();
    }
  }
}

// ---------------------------------------------------------------- K4 segment seams
// A long channel's segments were rendered from zero LP state (K3).  With the
// LP recursion linear, the true output of segment k is the zero-start output
// minus the free response of its true start state t_k, and
// t_k = e_(k-1) + M^len(k-1) t_(k-1) (e = zero-start end state, M^len by
// squaring M^kTile).  One warp per channel applies -scale * LPfree to the
// segment's tiles until the response is below 2^-44 of t_k.  (The response
// is at most the size of the low-pass branch, so the FP32 rounding of the
// zero-start output costs ~1 ulp of the channel's peak.)
struct SeamArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  Workspace ws;
  SegWs sw;
  DevPlan plan;
  float* out_full;
  float* out_early;
  int total_channels;
};

__global__ void __launch_bounds__(256) seam_kernel(const __grid_constant__ SeamArgs A) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= A.total_channels) return;
  const frir_job& J = A.jobs[A.chan_job[c]];
  const int n2 = J.n2;
  const int nseg = A.sw.seg[(size_t)c * kSegInts + 63];  // K2's seg_count
  if (nseg == 1) return;
  const int m = c - J.chan_off;
  const double scale = (double)A.ws.chan_scale[c];
  const int* seg = A.sw.seg + (size_t)c * kSegInts;
  const double* est = A.sw.state + (size_t)c * kMaxSeg * 4;
  const double* Mt = A.plan.mt;
  const double* fr = A.plan.scan + kScanFree + 2 * kChunk * lane;
  double f[2 * kChunk];
#pragma unroll
  for (int k = 0; k < 2 * kChunk; ++k) f[k] = fr[k];
  const int V = A.out_early ? 2 : 1;
  for (int v = 0; v < V; ++v) {
    float* out = (v ? A.out_early : A.out_full) + J.out_off + (size_t)m * J.out_stride;
    double t0 = 0.0, t1 = 0.0;  // true start state of segment k
    for (int k = 1; k < nseg; ++k) {
      double x0 = t0, x1 = t1;  // M^(kTile * tiles) t
      double p0 = Mt[0], p1 = Mt[1], p2 = Mt[2], p3 = Mt[3];
      for (int e = (seg[k] - seg[k - 1]) / kTileWin; e; e >>= 1) {
        if (e & 1) {
          const double y0 = fma(p0, x0, p1 * x1), y1 = fma(p2, x0, p3 * x1);
          x0 = y0; x1 = y1;
        }
        const double q0 = fma(p0, p0, p1 * p2), q1 = fma(p0, p1, p1 * p3);
        const double q2 = fma(p2, p0, p3 * p2), q3 = fma(p2, p1, p3 * p3);
        p0 = q0; p1 = q1; p2 = q2; p3 = q3;
      }
      t0 = est[4 * (k - 1) + 2 * v] + x0;
      t1 = est[4 * (k - 1) + 2 * v + 1] + x1;
      double s0 = t0, s1 = t1;
      const double cut = 0x1p-44 * (fabs(t0) + fabs(t1));
      for (int tw = seg[k]; tw < seg[k + 1]; tw += kTileWin) {
        if (!(fabs(s0) + fabs(s1) > cut)) break;  // warp-uniform
        const int n0 = tw * kWin - kExt + kChunk * lane;
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) {
          const int n = n0 + kk;
          if (n >= 0 && n < n2)
            out[n] = (float)((double)out[n] - scale * fma(f[2 * kk], s0, f[2 * kk + 1] * s1));
        }
        const double y0 = fma(Mt[0], s0, Mt[1] * s1), y1 = fma(Mt[2], s0, Mt[3] * s1);
        s0 = y0; s1 = y1;
      }
    }
  }
}

// ---------------------------------------------------------------- stage API kernels
// sample_image_geometry (core.py:131-183) for every job of a native-draw
// batch: the ImageSet rows K1 renders from -- distances, azimuths,
// elevations, distance ratios at img_off + i, per-mic distances at
// item_off + i * M + m (row-major (I + 1, M) like the reference), and, when
// `with_refl`, the reflection counts of sample_reflection_counts (core.py:
// 195-221) from the stage-1 stream (else NaN, as the reference leaves them).
struct ImageSetOut {
  double *dist, *az, *el, *ratio, *refl, *mic_dist;
  int with_refl;
};

__global__ void __launch_bounds__(128) image_set_kernel(GeomArgs A, ImageSetOut O) {
  const int j = blockIdx.x;
  const frir_job& J = A.jobs[j];
  const int I = J.n_images, M = J.n_mics;
  const int g = blockIdx.y * blockDim.x + threadIdx.x;
  const double* mics = A.mics + 3 * (size_t)J.mic_off;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  auto mic_row = [&](size_t i, double x, double y, double z) {  // params.py:162-171 distances_to_mics
    for (int m = 0; m < M; ++m) {
      const double dx = __dsub_rn(x, mics[3 * m]), dy = __dsub_rn(y, mics[3 * m + 1]), dz = __dsub_rn(z, mics[3 * m + 2]);
      O.mic_dist[J.item_off + i * M + m] =
          __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    }
  };
  if (g == 0) {  // row 0: the direct path (core.py:163-169)
    double x, y, z;
    image_position(J, J.d0, J.az, J.el, &x, &y, &z);
    const size_t o = J.img_off;
    O.dist[o] = J.d0; O.az[o] = J.az; O.el[o] = J.el; O.ratio[o] = 1.0; O.refl[o] = 0.0;
    mic_row(0, x, y, z);
  }
  if (g >= (I + 3) / 4) return;
  double px[4], py[4], pz[4];
  float lg[4];
  ImageDraws d;
  image_group(A, J, g, px, py, pz, lg, &d);
  const int nk = min(4, I - 4 * g);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= nk) break;
    const size_t i = 4 * (size_t)g + k + 1, o = J.img_off + i;
    O.dist[o] = d.dist[k]; O.az[o] = d.az[k]; O.el[o] = d.el[k]; O.ratio[o] = d.ratio[k];
    O.refl[o] = O.with_refl ? d.refl[k] : nan;
    mic_row(i, px[k], py[k], pz[k]);
  }
}

// Sparse items of explicit high-rate trains (downsample_highpass_downsample
// on a HighRateTrain or (M, L) array, resample.py:81-136): channel c of the
// batch is row c of `train`; its samples with sign * x > 0 become items
// (index n, amplitude sign * x[n]) in index order, the rest of the row's item
// slots go to the dropped bucket.  One CTA per channel, ordered compaction.
constexpr int kTrainThreads = 256;
__global__ void __launch_bounds__(kTrainThreads) train_items_kernel(const double* __restrict__ train, long ld,
                                                                     int sign, const frir_job* jobs,
                                                                     const int32_t* chan_job, Workspace ws, int r_h,
                                                                     int t0, unsigned magic) {
  __shared__ int s_w[kTrainThreads / 32];
  __shared__ int s_base;
  const int c = blockIdx.x;
  const frir_job& J = jobs[chan_job[c]];
  const int m = c - J.chan_off, rows = J.n_images + 1, L = J.L;
  const double* x = train + (size_t)c * ld;
  int2* out = ws.items_raw + J.item_off + (size_t)m * rows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_base = 0;
    ws.chan_q0[c] = 0;
    ws.chan_scale[c] = 1.0f;
    ws.chan_row[c] = make_longlong2((long long)J.item_off + (long long)m * rows, rows);
  }
  __syncthreads();
  for (int n0 = 0; n0 < L; n0 += kTrainThreads) {
    const int n = n0 + threadIdx.x;
    const double v = n < L ? sign * x[n] : 0.0;
    const bool keep = v > 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    int off = s_base;
    for (int w2 = 0; w2 < warp; ++w2) off += s_w[w2];
    if (keep) {
      const int pos = off + __popc(bal & ((1u << lane) - 1u));
      FRIR_CHECK(pos < rows);
      out[pos] = make_item(n, (float)v, r_h, t0, magic);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w2 = 0; w2 < kTrainThreads / 32; ++w2) t += s_w[w2];
      s_base += t;
    }
    __syncthreads();
  }
  for (int p = s_base + threadIdx.x; p < rows; p += kTrainThreads) out[p] = dropped_item(J.n2);
}

// Nonzeros with sign * x > 0 per row (the item count of train_items_kernel).
__global__ void __launch_bounds__(kTrainThreads) train_count_kernel(const double* __restrict__ train, long ld, int L,
                                                                     int sign, int32_t* counts) {
  const double* x = train + (size_t)blockIdx.x * ld;
  int n = 0;
  for (int i = threadIdx.x; i < L; i += kTrainThreads) n += sign * x[i] > 0.0;
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(counts + blockIdx.x, n);
}

}  // namespace

// ---------------------------------------------------------------- host launcher
int check_line() {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_frir_check_line, sizeof(int));
  return v;
}

size_t workspace_bytes(const frir_batch* b) {
  size_t n = align_up((size_t)b->total_items * 8) + raw_bytes(b) + 4 * align_up((size_t)b->total_channels * 4) +
             align_up((size_t)b->total_channels * 8) + align_up((size_t)b->total_channels * 64 * 8) +
             align_up((size_t)b->total_channels * 16) + 256;
  const int smax = batch_seg_max(b);
  if (smax > 1)
    n += align_up((size_t)b->total_channels * kSegInts * 4) + align_up((size_t)b->total_channels * kMaxSeg * 4 * 8) +
         align_up((size_t)b->total_channels * kMaxSeg * 4) + 256;
  return n;
}

static int table_blocks(const frir_plan_desc& d) { return (d.sup + 31) / 32; }
constexpr int kDynSlack = 1024;  // >= any kernel's static smem; launches check sizes against optin - slack
constexpr int kSortStageRows = 4608;  // sorted rows staged in shared memory up to this length (measured: helps config 2, not config 5)

static size_t render_smem(const frir_plan_desc& d, bool early) {
  const int v = early ? 2 : 1;
  return (size_t)d.r_h * 64 * table_blocks(d) * 8 + (size_t)kWarps * v * 32 * 8 +
         (size_t)kWarps * v * 2 * kTileRow * 4 + (size_t)kWarps * 32 * 8 +
         (size_t)kWarps * v * 2 * 64 * 4;
}

// Dynamic smem cap of every kernel: the opt-in maximum minus its static smem.
template <typename K>
static cudaError_t allow_smem(K k, int optin) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, k);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

// Every kernel that takes dynamic shared memory gets the device's opt-in
// maximum once here, and the render kernels' residency is queried once, so a
// launch issues no attribute or occupancy calls (plan = one device).
template <bool EARLY, int NBK, bool SEG, bool EONLY = false>
static cudaError_t init_render(frir_plan* p) {
  auto k = render_kernel<EARLY, NBK, SEG, EONLY>;
  const size_t smem = render_smem(p->dev.d, EARLY);
  int& per_sm = EONLY ? p->lc.render_e_per_sm[NBK - 1] : p->lc.render_per_sm[EARLY][NBK - 1][SEG];
  per_sm = 0;
  if ((int)smem > p->lc.smem_optin - kDynSlack) return cudaSuccess;  // 0: this plan cannot launch it
  // the cap is per kernel, not per plan: plans of other rates launch it with other sizes
  cudaError_t e = allow_smem(k, p->lc.smem_optin);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kRenderThreads, smem);
  return e;
}

cudaError_t init_launch_cache(frir_plan* p) {
  LaunchCache& lc = p->lc;
  cudaError_t e = cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, p->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&lc.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
  const int mx = lc.smem_optin;
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 8, false>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 16, false>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint32_t, 8, false>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint32_t, 16, false>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 8, true>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 16, true>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint32_t, 8, true>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint32_t, 16, true>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 8, false, 8>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 8, false, 17>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 16, false, 8>, mx);
  if (e == cudaSuccess) e = allow_smem(sort_kernel<uint16_t, 16, false, 17>, mx);
  if (e == cudaSuccess) e = allow_smem(tail_kernel<false>, mx);
  if (e == cudaSuccess) e = allow_smem(tail_kernel<true>, mx);
  if (e == cudaSuccess) e = init_render<true, 1, false>(p);
  if (e == cudaSuccess) e = init_render<true, 1, true>(p);
  if (e == cudaSuccess) e = init_render<false, 1, false>(p);
  if (e == cudaSuccess) e = init_render<false, 1, true>(p);
  if (e == cudaSuccess) e = init_render<true, 2, false>(p);
  if (e == cudaSuccess) e = init_render<true, 2, true>(p);
  if (e == cudaSuccess) e = init_render<false, 2, false>(p);
  if (e == cudaSuccess) e = init_render<false, 2, true>(p);
  if (e == cudaSuccess) e = init_render<false, 1, false, true>(p);
  if (e == cudaSuccess) e = init_render<false, 2, false, true>(p);
  return e;
}

template <bool EARLY, int NBK, bool SEG, bool EONLY = false>
static cudaError_t launch_render(const frir_plan* plan, const RenderArgs& ra, long channels, cudaStream_t st) {
  const size_t smem = render_smem(plan->dev.d, EARLY);
  const int per_sm = EONLY ? plan->lc.render_e_per_sm[NBK - 1] : plan->lc.render_per_sm[EARLY][NBK - 1][SEG];
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long want = (channels * ra.seg_max + kWarps - 1) / kWarps;  // upper bound of the work units
  int grid = (int)std::min<long>((long)plan->lc.sms * per_sm, want);
  if (!EONLY) {
    render_kernel<EARLY, NBK, SEG, EONLY><<<grid, kRenderThreads, smem, st>>>(ra);
    return cudaGetLastError();
  }
  // The early pass reads only K2 / K2b outputs and writes only the early rows,
  // so it need not wait for the full pass: a programmatic dependent launch
  // (the full pass triggers it at its start) lets its CTAs take the SMs the
  // full pass's CTAs leave as its work queue drains.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRenderThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, render_kernel<EARLY, NBK, SEG, EONLY>, ra);
}

#ifndef FRIR_SPLIT_EARLY_CHANNELS
#define FRIR_SPLIT_EARLY_CHANNELS 1024
#endif
constexpr long kSplitEarlyChannels = FRIR_SPLIT_EARLY_CHANNELS;
static bool split_early(const frir_batch* b) {
  return batch_seg_max(b) <= 1 && (long)b->total_channels >= kSplitEarlyChannels;
}

int launches(const frir_batch* b, int early) {
  // geom, sort, tail, render (plus one memset of the work counters); the split
  // tail and the seam kernel when the batch may hold segmented (long) channels;
  // the early pass when it is split from the full one
  return 4 + (batch_seg_max(b) > 1 ? 2 : 0) + (early && split_early(b) ? 1 : 0);
}

int launch_simulate(const frir_plan* plan, const frir_batch* b, void* wsp, size_t ws_bytes,
                    float* out_full, float* out_early, int32_t* direct_index, cudaStream_t st,
                    int stages) {
  const frir_plan_desc& d = plan->dev.d;
  if (ws_bytes < workspace_bytes(b)) {
    set_error("workspace too small: need " + std::to_string(workspace_bytes(b)) + " bytes");
    return FRIR_ENOMEM;
  }
  if (b->max_rows > kMaxRows) {
    set_error("num_images + 1 = " + std::to_string(b->max_rows) + " exceeds the kernel limit " +
              std::to_string(kMaxRows));
    return FRIR_ERANGE;
  }
  if (b->n_jobs == 0 || b->total_channels == 0) return FRIR_OK;
  Workspace ws = carve(wsp, b);
  const SegWs sw = carve_seg(wsp, b);
  cudaError_t e = cudaSuccess;

  const int rate = d.r_h * d.sample_rate;
  GeomArgs ga;
  ga.jobs = b->jobs; ga.mics = b->mics;
  ga.draw_dist = b->draw_dist; ga.draw_az = b->draw_az; ga.draw_el = b->draw_el; ga.draw_refl = b->draw_refl;
  ga.ws = ws; ga.direct_index = direct_index;
  ga.r_h = d.r_h; ga.t0 = d.t0;
  ga.rh_magic = (unsigned)((0x100000000ull + d.r_h - 1) / d.r_h);
  ga.rate = (double)rate;
  if (stages & FRIR_STAGE_GEOM) {  // K1: draws, geometry, delays, items
    int maxg = (b->max_rows - 1 + 3) / 4;
    dim3 g1(b->n_jobs, maxg > 0 ? (maxg + 127) / 128 : 1);
    geom_kernel<<<g1, 128, 0, st>>>(ga);
    e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(std::string("geom_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  }

  if (stages & FRIR_STAGE_DELAY) {  // K2: early flags + stable bucket sort per channel
    {
      SortArgs sa;
      sa.jobs = b->jobs; sa.chan_job = b->chan_job; sa.ws = ws; sa.sw = sw;
      sa.r_h = d.r_h; sa.t0 = d.t0; sa.plan = plan->dev;
      // ranks by shared-memory atomics (default) or by ballots (FRIR_SORT_BALLOT=1,
      // the reference ordering the tests compare against bit for bit)
      static const int ballot = getenv("FRIR_SORT_BALLOT") ? atoi(getenv("FRIR_SORT_BALLOT")) : 0;
      sa.atom_ranks = ballot ? 0 : 1;
      const int nbk = ((b->max_windows * kWin + kSpBias) >> 5) + 3;
      if (sw.nextra) {
        e = cudaMemsetAsync(sw.nextra, 0, sizeof(int), st);
        if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FRIR_ECUDA; }
      }
      const bool wide = b->max_rows > 65535;  // sorted positions need 32-bit counters
      const bool big = b->total_items >= 4096LL * b->total_channels;  // long rows on average: 16 warps
      int nw = big ? 16 : 8;  // (measured: 8 warps 1.28x slower on config 5, 16 warps 1.14x slower on config 2)
      size_t smem = align16((size_t)nbk * nw * (wide ? 4 : 2));
      const size_t cap = (size_t)(plan->lc.smem_optin - kDynSlack);
      if (smem > cap && nw == 16) {  // fewer warps, fewer counters
        nw = 8;
        smem = align16((size_t)nbk * nw * (wide ? 4 : 2));
      }
      if (smem > cap) {
        set_error("RIR too long for the per-channel sort: " + std::to_string(nbk) + " buckets need " +
                  std::to_string(smem) + " bytes of shared memory");
        return FRIR_ERANGE;
      }
      // short rows: the scatter goes to shared memory first (<= 36 KB) and the
      // sorted row leaves in coalesced stores (longer rows: the buffer costs
      // more residency than the scattered stores)
      const size_t stage = (size_t)b->max_rows * 8 + 16;  // (+16: the K > 0 path's aligned TMA cover)
      sa.stage_off = 0;
      // rows that fit nw * 32 * K registers: read once into registers (K > 0; K = 17
      // covers config 5's longest rows, I = 8192 -> 8193 rows, with 16 warps)
      const int kreg = (!sa.atom_ranks || wide || sw.seg || smem + stage > cap) ? 0
                       : b->max_rows <= nw * 32 * 8 ? 8 : b->max_rows <= nw * 32 * 17 ? 17 : 0;
      if (kreg || (sa.atom_ranks && b->max_rows <= kSortStageRows && smem + stage <= cap)) {
        sa.stage_off = (int)smem;
        smem += stage;
      }
      auto kern = kreg ? (nw == 16 ? (kreg == 8 ? sort_kernel<uint16_t, 16, false, 8> : sort_kernel<uint16_t, 16, false, 17>)
                                   : (kreg == 8 ? sort_kernel<uint16_t, 8, false, 8> : sort_kernel<uint16_t, 8, false, 17>))
                 : sw.seg ? (wide ? (nw == 16 ? sort_kernel<uint32_t, 16, true> : sort_kernel<uint32_t, 8, true>)
                                 : (nw == 16 ? sort_kernel<uint16_t, 16, true> : sort_kernel<uint16_t, 8, true>))
                         : (wide ? (nw == 16 ? sort_kernel<uint32_t, 16, false> : sort_kernel<uint32_t, 8, false>)
                                 : (nw == 16 ? sort_kernel<uint16_t, 16, false> : sort_kernel<uint16_t, 8, false>));
      kern<<<b->total_channels, nw * 32, smem, st>>>(sa);
      e = cudaGetLastError();
      if (e != cudaSuccess) { set_error(std::string("sort_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
    }
    TailArgs ta;  // K2b: tail corrections from the sorted rows
    ta.jobs = b->jobs; ta.chan_job = b->chan_job; ta.ws = ws; ta.sw = sw; ta.plan = plan->dev;
    ta.total_channels = b->total_channels;
    const size_t tsm = tail_smem(d);
    tail_kernel<false><<<(b->total_channels + kTailWarps - 1) / kTailWarps, kTailThreads, tsm, st>>>(ta);
    if (sw.seg) tail_kernel<true><<<b->total_channels, kTailThreads, tsm, st>>>(ta);  // long channels
    e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(std::string("tail_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  }

  if (stages & FRIR_STAGE_RENDER) {  // K3
    e = cudaMemsetAsync(ws.counter, 0, 2 * sizeof(int), st);  // [full / both, early pass]
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FRIR_ECUDA; }
    RenderArgs ra;
    ra.jobs = b->jobs; ra.chan_job = b->chan_job; ra.chan_order = b->chan_order;
    ra.total_channels = b->total_channels; ra.ws = ws; ra.sw = sw; ra.plan = plan->dev;
    ra.out_full = out_full; ra.out_early = out_early;
    ra.seg_max = batch_seg_max(b);
    const bool early = out_early != nullptr;
    const int nbk = table_blocks(d);
    const bool seg = ra.seg_max > 1;
    const long ch = b->total_channels;
    // batches of >= kSplitEarlyChannels channels without segmented ones
    // render the full variant and then the early variant in a second pass over
    // the early buckets only (identical bits to one full + early sweep; render
    // -4% on config 5, -6% config 3, -10% config 4; config 2's 6,144-channel
    // launches: +3% alone on one stream, but +2.2% throughput in the 2-deep
    // launch pipeline, where the early pass overlaps the other stream's work);
    // smaller batches (the per-call drop-in) sweep both variants at once
    const bool split = early && split_early(b);
    const bool both = early && !split;
    if (nbk == 1)
      e = both ? (seg ? launch_render<true, 1, true>(plan, ra, ch, st) : launch_render<true, 1, false>(plan, ra, ch, st))
               : (seg ? launch_render<false, 1, true>(plan, ra, ch, st) : launch_render<false, 1, false>(plan, ra, ch, st));
    else
      e = both ? (seg ? launch_render<true, 2, true>(plan, ra, ch, st) : launch_render<true, 2, false>(plan, ra, ch, st))
               : (seg ? launch_render<false, 2, true>(plan, ra, ch, st) : launch_render<false, 2, false>(plan, ra, ch, st));
    if (e == cudaSuccess && split)
      e = nbk == 1 ? launch_render<false, 1, false, true>(plan, ra, ch, st) : launch_render<false, 2, false, true>(plan, ra, ch, st);
    if (e != cudaSuccess) { set_error(std::string("render_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
    if (ra.seg_max > 1) {  // K4: seams of segmented channels
      SeamArgs sa;
      sa.jobs = b->jobs; sa.chan_job = b->chan_job; sa.ws = ws; sa.sw = sw; sa.plan = plan->dev;
      sa.out_full = out_full; sa.out_early = out_early; sa.total_channels = b->total_channels;
      seam_kernel<<<(b->total_channels + 7) / 8, 256, 0, st>>>(sa);
      e = cudaGetLastError();
      if (e != cudaSuccess) { set_error(std::string("seam_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
    }
  }
  return FRIR_OK;
}


static GeomArgs geom_args(const frir_plan* plan, const frir_batch* b, Workspace ws, int32_t* direct_index) {
  const frir_plan_desc& d = plan->dev.d;
  GeomArgs ga;
  ga.jobs = b->jobs; ga.mics = b->mics;
  ga.draw_dist = b->draw_dist; ga.draw_az = b->draw_az; ga.draw_el = b->draw_el; ga.draw_refl = b->draw_refl;
  ga.ws = ws; ga.direct_index = direct_index;
  ga.r_h = d.r_h; ga.t0 = d.t0;
  ga.rh_magic = (unsigned)((0x100000000ull + d.r_h - 1) / d.r_h);
  ga.rate = (double)d.r_h * d.sample_rate;
  return ga;
}

int launch_image_set(const frir_plan* plan, const frir_batch* b, double* dist, double* az, double* el,
                     double* ratio, double* refl, double* mic_dist, int with_refl, cudaStream_t st) {
  if (b->n_jobs == 0) return FRIR_OK;
  Workspace ws{};
  GeomArgs ga = geom_args(plan, b, ws, nullptr);
  ImageSetOut o{dist, az, el, ratio, refl, mic_dist, with_refl};
  const int maxg = (b->max_rows - 1 + 3) / 4;
  image_set_kernel<<<dim3(b->n_jobs, maxg > 0 ? (maxg + 127) / 128 : 1), 128, 0, st>>>(ga, o);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("image_set_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

int train_nonzeros(const double* train, int64_t ld, int32_t rows, int32_t L, int32_t sign, int32_t* counts,
                   cudaStream_t st) {
  if (rows <= 0) return FRIR_OK;
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int32_t) * rows, st);
  if (e == cudaSuccess) {
    train_count_kernel<<<rows, kTrainThreads, 0, st>>>(train, (long)ld, L, sign, counts);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) { set_error(std::string("train_count_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

int launch_simulate_train(const frir_plan* plan, const frir_batch* b, void* wsp, size_t ws_bytes,
                          const double* train, int64_t ld, int32_t sign, float* out_full, int32_t* direct_scratch,
                          cudaStream_t st) {
  if (ws_bytes < workspace_bytes(b)) {
    set_error("workspace too small: need " + std::to_string(workspace_bytes(b)) + " bytes");
    return FRIR_ENOMEM;
  }
  if (b->n_jobs == 0 || b->total_channels == 0) return FRIR_OK;
  const Workspace ws = carve(wsp, b);
  const GeomArgs ga = geom_args(plan, b, ws, direct_scratch);
  train_items_kernel<<<b->total_channels, kTrainThreads, 0, st>>>(train, (long)ld, sign, b->jobs, b->chan_job, ws,
                                                                   ga.r_h, ga.t0, ga.rh_magic);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("train_items_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return launch_simulate(plan, b, wsp, ws_bytes, out_full, nullptr, direct_scratch, st,
                         FRIR_STAGE_DELAY | FRIR_STAGE_RENDER);
}

}  // namespace frir
