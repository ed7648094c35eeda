// sm_100a kernels of the FRAM-RIR hot path.
//
//   K1 geom_kernel    per (job, 4 images): Philox draws (or oracle draws) ->
//                     image position + r^g in FP64          core.py:131-221
//   K2 delay_kernel   per channel (job, mic): FP64 distance -> integer delay q,
//                     FP32 gain, early flag, output-rate start/phase; block
//                     radix sort by 32-sample window          core.py:228-265
//   K3 render_kernel  persistent warps, one channel at a time: gather the
//                     composite decimation/low-pass tables into 32-sample
//                     windows (FP32), FP64 output-rate LP scan, exact tail
//                     correction, coalesced full + early stores
//                                                             resample.py:81-136
// No atomics touch sample values, so outputs are bit-reproducible.
#include <cub/block/block_radix_sort.cuh>

#include "frir_internal.h"
#include "frir_philox.cuh"

namespace frir {
namespace {

constexpr double kTwoPi = 6.283185307179586;       // 2.0 * np.pi
constexpr double kHalfPi = 1.5707963267948966;     // np.pi / 2.0
constexpr double kPi = 3.141592653589793;          // np.pi/2 - (-np.pi/2)

struct Workspace {
  double* px;
  double* py;
  double* pz;
  double* lg;
  int2* items;
  int* chan_q0;
  int* counter;
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

Workspace carve(void* base, const frir_batch* b) {
  char* p = (char*)base;
  Workspace w;
  size_t ni = (size_t)b->total_images;
  w.px = (double*)p; p += align_up(ni * 8);
  w.py = (double*)p; p += align_up(ni * 8);
  w.pz = (double*)p; p += align_up(ni * 8);
  w.lg = (double*)p; p += align_up(ni * 8);
  w.items = (int2*)p; p += align_up((size_t)b->total_items * 8);
  w.chan_q0 = (int*)p; p += align_up((size_t)b->total_channels * 4);
  w.counter = (int*)p;
  return w;
}

// ---------------------------------------------------------------- K1 geometry
// numpy operation order is kept with explicit _rn intrinsics (no FMA
// contraction): positions/distances feed the exact integer delays.
__device__ __forceinline__ void image_position(const frir_job& J, double dist, double az,
                                               double el, double* x, double* y, double* z) {
  // params.py:138-146 sph_to_cart; params.py:149-159 center + offset
  double ce = cos(el), se = sin(el), ca = cos(az), sa = sin(az);
  double dce = __dmul_rn(dist, ce);
  *x = __dadd_rn(J.center[0], __dmul_rn(dce, ca));
  *y = __dadd_rn(J.center[1], __dmul_rn(dce, sa));
  *z = __dadd_rn(J.center[2], __dmul_rn(dist, se));
}

__global__ void __launch_bounds__(128) geom_kernel(const frir_job* __restrict__ jobs,
                                                   const double* __restrict__ draw_dist,
                                                   const double* __restrict__ draw_az,
                                                   const double* __restrict__ draw_el,
                                                   const double* __restrict__ draw_refl,
                                                   Workspace ws) {
  const int j = blockIdx.x;
  const frir_job& J = jobs[j];
  const int I = J.n_images;
  const int g = blockIdx.y * blockDim.x + threadIdx.x;  // group of 4 images
  const int ngroups = (I + 3) / 4;
  if (g == 0) {  // row 0: direct path (core.py:169, params.py:156-159)
    double x, y, z;
    image_position(J, J.d0, J.az, J.el, &x, &y, &z);
    size_t o = (size_t)J.img_off;
    ws.px[o] = x; ws.py[o] = y; ws.pz[o] = z;
    ws.lg[o] = 1.0;  // r ** 0.0
  }
  if (g >= ngroups) return;
  const double c_max = __dmul_rn(J.c0, J.t60);
  double th[4], ph[4], dist[4], refl[4];
  const bool oracle = draw_dist != nullptr;
  if (oracle) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int i = 4 * g + k + 1;
      size_t o = (size_t)J.img_off + (i <= I ? i : 0);
      dist[k] = draw_dist[o]; th[k] = draw_az[o]; ph[k] = draw_el[o]; refl[k] = draw_refl[o];
    }
  } else {
    // stage-0 stream: theta words [0, I), phi words [I, 2I), u words [2I, 3I)
    const uint64_t k0[2] = {J.key[0], J.key[1]};
    const uint64_t k1[2] = {J.key[2], J.key[3]};
    const uint64_t w0 = 4ull * g;
    u64x4 bt = philox4x64_10((uint64_t)g + 1, 0, 0, 0, k0[0], k0[1]);
    uint64_t wp = (uint64_t)I + w0, wu = 2ull * I + w0;
    u64x4 bp0 = philox4x64_10(wp / 4 + 1, 0, 0, 0, k0[0], k0[1]);
    u64x4 bp1 = bp0;
    if (wp & 3) bp1 = philox4x64_10(wp / 4 + 2, 0, 0, 0, k0[0], k0[1]);
    u64x4 bu0 = philox4x64_10(wu / 4 + 1, 0, 0, 0, k0[0], k0[1]);
    u64x4 bu1 = bu0;
    if (wu & 3) bu1 = philox4x64_10(wu / 4 + 2, 0, 0, 0, k0[0], k0[1]);
    u64x4 bq = philox4x64_10((uint64_t)g + 1, 0, 0, 0, k1[0], k1[1]);
    const double alpha = J.alpha, beta = J.beta;
    const double kres = __ddiv_rn(alpha, __dsub_rn(beta, alpha));
    const double mr1 = __dsub_rn(__ddiv_rn(c_max, J.d0), 1.0);
    const double rrm1 = __dsub_rn(J.rr_max, 1.0);
    const double prange = __dsub_rn(J.perturb_hi, J.perturb_lo);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int ip = (int)((wp & 3) + k), iu = (int)((wu & 3) + k);
      uint64_t wpk = ip < 4 ? bp0.v[ip] : bp1.v[ip - 4];
      uint64_t wuk = iu < 4 ? bu0.v[iu] : bu1.v[iu - 4];
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
      double gg = __dadd_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(qq, qq), rrm1)),
                            __dmul_rn(pr, pow(dr, J.tau)));
      gg = fmin(fmax(gg, 1.0), J.rr_max);
      dist[k] = dd;
      refl[k] = gg;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int i = 4 * g + k + 1;
    if (i > I) break;
    double x, y, z;
    image_position(J, dist[k], th[k], ph[k], &x, &y, &z);
    size_t o = (size_t)J.img_off + i;
    ws.px[o] = x; ws.py[o] = y; ws.pz[o] = z;
    ws.lg[o] = pow(J.r, refl[k]);  // core.py:246 r ** g
  }
}

// ---------------------------------------------------------------- K2 delays + sort
struct DelayArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  const double* mics;
  Workspace ws;
  int32_t* direct_index;
  frir_plan_desc d;
  int end_bit;
};

__device__ __forceinline__ int ceil_div_i(int a, int b) {  // b > 0, any sign of a
  return a >= 0 ? (a + b - 1) / b : -((-a) / b);
}

template <int THREADS, int IPT>
__global__ void __launch_bounds__(THREADS) delay_kernel(DelayArgs A) {
  using Sort = cub::BlockRadixSort<uint32_t, THREADS, IPT, uint2>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typename Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(smem_raw);
  __shared__ int s_q0;

  const int c = blockIdx.x;
  const int j = A.chan_job[c];
  const frir_job& J = A.jobs[j];
  const int m = c - J.chan_off;
  const int rows = J.n_images + 1;
  const double* mic = A.mics + 3 * (size_t)(J.mic_off + m);
  const double mx = mic[0], my = mic[1], mz = mic[2];
  const double rate = (double)A.d.r_h * (double)A.d.sample_rate;
  const int lo = (6 * A.d.r_h * A.d.sample_rate + 999) / 1000;   // core.py:257
  const int hi = (50 * A.d.r_h * A.d.sample_rate + 999) / 1000;  // core.py:258
  const int r_h = A.d.r_h, t0 = A.d.t0;

  int q[IPT];
  float a[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int r = threadIdx.x * IPT + k;
    q[k] = 0;
    a[k] = 0.f;
    if (r < rows) {
      size_t o = (size_t)J.img_off + r;
      // params.py:162-171 distances_to_mics; core.py:242-246
      double dx = __dsub_rn(A.ws.px[o], mx), dy = __dsub_rn(A.ws.py[o], my),
             dz = __dsub_rn(A.ws.pz[o], mz);
      double D = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      double qd = ceil(__dmul_rn(__ddiv_rn(D, J.c0), rate));
      int qi = qd >= (double)(J.L - 1) ? J.L - 1 : (int)qd;
      q[k] = qi;
      a[k] = (float)__ddiv_rn(A.ws.lg[o], D);
      if (r == 0) s_q0 = qi;
    }
  }
  __syncthreads();
  const int q0 = s_q0;
  if (threadIdx.x == 0) {
    A.ws.chan_q0[c] = q0;
    // resample.py:115-119 direct = clip(round(q0 / r_h), 0, n2 - 1), half-even
    double dv = rint(__ddiv_rn((double)q0, (double)r_h));
    int di = (int)dv;
    di = di < 0 ? 0 : (di > J.n2 - 1 ? J.n2 - 1 : di);
    A.direct_index[c] = di;
  }
  uint32_t key[IPT];
  uint2 val[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int r = threadIdx.x * IPT + k;
    if (r < rows) {
      int rel = q[k] - q0;
      bool early = rel >= -lo && rel <= hi;  // core.py:259-264
      int s = ceil_div_i(q[k] + t0, r_h);
      uint32_t spb = (uint32_t)(s + kExt + kSpBias);  // biased output-rate start, >= 0
      uint32_t off = (uint32_t)(r_h * s - q[k] - t0);  // phase, < r_h <= 1023
      key[k] = spb >> 5;
      // early flag rides in the sign of the (positive) gain
      val[k] = make_uint2(spb | (off << 20), __float_as_uint(early ? -a[k] : a[k]));
    } else {
      key[k] = 0xffffffffu;
      val[k] = make_uint2(0u, 0u);
    }
  }
  __syncthreads();  // s_q0 read before TempStorage reuse (distinct storage, kept for clarity)
  Sort(tmp).SortBlockedToStriped(key, val, 0, A.end_bit);
  int2* out = A.ws.items + J.item_off + (size_t)m * rows;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int r = k * THREADS + threadIdx.x;
    if (r < rows) out[r] = make_int2((int)val[k].x, (int)val[k].y);
  }
}

// ---------------------------------------------------------------- K3 render
struct RenderArgs {
  const frir_job* jobs;
  const int32_t* chan_job;
  const int32_t* chan_order;
  int total_channels;
  Workspace ws;
  DevPlan plan;
  float* out_full;
  float* out_early;
};

constexpr int kRenderThreads = 256;
constexpr int kWarps = kRenderThreads / 32;
constexpr int kPad = kChunk + 1;
constexpr int kWarpBuf = 32 * kPad;  // doubles per variant per warp

__device__ __forceinline__ int pidx(int o) { return (o / kChunk) * kPad + (o % kChunk); }

struct Cplx {
  double re, im;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }

// One variant's LP scan over a tile held (as doubles) in buf; on return buf
// holds LP (FP64) for the tile and (s0, s1) the carried state (LP[last], LP[last-1]).
__device__ __forceinline__ void lp_scan_tile(double* buf, const double* scan, double c1, double c2,
                                             double& s0, double& s1, int lane) {
  double l[kChunk];
  const int base = lane * kPad;
#pragma unroll
  for (int k = 0; k < kChunk; ++k) {
    double x = buf[base + k];
    double p1 = k >= 1 ? l[k - 1] : 0.0, p2 = k >= 2 ? l[k - 2] : 0.0;
    l[k] = fma(c1, p1, fma(c2, p2, x));
  }
  // affine combine over lanes: E_L = sum_{i<=L} M^{C(L-i)} e_i
  double e0 = l[kChunk - 1], e1 = l[kChunk - 2];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int dd = 1 << s;
    double u0 = shfl_up_d(e0, dd), u1 = shfl_up_d(e1, dd);
    if (lane >= dd) {
      const double* Mp = scan + 4 * s;
      e0 = fma(Mp[0], u0, fma(Mp[1], u1, e0));
      e1 = fma(Mp[2], u0, fma(Mp[3], u1, e1));
    }
  }
  double x0 = shfl_up_d(e0, 1), x1 = shfl_up_d(e1, 1);
  if (lane == 0) { x0 = 0.0; x1 = 0.0; }
  const double* Ms = scan + 20 + 4 * lane;  // M^{C*lane}
  double t0 = fma(Ms[0], s0, fma(Ms[1], s1, x0));
  double t1 = fma(Ms[2], s0, fma(Ms[3], s1, x1));
  const double* fr = scan + 20 + 128;
#pragma unroll
  for (int k = 0; k < kChunk; ++k) {
    double v = l[k] + fma(fr[2 * k], t0, fr[2 * k + 1] * t1);
    l[k] = v;
    buf[base + k] = v;
  }
  s0 = shfl_d(l[kChunk - 1], 31);
  s1 = shfl_d(l[kChunk - 2], 31);
}

// Accumulate window w (outputs n' in [32w, 32w + 32), one per lane) from the
// bucket-sorted items.  Items are staged 32 at a time through per-warp shared
// memory and read back as broadcasts; each candidate costs one table LDS.64
// and two (four in early windows) FFMAs per lane.  Returns the new lower item
// bound for window w + 1.
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
  // one item: x = biased start | phase << 20, ae = +-gain (sign = early flag).
  // Lane L takes taps k0 + 32 j, k0 = (L - start) mod 32, of the item's phase
  // row; they land in windows j (k0 <= L) or j + 1 (k0 > L).  Selects instead
  // of branches keep the warp converged; only the early test branches, and
  // it is warp-uniform.
  template <bool EW>
  __device__ __forceinline__ void add(int x, float ae, int lane, const float2* __restrict__ s_comp) {
    const int k0 = (lane - x) & 31;
    const int idx = ((((unsigned)x >> 20) & 0x3FF) << (5 + (NBK - 1))) | k0;
    const bool hi = k0 > lane;
    const float a = fabsf(ae);
    const float alo = hi ? 0.f : a, ahi = hi ? a : 0.f;
#pragma unroll
    for (int j = 0; j < NBK; ++j) {
      const float2 t = s_comp[idx + 32 * j];
      dF[j] = fmaf(alo, t.x, dF[j]);
      wF[j] = fmaf(alo, t.y, wF[j]);
      dF[j + 1] = fmaf(ahi, t.x, dF[j + 1]);
      wF[j + 1] = fmaf(ahi, t.y, wF[j + 1]);
      if (EW && ae < 0.f) {
        dE[j] = fmaf(alo, t.x, dE[j]);
        wE[j] = fmaf(alo, t.y, wE[j]);
        dE[j + 1] = fmaf(ahi, t.x, dE[j + 1]);
        wE[j + 1] = fmaf(ahi, t.y, wE[j + 1]);
      }
    }
  }
};

template <bool EARLY, int NBK>
__global__ void __launch_bounds__(kRenderThreads) render_kernel(RenderArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const frir_plan_desc& d = A.plan.d;
  constexpr int kRow = 32 * NBK;
  const int ncomp = d.r_h * kRow;
  float2* s_comp = reinterpret_cast<float2*>(smem);
  double* s_scan = reinterpret_cast<double*>(smem + (size_t)ncomp * 8);
  double* s_warp = s_scan + kScanDoubles;  // per warp: W buffers (F[, E])
  float* s_dbuf = reinterpret_cast<float*>(s_warp + (size_t)kWarps * (EARLY ? 2 : 1) * kWarpBuf);
  int2* s_items = reinterpret_cast<int2*>(s_dbuf + (size_t)kWarps * (EARLY ? 2 : 1) * kTile);
  for (int i = threadIdx.x; i < ncomp; i += blockDim.x) s_comp[i] = A.plan.comp[i];
  for (int i = threadIdx.x; i < kScanDoubles; i += blockDim.x) s_scan[i] = A.plan.scan[i];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* bufF = s_warp + (size_t)warp * (EARLY ? 2 : 1) * kWarpBuf;
  double* bufE = bufF + kWarpBuf;
  float* dbF = s_dbuf + (size_t)warp * (EARLY ? 2 : 1) * kTile;
  float* dbE = dbF + kTile;
  int2* s_it = s_items + 32 * warp;
  const double c1 = A.plan.lp[0], c2 = A.plan.lp[1];
  const Cplx v0a = {A.plan.lp[2], A.plan.lp[3]}, v0b = {A.plan.lp[4], A.plan.lp[5]};
  const int sup = d.sup, r_h = d.r_h, up = d.up, down = d.down, half1 = d.half1;
  (void)sup;

  for (;;) {
    int ci = 0;
    if (lane == 0) ci = atomicAdd(A.ws.counter, 1);
    ci = __shfl_sync(0xffffffffu, ci, 0);
    if (ci >= A.total_channels) break;
    const int c = A.chan_order ? A.chan_order[ci] : ci;
    const int j = A.chan_job[c];
    const frir_job& J = A.jobs[j];
    const int m = c - J.chan_off;
    const int rows = J.n_images + 1;
    const int n1 = J.n1, n2 = J.n2;
    const int2* items = A.ws.items + J.item_off + (size_t)m * rows;
    float* outF = A.out_full + J.out_off + (size_t)m * J.out_stride;
    float* outE = EARLY ? A.out_early + J.out_off + (size_t)m * J.out_stride : nullptr;

    // ---- tail: HP state at n1 (modal sum) + taps past n1 (resample.py:107-113 truncation)
    Cplx zF = {0.0, 0.0}, zE = {0.0, 0.0};
    double xtF[2] = {0.0, 0.0}, xtE[2] = {0.0, 0.0};
    {
      const long kthr = (long)n1 - d.horizon;  // need k_hi >= kthr
      for (int base = rows; base > 0; base -= 32) {
        const int r = base - 32 + lane;
        int q = 0, early = 0, valid = 0;
        float a = 0.f;
        long khi = -1;
        if (r >= 0) {
          int2 it = items[r];
          int sp = (it.x & 0xFFFFF) - kSpBias;
          int phi = ((unsigned)it.x >> 20) & 0x3FF;
          float ae = __int_as_float(it.y);
          early = ae < 0.f;
          a = fabsf(ae);
          q = r_h * (sp - kExt) - d.t0 - phi;
          long e = (long)up * q + half1;
          khi = e >= 0 ? e / down : -((-e + down - 1) / down);
          valid = khi >= kthr;
          // bound for "everything below is past the horizon": max q of this bucket
          int bucket = (sp > 0 ? sp : 0) >> 5;
          long qmax = (long)r_h * (32L * bucket + 31 - kExt) - d.t0;
          long kmax = ((long)up * qmax + half1) / down;
          if (kmax >= kthr) valid |= 2;
        }
        if (valid & 1) {
          long e = (long)up * q + half1;
          if (khi < n1) {
            int rho = (int)(e - (long)down * khi);
            long mm = (long)n1 - 1 - khi;
            Cplx pm = {A.plan.ppow[2 * mm], A.plan.ppow[2 * mm + 1]};
            Cplx zr = {A.plan.zphase[2 * rho], A.plan.zphase[2 * rho + 1]};
            Cplx t = cmul(pm, zr);
            zF.re += a * t.re; zF.im += a * t.im;
            if (EARLY && early) { zE.re += a * t.re; zE.im += a * t.im; }
          } else {
            long klo = (long)up * q - half1;
            klo = klo >= 0 ? (klo + down - 1) / down : -((-klo) / down);
            for (long k = klo; k < n1; ++k) {
              long mm = (long)n1 - 1 - k;
              if (mm >= d.horizon) continue;
              double cc = (double)a * A.plan.h1up[(long)down * k + half1 - (long)up * q];
              double pr = A.plan.ppow[2 * mm], pi = A.plan.ppow[2 * mm + 1];
              zF.re += cc * pr; zF.im += cc * pi;
              if (EARLY && early) { zE.re += cc * pr; zE.im += cc * pi; }
            }
          }
        }
        // taps past n1, one straddler at a time (deterministic lane order)
        unsigned strad = __ballot_sync(0xffffffffu, (valid & 1) && khi >= n1);
        while (strad) {
          int src = __ffs(strad) - 1;
          strad &= strad - 1;
          int qs = __shfl_sync(0xffffffffu, q, src);
          float as = __shfl_sync(0xffffffffu, a, src);
          int es = __shfl_sync(0xffffffffu, early, src);
          long khs = (long)((long)up * qs + half1) / down;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int l = lane + 32 * h;
            long k = (long)n1 + l;
            if (l < d.lt_max && k <= khs) {
              long idx = (long)down * k + half1 - (long)up * qs;
              if (idx >= 0 && idx < d.len1) {
                double cc = (double)as * A.plan.h1up[idx];
                xtF[h] += cc;
                if (EARLY && es) xtE[h] += cc;
              }
            }
          }
        }
        if (!__any_sync(0xffffffffu, valid & 2)) break;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      zF.re += __shfl_xor_sync(0xffffffffu, zF.re, o);
      zF.im += __shfl_xor_sync(0xffffffffu, zF.im, o);
      if (EARLY) {
        zE.re += __shfl_xor_sync(0xffffffffu, zE.re, o);
        zE.im += __shfl_xor_sync(0xffffffffu, zE.im, o);
      }
    }
    // state s = 2 Re(v0 zeta); corrections for outputs n >= n_c
    const int n_c = n1 - d.half2 > 0 ? (n1 - d.half2 + d.r_l - 1) / d.r_l : 0;
    double corrF = 0.0, corrE = 0.0;
    {
      Cplx ta = cmul(v0a, zF), tb = cmul(v0b, zF);
      double sF0 = 2.0 * ta.re, sF1 = 2.0 * tb.re;
      double sE0 = 0.0, sE1 = 0.0;
      if (EARLY) {
        Cplx ea = cmul(v0a, zE), eb = cmul(v0b, zE);
        sE0 = 2.0 * ea.re;
        sE1 = 2.0 * eb.re;
      }
      const int n = n_c + lane;
      const int e = d.r_l * n + d.half2 - n1;
      const bool act = n < n2 && e >= 0 && e < d.half2;
      if (act) {
        corrF = A.plan.kappa[2 * e] * sF0 + A.plan.kappa[2 * e + 1] * sF1;
        if (EARLY) corrE = A.plan.kappa[2 * e] * sE0 + A.plan.kappa[2 * e + 1] * sE1;
      }
      for (int l = 0; l < d.lt_max; ++l) {
        double xf = shfl_d(xtF[l >> 5], l & 31);
        double xe = EARLY ? shfl_d(xtE[l >> 5], l & 31) : 0.0;
        if (act && l <= e) {
          double uu = A.plan.u[e - l];
          corrF += xf * uu;
          if (EARLY) corrE += xe * uu;
        }
      }
    }

    // ---- ordered sweep: windows w = -2 .. nwin-1 over n' = n + 10
    const int nwin = (n2 + kExt + kWin - 1) / kWin;
    Channel<EARLY, NBK> ch;
    ch.clear();
    double sF0 = 0.0, sF1 = 0.0, sE0 = 0.0, sE1 = 0.0;
    int w = -2;     // window that the front accumulators (index 0) hold
    int slot = 0;   // next tile slot
    auto emit = [&]() {
      if (w >= 0) {
        dbF[slot * kWin + lane] = ch.dF[0];
        bufF[pidx(slot * kWin + lane)] = (double)ch.wF[0];
        if (EARLY) {
          dbE[slot * kWin + lane] = ch.dE[0];
          bufE[pidx(slot * kWin + lane)] = (double)ch.wE[0];
        }
        ++slot;
        if (slot == kTileWin || w == nwin - 1) {
          for (int s2 = slot; s2 < kTileWin; ++s2) {  // pad a partial last tile
            bufF[pidx(s2 * kWin + lane)] = 0.0;
            if (EARLY) bufE[pidx(s2 * kWin + lane)] = 0.0;
          }
          __syncwarp();
          lp_scan_tile(bufF, s_scan, c1, c2, sF0, sF1, lane);
          if (EARLY) lp_scan_tile(bufE, s_scan, c1, c2, sE0, sE1, lane);
          __syncwarp();
          const int w0 = w - slot + 1;
          for (int wi = 0; wi < slot; ++wi) {
            const int n = (w0 + wi) * kWin + lane - kExt;
            const bool tailwin = (w0 + wi) * kWin - kExt + 31 >= n_c;  // warp-uniform
            double cf = 0.0, ce = 0.0;
            if (tailwin) {
              int src = n - n_c;
              src = src < 0 ? 0 : (src > 31 ? 31 : src);
              cf = shfl_d(corrF, src);
              if (EARLY) ce = shfl_d(corrE, src);
            }
            if (n >= 0 && n < n2) {
              const bool fix = n >= n_c;
              const double yf = (double)dbF[wi * kWin + lane] - bufF[pidx(wi * kWin + lane)] - (fix ? cf : 0.0);
              outF[n] = (float)yf;
              if (EARLY) {
                const double ye = (double)dbE[wi * kWin + lane] - bufE[pidx(wi * kWin + lane)] - (fix ? ce : 0.0);
                outE[n] = (float)ye;
              }
            }
          }
          __syncwarp();
          slot = 0;
        }
      }
      ch.shift();
      ++w;
    };
    for (int p = 0; p < rows; p += 32) {
      const int pi = p + lane;
      const int2 mine = pi < rows ? items[pi] : make_int2(0xFFFFF, 0);  // sentinel: last bucket
      __syncwarp();
      s_it[lane] = mine;
      __syncwarp();
      const int bk = (mine.x & 0xFFFFF) >> 5;
      const int cnt = min(32, rows - p);
      const unsigned emask = EARLY ? __ballot_sync(0xffffffffu, pi < rows && mine.y < 0) : 0u;
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
            ch.template add<true>(it.x, __int_as_float(it.y), lane, s_comp);
          }
        } else {
#pragma unroll 4
          for (; jj < end; ++jj) {
            const int2 it = s_it[jj];
            ch.template add<false>(it.x, __int_as_float(it.y), lane, s_comp);
          }
        }
      }
    }
    while (w < nwin) emit();
  }
}

}  // namespace

// ---------------------------------------------------------------- host launcher
size_t workspace_bytes(const frir_batch* b) {
  size_t ni = (size_t)b->total_images;
  return 4 * align_up(ni * 8) + align_up((size_t)b->total_items * 8) +
         align_up((size_t)b->total_channels * 4) + 256;
}

static int table_blocks(const frir_plan_desc& d) { return (d.sup + 31) / 32; }

static size_t render_smem(const frir_plan_desc& d, bool early) {
  const int v = early ? 2 : 1;
  return (size_t)d.r_h * 32 * table_blocks(d) * 8 + kScanDoubles * 8 +
         (size_t)kWarps * v * kWarpBuf * 8 + (size_t)kWarps * v * kTile * 4 + (size_t)kWarps * 32 * 8;
}

template <bool EARLY, int NBK>
static cudaError_t launch_render(const RenderArgs& ra, const frir_plan_desc& d, long channels,
                                 cudaStream_t st) {
  size_t smem = render_smem(d, EARLY);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(render_kernel<EARLY, NBK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, render_kernel<EARLY, NBK>, kRenderThreads, smem);
  if (per_sm < 1) per_sm = 1;
  long want = (channels + kWarps - 1) / kWarps;
  int grid = (int)std::min<long>((long)sms * per_sm, want);
  render_kernel<EARLY, NBK><<<grid, kRenderThreads, smem, st>>>(ra);
  return cudaGetLastError();
}

template <int T, int IPT>
static cudaError_t launch_delay(const DelayArgs& a, int grid, cudaStream_t st) {
  using Sort = cub::BlockRadixSort<uint32_t, T, IPT, uint2>;
  size_t smem = sizeof(typename Sort::TempStorage);
  cudaError_t e = cudaFuncSetAttribute(delay_kernel<T, IPT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  delay_kernel<T, IPT><<<grid, T, smem, st>>>(a);
  return cudaGetLastError();
}

int launches(const frir_batch* b, int early) {
  (void)b;
  (void)early;
  return 3;  // geom, delay, render (plus one memset of the work counter)
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
  cudaError_t e = cudaSuccess;

  if (stages & FRIR_STAGE_GEOM) {  // K1
  int maxg = (b->max_rows - 1 + 3) / 4;
  dim3 g1(b->n_jobs, (maxg + 127) / 128 > 0 ? (maxg + 127) / 128 : 1);
  geom_kernel<<<g1, 128, 0, st>>>(b->jobs, b->draw_dist, b->draw_az, b->draw_el, b->draw_refl, ws);
  e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("geom_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  }

  if (stages & FRIR_STAGE_DELAY) {  // K2
  DelayArgs da;
  da.jobs = b->jobs; da.chan_job = b->chan_job; da.mics = b->mics; da.ws = ws;
  da.direct_index = direct_index; da.d = d;
  int maxb = b->max_windows + 2;
  int bits = 1;
  while ((1 << bits) <= maxb + 1) ++bits;
  da.end_bit = bits;
  int rows = b->max_rows, grid = b->total_channels;
  if (rows <= 1024) e = launch_delay<128, 8>(da, grid, st);
  else if (rows <= 2048) e = launch_delay<256, 8>(da, grid, st);
  else if (rows <= 4352) e = launch_delay<256, 17>(da, grid, st);
  else if (rows <= 8704) e = launch_delay<512, 17>(da, grid, st);
  else e = launch_delay<1024, 17>(da, grid, st);
  if (e != cudaSuccess) { set_error(std::string("delay_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  }

  if (stages & FRIR_STAGE_RENDER) {  // K3
  e = cudaMemsetAsync(ws.counter, 0, sizeof(int), st);
  if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FRIR_ECUDA; }
  RenderArgs ra;
  ra.jobs = b->jobs; ra.chan_job = b->chan_job; ra.chan_order = b->chan_order;
  ra.total_channels = b->total_channels; ra.ws = ws; ra.plan = plan->dev;
  ra.out_full = out_full; ra.out_early = out_early;
  const bool early = out_early != nullptr;
  const int nbk = table_blocks(d);
  if (nbk == 1) e = early ? launch_render<true, 1>(ra, d, b->total_channels, st)
                          : launch_render<false, 1>(ra, d, b->total_channels, st);
  else e = early ? launch_render<true, 2>(ra, d, b->total_channels, st)
                 : launch_render<false, 2>(ra, d, b->total_channels, st);
  if (e != cudaSuccess) { set_error(std::string("render_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  }
  return FRIR_OK;
}

}  // namespace frir
