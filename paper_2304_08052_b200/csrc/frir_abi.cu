// C-ABI entry points (include/frir.h).  Host bookkeeping only; the math of
// the hot path is in frir_kernels.cu and frir_design.cpp.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "frir_internal.h"
#include "frir_philox.cuh"

namespace frir {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static std::string fmt(const char* f, double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, f, v);
  return buf;
}

// 2x2 helpers for the LP scan constants.
struct M2 {
  double a, b, c, d;
};
static M2 mul(const M2& x, const M2& y) {
  return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c,
          x.c * y.b + x.d * y.d};
}
static M2 mpow(M2 m, int n) {
  M2 r{1, 0, 0, 1};
  for (int i = 0; i < n; ++i) r = mul(r, m);
  return r;
}

static std::vector<double> scan_constants(double c1, double c2) {
  std::vector<double> s(kScanDoubles, 0.0);
  M2 M{c1, c2, 1.0, 0.0};
  auto put = [&](int at, const M2& p) { s[at] = p.a; s[at + 1] = p.b; s[at + 2] = p.c; s[at + 3] = p.d; };
  for (int k = 0; k < 5; ++k) put(kScanKS + 4 * k, mpow(M, kChunk << k));
  for (int l = 0; l < 32; ++l) put(kScanStart + 4 * l, mpow(M, kChunk * l));
  M2 p{1, 0, 0, 1};
  for (int k = 0; k < kTile; ++k) {
    p = mul(p, M);  // M^(k+1)
    s[kScanFree + 2 * k] = p.a;
    s[kScanFree + 2 * k + 1] = p.b;
  }
  put(kScanTileM, p);  // M^kTile
  return s;
}

template <typename T>
static cudaError_t upload(T** dst, const T* src, size_t n) {
  cudaError_t e = cudaMalloc((void**)dst, n * sizeof(T) + 16);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace frir

using namespace frir;

extern "C" {

const char* frir_last_error(void) { return g_err.c_str(); }
int32_t frir_abi_version(void) { return FRIR_ABI_VERSION; }

int32_t frir_debug_status(void) { return check_line(); }

int64_t frir_struct_size(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(frir_job);
    case 1: return (int64_t)sizeof(frir_batch);
    case 2: return (int64_t)sizeof(frir_plan_desc);
    default: return -1;
  }
}

int frir_design_describe(int32_t fs, frir_plan_desc* out) {
  if (!out) { set_error("null output"); return FRIR_EINVAL; }
  Design D;
  std::string err;
  if (!design(fs, &D, &err)) { set_error(err); return FRIR_EINVAL; }
  *out = D.d;
  return FRIR_OK;
}

int frir_design_table(int32_t fs, int32_t which, double* out, int64_t cap, int64_t* n_out) {
  Design D;
  std::string err;
  if (!design(fs, &D, &err)) { set_error(err); return FRIR_EINVAL; }
  std::vector<double> v;
  switch (which) {
    case FRIR_TAB_H1: v = D.h1; break;
    case FRIR_TAB_H2: v = D.h2; break;
    case FRIR_TAB_SOS: v.assign(D.d.sos, D.d.sos + 6); break;
    case FRIR_TAB_COMP_D: v = D.comp_d; break;
    case FRIR_TAB_COMP_W: v = D.comp_w; break;
    case FRIR_TAB_KAPPA: v = D.kappa; break;
    case FRIR_TAB_U: v = D.u; break;
    case FRIR_TAB_ZPHASE: v = D.zphase; break;
    case FRIR_TAB_PPOW: v = D.ppow; break;
    case FRIR_TAB_LPCOEF: v = D.lpcoef; break;
    case FRIR_TAB_GW: v = D.gw; break;
    default: set_error("unknown table id"); return FRIR_EINVAL;
  }
  if (n_out) *n_out = (int64_t)v.size();
  if (out) {
    if (cap < (int64_t)v.size()) { set_error("table buffer too small"); return FRIR_ENOMEM; }
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  }
  return FRIR_OK;
}

int frir_philox_doubles(uint64_t seed, uint64_t k, uint64_t stage, uint64_t first, int64_t n,
                        double* out) {
  if (n < 0 || (n > 0 && !out)) { set_error("bad output buffer"); return FRIR_EINVAL; }
  uint64_t key[2];
  seed_keys(seed, k, stage, key);
  for (int64_t i = 0; i < n; ++i) out[i] = u64_to_unit(stream_word(key, first + (uint64_t)i));
  return FRIR_OK;
}

int frir_plan_create(int32_t fs, frir_plan** out) {
  if (!out) { set_error("null plan output"); return FRIR_EINVAL; }
  *out = nullptr;
  frir_plan* p = new frir_plan();
  std::string err;
  if (!design(fs, &p->design, &err)) { delete p; set_error(err); return FRIR_EINVAL; }
  if (p->design.d.r_h > 1023 || p->design.d.sup > 64 || p->design.d.lt_max > kLtMax) {
    delete p;
    set_error("sample_rate " + std::to_string(fs) + " is outside the supported range (r_h <= 1023, <= 64 taps)");
    return FRIR_ERANGE;
  }
  const Design& D = p->design;
  DevPlan& dv = p->dev;
  std::memset(&dv, 0, sizeof dv);
  dv.d = D.d;
  cudaGetDevice(&p->device);
  // phase-major rows of ceil(sup / 32) blocks; block j holds taps 32 j .. 32 j + 31
  // TWICE (64 entries, zeros past sup) so the render kernel indexes it without
  // wrapping (csrc/frir_kernels.cu Channel::add)
  const int nbk = (D.d.sup + 31) / 32, row = 64 * nbk;
  std::vector<float2> comp((size_t)D.d.r_h * row, make_float2(0.f, 0.f));
  for (int ph = 0; ph < D.d.r_h; ++ph)
    for (int j = 0; j < nbk; ++j)
      for (int e = 0; e < 64; ++e) {
        int k = 32 * j + (e & 31);
        if (k >= D.d.sup) continue;
        size_t t = (size_t)ph + (size_t)D.d.r_h * k;  // t - t0
        comp[(size_t)ph * row + 64 * j + e] = make_float2((float)D.comp_d[t], (float)D.comp_w[t]);
      }
  std::vector<double> scan = scan_constants(D.d.c1, D.d.c2);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&dv.comp, comp.data(), comp.size());
  if (e == cudaSuccess) e = upload(&dv.h1up, D.h1up.data(), D.h1up.size());
  if (e == cudaSuccess) e = upload(&dv.h2, D.h2.data(), D.h2.size());
  if (e == cudaSuccess) e = upload(&dv.gw, D.gw.data(), D.gw.size());
  if (e == cudaSuccess) e = upload(&dv.ppow, D.ppow.data(), D.ppow.size());
  if (e == cudaSuccess) e = upload(&dv.ppow_lo, D.ppow_lo.data(), D.ppow_lo.size());
  if (e == cudaSuccess) e = upload(&dv.ppow_hi, D.ppow_hi.data(), D.ppow_hi.size());
  if (e == cudaSuccess) e = upload(&dv.zphase, D.zphase.data(), D.zphase.size());
  if (e == cudaSuccess) e = upload(&dv.kappa, D.kappa.data(), D.kappa.size());
  if (e == cudaSuccess) e = upload(&dv.u, D.u.data(), D.u.size());
  if (e == cudaSuccess) e = upload(&dv.scan, scan.data(), scan.size());
  for (int i = 0; i < 6; ++i) dv.lp[i] = D.lpcoef[i];
  for (int i = 0; i < 20; ++i) dv.ks[i] = scan[kScanKS + i];
  for (int i = 0; i < 4; ++i) dv.mc[i] = scan[kScanStart + 4 + i];  // M^(C * 1)
  for (int i = 0; i < 2 * kChunk; ++i) dv.fr0[i] = scan[kScanFree + i];
  for (int i = 0; i < 4; ++i) dv.mt[i] = scan[kScanTileM + i];
  if (e == cudaSuccess) e = init_launch_cache(p);
  if (e == cudaSuccess && p->lc.render_per_sm[0][(D.d.sup + 31) / 32 - 1][0] < 1) {
    frir_plan_destroy(p);
    set_error("sample_rate " + std::to_string(fs) + ": the render kernel's filter tables exceed the device's shared memory");
    return FRIR_ERANGE;
  }
  if (e != cudaSuccess) {
    set_error(std::string("plan upload: ") + cudaGetErrorString(e));
    frir_plan_destroy(p);
    return FRIR_ECUDA;
  }
  *out = p;
  return FRIR_OK;
}

int frir_plan_describe(const frir_plan* p, frir_plan_desc* out) {
  if (!p || !out) { set_error("null argument"); return FRIR_EINVAL; }
  *out = p->design.d;
  return FRIR_OK;
}

int frir_plan_destroy(frir_plan* p) {
  if (!p) return FRIR_OK;
  DevPlan& dv = p->dev;
  cudaFree(dv.comp); cudaFree(dv.h1up); cudaFree(dv.ppow); cudaFree(dv.zphase);
  cudaFree(dv.ppow_lo); cudaFree(dv.ppow_hi); cudaFree(dv.h2); cudaFree(dv.gw);
  cudaFree(dv.kappa); cudaFree(dv.u); cudaFree(dv.scan);
  delete p;
  return FRIR_OK;
}

static int64_t ceil_div64(int64_t a, int64_t b) { return a / b + (a % b != 0); }

int frir_jobs_prepare(int32_t sample_rate, frir_job* jobs, int32_t n_jobs, int32_t padded,
                      frir_batch* batch, int32_t* chan_job, int32_t* chan_order) {
  if (!batch || (n_jobs > 0 && !jobs) || n_jobs < 0) {
    set_error("null argument");
    return FRIR_EINVAL;
  }
  frir_plan_desc d;
  {
    std::string err;
    if (!rate_constants(sample_rate, &d, &err)) { set_error(err); return FRIR_EINVAL; }
  }
  const int64_t rate = (int64_t)d.r_h * d.sample_rate;
  int64_t img = 0, item = 0, out = 0;
  int32_t chan = 0, max_rows = 0, max_n2 = 0;
  for (int32_t j = 0; j < n_jobs; ++j) {
    frir_job& J = jobs[j];
    std::string pre = "job " + std::to_string(j) + ": ";
    if (J.kind != FRIR_KIND_FRAM && J.kind != FRIR_KIND_ISM && J.kind != FRIR_KIND_TRAIN) {
      set_error(pre + "unknown job kind " + std::to_string(J.kind));
      return FRIR_EINVAL;
    }
    const bool ism = J.kind == FRIR_KIND_ISM;
    const bool train = J.kind == FRIR_KIND_TRAIN;
    if (train) {
      // an explicit high-rate train of `duration` samples (frir_simulate_train)
      if (!(J.duration >= 1.0 && J.duration == std::floor(J.duration))) {
        set_error(pre + "a train job needs its length in samples as duration");
        return FRIR_EINVAL;
      }
      if (J.n_mics < 1 || J.n_images < 0) { set_error(pre + "a train job needs rows and channels"); return FRIR_EINVAL; }
      J.t60 = 1.0;
      J.r = 0.5;
      J.rr_max = 0.0;
      J.normalize = 0;
    } else if (ism) {
      // IsmConfig / ism_rir (ism.py:39-60, 63-78, 118-126); positions come as draws
      if (!(J.t60 > 0)) { set_error(pre + "t60 must be > 0"); return FRIR_EINVAL; }
      if (!(J.c0 > 0)) { set_error(pre + "sound_speed must be > 0"); return FRIR_EINVAL; }
      for (int k = 0; k < 3; ++k)
        if (!(J.room[k] > 0)) { set_error(pre + "room_dims must be 3 positive lengths"); return FRIR_EINVAL; }
      if (J.n_mics < 1) { set_error(pre + "mic_positions must be an (M, 3) array with M >= 1"); return FRIR_EINVAL; }
      if (J.lattice < 0) { set_error(pre + "max_order must be >= 0"); return FRIR_EINVAL; }
      if (J.lattice > 0) {  // device lattice: (2K + 1)^3 points without the origin (row 0)
        const int64_t n = 2 * (int64_t)(J.lattice - 1) + 1;
        if (n > 1023 || n * n * n - 1 >= (int64_t)kMaxRows) {
          set_error(pre + "image lattice of order " + std::to_string(J.lattice - 1) + " has too many points");
          return FRIR_ERANGE;
        }
        J.n_images = (int32_t)(n * n * n - 1);
        J.n_images_hi = 0;
      }
      if (J.n_images < 0 || J.n_images_hi > J.n_images) { set_error(pre + "image count must be >= 0"); return FRIR_EINVAL; }
      if (!(J.duration >= 0) || !(J.reflection >= 0)) {
        set_error(pre + "duration and reflection must be >= 0 (0 = default)");
        return FRIR_EINVAL;
      }
      if (J.normalize != 0) { set_error(pre + "normalize is not defined for ISM jobs"); return FRIR_EINVAL; }
      const double lx = J.room[0], ly = J.room[1], lz = J.room[2];
      const double ratio = (lx * ly * lz) / (2.0 * (lx * ly + lx * lz + ly * lz));
      J.r = J.reflection > 0 ? J.reflection : std::exp(-0.0805 * ratio / J.t60);
      if (!(0.0 < J.r && J.r < 1.0)) {
        set_error(pre + "reflection coefficient must be in (0, 1), got " + fmt("%.17g", J.r));
        return FRIR_EINVAL;
      }
      J.rr_max = 0.0;
    } else {
      // extension: I ~ U{n_images .. n_images_hi} from the job's own stream (seed, k, 2)
      if (J.n_images_hi > J.n_images && J.n_images >= 0) {
        uint64_t k2[2];
        seed_keys(J.seed, (uint64_t)J.source_index, 2, k2);
        const double u = u64_to_unit(stream_word(k2, 0));
        J.n_images += (int32_t)(u * (double)(J.n_images_hi - J.n_images + 1));
        J.n_images_hi = J.n_images;  // idempotent: a prepared table keeps its draw
      }
      // SimParams.__post_init__ (params.py:49-65)
      if (!(J.t60 > 0)) { set_error(pre + "t60 must be > 0, got " + fmt("%g", J.t60)); return FRIR_EINVAL; }
      if (J.n_images < 0) { set_error(pre + "num_images must be >= 0"); return FRIR_EINVAL; }
      if (!(0.0 <= J.alpha && J.alpha < J.beta && J.beta <= 1.0)) {
        set_error(pre + "need 0 <= alpha < beta <= 1, got alpha=" + fmt("%g", J.alpha) + " beta=" + fmt("%g", J.beta));
        return FRIR_EINVAL;
      }
      if (J.perturb_lo > J.perturb_hi) { set_error(pre + "perturb_lo must be <= perturb_hi"); return FRIR_EINVAL; }
      if (!(J.tau > 0)) { set_error(pre + "tau must be > 0, got " + fmt("%g", J.tau)); return FRIR_EINVAL; }
      if (!(J.c0 > 0)) { set_error(pre + "sound_speed must be > 0"); return FRIR_EINVAL; }
      // Scene (params.py:82-93)
      for (int k = 0; k < 3; ++k)
        if (!(J.room[k] > 0)) { set_error(pre + "room_dims must be 3 positive lengths"); return FRIR_EINVAL; }
      if (J.n_mics < 1) { set_error(pre + "mic_positions must be an (M, 3) array with M >= 1"); return FRIR_EINVAL; }
      if (!(J.d0 > 0)) { set_error(pre + "source distances must be > 0"); return FRIR_EINVAL; }
      // reflection_coefficient (core.py:113-128)
      double lx = J.room[0], ly = J.room[1], lz = J.room[2];
      double volume = lx * ly * lz;
      double surface = 2.0 * (lx * ly + lx * lz + ly * lz);
      double ratio = volume / surface;
      double t = 1.0 - std::exp(-0.16 * ratio / J.t60);
      J.r = std::sqrt(1.0 - t * t);
      // sample_image_geometry (core.py:140-148)
      if (J.alpha == 0.0) { set_error(pre + "alpha must be > 0 to sample image distances"); return FRIR_EINVAL; }
      double c_max = J.c0 * J.t60;
      if (c_max <= J.d0) {
        set_error(pre + "c0*t60 = " + fmt("%.3f", c_max) + " m must exceed the direct distance " + fmt("%.3f", J.d0) + " m");
        return FRIR_EINVAL;
      }
      J.rr_max = 0.0;
      if (J.n_images > 0) {  // core.py:295-299
        if (!(0.0 < J.r && J.r < 1.0)) {
          set_error(pre + "reflection coefficient must be in (0, 1), got " + fmt("%.17g", J.r));
          return FRIR_EINVAL;
        }
        J.rr_max = (std::log10(J.c0 * J.t60) - std::log10(J.d0) - 3.0) / std::log10(J.r);
        if (J.rr_max < 1.0) {
          set_error(pre + "rr_max must be >= 1, got " + fmt("%.17g", J.rr_max));
          return FRIR_EINVAL;
        }
      }
    }
    J.log2r = std::log2(J.r);
    // early window (core.py:257-258: -ceil(6 rate / 1000) .. +ceil(50 rate / 1000))
    if (J.early_lo_ms == 0.0 && J.early_hi_ms == 0.0) {
      J.e_lo = (int32_t)((6 * rate + 999) / 1000);
      J.e_hi = (int32_t)((50 * rate + 999) / 1000);
    } else {
      if (!(J.early_lo_ms >= 0.0 && J.early_hi_ms >= 0.0 && J.early_lo_ms < 1e6 && J.early_hi_ms < 1e6)) {
        set_error(pre + "early window must be non-negative milliseconds");
        return FRIR_EINVAL;
      }
      J.e_lo = (int32_t)std::ceil(J.early_lo_ms * (double)rate / 1000.0);
      J.e_hi = (int32_t)std::ceil(J.early_hi_ms * (double)rate / 1000.0);
    }
    if (J.normalize < 0 || J.normalize > 1) { set_error(pre + "normalize must be 0 or 1"); return FRIR_EINVAL; }
    J.alpha3 = std::pow(J.alpha, 3.0);
    J.b3a3 = std::pow(J.beta, 3.0) - J.alpha3;
    uint64_t key[2];
    seed_keys(J.seed, (uint64_t)J.source_index, 0, key);
    J.key[0] = key[0]; J.key[1] = key[1];
    seed_keys(J.seed, (uint64_t)J.source_index, 1, key);
    J.key[2] = key[0]; J.key[3] = key[1];
    // lengths (core.py:239, scipy resample_poly output lengths)
    double Ld = train ? J.duration : std::ceil((ism && J.duration > 0 ? J.duration : J.t60) * (double)rate);
    if (!(Ld >= 1.0 && Ld < 2.0e9)) { set_error(pre + "RIR length out of range"); return FRIR_ERANGE; }
    J.L = (int32_t)Ld;
    int64_t n1 = ceil_div64((int64_t)J.L * d.up, d.down);
    int64_t n2 = ceil_div64(n1, d.r_l);
    if (n2 + kExt + kSpBias + 64 >= (1 << 20)) { set_error(pre + "RIR too long for the packed layout"); return FRIR_ERANGE; }
    if (((int64_t)J.L + 66LL * d.r_h) * d.r_h >= (1LL << 32)) {
      set_error(pre + "RIR too long for the delay arithmetic");
      return FRIR_ERANGE;
    }
    J.n1 = (int32_t)n1;
    J.n2 = (int32_t)n2;
    int rows = J.n_images + 1;
    if (rows > kMaxRows) {
      set_error(pre + "num_images " + std::to_string(J.n_images) + " exceeds the supported maximum " + std::to_string(kMaxRows - 1));
      return FRIR_ERANGE;
    }
    J.img_off = img;
    J.item_off = item;
    J.chan_off = chan;
    img += rows;
    item += (int64_t)rows * J.n_mics;
    if (chan_job)
      for (int m = 0; m < J.n_mics; ++m) chan_job[chan + m] = j;
    chan += J.n_mics;
    max_rows = std::max(max_rows, rows);
    max_n2 = std::max(max_n2, J.n2);
  }
  for (int32_t j = 0; j < n_jobs; ++j) {
    frir_job& J = jobs[j];
    // rows start 16-byte aligned (the render kernel stores float4s)
    J.out_stride = ((padded ? max_n2 : J.n2) + 3) & ~3;
    J.out_off = out;
    out += (int64_t)J.out_stride * J.n_mics;
  }
  if (chan_order) {
    std::vector<int64_t> cost(chan);
    for (int32_t j = 0; j < n_jobs; ++j)
      for (int m = 0; m < jobs[j].n_mics; ++m)
        cost[jobs[j].chan_off + m] = 2 * (int64_t)(jobs[j].n_images + 1) + jobs[j].n2;
    std::vector<int32_t> ord(chan);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
    std::memcpy(chan_order, ord.data(), ord.size() * sizeof(int32_t));
  }
  batch->n_jobs = n_jobs;
  batch->total_channels = chan;
  batch->total_images = img;
  batch->total_items = item;
  batch->total_out = out;
  batch->max_rows = max_rows;
  batch->max_windows = (int32_t)((max_n2 + kExt + kWin - 1) / kWin);
  return FRIR_OK;
}

size_t frir_workspace_size(const frir_plan* plan, const frir_batch* b) {
  (void)plan;
  if (!b) return 0;
  return workspace_bytes(b);
}

int frir_simulate_stages(const frir_plan* plan, const frir_batch* b, void* ws, size_t ws_bytes,
                         float* out_full, float* out_early, int32_t* direct_index, void* stream,
                         int32_t stages) {
  if (!plan || !b) { set_error("null argument"); return FRIR_EINVAL; }
  if (b->n_jobs > 0 && (!b->jobs || !b->chan_job || !b->mics || !out_full || !direct_index || !ws)) {
    set_error("null device pointer in batch");
    return FRIR_EINVAL;
  }
  if (stages <= 0 || stages > FRIR_STAGE_ALL) { set_error("bad stage mask"); return FRIR_EINVAL; }
  // TMA bulk copies and float4 row stores: a cudaMalloc'd (256-byte aligned)
  // workspace and 16-byte aligned output buffers
  if (((uintptr_t)ws & 255) || ((uintptr_t)out_full & 15) || ((uintptr_t)out_early & 15)) {
    set_error("workspace must be 256-byte aligned and outputs 16-byte aligned (cudaMalloc'd buffers)");
    return FRIR_EINVAL;
  }
  const bool oracle = b->draw_dist || b->draw_az || b->draw_el || b->draw_refl;
  if (oracle && !(b->draw_dist && b->draw_az && b->draw_el && b->draw_refl)) {
    set_error("oracle mode needs all four draw arrays");
    return FRIR_EINVAL;
  }
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != plan->device) {
    set_error("plan was created on device " + std::to_string(plan->device) + ", current device is " + std::to_string(dev));
    return FRIR_EINVAL;
  }
  return launch_simulate(plan, b, ws, ws_bytes, out_full, out_early, direct_index,
                         (cudaStream_t)stream, stages);
}

int frir_simulate(const frir_plan* plan, const frir_batch* b, void* ws, size_t ws_bytes,
                  float* out_full, float* out_early, int32_t* direct_index, void* stream) {
  return frir_simulate_stages(plan, b, ws, ws_bytes, out_full, out_early, direct_index, stream,
                              FRIR_STAGE_ALL);
}

int32_t frir_launch_count(const frir_plan* plan, const frir_batch* b, int32_t early) {
  (void)plan;
  if (!b || b->n_jobs == 0) return 0;
  return launches(b, early);
}

}  // extern "C"
