// sm_100a kernels behind the reference's public stage functions
// (framrir/__init__.py:15-28: quadratic_ratio_sample, rescale_distance_ratio,
// sample_image_geometry, sample_reflection_counts, build_impulse_train,
// early_reverb_train, downsample_highpass_downsample).  The batched hot path
// (frir_simulate) never builds these intermediates; these entry points exist
// so code written against the reference's stage API runs on the device with
// the same arithmetic (FP64 in numpy's operation order) and no CPU fallback.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"
#include "frir_philox.cuh"

namespace frir {
namespace {

// Elementwise stage arithmetic (op codes in include/frir.h).
__global__ void stage_eval_kernel(int op, const double* __restrict__ x0, const double* __restrict__ x1,
                                  const double* __restrict__ x2, long n, double p0, double p1, double p2, double p3,
                                  double* __restrict__ out) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (op == FRIR_STAGE_RATIO_SAMPLE) {  // core.py:94-100, p0 = alpha**3, p1 = beta**3 (host pow)
    out[i] = cbrt(__dadd_rn(p0, __dmul_rn(__dsub_rn(1.0, x0[i]), __dsub_rn(p1, p0))));
  } else if (op == FRIR_STAGE_RESCALE) {  // core.py:103-110, p0 = alpha, p1 = beta, p2 = max_ratio
    const double k = __ddiv_rn(p0, __dsub_rn(p1, p0));
    out[i] = __dadd_rn(1.0, __dmul_rn(__dmul_rn(k, __dsub_rn(__ddiv_rn(x0[i], p0), 1.0)), __dsub_rn(p2, 1.0)));
  } else {  // FRIR_STAGE_REFLECTIONS, core.py:213-220: x0 = D, x1 = DR, x2 = p; p0 = c_max, p1 = rr_max, p2 = tau
    const double q = __ddiv_rn(x0[i], p0);
    const double drt = p2 == 0.25 ? __dsqrt_rn(__dsqrt_rn(x1[i])) : pow(x1[i], p2);
    const double g = __dadd_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(q, q), __dsub_rn(p1, 1.0))), __dmul_rn(x2[i], drt));
    out[i] = fmin(fmax(g, 1.0), p1);
  }
}

// Generator(Philox(SeedSequence((seed, k, stage)))).uniform(lo, hi) words
// [first, first + n) (numpy: lo + (hi - lo) * random()).
__global__ void philox_uniform_kernel(uint64_t k0, uint64_t k1, long first, long n, double lo, double hi,
                                      double* __restrict__ out) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t key[2] = {k0, k1};
  out[i] = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u64_to_unit(stream_word(key, (uint64_t)(first + i)))));
}

// build_impulse_train (core.py:228-251), pass A: q = min(ceil(D / c0 * rate),
// L - 1) and amp = r ** g / D per (image, mic) in FP64, plus per-(mic, sample)
// arrival counts and the first arriving image.
__global__ void train_arrivals_kernel(const double* __restrict__ mic_dist, const double* __restrict__ refl, int rows,
                                      int M, double r, double c0, double rate, int L, int32_t* __restrict__ q,
                                      double* __restrict__ amp, int32_t* __restrict__ cnt, int32_t* __restrict__ first) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)rows * M) return;
  const int i = (int)(t / M), m = (int)(t % M);
  const double D = mic_dist[t];
  const double x = ceil(__dmul_rn(__ddiv_rn(D, c0), rate));
  const int qi = x >= (double)(L - 1) ? L - 1 : (int)x;
  q[t] = qi;
  amp[t] = __ddiv_rn(pow(r, refl[i]), D);
  const long s = (long)m * L + qi;
  atomicAdd(cnt + s, 1);
  atomicMin(first + s, i);
}

// Pass B: np.add.at order -- a sample with one arrival takes its amplitude;
// with several, the first image sums them in row order (0 + a_i1 + a_i2 ...).
__global__ void train_assemble_kernel(int rows, int M, int L, const int32_t* __restrict__ q,
                                      const double* __restrict__ amp, const int32_t* __restrict__ cnt,
                                      const int32_t* __restrict__ first, double* __restrict__ train) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)rows * M) return;
  const int i = (int)(t / M), m = (int)(t % M);
  const long s = (long)m * L + q[t];
  const int c = cnt[s];
  if (c == 1) {
    train[s] = 0.0 + amp[t];
  } else if (first[s] == i) {
    double acc = 0.0;
    int seen = 0;
    for (int j = i; j < rows && seen < c; ++j)
      if (q[(long)j * M + m] == q[t]) {
        acc += amp[(long)j * M + m];
        ++seen;
      }
    train[s] = acc;
  }
}

// early_reverb_train (core.py:254-265): keep n with -lo <= n - q0[m] <= hi.
__global__ void early_window_kernel(const double* __restrict__ x, int M, long L, const int32_t* __restrict__ q0,
                                    long lo, long hi, double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)M * L) return;
  const long rel = t % L - q0[t / L];
  out[t] = (rel >= -lo && rel <= hi) ? x[t] : 0.0;
}

inline int blocks(long n, int t) { return (int)((n + t - 1) / t); }

int cuda_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return FRIR_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FRIR_ECUDA;
}

}  // namespace
}  // namespace frir

using namespace frir;

extern "C" {

int frir_stage_eval(int32_t op, const double* x0, const double* x1, const double* x2, int64_t n,
                    const double* params, double* out, void* stream) {
  if (op < FRIR_STAGE_RATIO_SAMPLE || op > FRIR_STAGE_REFLECTIONS || n < 0 || !params || (n > 0 && (!x0 || !out)) ||
      (op == FRIR_STAGE_REFLECTIONS && n > 0 && (!x1 || !x2))) {
    set_error("frir_stage_eval: invalid argument");
    return FRIR_EINVAL;
  }
  if (n == 0) return FRIR_OK;
  stage_eval_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(op, x0, x1, x2, (long)n, params[0], params[1],
                                                                      params[2], params[3], out);
  return cuda_status("stage_eval_kernel");
}

int frir_philox_uniform(uint64_t seed, uint64_t source_index, uint64_t stage, int64_t first_word, int64_t n,
                        double lo, double hi, double* out, void* stream) {
  if (n < 0 || first_word < 0 || (n > 0 && !out)) {
    set_error("frir_philox_uniform: invalid argument");
    return FRIR_EINVAL;
  }
  if (n == 0) return FRIR_OK;
  uint64_t key[2];
  seed_keys(seed, source_index, stage, key);  // SeedSequence hashing: host bookkeeping
  philox_uniform_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(key[0], key[1], (long)first_word, (long)n,
                                                                          lo, hi, out);
  return cuda_status("philox_uniform_kernel");
}

int frir_image_set(const frir_plan* plan, const frir_batch* batch, double* dist, double* az, double* el,
                   double* ratio, double* refl, double* mic_dist, int32_t with_reflections, void* stream) {
  if (!plan || !batch || !dist || !az || !el || !ratio || !refl || !mic_dist) {
    set_error("frir_image_set: null argument");
    return FRIR_EINVAL;
  }
  if (batch->draw_dist) {
    set_error("frir_image_set: native-draw batches only");
    return FRIR_EINVAL;
  }
  return launch_image_set(plan, batch, dist, az, el, ratio, refl, mic_dist, with_reflections,
                          (cudaStream_t)stream);
}

int64_t frir_impulse_train_scratch(int32_t rows, int32_t n_mics, int32_t length) {
  if (rows < 0 || n_mics < 0 || length < 1) return -1;
  const int64_t rm = (int64_t)rows * n_mics, ml = (int64_t)n_mics * length;
  return rm * (4 + 8) + ml * (4 + 4) + 256;
}

int frir_impulse_train(const double* mic_dist, const double* refl, int32_t rows, int32_t n_mics, double r,
                       double sound_speed, int64_t rate, int32_t length, double* train, int32_t* q, void* scratch,
                       int64_t scratch_bytes, void* stream) {
  if (!mic_dist || !refl || !train || !q || !scratch || rows < 1 || n_mics < 1 || length < 1 ||
      scratch_bytes < frir_impulse_train_scratch(rows, n_mics, length)) {
    set_error("frir_impulse_train: invalid argument");
    return FRIR_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rm = (int64_t)rows * n_mics, ml = (int64_t)n_mics * length;
  char* p = (char*)scratch;
  double* amp = (double*)p; p += rm * 8;
  int32_t* cnt = (int32_t*)p; p += ml * 4;
  int32_t* first = (int32_t*)p;
  cudaError_t e = cudaMemsetAsync(train, 0, ml * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, ml * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(first, 0x7f, ml * 4, st);  // 0x7f7f7f7f > any row
  if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FRIR_ECUDA; }
  train_arrivals_kernel<<<blocks(rm, 256), 256, 0, st>>>(mic_dist, refl, rows, n_mics, r, sound_speed, (double)rate,
                                                         length, q, amp, cnt, first);
  int s = cuda_status("train_arrivals_kernel");
  if (s) return s;
  train_assemble_kernel<<<blocks(rm, 256), 256, 0, st>>>(rows, n_mics, length, q, amp, cnt, first, train);
  return cuda_status("train_assemble_kernel");
}

int frir_early_window(const double* train, int32_t n_mics, int64_t length, const int32_t* q0, int64_t lo, int64_t hi,
                      double* out, void* stream) {
  if (!train || !q0 || !out || n_mics < 0 || length < 0) {
    set_error("frir_early_window: invalid argument");
    return FRIR_EINVAL;
  }
  const long n = (long)n_mics * length;
  if (n == 0) return FRIR_OK;
  early_window_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(train, n_mics, (long)length, q0, (long)lo,
                                                                        (long)hi, out);
  return cuda_status("early_window_kernel");
}

int frir_train_nonzeros(const double* train, int64_t ld, int32_t rows, int32_t length, int32_t sign, int32_t* counts,
                        void* stream) {
  if (!train || !counts || rows < 0 || length < 0 || ld < length || (sign != 1 && sign != -1)) {
    set_error("frir_train_nonzeros: invalid argument");
    return FRIR_EINVAL;
  }
  return train_nonzeros(train, ld, rows, length, sign, counts, (cudaStream_t)stream);
}

int frir_simulate_train(const frir_plan* plan, const frir_batch* batch, void* workspace, size_t workspace_bytes,
                        const double* train, int64_t ld, int32_t sign, float* out_full, int32_t* direct_scratch,
                        void* stream) {
  if (!plan || !batch || !workspace || !train || !out_full || !direct_scratch || (sign != 1 && sign != -1)) {
    set_error("frir_simulate_train: invalid argument");
    return FRIR_EINVAL;
  }
  return launch_simulate_train(plan, batch, workspace, workspace_bytes, train, ld, sign, out_full, direct_scratch,
                               (cudaStream_t)stream);
}

}  // extern "C"
