// sm_100a kernels of the spatialise-and-mix consumer:
// reference framrir/mixture.py:216-222 (_convolve_multichannel, _power) and
// :225-332 (spatialize_and_mix).  The FFTs of the batched convolution run in
// cuFFT (through torch on the host side); these kernels do everything around
// them: the per-filter spectral products, the reference-channel powers, the
// SIR/SNR gains and the scaled outputs plus the mixture.  FP32 samples, FP64
// powers and gains (the reference computes in FP64), fixed-order reductions.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"

namespace frir {
namespace {

// spec[b][j][f] *= dry[b][src_of[j]][f], complex64 interleaved, f < Fc.
__global__ void mix_spectra_kernel(float2* __restrict__ spec, const float2* __restrict__ dry,
                                   const int32_t* __restrict__ src_of, int J, int K, long Fc) {
  const long per_item = (long)J * Fc;
  const int b = blockIdx.y;
  float2* s = spec + (size_t)b * per_item;
  const float2* x = dry + (size_t)b * K * Fc;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < per_item; i += (long)gridDim.x * blockDim.x) {
    const int j = (int)(i / Fc);
    const long f = i - (long)j * Fc;
    const float2 h = s[i], d = x[(size_t)src_of[j] * Fc + f];
    s[i] = make_float2(h.x * d.x - h.y * d.y, h.x * d.y + h.y * d.x);
  }
}

// Mean of squares over [lo, hi) of one row per request, FP64, fixed order.
// req[r] = {row index into y (absolute), lo, hi}; y rows have length F.
__global__ void mix_power_kernel(const float* __restrict__ y, const int64_t* __restrict__ req_row,
                                 const int32_t* __restrict__ req_lo, const int32_t* __restrict__ req_hi,
                                 long F, double* __restrict__ out) {
  const int r = blockIdx.x;
  const float* row = y + (size_t)req_row[r] * F;
  const int lo = req_lo[r], hi = req_hi[r];
  double acc = 0.0;
  for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
    const double v = (double)row[t];
    acc = fma(v, v, acc);
  }
  __shared__ double s[256];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = hi > lo ? s[0] / (double)(hi - lo) : 0.0 / 0.0;
}

// Gains of mixture.py:285-311 per item from the power table
// pw[b] = {p_ref, (p_int_k, p_tgt_k) for k = 1..S-1, p_noise}:
//   g_0 = 1, g_k = sqrt(p_tgt / (p_int 10^(sir_k/10))), g_noise = sqrt(p_ref / (p_noise 10^(snr/10))).
__global__ void mix_gains_kernel(const double* __restrict__ pw, const double* __restrict__ sir_db,
                                 const double* __restrict__ snr_db, int B, int S, double* __restrict__ gains) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* p = pw + (size_t)b * 2 * S;
  double* g = gains + (size_t)b * (S + 1);
  g[0] = 1.0;
  for (int k = 1; k < S; ++k) {
    const double p_int = p[2 * k - 1], p_tgt = p[2 * k];
    g[k] = sqrt(p_tgt / (p_int * pow(10.0, sir_db[(size_t)b * (S > 1 ? S - 1 : 1) + (k - 1)] / 10.0)));
  }
  g[S] = sqrt(p[0] / (p[2 * S - 1] * pow(10.0, snr_db[b] / 10.0)));
}

// Scaled outputs and the mixture (mixture.py:293-313):
//   sources[b][k][m][t] = g_k y[b][kM + m][t], early[b][k][m][t] = g_k y[b][(S + k)M + m][t],
//   noise[b][m][t] = g_n y[b][2SM + m][t], mixture = sum_k sources + noise,
// for t < total_b (zeros up to T).
__global__ void mix_combine_kernel(const float* __restrict__ y, const double* __restrict__ gains,
                                   const int32_t* __restrict__ total, int S, int M, long F, long T,
                                   float* __restrict__ mixture, float* __restrict__ sources,
                                   float* __restrict__ early, float* __restrict__ noise) {
  const int b = blockIdx.y;
  const long per_item = (long)M * T;
  const int J = (2 * S + 1) * M;
  const float* yb = y + (size_t)b * J * F;
  const double* g = gains + (size_t)b * (S + 1);
  const int tot = total[b];
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < per_item; i += (long)gridDim.x * blockDim.x) {
    const int m = (int)(i / T);
    const long t = i - (long)m * T;
    const bool in = t < tot;
    float mix = 0.f;
    for (int k = 0; k < S; ++k) {
      const float gk = (float)g[k];
      const float vf = in ? gk * yb[(size_t)(k * M + m) * F + t] : 0.f;
      const float ve = in ? gk * yb[(size_t)((S + k) * M + m) * F + t] : 0.f;
      sources[(((size_t)b * S + k) * M + m) * T + t] = vf;
      early[(((size_t)b * S + k) * M + m) * T + t] = ve;
      mix += vf;
    }
    const float vn = in ? (float)g[S] * yb[(size_t)(2 * S * M + m) * F + t] : 0.f;
    noise[((size_t)b * M + m) * T + t] = vn;
    mixture[((size_t)b * M + m) * T + t] = mix + vn;
  }
}

int grid_for(long n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long want = (n + threads - 1) / threads;
  return (int)(want < 8L * sms ? (want > 0 ? want : 1) : 8L * sms);
}

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return FRIR_ECUDA;
  }
  return FRIR_OK;
}

}  // namespace
}  // namespace frir

using namespace frir;

extern "C" {

int frir_mix_spectra(void* filt_spec, const void* dry_spec, const int32_t* src_of, int32_t B,
                     int32_t J, int32_t K, int64_t Fc, void* stream) {
  if (!filt_spec || !dry_spec || !src_of || B < 0 || J < 0 || K < 1 || Fc < 1) {
    set_error("frir_mix_spectra: invalid argument");
    return FRIR_EINVAL;
  }
  if (B == 0 || J == 0) return FRIR_OK;
  dim3 grid(grid_for((long)J * Fc, 256) / (B > 8 ? 8 : 1) + 1, B);
  mix_spectra_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((float2*)filt_spec, (const float2*)dry_spec,
                                                            src_of, J, K, (long)Fc);
  return launched("mix_spectra_kernel");
}

int frir_mix_powers(const float* y, int64_t F, const int64_t* req_row, const int32_t* req_lo,
                    const int32_t* req_hi, int32_t n_req, double* out, void* stream) {
  if (!y || !req_row || !req_lo || !req_hi || !out || n_req < 0 || F < 1) {
    set_error("frir_mix_powers: invalid argument");
    return FRIR_EINVAL;
  }
  if (n_req == 0) return FRIR_OK;
  mix_power_kernel<<<n_req, 256, 0, (cudaStream_t)stream>>>(y, req_row, req_lo, req_hi, (long)F, out);
  return launched("mix_power_kernel");
}

int frir_mix_gains(const double* powers, const double* sir_db, const double* snr_db, int32_t B,
                   int32_t S, double* gains, void* stream) {
  if (!powers || !sir_db || !snr_db || !gains || B < 0 || S < 1) {
    set_error("frir_mix_gains: invalid argument");
    return FRIR_EINVAL;
  }
  if (B == 0) return FRIR_OK;
  mix_gains_kernel<<<(B + 127) / 128, 128, 0, (cudaStream_t)stream>>>(powers, sir_db, snr_db, B, S, gains);
  return launched("mix_gains_kernel");
}

int frir_mix_combine(const float* y, const double* gains, const int32_t* total, int32_t B, int32_t S,
                     int32_t M, int64_t F, int64_t T, float* mixture, float* sources, float* early,
                     float* noise, void* stream) {
  if (!y || !gains || !total || !mixture || !sources || !early || !noise || B < 0 || S < 1 || M < 1 ||
      T < 0 || F < T) {
    set_error("frir_mix_combine: invalid argument");
    return FRIR_EINVAL;
  }
  if (B == 0 || T == 0) return FRIR_OK;
  dim3 grid(grid_for((long)M * T, 256) / (B > 8 ? 8 : 1) + 1, B);
  mix_combine_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(y, gains, total, S, M, (long)F, (long)T,
                                                            mixture, sources, early, noise);
  return launched("mix_combine_kernel");
}

}  // extern "C"
