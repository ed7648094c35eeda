// sm_100a kernels of the spatialise-and-mix consumer:
// reference framrir/mixture.py:216-222 (_convolve_multichannel, _power) and
// :225-332 (spatialize_and_mix).  The batched convolution itself is
// frir_fftconv.cu; these kernels do everything after it: the reference-channel
// powers, the SIR/SNR gains and the scaled outputs plus the mixture.  FP32 samples, FP64
// powers and gains (the reference computes in FP64), fixed-order reductions.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"

namespace frir {
namespace {

// Sums of squares over [lo, hi) of one row per request, split into kPowChunks
// chunks (grid (chunks, requests)); FP64, fixed order: each chunk's block
// reduction, then mix_gains_kernel adds the chunks in order.
constexpr int kPowChunks = FRIR_MIX_POWER_CHUNKS;
__global__ void mix_power_kernel(const float* __restrict__ y, const int64_t* __restrict__ req_row,
                                 const int32_t* __restrict__ req_lo, const int32_t* __restrict__ req_hi,
                                 long F, double* __restrict__ part) {
  const int r = blockIdx.y, c = blockIdx.x;
  const float* __restrict__ row = y + (size_t)req_row[r] * F;
  const int lo = req_lo[r], hi = req_hi[r];
  const int span = (hi - lo + kPowChunks - 1) / kPowChunks;
  const int a = lo + c * span, e = min(hi, a + span);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // four independent loads in flight per thread
  int t = a + threadIdx.x;
  for (; t + 3 * 256 < e; t += 4 * 256) {
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = row[t + i * 256];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = fma((double)v[i], (double)v[i], acc[i]);
  }
  for (int i = 0; t < e; t += 256, ++i) acc[i] = fma((double)row[t], (double)row[t], acc[i]);
  __shared__ double s[256];
  s[threadIdx.x] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)r * kPowChunks + c] = s[0];
}

// Means from the chunk sums (fixed order).
__global__ void mix_power_finish_kernel(const double* __restrict__ part, const int32_t* __restrict__ req_lo,
                                        const int32_t* __restrict__ req_hi, int n_req, double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  double t = 0.0;
  for (int c = 0; c < kPowChunks; ++c) t += part[(size_t)r * kPowChunks + c];
  const int n = req_hi[r] - req_lo[r];
  out[r] = n > 0 ? t / (double)n : 0.0 / 0.0;
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
// for t < total_b (zeros up to T).  Grid (T / (256 kCombineU), M, B): each
// thread takes kCombineU samples 256 apart, all loads issued before the stores.
constexpr int kCombineU = 4;
__global__ void __launch_bounds__(256) mix_combine_kernel(const float* __restrict__ y, const double* __restrict__ gains,
                                   const int32_t* __restrict__ total, int S, int M, long F, long T,
                                   float* __restrict__ mixture, float* __restrict__ sources,
                                   float* __restrict__ early, float* __restrict__ noise) {
  const int m = blockIdx.y, b = blockIdx.z;
  const int J = (2 * S + 1) * M;
  const float* yb = y + (size_t)b * J * F;
  const double* g = gains + (size_t)b * (S + 1);
  const long tot = total[b];
  const long t0 = (long)blockIdx.x * (256 * kCombineU) + threadIdx.x;
  float mix[kCombineU], nv[kCombineU], v[kCombineU];
  const float gn = (float)g[S];
  const float* yn = yb + (size_t)(2 * S * M + m) * F;
#pragma unroll
  for (int i = 0; i < kCombineU; ++i) {
    const long t = t0 + i * 256;
    nv[i] = t < tot ? gn * yn[t] : 0.f;
    mix[i] = 0.f;
  }
#pragma unroll
  for (int i = 0; i < kCombineU; ++i) {
    const long t = t0 + i * 256;
    if (t < T) noise[((size_t)b * M + m) * T + t] = nv[i];
  }
  for (int k = 0; k < S; ++k) {
    const float gk = (float)g[k];
    const float* yf = yb + (size_t)(k * M + m) * F;
    const float* ye = yb + (size_t)((S + k) * M + m) * F;
    float* so = sources + (((size_t)b * S + k) * M + m) * T;
    float* eo = early + (((size_t)b * S + k) * M + m) * T;
#pragma unroll
    for (int i = 0; i < kCombineU; ++i) {
      const long t = t0 + i * 256;
      v[i] = t < tot ? gk * yf[t] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kCombineU; ++i) {
      const long t = t0 + i * 256;
      if (t < T) so[t] = v[i];
      mix[i] += v[i];
    }
#pragma unroll
    for (int i = 0; i < kCombineU; ++i) {
      const long t = t0 + i * 256;
      v[i] = t < tot ? gk * ye[t] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kCombineU; ++i) {
      const long t = t0 + i * 256;
      if (t < T) eo[t] = v[i];
    }
  }
#pragma unroll
  for (int i = 0; i < kCombineU; ++i) {
    const long t = t0 + i * 256;
    if (t < T) mixture[((size_t)b * M + m) * T + t] = mix[i] + nv[i];  // sum of the sources, then the noise
  }
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

int frir_mix_powers(const float* y, int64_t F, const int64_t* req_row, const int32_t* req_lo,
                    const int32_t* req_hi, int32_t n_req, double* scratch, double* out, void* stream) {
  if (!y || !req_row || !req_lo || !req_hi || !scratch || !out || n_req < 0 || F < 1) {
    set_error("frir_mix_powers: invalid argument");
    return FRIR_EINVAL;
  }
  if (n_req == 0) return FRIR_OK;
  mix_power_kernel<<<dim3(kPowChunks, n_req), 256, 0, (cudaStream_t)stream>>>(y, req_row, req_lo, req_hi,
                                                                             (long)F, scratch);
  mix_power_finish_kernel<<<(n_req + 127) / 128, 128, 0, (cudaStream_t)stream>>>(scratch, req_lo, req_hi,
                                                                                n_req, out);
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
  dim3 grid((unsigned)((T + 256 * kCombineU - 1) / (256 * kCombineU)), M, B);
  mix_combine_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(y, gains, total, S, M, (long)F, (long)T,
                                                            mixture, sources, early, noise);
  return launched("mix_combine_kernel");
}

}  // extern "C"
