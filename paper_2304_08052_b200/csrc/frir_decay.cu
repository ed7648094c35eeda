// sm_100a kernels of the batched decay measurement:
// reference framrir/decay.py:8-49 (schroeder_curve, measure_t60).
//
// One thread per channel walks its row backwards in FP64 exactly like
// numpy's sequential cumsum of the reversed squared response, so the energy
// decay curve is bit-identical to the reference's; rows are staged through
// shared memory in 32-sample tiles so the global loads stay coalesced.  The
// T60 kernel then finds the direct-path index, the adaptive drop and the
// first crossing (binary search: the curve is monotone) per channel.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"

namespace frir {
namespace {

constexpr int kEdcThreads = 128;  // channels per CTA
constexpr int kEdcTile = 32;      // samples per staged tile

// edc[c][i] = sum_{j >= i} h[c][j]^2 (FP64, sequential from the end) for
// i < len[c]; amax[c] = max |h[c][i]|.  Rows are float32 with stride `ld`.
__global__ void __launch_bounds__(kEdcThreads) edc_kernel(const float* __restrict__ h, long ld,
                                                        const int32_t* __restrict__ len, int C,
                                                        double* __restrict__ edc, long ld_out,
                                                        double* __restrict__ amax) {
  __shared__ float tile[kEdcThreads][kEdcTile + 1];
  const int c0 = blockIdx.x * kEdcThreads;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = c0 + threadIdx.x;
  const int n = c < C ? len[c] : 0;
  // longest row of the CTA (tiles run to its start)
  int nmax = n;
  for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
  __shared__ int s_nmax[kEdcThreads / 32];
  if (lane == 0) s_nmax[warp] = nmax;
  __syncthreads();
  nmax = 0;
  for (int w = 0; w < kEdcThreads / 32; ++w) nmax = max(nmax, s_nmax[w]);
  double acc = 0.0, mx = 0.0;
  const int ntile = (nmax + kEdcTile - 1) / kEdcTile;
  for (int t = ntile - 1; t >= 0; --t) {
    const int base = t * kEdcTile;
    __syncthreads();
    // warp w stages rows w, w + 4, ...: lane = sample within the tile (coalesced)
    for (int r = warp; r < kEdcThreads; r += kEdcThreads / 32) {
      const int cr = c0 + r;
      float v = 0.f;
      if (cr < C && base + lane < len[cr]) v = h[(size_t)cr * ld + base + lane];
      tile[r][lane] = v;
    }
    __syncthreads();
    if (c < C) {
      for (int k = kEdcTile - 1; k >= 0; --k) {
        const int i = base + k;
        if (i < n) {
          const double v = (double)tile[threadIdx.x][k];
          acc += v * v;  // numpy: cumsum(h[::-1] ** 2), sequential
          edc[(size_t)c * ld_out + i] = acc;
          mx = fmax(mx, fabs(v));
        }
      }
    }
  }
  if (c < C) amax[c] = mx;
}

__device__ __forceinline__ double db_of(double e, double e0) {
  return 10.0 * log10(fmax(e / e0, 1e-300));  // decay.py:39
}

// measure_t60 (decay.py:20-49) per channel from the EDC and |h|.
__global__ void t60_kernel(const float* __restrict__ h, long ld, const int32_t* __restrict__ len, int C,
                           const double* __restrict__ edc, long ld_e, const double* __restrict__ amax,
                           double fs, double max_drop, double floor_margin, double min_drop,
                           double* __restrict__ t60) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int n = len[c];
  const double* e = edc + (size_t)c * ld_e;
  if (n <= 0 || !(e[0] > 0.0)) {  // schroeder_curve raises; the batch reports NaN
    t60[c] = 0.0 / 0.0;
    return;
  }
  const double e0 = e[0];
  const double half = 0.5 * amax[c];
  const float* row = h + (size_t)c * ld;
  int direct = 0;
  while (direct < n && !(fabs((double)row[direct]) >= half)) ++direct;
  const double d0 = db_of(e[direct], e0);
  // rel is non-increasing: its minimum is the last sample
  const double drop = fmin(max_drop, -(db_of(e[n - 1], e0) - d0) - floor_margin);
  if (drop < min_drop) {
    t60[c] = 0.0 / 0.0;
    return;
  }
  int lo = direct, hi = n - 1;  // first i with db[i] - d0 <= -drop (exists: the last one)
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if (db_of(e[mid], e0) - d0 <= -drop) hi = mid; else lo = mid + 1;
  }
  t60[c] = (double)(lo - direct) / fs * (60.0 / drop);
}

}  // namespace
}  // namespace frir

using namespace frir;

extern "C" {

int frir_edc(const float* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
             double* amax, void* stream) {
  if (!h || !len || !edc || !amax || C < 0 || ld < 0 || ld_out < 0) {
    set_error("frir_edc: invalid argument");
    return FRIR_EINVAL;
  }
  if (C == 0) return FRIR_OK;
  edc_kernel<<<(C + kEdcThreads - 1) / kEdcThreads, kEdcThreads, 0, (cudaStream_t)stream>>>(
      h, (long)ld, len, C, edc, (long)ld_out, amax);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("edc_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

int frir_t60(const float* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
             const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
             double* t60, void* stream) {
  if (!h || !len || !edc || !amax || !t60 || C < 0 || !(sample_rate > 0)) {
    set_error("frir_t60: invalid argument");
    return FRIR_EINVAL;
  }
  if (C == 0) return FRIR_OK;
  t60_kernel<<<(C + 127) / 128, 128, 0, (cudaStream_t)stream>>>(h, (long)ld, len, C, edc, (long)ld_e, amax,
                                                                sample_rate, max_drop, floor_margin, min_drop,
                                                                t60);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("t60_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

}  // extern "C"
