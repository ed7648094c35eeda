// sm_100a kernels of the batched decay measurement:
// reference framrir/decay.py:8-49 (schroeder_curve, measure_t60).
//
// One lane per channel walks its row backwards in FP64 exactly like numpy's
// sequential cumsum of the reversed squared response, so the energy decay
// curve is bit-identical to the reference's; rows are staged through shared
// memory in 64-sample tiles both ways (a cp.async ring in, row-contiguous
// stores out) by a second warp, so loads and stores stay coalesced and off
// the serial sums.  The
// T60 kernel then finds the direct-path index, the adaptive drop and the
// first crossing (binary search: the curve is monotone) per channel.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"

namespace frir {
namespace {

constexpr int kEdcRows = 32;    // channels per CTA; lane = channel in the sums
constexpr int kEdcTile = 64;    // samples per staged tile
constexpr int kEdcStages = 8;   // input tiles in flight (cp.async ring)
constexpr int kEdcOut = kEdcTile + 2;  // padded output row: 16-byte aligned
constexpr int kEdcIo = 4;               // I/O warps per CTA (plus one summing warp)
// Input samples are float32 (renderer output) or float64 (any caller's rows,
// e.g. the reference's own RIRs): VEC elements per 16-byte copy, padded rows.
template <typename T>
struct EdcIn {
  static constexpr int kVec = 16 / (int)sizeof(T);
  static constexpr int kRow = kEdcTile + kVec;  // padded input row: 16-byte aligned
  static constexpr size_t kSmem = (size_t)kEdcStages * kEdcRows * kRow * sizeof(T) +
                                  2 * (size_t)kEdcRows * kEdcOut * 8 + kEdcRows * 4;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// edc[c][i] = sum_{j >= i} h[c][j]^2 (FP64, sequential from the end) for
// i < len[c], zeros for len[c] <= i < ld_out; amax[c] = max |h[c][i]|.  Rows
// are float32 with stride `ld`.  Per 32 channels, warp 0 runs each lane's row
// sum in numpy's order over tiles of 64 samples; four I/O warps stream the
// tiles in through an 8-deep cp.async ring (16-byte row-contiguous copies,
// zero-filled past each length; scalar loads when rows are not 16-byte
// aligned) and writes the previous EDC tile out row-contiguous, so the serial
// sums never wait on memory.
template <typename T>
__global__ void __launch_bounds__(32 * (1 + kEdcIo)) edc_kernel(const T* __restrict__ h, long ld,
                                                 const int32_t* __restrict__ len, int C,
                                                 double* __restrict__ edc, long ld_out,
                                                 double* __restrict__ amax) {
  constexpr int kEdcIn = EdcIn<T>::kRow, kVec = EdcIn<T>::kVec;
  extern __shared__ __align__(16) unsigned char edc_smem[];
  T(*tin)[kEdcRows][kEdcIn] = reinterpret_cast<T(*)[kEdcRows][kEdcIn]>(edc_smem);
  double(*tout)[kEdcRows][kEdcOut] =
      reinterpret_cast<double(*)[kEdcRows][kEdcOut]>(edc_smem + (size_t)kEdcStages * kEdcRows * kEdcIn * sizeof(T));
  int* s_len = reinterpret_cast<int*>(edc_smem + (size_t)kEdcStages * kEdcRows * kEdcIn * sizeof(T) +
                                      2 * (size_t)kEdcRows * kEdcOut * 8);
  const int c0 = blockIdx.x * kEdcRows;
  const int lane = threadIdx.x & 31;
  const bool io = threadIdx.x >= 32;
  const int iw = (threadIdx.x >> 5) - 1;  // I/O warp index
  if (!io) s_len[lane] = c0 + lane < C ? len[c0 + lane] : 0;
  __syncthreads();
  int nmax = 0;
  for (int r = 0; r < kEdcRows; ++r) nmax = max(nmax, s_len[r]);
  const int ntile = (int)((max((long)nmax, ld_out) + kEdcTile - 1) / kEdcTile);
  const int nlive = (nmax + kEdcTile - 1) / kEdcTile;  // tiles holding samples
  const bool vec_in = (ld % kVec == 0) && (((uintptr_t)h & 15) == 0);
  const bool vec_out = (ld_out % 2 == 0) && (((uintptr_t)edc & 15) == 0);

  auto stage = [&](int t) {  // I/O warp: tile t into ring slot t % kEdcStages
    if (t >= 0 && t < nlive) {
      const int base = t * kEdcTile;
      T(*dst)[kEdcIn] = tin[t % kEdcStages];
      constexpr int kPerRow = kEdcTile / kVec;  // 16-byte copies per row
#pragma unroll
      for (int i = 0; i < kEdcRows * kPerRow / (32 * kEdcIo); ++i) {
        const int q = (i * kEdcIo + iw) * 32 + lane, r = q / kPerRow, col = (q % kPerRow) * kVec;
        const int nr = s_len[r];
        const long off = (long)(c0 + r) * ld + base + col;
        if (vec_in) {
          const int bytes = max(0, min(16, (nr - base - col) * (int)sizeof(T)));
          cp_async16(&dst[r][col], bytes > 0 ? (const void*)(h + off) : (const void*)h, bytes);
        } else {
#pragma unroll
          for (int e = 0; e < kVec; ++e) dst[r][col + e] = base + col + e < nr ? h[off + e] : (T)0;
        }
      }
    }
    cp_async_commit();
  };
  auto store = [&](int t) {  // I/O warp: EDC tile t (zeros for tiles past every length)
    if (t < 0 || t >= ntile) return;
    const int base = t * kEdcTile, k2 = 2 * lane;
    for (int r = iw; r < kEdcRows && c0 + r < C; r += kEdcIo) {
      double* out = edc + (size_t)(c0 + r) * ld_out + base;
      const double2 v = t < nlive ? *reinterpret_cast<const double2*>(&tout[t & 1][r][k2]) : make_double2(0.0, 0.0);
      if (vec_out && base + k2 + 1 < ld_out) {
        *reinterpret_cast<double2*>(out + k2) = v;
      } else {
        if (base + k2 < ld_out) out[k2] = v.x;
        if (base + k2 + 1 < ld_out) out[k2 + 1] = v.y;
      }
    }
  };

  if (io) {
    for (int k = 0; k < kEdcStages - 1; ++k) stage(nlive - 1 - k);
    cp_async_wait<kEdcStages - 2>();  // tile nlive - 1 has landed
    __syncwarp();
  }
  double acc = 0.0;
  T mx = 0;  // max |h|, exact in the input type
  for (int t = ntile - 1; t >= -1; --t) {
    __syncthreads();  // tile t staged; tout[t & 1] free (its store was two rounds ago)
    if (!io) {
      if (t >= 0 && t < nlive) {
        const T(*src)[kEdcIn] = tin[t % kEdcStages];
        double* dst = tout[t & 1][lane];
        // No length tests: samples past a row's end were staged as zeros and
        // come first in the backward walk, so they leave acc at +0.0 and
        // their EDC entries are the zeros the contract asks for.
        // Warps issue in order: the independent loads, conversions and
        // squares of a half tile go first, then the dependent adds back to
        // back (one FP64 add latency per sample).
#pragma unroll
        for (int hh = 1; hh >= 0; --hh) {
          double sq[kEdcTile / 2];
#pragma unroll
          for (int k = 0; k < kEdcTile / 2; k += kVec) {  // 16-byte reads (registers, no local array)
            if constexpr (sizeof(T) == 4) {
              const float4 f4 = *reinterpret_cast<const float4*>(&src[lane][hh * (kEdcTile / 2) + k]);
              const float f[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const double v = (double)f[e];
                sq[k + e] = v * v;  // numpy: h ** 2 in FP64 (exact for float32 samples)
                mx = fmaxf(mx, fabsf(f[e]));
              }
            } else {
              const double2 f2 = *reinterpret_cast<const double2*>(&src[lane][hh * (kEdcTile / 2) + k]);
              sq[k] = f2.x * f2.x;
              sq[k + 1] = f2.y * f2.y;
              mx = fmax(mx, fmax(fabs(f2.x), fabs(f2.y)));
            }
          }
#pragma unroll
          for (int k = kEdcTile / 2 - 2; k >= 0; k -= 2) {
            const double a1 = acc + sq[k + 1];  // numpy: cumsum(h[::-1] ** 2), sequential
            acc = a1 + sq[k];
            *reinterpret_cast<double2*>(&dst[hh * (kEdcTile / 2) + k]) = make_double2(acc, a1);
          }
        }
      }
    } else {
      store(t + 1);                        // the tile computed last round
      if (t >= 0 && t < nlive) {
        stage(t - (kEdcStages - 1));       // keep the ring full
        cp_async_wait<kEdcStages - 2>();   // tile t - 1 has landed
      }
      __syncwarp();
    }
  }
  if (!io && c0 + lane < C) amax[c0 + lane] = (double)mx;
}

__device__ __forceinline__ double db_of(double e, double e0) {
  return 10.0 * log10(fmax(e / e0, 1e-300));  // decay.py:39
}

// measure_t60 (decay.py:20-49) per channel from the EDC and |h|.
template <typename T>
__global__ void t60_kernel(const T* __restrict__ h, long ld, const int32_t* __restrict__ len, int C,
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
  const T* row = h + (size_t)c * ld;
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

template <typename T>
static int edc_impl(const T* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
                    double* amax, void* stream) {
  if (!h || !len || !edc || !amax || C < 0 || ld < 0 || ld_out < 0) {
    set_error("frir_edc: invalid argument");
    return FRIR_EINVAL;
  }
  if (C == 0) return FRIR_OK;
  // > 48 KB of dynamic shared memory (per device and function: set every call)
  cudaFuncSetAttribute(edc_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EdcIn<T>::kSmem);
  edc_kernel<T><<<(C + kEdcRows - 1) / kEdcRows, 32 * (1 + kEdcIo), EdcIn<T>::kSmem, (cudaStream_t)stream>>>(
      h, (long)ld, len, C, edc, (long)ld_out, amax);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("edc_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

template <typename T>
static int t60_impl(const T* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
                    const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
                    double* t60, void* stream) {
  if (!h || !len || !edc || !amax || !t60 || C < 0 || !(sample_rate > 0)) {
    set_error("frir_t60: invalid argument");
    return FRIR_EINVAL;
  }
  if (C == 0) return FRIR_OK;
  t60_kernel<T><<<(C + 127) / 128, 128, 0, (cudaStream_t)stream>>>(h, (long)ld, len, C, edc, (long)ld_e, amax,
                                                                   sample_rate, max_drop, floor_margin, min_drop,
                                                                   t60);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("t60_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

extern "C" {

int frir_edc(const float* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
             double* amax, void* stream) {
  return edc_impl(h, ld, len, C, edc, ld_out, amax, stream);
}

int frir_edc_f64(const double* h, int64_t ld, const int32_t* len, int32_t C, double* edc, int64_t ld_out,
                 double* amax, void* stream) {
  return edc_impl(h, ld, len, C, edc, ld_out, amax, stream);
}

int frir_t60(const float* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
             const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
             double* t60, void* stream) {
  return t60_impl(h, ld, len, C, edc, ld_e, amax, sample_rate, max_drop, floor_margin, min_drop, t60, stream);
}

int frir_t60_f64(const double* h, int64_t ld, const int32_t* len, int32_t C, const double* edc, int64_t ld_e,
                 const double* amax, double sample_rate, double max_drop, double floor_margin, double min_drop,
                 double* t60, void* stream) {
  return t60_impl(h, ld, len, C, edc, ld_e, amax, sample_rate, max_drop, floor_margin, min_drop, t60, stream);
}

}  // extern "C"
