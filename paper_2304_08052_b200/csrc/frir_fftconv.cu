// Hand-written FFT convolution for the spatialise-and-mix consumer (SURVEY
// §8f row 1; reference framrir/mixture.py:216-218 _convolve_multichannel,
// scipy fftconvolve): uniformly partitioned overlap-save with 8192-point
// complex FFTs computed in shared memory.
//
//   block size P = 4096, FFT size N = 2P; the filter is cut into Q
//   partitions of P taps, the input into blocks of P samples:
//   y[tP + n] = last P samples of IFFT( sum_p X_{t-p} . H_p ),  n < P,
//   X_s = FFT(x[(s-1)P, (s+1)P)),  H_p = FFT(h[pP, pP + P) zero-padded).
//
// Two real filter rows that share a source (mics 2h, 2h + 1 of one filter
// group: a speaker's full filters, its early filters, or the noise) ride in
// one complex transform, H = FFT(h_a + i h_b), so IFFT(X . H) = y_a + i y_b;
// all-zero filter partitions (early filters end early) are skipped.  The FFT is a radix
// 16 * 16 * 16 * 2 Stockham in place in 64 KB of swizzled shared memory, 512
// threads, twiddles from an FP64-computed table.  FP32 throughout (the
// reference is FP64; the mixing tests hold the result to 1e-5 of the peak).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/frir.h"
#include "frir_internal.h"

namespace frir {
namespace {

constexpr int kFftN = 8192;            // transform length
constexpr int kFftP = kFftN / 2;       // hop / partition length
constexpr int kFftThreads = 512;

// (the library builds with -fmad=false for the FP64 geometry; the FFTs fuse explicitly)
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 addf(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 subf(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

// Size-4 DFT in place (forward).
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 t0 = addf(a0, a2), t1 = subf(a0, a2), t2 = addf(a1, a3), t3 = mul_mi(subf(a1, a3));
  a0 = addf(t0, t2);
  a2 = subf(t0, t2);
  a1 = addf(t1, t3);
  a3 = subf(t1, t3);
}
__device__ __forceinline__ float2 cmulc(float2 a, float wr, float wi) {
  return make_float2(fmaf(a.x, wr, -a.y * wi), fmaf(a.x, wi, a.y * wr));
}

// Size-16 DFT in registers, natural order in and out (4 x 4: DFTs over n1 of
// x[4 n1 + n2], twiddles W16^(n2 k1), DFTs over n2, transpose).
__device__ __forceinline__ void dft16(const float2 (&x)[16], float2 (&o)[16]) {
  float2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = x[i];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  const float c = 0.92387953251128674f, s = 0.38268343236508977f, h = 0.70710678118654752f;
  v[5] = cmulc(v[5], c, -s);     // W16^1
  v[6] = cmulc(v[6], h, -h);     // W16^2
  v[7] = cmulc(v[7], s, -c);     // W16^3
  v[9] = cmulc(v[9], h, -h);     // W16^2
  v[10] = mul_mi(v[10]);         // W16^4
  v[11] = cmulc(v[11], -h, -h);  // W16^6
  v[13] = cmulc(v[13], s, -c);   // W16^3
  v[14] = cmulc(v[14], -h, -h);  // W16^6
  v[15] = cmulc(v[15], -c, s);   // W16^9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) o[k1 + 4 * k2] = v[4 * k1 + k2];
}

// Shared-memory layout of the transform: an XOR swizzle of the low four bits
// of the float2 index with bits 4..7.  Every access of the passes below --
// consecutive reads (j + 512 r), the stride-16 stores of pass 1, the 16-runs
// at stride 256 of pass 2 and the 256-runs of pass 3 -- is free of bank
// conflicts (checked exhaustively offline), and reads at j + 512 r are
// swz(j) + 512 r (immediate offsets).
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 15); }
constexpr int kTwN = kFftN / 8;  // smem twiddle table: W^m, m < N / 8

// The forward 8192-point FFT is a radix 16 * 16 * 16 * 2 Stockham
// decomposition, 512 threads, one butterfly per thread per radix-16 pass:
//   fft_first(buf, x): pass 1 of butterfly j = threadIdx.x from registers,
//     x[r] = input[j + 512 r]; results to buf.
//   fft_mid(buf, tws): passes 2 and 3 (after a barrier; ends with one).
//   fft_last(buf, tws, f): pass 4 (radix 2), f(j, X[j], X[j + N/2]) for the
//     thread's eight butterflies j < N/2, straight to the caller.
// The kernels feed pass 1 from global memory and take pass 4 to global memory,
// so only passes 2-3 make a full shared-memory round trip.
__device__ __forceinline__ void fft_first(float2* buf, const float2 (&x)[16]) {
  const int j = threadIdx.x;
  float2 o[16];
  dft16(x, o);
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[16 * j + (r ^ (j & 15))] = o[r];  // swz(16 j + r)
}
// Radix-16 pass over NS-point sub-transforms (NS = 16, 256): twiddles W^{r k step},
// w1 = W^{k step} (k step < 512) from the table, w_r = w1^r.
template <int NS>
__device__ __forceinline__ void pass16(float2* buf, const float2* tws) {
  constexpr int step = kFftN / (NS * 16);
  const int j = threadIdx.x;
  const int k = j & (NS - 1);
  const int sj = swz(j);
  float2 x[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = buf[sj + 512 * r];
  const float2 w1 = tws[k * step];
  float2 w = w1;
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    x[r] = cmulf(x[r], w);
    if (r + 1 < 16) w = cmulf(w, w1);
  }
  __syncthreads();
  float2 o[16];
  dft16(x, o);
  const int d = (j / NS) * NS * 16 + k;
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[swz(d + r * NS)] = o[r];
  __syncthreads();
}
__device__ __forceinline__ void fft_mid(float2* buf, const float2* tws) {
  __syncthreads();
  pass16<16>(buf, tws);
  pass16<256>(buf, tws);
}
// Pass 4 for the butterflies j = threadIdx.x + 512 b, b < 8: f(j, X[j], X[j + N/2]).
// W^j = W^t * W^{512 b}: one table read per thread, the eight W^{512 b} are
// constants.
template <typename F>
__device__ __forceinline__ void fft_last(const float2* buf, const float2* tws, F&& f) {
  constexpr float kC[8] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                           0.f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f};
  constexpr float kS[8] = {0.f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f,
                           1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f};
  const int t = threadIdx.x;
  const float2 wt = tws[t];
  const int st = swz(t);  // swz(t + 512 b) = swz(t) + 512 b
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const float2 w = b == 0 ? wt : cmulc(wt, kC[b], -kS[b]);
    const float2 a = buf[st + 512 * b];
    const float2 c = cmulf(buf[st + 512 * b + kFftP], w);
    f(t + 512 * b, addf(a, c), subf(a, c));
  }
}

// Shared memory of the FFT kernels: the padded transform, then the twiddles.
__device__ __forceinline__ float2* load_twiddles(float2* smem_base, const float2* __restrict__ tw) {
  float2* tws = smem_base + kFftN;
  for (int i = threadIdx.x; i < kTwN; i += kFftThreads) tws[i] = __ldg(tw + i);
  return tws;
}
constexpr size_t kFftSmem = (size_t)(kFftN + kTwN) * sizeof(float2);

struct ConvArgs {
  const float* dry;
  long dry_sb, dry_sk;
  const float* noise;
  long noise_sb;
  const int32_t* off;
  const int32_t* len;
  const int32_t* nlen;
  const int32_t* dlen;
  const float* rir_full;
  long full_sb;
  const float* rir_early;
  long early_sb;
  const int32_t* rlen;
  int S, M, R, nb, Q, npairs;
  int hm;      // row pairs per filter group: ceil(M / 2)
  const float2* tw;
  float2* X;   // [B][S+1][nb][N]
  float2* H;   // [B][npairs][Q][N]
  int32_t* live;  // [B][npairs][Q]: partition has a non-zero tap
  float* y;    // [B][J][y_stride]
  long y_stride;
};

// Row pairs: filter group g (g < S: full filters of speaker g, S <= g < 2S:
// early filters of speaker g - S, g = 2S: the noise) pairs mics 2h and 2h + 1,
// so both rows of a pair convolve the same source and the short early
// filters pair with each other (their zero partitions are skipped).  Without
// early filters the early groups are not run: the full pair writes both.
struct Pair {
  int ja, jb, src;  // rows (jb = -1: no partner) and source
  bool dup;         // also write rows ja + S M, jb + S M (early == full)
};
__device__ __forceinline__ Pair pair_rows(int pi, const ConvArgs& A) {
  int g = pi / A.hm;
  const int h = pi - g * A.hm;
  if (!A.rir_early && g >= A.S) g += A.S;
  Pair P;
  P.ja = g * A.M + 2 * h;
  P.jb = 2 * h + 1 < A.M ? P.ja + 1 : -1;
  P.src = g < A.S ? g : g < 2 * A.S ? g - A.S : A.S;
  P.dup = !A.rir_early && g < A.S;
  return P;
}

// Samples base + threadIdx.x + 512 i (i < 16) of source k of item b: speaker k
// placed at its offset, or (k = S) the point noise tiled to the dry length.
__device__ __forceinline__ void load_block(const ConvArgs& A, int k, int b, long base, float (&vals)[16]) {
  if (k < A.S) {
    const long o = A.off[b * A.S + k], n = A.len[b * A.S + k];
    const float* src = A.dry + (size_t)b * A.dry_sb + (size_t)k * A.dry_sk;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const long q = base + threadIdx.x + i * kFftThreads - o;
      vals[i] = q >= 0 && q < n ? __ldg(src + q) : 0.f;
    }
  } else {
    const long dl = A.dlen[b], nl = A.nlen[b];
    const float* src = A.noise + (size_t)b * A.noise_sb;
    long pos = base + threadIdx.x;
    long q = pos >= 0 ? pos % nl : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i, pos += kFftThreads) {
      vals[i] = pos >= 0 && pos < dl ? __ldg(src + q) : 0.f;
      if (pos >= 0) {
        q += kFftThreads;
        while (q >= nl) q -= nl;
      } else if (pos + kFftThreads >= 0) {
        q = (pos + kFftThreads) % nl;
      }
    }
  }
}

// Pass 4 of a transform whose input was two real blocks packed as z = a + i b,
// split into their spectra: X_a[f] = (Z[f] + conj Z[N-f]) / 2 and
// X_b[f] = (Z[f] - conj Z[N-f]) / 2i.  Thread t takes the butterflies
// j = t + 512 q (q < 4) and their mirrors P - j (twiddle W^{P-j} = -conj W^j),
// so Z[f] and Z[N-f] meet in one thread; butterflies 0 and 2048 are their own
// mirrors (thread 0).  xb may be null (no second block).
__device__ __forceinline__ void fft_last_real_pair(const float2* buf, const float2* tws, float2* xa, float2* xb) {
  constexpr float kC[4] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f};
  constexpr float kS[4] = {0.f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  const int t = threadIdx.x;
  const float2 wt = tws[t];
  auto bfly = [&](int j, float2 w, float2& z0, float2& z1) {  // Z[j], Z[j + P]
    const int sj = swz(j);
    const float2 a = buf[sj], c = cmulf(buf[sj + kFftP], w);
    z0 = addf(a, c);
    z1 = subf(a, c);
  };
  auto emit = [&](int f, float2 zf, float2 zm) {  // zm = Z[N - f]
    xa[f] = make_float2(0.5f * (zf.x + zm.x), 0.5f * (zf.y - zm.y));
    if (xb) xb[f] = make_float2(0.5f * (zf.y + zm.y), 0.5f * (zm.x - zf.x));
  };
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j1 = t + 512 * q;
    const float2 w1 = q == 0 ? wt : cmulc(wt, kC[q], -kS[q]);  // W^{j1}
    float2 z1a, z1b;
    bfly(j1, w1, z1a, z1b);
    if (j1 == 0) {
      emit(0, z1a, z1a);
      emit(kFftP, z1b, z1b);
      float2 za, zb;
      bfly(2048, make_float2(0.f, -1.f), za, zb);  // W^2048 = -i
      emit(2048, za, zb);
      emit(2048 + kFftP, zb, za);
    } else {
      const int j2 = kFftP - j1;
      float2 z2a, z2b;
      bfly(j2, make_float2(-w1.x, w1.y), z2a, z2b);
      emit(j1, z1a, z2b);
      emit(j1 + kFftP, z1b, z2a);
      emit(j2, z2a, z1b);
      emit(j2 + kFftP, z2b, z1a);
    }
  }
}

// X_t = FFT of the placed dry signal (speaker k at its offset, or the tiled
// noise) over [(t-1)P, (t+1)P).  Blocks 2u and 2u + 1 ride in one complex
// transform (real and imaginary parts).  Grid (ceil(nb / 2), S+1, B).
__global__ void __launch_bounds__(kFftThreads, 2) fft_in_kernel(ConvArgs A) {
  extern __shared__ __align__(16) float2 buf[];
  const int u = blockIdx.x, k = blockIdx.y, b = blockIdx.z;
  const int t0 = 2 * u;
  const bool two = t0 + 1 < A.nb;
  const float2* tws = load_twiddles(buf, A.tw);
  {  // butterfly j = threadIdx.x of pass 1 reads samples j + 512 r
    float va[16], vb[16];
    load_block(A, k, b, (long)(t0 - 1) * kFftP, va);
    if (two) {
      load_block(A, k, b, (long)t0 * kFftP, vb);
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) vb[r] = 0.f;
    }
    float2 x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = make_float2(va[r], vb[r]);
    fft_first(buf, x);
  }
  fft_mid(buf, tws);
  float2* out = A.X + (((size_t)b * (A.S + 1) + k) * A.nb + t0) * kFftN;
  fft_last_real_pair(buf, tws, out, two ? out + kFftN : nullptr);
}

// H_p = FFT(h_a + i h_b) over taps [pP, pP + P).  Grid (Q, npairs, B).
__global__ void __launch_bounds__(kFftThreads, 2) fft_filt_kernel(ConvArgs A) {
  extern __shared__ __align__(16) float2 buf[];
  const int p = blockIdx.x, pi = blockIdx.y, b = blockIdx.z;
  const int M = A.M, S = A.S, r = A.rlen[b];
  if (p * kFftP >= r) return;  // partitions past this item's filter length are never read
  const Pair pr = pair_rows(pi, A);
  const int ja = pr.ja, jb = pr.jb;
  auto row = [&](int j) -> const float* {
    if (j < S * M) return A.rir_full + (size_t)b * A.full_sb + (size_t)j * A.R;
    if (j < 2 * S * M) {
      const int jj = j - S * M;
      return A.rir_early ? A.rir_early + (size_t)b * A.early_sb + (size_t)jj * A.R
                         : A.rir_full + (size_t)b * A.full_sb + (size_t)jj * A.R;
    }
    return A.rir_full + (size_t)b * A.full_sb + ((size_t)S * M + (j - 2 * S * M)) * A.R;
  };
  const float* ha = row(ja);
  const float* hb = jb >= 0 ? row(jb) : nullptr;
  const float2* tws = load_twiddles(buf, A.tw);
  {
    const int j = threadIdx.x;
    float2 x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {  // taps j + 512 q of the partition; the upper half is padding
      const int u = j + q * kFftThreads, tap = p * kFftP + u;
      float va = 0.f, vb = 0.f;
      if (q < 8 && tap < r) {
        va = __ldg(ha + tap);
        if (hb) vb = __ldg(hb + tap);
      }
      x[q] = make_float2(va, vb);
    }
    bool nz = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) nz |= x[q].x != 0.f || x[q].y != 0.f;
    const bool live = __syncthreads_or(nz);
    if (threadIdx.x == 0) A.live[((size_t)b * A.npairs + pi) * A.Q + p] = live;
    if (!live) return;  // all-zero partition (the tail of an early filter): skipped by the convolution
    fft_first(buf, x);
  }
  fft_mid(buf, tws);
  float2* out = A.H + (((size_t)b * A.npairs + pi) * A.Q + p) * kFftN;
  fft_last(buf, tws, [&](int j, float2 x0, float2 x1) {
    out[j] = x0;
    out[j + kFftP] = x1;
  });
}

// Output block t of a pair: sum_p X_{t-p} H_p, inverse FFT (conj trick),
// last P samples -> y_a (real), y_b (imag).  Grid (nb, npairs, B).
__global__ void __launch_bounds__(kFftThreads, 2) fft_conv_kernel(ConvArgs A) {
  extern __shared__ __align__(16) float2 buf[];
  const int t = blockIdx.x, pi = blockIdx.y, b = blockIdx.z;
  const Pair pr = pair_rows(pi, A);
  const int ja = pr.ja, jb = pr.jb;
  const float2* Xs = A.X + ((size_t)b * (A.S + 1) + pr.src) * A.nb * kFftN;
  const int32_t* live = A.live + ((size_t)b * A.npairs + pi) * A.Q;
  const float2* Hs = A.H + ((size_t)b * A.npairs + pi) * A.Q * kFftN;
  const int qb = (A.rlen[b] + kFftP - 1) / kFftP;  // this item's non-zero partitions
  const int qmax = min(qb - 1, t);
  const float2* tws = load_twiddles(buf, A.tw);
  {  // butterfly j = threadIdx.x of pass 1 reads bins j + 512 r
    const int j = threadIdx.x;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = make_float2(0.f, 0.f);
    for (int p = 0; p <= qmax; ++p) {
      if (!live[p]) continue;  // block-uniform
      const float2* xp = Xs + (size_t)(t - p) * kFftN + j;
      const float2* hp = Hs + (size_t)p * kFftN + j;
#pragma unroll
      for (int c = 0; c < 16; c += 8) {
        float2 x[8], hh[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          x[r] = __ldg(xp + (c + r) * kFftThreads);
          hh[r] = __ldg(hp + (c + r) * kFftThreads);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          v[c + r].x = fmaf(x[r].x, hh[r].x, fmaf(-x[r].y, hh[r].y, v[c + r].x));
          v[c + r].y = fmaf(x[r].x, hh[r].y, fmaf(x[r].y, hh[r].x, v[c + r].y));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r].y = -v[r].y;  // conj: IFFT(z) = conj(FFT(conj(z))) / N
    fft_first(buf, v);
  }
  fft_mid(buf, tws);
  const float inv = 1.0f / kFftN;
  float* ya = A.y + ((size_t)b * ((2 * A.S + 1) * A.M) + ja) * A.y_stride + (size_t)t * kFftP;
  float* yb = jb >= 0 ? A.y + ((size_t)b * ((2 * A.S + 1) * A.M) + jb) * A.y_stride + (size_t)t * kFftP : nullptr;
  const size_t dup = pr.dup ? (size_t)A.S * A.M * A.y_stride : 0;  // early rows = full rows
  fft_last(buf, tws, [&](int n, float2, float2 z1) {  // the last P outputs: X[n + P]
    ya[n] = z1.x * inv;
    if (yb) yb[n] = -z1.y * inv;
    if (dup) {
      ya[dup + n] = z1.x * inv;
      if (yb) yb[dup + n] = -z1.y * inv;
    }
  });
}

// Twiddle table exp(-2 pi i m / N), m < N, per device (FP64-computed).
const float2* twiddles(std::string* err) {
  static std::mutex mu;
  static const float2* tab[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (dev < 0 || dev >= 64) { *err = "device index out of range"; return nullptr; }
  if (!tab[dev]) {
    std::vector<float2> h(kFftN);
    for (int m = 0; m < kFftN; ++m) {
      const double a = -2.0 * M_PI * (double)m / (double)kFftN;
      h[m] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    float2* d = nullptr;
    cudaError_t e = cudaMalloc((void**)&d, kFftN * sizeof(float2));
    if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), kFftN * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return nullptr; }
    tab[dev] = d;
  }
  return tab[dev];
}

}  // namespace
}  // namespace frir

using namespace frir;

extern "C" {

int64_t frir_mix_convolve_scratch(int32_t B, int32_t S, int32_t M, int64_t R, int64_t T, int64_t* y_stride) {
  if (B < 0 || S < 1 || M < 1 || R < 1 || T < 1) return -1;
  const int64_t nb = (T + kFftP - 1) / kFftP;
  const int64_t Q = (R + kFftP - 1) / kFftP;
  const int64_t npairs = (int64_t)(2 * S + 1) * ((M + 1) / 2);
  if (y_stride) *y_stride = nb * kFftP;
  const int64_t flags = ((int64_t)B * npairs * Q * 4 + 255) & ~(int64_t)255;
  return ((int64_t)B * (S + 1) * nb + (int64_t)B * npairs * Q) * kFftN * (int64_t)sizeof(float2) + flags;
}

int frir_mix_convolve(const float* dry, int64_t dry_stride_b, int64_t dry_stride_k, const float* noise,
                      int64_t noise_stride, const int32_t* offsets, const int32_t* lengths, const int32_t* noise_len,
                      const int32_t* dry_len, const float* rir_full, int64_t full_stride_b, const float* rir_early,
                      int64_t early_stride_b, const int32_t* rir_len, int32_t B, int32_t S, int32_t M, int64_t R,
                      int64_t T, void* scratch, int64_t scratch_bytes, float* y, int64_t y_stride, void* stream) {
  int64_t ys = 0;
  const int64_t need = frir_mix_convolve_scratch(B, S, M, R, T, &ys);
  if (!dry || !noise || !offsets || !lengths || !noise_len || !dry_len || !rir_full || !rir_len || !scratch || !y ||
      need < 0 || scratch_bytes < need || y_stride < ys) {
    set_error("frir_mix_convolve: invalid argument or scratch/y too small");
    return FRIR_EINVAL;
  }
  if (B == 0) return FRIR_OK;
  std::string err;
  const float2* tw = twiddles(&err);
  if (!tw) { set_error("frir_mix_convolve: " + err); return FRIR_ECUDA; }
  ConvArgs a;
  a.dry = dry; a.dry_sb = (long)dry_stride_b; a.dry_sk = (long)dry_stride_k;
  a.noise = noise; a.noise_sb = (long)noise_stride;
  a.off = offsets; a.len = lengths; a.nlen = noise_len; a.dlen = dry_len;
  a.rir_full = rir_full; a.full_sb = (long)full_stride_b; a.rir_early = rir_early; a.early_sb = (long)early_stride_b;
  a.rlen = rir_len;
  a.S = S; a.M = M; a.R = (int)R;
  a.nb = (int)((T + kFftP - 1) / kFftP);
  a.Q = (int)((R + kFftP - 1) / kFftP);
  a.hm = (M + 1) / 2;
  a.npairs = (rir_early ? 2 * S + 1 : S + 1) * a.hm;  // no early filters: the full pairs write both
  a.tw = tw;
  a.X = (float2*)scratch;
  a.H = a.X + (size_t)B * (S + 1) * a.nb * kFftN;
  a.live = (int32_t*)(a.H + (size_t)B * a.npairs * a.Q * kFftN);
  a.y = y; a.y_stride = (long)y_stride;
  const size_t smem = kFftSmem;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  for (auto k : {(const void*)fft_in_kernel, (const void*)fft_filt_kernel, (const void*)fft_conv_kernel}) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) break;
  }
  if (e == cudaSuccess) {
    fft_in_kernel<<<dim3((a.nb + 1) / 2, S + 1, B), kFftThreads, smem, st>>>(a);
    fft_filt_kernel<<<dim3(a.Q, a.npairs, B), kFftThreads, smem, st>>>(a);
    fft_conv_kernel<<<dim3(a.nb, a.npairs, B), kFftThreads, smem, st>>>(a);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) { set_error(std::string("frir_mix_convolve: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

}  // extern "C"
