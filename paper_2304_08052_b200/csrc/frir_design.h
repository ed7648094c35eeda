// Host-side filter design for one sample rate (FP64).  Restates, without
// scipy, the tables the reference builds per call:
//   resample.py:59-71   rate_factors
//   resample.py:74-78   _decimation_taps -> scipy.signal.firwin(kaiser 7.0)
//   resample.py:107     resample_poly(x, r_l, r_h) conventions (gcd, gain, offsets)
//   resample.py:109-110 butter(2, 80, 'highpass', fs=r_l*fs, output='sos')
//   resample.py:113     resample_poly(y, 1, r_l)
// and derives from them the output-rate composite tables the render kernel
// gathers.
#pragma once
#include <complex>
#include <string>
#include <vector>

#include "../../include/frir.h"

namespace frir {

struct Design {
  frir_plan_desc d{};
  std::vector<double> h1, h2;          // Kaiser taps (firwin-normalised, unscaled by up)
  std::vector<double> comp_d, comp_w;  // r_h*sup entries each, index t - t0
  std::vector<double> kappa;           // [half2][2]
  std::vector<double> u;               // [half2]
  std::vector<double> zphase;          // [down][2]
  std::vector<double> ppow;            // [horizon][2]
  std::vector<double> ppow_lo, ppow_hi; // p^i (i < 128), p^(128 j) (j <= horizon / 128): [][2]
  std::vector<double> lpcoef;          // c1, c2, v0 (re0, im0, re1, im1)
  std::vector<double> h1up;            // up * h1 (stage-1 taps as applied)
  std::vector<double> gw;              // h2 * N * B' (low-pass branch filter, len2 + 2 r_l)
};

// Returns false and sets *err on an invalid sample rate (rate_factors rules).
bool design(int sample_rate, Design* out, std::string* err);
// Only the integer rate constants (r_h, r_l, up, down, filter lengths).
bool rate_constants(int sample_rate, frir_plan_desc* d, std::string* err);

}  // namespace frir
