// Host filter design: see frir_design.h.  Everything here runs once per plan.
#include "frir_design.h"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace frir {
namespace {

using cplx = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;

// Modified Bessel I0 by its power series in long double (scipy.special.i0 is a
// Cephes Chebyshev fit; both are accurate to ~1 ulp in double).
double bessel_i0(double x) {
  long double half = (long double)x / 2.0L, term = 1.0L, sum = 1.0L;
  for (int k = 1; k < 500; ++k) {
    term *= (half / k) * (half / k);
    sum += term;
    if (term < sum * 1e-21L) break;
  }
  return (double)sum;
}

// scipy.signal.windows.kaiser(M, beta, sym=True)
std::vector<double> kaiser(int m, double beta) {
  std::vector<double> w(m);
  double alpha = (m - 1) / 2.0, den = bessel_i0(beta);
  for (int n = 0; n < m; ++n) {
    double r = (n - alpha) / alpha;
    w[n] = bessel_i0(beta * std::sqrt(1.0 - r * r)) / den;
  }
  return w;
}

double np_sinc(double x) {
  double y = kPi * (x == 0.0 ? 1.0e-20 : x);
  return std::sin(y) / y;
}

// scipy.signal.firwin(numtaps, cutoff, window=('kaiser', beta)) with the
// default pass_zero=True, scale=True, fs=2 (cutoff relative to Nyquist).
std::vector<double> firwin_kaiser(int numtaps, double cutoff, double beta) {
  std::vector<double> h(numtaps), win = kaiser(numtaps, beta);
  double alpha = 0.5 * (numtaps - 1);
  long double s = 0.0L;
  for (int n = 0; n < numtaps; ++n) {
    double m = n - alpha;
    h[n] = cutoff * np_sinc(cutoff * m) * win[n];
    s += h[n];
  }
  for (double& v : h) v /= (double)s;
  return h;
}

// Direct-form polynomial of a set of complex roots (numpy.poly).
std::vector<cplx> poly(const std::vector<cplx>& roots) {
  std::vector<cplx> c{1.0};
  for (const cplx& r : roots) {
    std::vector<cplx> n(c.size() + 1, 0.0);
    for (size_t i = 0; i < c.size(); ++i) {
      n[i] += c[i];
      n[i + 1] -= r * c[i];
    }
    c.swap(n);
  }
  return c;
}

// scipy.signal.butter(2, f, 'highpass', fs=fs, output='sos'): buttap ->
// lp2hp_zpk -> bilinear_zpk -> zpk2sos (one section).
void butter2_highpass(double f, double fs, double sos[6]) {
  const int order = 2;
  double wn = 2.0 * f / fs;
  double fs_int = 2.0;
  double warped = 2.0 * fs_int * std::tan(kPi * wn / fs_int);
  std::vector<cplx> p;
  for (int m = -order + 1; m < order; m += 2)
    p.push_back(-std::exp(cplx(0.0, 1.0) * (kPi * m / (2.0 * order))));
  // lp2hp_zpk: z = [0, 0], p = wo / p, k = real(1 / prod(-p))
  cplx prod_negp = 1.0;
  for (const cplx& v : p) prod_negp *= -v;
  double k_hp = std::real(cplx(1.0) / prod_negp);
  std::vector<cplx> p_hp, z_hp(order, 0.0);
  for (const cplx& v : p) p_hp.push_back(warped / v);
  // bilinear_zpk, fs = 2 -> fs2 = 4
  double fs2 = 2.0 * fs_int;
  std::vector<cplx> z_z, p_z;
  cplx num = 1.0, den = 1.0;
  for (const cplx& z : z_hp) {
    z_z.push_back((fs2 + z) / (fs2 - z));
    num *= (fs2 - z);
  }
  for (const cplx& v : p_hp) {
    p_z.push_back((fs2 + v) / (fs2 - v));
    den *= (fs2 - v);
  }
  double k_z = k_hp * std::real(num / den);
  std::vector<cplx> b = poly(z_z), a = poly(p_z);
  for (int i = 0; i < 3; ++i) sos[i] = k_z * std::real(b[i]);
  sos[3] = std::real(a[0]);
  sos[4] = std::real(a[1]);
  sos[5] = std::real(a[2]);
}

std::vector<double> convolve(const std::vector<double>& a, const std::vector<double>& b) {
  std::vector<double> c(a.size() + b.size() - 1, 0.0);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) c[i + j] += a[i] * b[j];
  return c;
}

int floordiv(long a, long b) { return (int)((a >= 0) ? a / b : -((-a + b - 1) / b)); }

}  // namespace

bool rate_constants(int fs, frir_plan_desc* dp, std::string* err) {
  if (fs <= 0) {
    *err = "sample_rate must be > 0, got " + std::to_string(fs);
    return false;
  }
  frir_plan_desc& d = *dp;
  d = frir_plan_desc{};
  d.sample_rate = fs;
  d.r_h = 1000000 / fs;
  d.r_l = (int)std::floor(std::sqrt((double)d.r_h));
  while ((long)(d.r_l + 1) * (d.r_l + 1) <= d.r_h) ++d.r_l;
  while ((long)d.r_l * d.r_l > d.r_h) --d.r_l;
  if (!(1 < d.r_l && d.r_l < d.r_h)) {
    *err = "sample_rate " + std::to_string(fs) + " leaves no room for the two-stage chain (r_h=" +
           std::to_string(d.r_h) + ", r_l=" + std::to_string(d.r_l) + ")";
    return false;
  }
  const int taps_per_phase = 10;
  int g = std::gcd(d.r_l, d.r_h);
  d.up = d.r_l / g;
  d.down = d.r_h / g;
  int m1 = std::max(d.r_l, d.r_h);
  d.len1 = 2 * taps_per_phase * m1 + 1;
  d.half1 = (d.len1 - 1) / 2;
  d.len2 = 2 * taps_per_phase * d.r_l + 1;
  d.half2 = (d.len2 - 1) / 2;
  return true;
}

bool design(int fs, Design* out, std::string* err) {
  Design& D = *out;
  if (!rate_constants(fs, &D.d, err)) return false;
  frir_plan_desc& d = D.d;
  const double beta = 7.0;
  int m1 = std::max(d.r_l, d.r_h);
  D.h1 = firwin_kaiser(d.len1, 1.0 / m1, beta);
  D.h2 = firwin_kaiser(d.len2, 1.0 / d.r_l, beta);
  D.h1up.resize(d.len1);
  for (int i = 0; i < d.len1; ++i) D.h1up[i] = D.h1[i] * d.up;  // resample_poly: h *= up
  butter2_highpass(80.0, (double)d.r_l * fs, d.sos);

  const double b0 = d.sos[0], b1 = d.sos[1], b2 = d.sos[2], a1 = d.sos[4], a2 = d.sos[5];
  // LP = 1 - HP = N(z)/A(z);  1/A(z) = B'(z) / A_R(z^{r_l})
  std::vector<double> nlp = {1.0 - b0, a1 - b1, a2 - b2};
  cplx disc = std::sqrt(cplx(a1 * a1 - 4.0 * a2, 0.0));
  cplx pole = (-a1 + disc) / 2.0;  // upper-half-plane pole p
  cplx poles[2] = {pole, std::conj(pole)};
  std::vector<cplx> bp{1.0};
  for (const cplx& pl : poles) {
    std::vector<cplx> geo(d.r_l), nb(bp.size() + d.r_l - 1, 0.0);
    cplx pk = 1.0;
    for (int k = 0; k < d.r_l; ++k) { geo[k] = pk; pk *= pl; }
    for (size_t i = 0; i < bp.size(); ++i)
      for (int k = 0; k < d.r_l; ++k) nb[i + k] += bp[i] * geo[k];
    bp.swap(nb);
  }
  std::vector<double> bpr(bp.size());
  for (size_t i = 0; i < bp.size(); ++i) bpr[i] = std::real(bp[i]);
  cplx P = std::pow(pole, d.r_l);
  d.c1 = 2.0 * std::real(P);
  d.c2 = -std::norm(P);
  std::vector<double> gfilt = convolve(convolve(D.h2, nlp), bpr);
  D.gw = gfilt;

  // Composite tables T(t) = up * sum_k h1[down k + half1 + up t] * F[half2 - k].
  auto composite = [&](const std::vector<double>& filt, int tmin, int tmax) {
    std::vector<double> T(tmax - tmin + 1, 0.0);
    int fl = (int)filt.size();
    for (int t = tmin; t <= tmax; ++t) {
      long double s = 0.0L;
      for (int j = 0; j < fl; ++j) {  // j = half2 - k
        int k = d.half2 - j;
        long idx = (long)d.down * k + d.half1 + (long)d.up * t;
        if (idx < 0 || idx >= d.len1) continue;
        s += (long double)D.h1[idx] * filt[j];
      }
      T[t - tmin] = (double)(s * d.up);
    }
    return T;
  };
  // Bounds: h1 index within [0, len1) for some k in [half2 - fl + 1, half2].
  int fl_w = (int)gfilt.size();
  int kmin = d.half2 - fl_w + 1, kmax = d.half2;
  int tmin = floordiv(-(long)d.half1 - (long)d.down * kmax, d.up) - 1;
  int tmax = floordiv((long)d.len1 - d.half1 - (long)d.down * kmin, d.up) + 1;
  std::vector<double> TD = composite(D.h2, tmin, tmax), TW = composite(gfilt, tmin, tmax);
  int first = (int)TD.size(), last = -1;
  for (int i = 0; i < (int)TD.size(); ++i)
    if (TD[i] != 0.0 || TW[i] != 0.0) { first = std::min(first, i); last = i; }
  d.t0 = tmin + first;
  int span = last - first + 1;
  d.sup = (span + d.r_h - 1) / d.r_h;
  D.comp_d.assign((size_t)d.r_h * d.sup, 0.0);
  D.comp_w.assign((size_t)d.r_h * d.sup, 0.0);
  for (int i = 0; i < span; ++i) {
    D.comp_d[i] = TD[first + i];
    D.comp_w[i] = TW[first + i];
  }
  d.nb = (d.sup - 1 + 31) / 32;
  if (d.nb < 1) d.nb = 1;

  // Tail correction (truncation of the mid-rate signal at n1, resample.py:107-113).
  // TDF-II state s(n+1) = A s(n) + B x(n), z(n) = b0 x(n) + s1(n).
  double A[2][2] = {{-a1, 1.0}, {-a2, 0.0}};
  double B[2] = {b1 - a1 * b0, b2 - a2 * b0};
  // eigenvector of A for eigenvalue p: (1, p + a1); s = 2 Re(v0 * zeta)
  cplx v0a = 1.0, v0b = pole + a1;
  cplx v1a = 1.0, v1b = std::conj(pole) + a1;
  cplx det = v0a * v1b - v1a * v0b;  // V = [[v0a v1a],[v0b v1b]]
  cplx w0 = (v1b * B[0] - v1a * B[1]) / det;  // first row of V^-1 times B
  cplx v0[2] = {v0a * w0, v0b * w0};
  D.lpcoef = {d.c1, d.c2, std::real(v0[0]), std::imag(v0[0]), std::real(v0[1]), std::imag(v0[1])};

  double rho = std::abs(pole);
  d.horizon = (int)std::ceil(std::log(1e-9) / std::log(rho));  // items beyond feed < 1e-9 of their amplitude
  D.ppow.resize((size_t)2 * d.horizon);
  {
    cplx pm = 1.0;
    for (int m = 0; m < d.horizon; ++m) {
      if (m % 64 == 0) pm = std::pow(pole, m);  // re-anchor to limit drift
      D.ppow[2 * m] = std::real(pm);
      D.ppow[2 * m + 1] = std::imag(pm);
      pm *= pole;
    }
  }
  {  // two-level power table for the render kernel: p^m = hi[m >> 7] * lo[m & 127]
    const int nhi = d.horizon / 128 + 1;
    D.ppow_lo.resize(256);
    D.ppow_hi.resize((size_t)2 * nhi);
    for (int i = 0; i < 128; ++i) {
      cplx v = std::pow(pole, i);
      D.ppow_lo[2 * i] = std::real(v);
      D.ppow_lo[2 * i + 1] = std::imag(v);
    }
    for (int j = 0; j < nhi; ++j) {
      cplx v = std::pow(pole, 128 * j);
      D.ppow_hi[2 * j] = std::real(v);
      D.ppow_hi[2 * j + 1] = std::imag(v);
    }
  }
  // Z[rho] = sum_{j>=0} p^j * up*h1[2 half1 - rho - down j]
  D.zphase.assign((size_t)2 * d.down, 0.0);
  for (int ph = 0; ph < d.down; ++ph) {
    cplx s = 0.0, pj = 1.0;
    for (int j = 0;; ++j) {
      long idx = 2L * d.half1 - ph - (long)d.down * j;
      if (idx < 0) break;
      s += pj * D.h1up[idx];
      pj *= pole;
    }
    D.zphase[2 * ph] = std::real(s);
    D.zphase[2 * ph + 1] = std::imag(s);
  }
  // HP impulse response and the two tail tables over e in [0, half2).
  int ne = d.half2;
  std::vector<double> hhp(ne + 1);
  {
    double s[2] = {B[0], B[1]};
    hhp[0] = b0;
    for (int j = 1; j <= ne; ++j) {
      hhp[j] = s[0];
      double t0v = A[0][0] * s[0] + A[0][1] * s[1], t1v = A[1][0] * s[0] + A[1][1] * s[1];
      s[0] = t0v;
      s[1] = t1v;
    }
  }
  D.kappa.assign((size_t)2 * ne, 0.0);
  D.u.assign(ne, 0.0);
  for (int e = 0; e < ne; ++e) {
    double r0[2] = {1.0, 0.0};  // [1 0] A^j
    double k0 = 0.0, k1 = 0.0;
    for (int j = 0; j <= e; ++j) {
      k0 += D.h2[e - j] * r0[0];
      k1 += D.h2[e - j] * r0[1];
      double n0 = r0[0] * A[0][0] + r0[1] * A[1][0], n1 = r0[0] * A[0][1] + r0[1] * A[1][1];
      r0[0] = n0;
      r0[1] = n1;
    }
    D.kappa[2 * e] = k0;
    D.kappa[2 * e + 1] = k1;
    double uu = 0.0;
    for (int j = 0; j <= e; ++j) uu += D.h2[e - j] * hhp[j];
    D.u[e] = uu;
  }
  d.lt_max = (d.half1 - d.up) / d.down + 2;
  if (d.lt_max < 1) d.lt_max = 1;
  return true;
}

}  // namespace frir
