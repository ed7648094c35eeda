// Internal structures shared by the C-ABI layer and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_design.h"

namespace frir {

constexpr int kWin = 32;        // outputs per gather window (one per lane)
constexpr int kTileWin = 4;     // windows per LP-scan tile
constexpr int kTile = kWin * kTileWin;
constexpr int kChunk = kTile / 32;  // serial outputs per lane in the scan
// Output-rate grid offset n'' = n + kExt.  The LP recursion needs W from
// n = -half2 / r_l = -10 on (zero before that); 32 keeps n'' windows aligned
// with output windows so the scan can store float4s.
constexpr int kExt = 32;
constexpr int kSpBias = 64;     // bias of the packed start index
constexpr int kMaxRows = 1 << 22;  // max images + 1 per job (item index arithmetic)
constexpr int kLtMax = 128;     // max stage-1 taps past n1 (lt_max = (half1 - up) / down + 2, 91 at 11025 Hz)
// Per-warp row length of the render kernel's past-n1 tap sums, sized per rate
// so the 16 kHz plan keeps two CTAs per SM.
__host__ __device__ inline int lt_cap(const frir_plan_desc& d) { return (d.lt_max + 31) & ~31; }

// Device-resident, read-only per-plan data (uploaded once by frir_plan_create).
struct DevPlan {
  frir_plan_desc d;
  float2* comp;        // [r_h][sup] (TD, TW), phase-major
  double* h1up;        // [len1]
  double* h2;          // [len2]
  double* gw;          // [len2 + 2 r_l]
  double* ppow;        // [horizon][2]
  double* ppow_lo;     // [128][2]   p^i
  double* ppow_hi;     // [nhi][2]   p^(128 j), nhi = horizon / 128 + 1
  double* zphase;      // [down][2]
  double* kappa;       // [half2][2]
  double* u;           // [half2]
  double* scan;        // LP scan constants, see kernels (kScanDoubles)
  double lp[6];        // c1, c2, v0
  // LP scan constants the render kernel reads as kernel parameters (constant
  // bank operands, no shared-memory traffic); see lp_scan_tile
  double ks[20];        // Kogge-Stone powers M^(C 2^s), s < 5
  double mc[4];         // M^C (one chunk)
  double fr0[2 * kChunk];  // row0(M^(k+1)), k < C
  double mt[4];         // M^kTile
};

// LP scan constants: KS powers M^(C 2^s) (5 x 4), M^(C L) (32 x 4), free
// response row0(M^(k+1)) for k < kTile (kTile x 2), M^kTile (4).
constexpr int kScanKS = 0, kScanStart = 20, kScanFree = 20 + 128, kScanTileM = kScanFree + 2 * kTile;
constexpr int kScanDoubles = kScanTileM + 4;

// Device facts and kernel attributes queried once per plan (frir_plan_create),
// so launches issue no attribute or occupancy queries.
struct LaunchCache {
  int sms = 148;
  int smem_optin = 227 * 1024;  // max dynamic smem per block (opt-in)
  int render_per_sm[2][2][2] = {};  // [EARLY][NBK - 1][SEG]: resident render CTAs per SM
  int render_e_per_sm[2] = {};      // [NBK - 1]: the early pass
};

}  // namespace frir

struct frir_plan {
  frir::Design design;
  frir::DevPlan dev;
  int device;
  frir::LaunchCache lc;
};

namespace frir {
void set_error(const std::string& msg);
int launch_simulate(const frir_plan* plan, const frir_batch* b, void* ws, size_t ws_bytes,
                    float* out_full, float* out_early, int32_t* direct_index, cudaStream_t st,
                    int stages);
size_t workspace_bytes(const frir_batch* b);
int launches(const frir_batch* b, int early);
cudaError_t init_launch_cache(frir_plan* plan);
int launch_image_set(const frir_plan* plan, const frir_batch* b, double* dist, double* az, double* el,
                     double* ratio, double* refl, double* mic_dist, int with_refl, cudaStream_t st);
int train_nonzeros(const double* train, int64_t ld, int32_t rows, int32_t L, int32_t sign, int32_t* counts,
                   cudaStream_t st);
int launch_simulate_train(const frir_plan* plan, const frir_batch* b, void* ws, size_t ws_bytes,
                          const double* train, int64_t ld, int32_t sign, float* out_full, int32_t* direct_scratch,
                          cudaStream_t st);
int check_line();
}  // namespace frir
