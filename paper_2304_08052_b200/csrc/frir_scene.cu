// On-device scene sampler: the reference's sample_scene
// (framrir/mixture.py:171-213) for a range of item indices, written straight
// into render jobs -- no host work per room.
//
// Item i draws from Philox(SeedSequence((seed, first + i))) exactly like
// numpy's Generator in sample_scene: room (3 uniforms), T60, then per source
// (the speakers, then the point noise) distance / azimuth / elevation, then the
// simulation seed rng.integers(2**63) (Lemire's bounded draw with range 2^63
// is the raw word >> 1).  Every uniform is low + (high - low) * u with
// u = (word >> 11) * 2^-53, one word each, so the draws are bit-identical to
// the host's.  The derived job fields follow frir_jobs_prepare (SimParams
// defaults, reference rules); rows are laid out with a fixed stride sized
// for the spec's longest T60, so no prefix sum is needed.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/frir.h"
#include "frir_internal.h"
#include "frir_philox.cuh"

namespace frir {
namespace {

__device__ __forceinline__ double uniform_rn(const uint64_t key[2], uint64_t w, double lo, double hi) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u64_to_unit(stream_word(key, w))));
}

struct SceneArgs {
  frir_scene_spec S;
  uint64_t seed;
  int64_t first;
  int count;
  int r_h, r_l, up, down, rate;
  frir_job* jobs;
  int32_t* chan_job;
  int32_t* status;
};

__global__ void scene_jobs_kernel(const __grid_constant__ SceneArgs A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.count) return;
  const frir_scene_spec& S = A.S;
  const uint64_t vals[2] = {A.seed, (uint64_t)(A.first + i)};
  uint64_t key[2];
  seed_keys_n(vals, 2, key);
  double room[3];
  room[0] = uniform_rn(key, 0, S.room_length[0], S.room_length[1]);
  room[1] = uniform_rn(key, 1, S.room_width[0], S.room_width[1]);
  room[2] = uniform_rn(key, 2, S.room_height[0], S.room_height[1]);
  const double t60 = uniform_rn(key, 3, S.t60[0], S.t60[1]);
  const int S1 = S.n_sources;
  const uint64_t sim_seed = stream_word(key, 4 + 3 * (uint64_t)S1) >> 1;  // rng.integers(2**63)
  // reflection coefficient (core.py:113-128)
  const double lx = room[0], ly = room[1], lz = room[2];
  const double ratio = __ddiv_rn(lx * ly * lz, 2.0 * (lx * ly + lx * lz + ly * lz));
  const double tt = 1.0 - exp(-0.16 * ratio / t60);
  const double r = sqrt(1.0 - tt * tt);
  const double c0 = S.c0;
  const int L = (int)ceil(t60 * (double)A.rate);
  const int64_t n1 = ((int64_t)L * A.up + A.down - 1) / A.down;
  const int n2 = (int)((n1 + A.r_l - 1) / A.r_l);
  int st = 0;
  if (!(S.aperture < fmin(lx, fmin(ly, lz)))) st = 1;  // Scene aperture rule (params.py:94-99)
  if (n2 > S.out_stride) st = 4;
  const int rows = S.num_images + 1;
  const int M = S.n_mics;
  for (int k = 0; k < S1; ++k) {
    const double d0 = uniform_rn(key, 4 + 3 * k, S.distance[0], S.distance[1]);
    const double az = uniform_rn(key, 5 + 3 * k, 0.0, 6.283185307179586);
    const double el = uniform_rn(key, 6 + 3 * k, S.elevation[0], S.elevation[1]);
    const int j = i * S1 + k;
    frir_job J;
    memset(&J, 0, sizeof(J));
    J.room[0] = lx; J.room[1] = ly; J.room[2] = lz;
    J.center[0] = S.center[0]; J.center[1] = S.center[1]; J.center[2] = S.center[2];
    J.d0 = d0; J.az = az; J.el = el;
    J.t60 = t60;
    J.c0 = c0;
    J.alpha = 0.1; J.beta = 1.0; J.perturb_lo = -2.0; J.perturb_hi = 2.0; J.tau = 0.25;  // SimParams defaults
    J.seed = sim_seed;
    J.source_index = k;
    J.n_images = S.num_images;
    J.mic_off = 0;
    J.n_mics = M;
    // layout: fixed per-job sizes
    J.img_off = (int64_t)j * rows;
    J.item_off = (int64_t)j * rows * M;
    J.chan_off = j * M;
    J.out_stride = S.out_stride;
    J.out_off = (int64_t)j * M * S.out_stride;
    J.L = L;
    J.n1 = (int)n1;
    J.n2 = n2;
    // derived (frir_jobs_prepare, core.py:140-148, 186-192, 295-299)
    J.r = r;
    if (!(c0 * t60 > d0)) st = st ? st : 2;
    J.rr_max = 0.0;
    if (S.num_images > 0) {
      J.rr_max = (log10(c0 * t60) - log10(d0) - 3.0) / log10(r);
      if (!(0.0 < r && r < 1.0) || !(J.rr_max >= 1.0)) st = st ? st : 3;
    }
    J.log2r = log2(r);
    J.e_lo = (int32_t)((6LL * A.rate + 999) / 1000);
    J.e_hi = (int32_t)((50LL * A.rate + 999) / 1000);
    J.alpha3 = S.alpha3;  // host pow(alpha, 3), as frir_jobs_prepare
    J.b3a3 = S.b3a3;
    uint64_t kk[2];
    seed_keys(sim_seed, (uint64_t)k, 0, kk);
    J.key[0] = kk[0]; J.key[1] = kk[1];
    seed_keys(sim_seed, (uint64_t)k, 1, kk);
    J.key[2] = kk[0]; J.key[3] = kk[1];
    A.jobs[j] = J;
    for (int m = 0; m < M; ++m) A.chan_job[j * M + m] = j;
  }
  A.status[i] = st;
}

}  // namespace
}  // namespace frir

using namespace frir;

extern "C" {

int frir_sample_scene_jobs(const frir_plan* plan, const frir_scene_spec* spec, uint64_t seed, int64_t first_index,
                           int32_t count, frir_job* jobs, int32_t* chan_job, int32_t* status, void* stream) {
  if (!plan || !spec || !jobs || !chan_job || !status || count < 0 || first_index < 0 || spec->n_sources < 1 ||
      spec->n_mics < 1 || spec->num_images < 0 || spec->out_stride < 4 || !(spec->c0 > 0)) {
    set_error("frir_sample_scene_jobs: invalid argument");
    return FRIR_EINVAL;
  }
  if (count == 0) return FRIR_OK;
  SceneArgs a;
  a.S = *spec;
  a.seed = seed;
  a.first = first_index;
  a.count = count;
  const frir_plan_desc& d = plan->dev.d;
  a.r_h = d.r_h; a.r_l = d.r_l; a.up = d.up; a.down = d.down; a.rate = d.r_h * d.sample_rate;
  a.jobs = jobs; a.chan_job = chan_job; a.status = status;
  scene_jobs_kernel<<<(count + 127) / 128, 128, 0, (cudaStream_t)stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("scene_jobs_kernel: ") + cudaGetErrorString(e)); return FRIR_ECUDA; }
  return FRIR_OK;
}

}  // extern "C"
