// Counter-based streams, bit-compatible with the reference's
//   np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, k, stage))))
// (core.py:86-91).  numpy 2.x semantics restated (numpy is not vendored in the
// reference; pinned only as numpy>=1.24, pkg/pyproject.toml:10-14; verified
// against numpy 2.3.5 in tests/test_host_abi.py):
//   * SeedSequence(entropy).generate_state(2, uint64): entropy words are the
//     little-endian 32-bit limbs of each int (0 -> one zero word), mixed into a
//     4-word pool with the hashmix/mix constants below;
//   * Philox4x64-10 keyed by those two words, counter starting at 0 and
//     incremented BEFORE each 4-word block;
//   * Generator.random() = (u64 >> 11) * 2^-53 and uniform(lo, hi) =
//     lo + (hi - lo) * random().
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define FRIR_HD __host__ __device__ __forceinline__
#else
#define FRIR_HD inline
#endif

namespace frir {

FRIR_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

struct u64x4 {
  uint64_t v[4];
};

// Random123 philox4x64 with 10 rounds.
FRIR_HD u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                            uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t lo0 = M0 * c0, hi0 = mulhi64(M0, c0);
    uint64_t lo1 = M1 * c2, hi1 = mulhi64(M1, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  u64x4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

struct SeedMixer {
  uint32_t hash_const;
  FRIR_HD uint32_t hashmix(uint32_t value) {
    value ^= hash_const;
    hash_const *= 0x931e8875u;
    value *= hash_const;
    value ^= value >> 16;
    return value;
  }
  FRIR_HD static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    r ^= r >> 16;
    return r;
  }
};

// SeedSequence((seed, k, stage)).generate_state(2, np.uint64)
// Keys of Philox(SeedSequence(tuple(vals[0:nv]))) for nv <= 3 non-negative
// 64-bit integers (numpy's entropy: each int as little-endian uint32 words).
FRIR_HD void seed_keys_n(const uint64_t* vals, int nv, uint64_t key[2]) {
  uint32_t ent[6];
  int n = 0;
  for (int v = 0; v < nv; ++v) {
    uint64_t x = vals[v];
    if (x == 0) {
      ent[n++] = 0;
    } else {
      while (x) {
        ent[n++] = (uint32_t)(x & 0xffffffffu);
        x >>= 32;
      }
    }
  }
  SeedMixer m{0x43b0d7e5u};
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = m.hashmix(i < n ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = SeedMixer::mix(pool[d], m.hashmix(pool[s]));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = SeedMixer::mix(pool[d], m.hashmix(ent[s]));
  uint32_t hc = 0x8b51f9ddu;
  uint32_t st[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hc;
    hc *= 0x58f38dedu;
    v *= hc;
    v ^= v >> 16;
    st[i] = v;
  }
  key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

FRIR_HD void seed_keys(uint64_t seed, uint64_t k, uint64_t stage, uint64_t key[2]) {
  const uint64_t vals[3] = {seed, k, stage};
  seed_keys_n(vals, 3, key);
}

// Word `w` of the stream keyed by `key`: block w/4 (counter w/4 + 1), lane w%4.
FRIR_HD uint64_t stream_word(const uint64_t key[2], uint64_t w) {
  u64x4 b = philox4x64_10(w / 4 + 1, 0, 0, 0, key[0], key[1]);
  return b.v[w & 3];
}

FRIR_HD double u64_to_unit(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

}  // namespace frir
