// Checks that sincos() returns bit-identical results to separate sin()/cos()
// in FP64 on this GPU (the geometry kernel relies on it).  Dev tool.
#include <cstdio>
#include <cstdint>
#include <cmath>
__global__ void k(unsigned long long seed, int n, unsigned long long* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long x = seed + 0x9E3779B97F4A7C15ull * (i + 1);
  x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27;
  double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
  double a = (i & 1) ? 6.283185307179586 * u : 3.141592653589793 * u - 1.5707963267948966;
  double s1 = sin(a), c1 = cos(a), s2, c2;
  sincos(a, &s2, &c2);
  if (__double_as_longlong(s1) != __double_as_longlong(s2) || __double_as_longlong(c1) != __double_as_longlong(c2))
    atomicAdd(bad, 1ull);
}
int main() {
  unsigned long long* bad; cudaMallocManaged(&bad, 8); *bad = 0;
  const int n = 1 << 24;
  for (int r = 0; r < 8; ++r) k<<<n / 256, 256>>>(1234567ull * (r + 1), n, bad);
  cudaDeviceSynchronize();
  printf("{\"checked\": %d, \"mismatches\": %llu}\n", 8 * n, *bad);
  return 0;
}
