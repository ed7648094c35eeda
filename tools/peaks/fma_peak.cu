// FP32 / FP64 CUDA-core FMA throughput microbenchmark (roofline denominators
// for the FRAM-RIR render kernel, which uses no tensor cores).
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == (T)123.456) out[threadIdx.x] = s;
}

template <typename T, int CHAINS>
double run(int sms, const char* name) {
  T* out; cudaMalloc(&out, 1024 * sizeof(T));
  int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) fma_loop<T, CHAINS><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) fma_loop<T, CHAINS><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * CHAINS * (double)iters * blocks * threads * reps;
  double tf = flops / (ms * 1e-3) / 1e12;
  printf("{\"kind\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f}\n", name, tf, ms);
  cudaFree(out);
  return tf;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"smem_per_block_optin\": %zu, \"l2\": %d}\n",
         p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin, p.l2CacheSize);
  run<float, 8>(p.multiProcessorCount, "fp32_ffma");
  run<double, 8>(p.multiProcessorCount, "fp64_dfma");
  run<float, 8>(p.multiProcessorCount, "fp32_ffma");
  run<double, 8>(p.multiProcessorCount, "fp64_dfma");
  return 0;
}
