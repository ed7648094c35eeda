// Dependent-chain latency of FP64 add / FP32 add / FP64 FMA and the F2F
// conversion on this GPU (one thread, clock64), plus FP64 add throughput with
// 32 warps.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64lat fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, float* outf, long long* cyc, double a, float af, int n) {
  double x = a;
  float y = af;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __fadd_rn(y, af);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __fma_rn(z, 0.999, a);
  long long t3 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) w = (double)(float)w + a;
  long long t4 = clock64();
  out[0] = x + z + w;
  outf[0] = y;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

__global__ void thru(double* out, double a, int n) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < n; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void f2f_thru(double* out, const float* in, int n) {
  float f0 = in[threadIdx.x], f1 = f0 * 1.1f, f2 = f0 * 1.2f, f3 = f0 * 1.3f;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < n; ++i) {
    acc0 += (double)f0; acc1 += (double)f1; acc2 += (double)f2; acc3 += (double)f3;
    f0 += 1.0f; f1 += 1.0f; f2 += 1.0f; f3 += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  double* d; float* f; long long* c;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 64); cudaMalloc(&c, 64);
  const int n = 4096;
  chain<<<1, 1>>>(d, f, c, 1e-3, 1e-3f, n);
  chain<<<1, 1>>>(d, f, c, 1e-3, 1e-3f, n);
  long long h[4];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: dadd %.2f  fadd %.2f  dfma %.2f  f2f+dadd %.2f\n", (double)h[0] / n,
         (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int m = 20000;
  thru<<<sms * 4, 256>>>(d, 1e-3, m);
  cudaEventRecord(e0);
  thru<<<sms * 4, 256>>>(d, 1e-3, m);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * 4 * 256 * m * 8;
  printf("FP64 add throughput: %.1f Gop/s (%.1f per SM per ns)\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
  float* fin;
  cudaMalloc(&fin, 1024 * 4);
  cudaMemset(fin, 0, 1024 * 4);
  f2f_thru<<<sms * 4, 256>>>(d, fin, m);
  cudaEventRecord(e0);
  f2f_thru<<<sms * 4, 256>>>(d, fin, m);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double cv = (double)sms * 4 * 256 * m * 4;
  printf("F2F.F64.F32 (+DADD +FADD) throughput: %.1f Gconv/s (%.1f per SM per ns)\n", cv / ms / 1e6, cv / ms / 1e6 / sms);
  return 0;
}
