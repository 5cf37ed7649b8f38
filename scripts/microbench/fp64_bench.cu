#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma(int iters, double* out) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void dmma(int iters, double* out) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int blocks : {sms * 4}) {
    dfma<<<blocks, 256>>>(10, o);
    cudaEventRecord(a); dfma<<<blocks, 256>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)blocks * 256;
    printf("DFMA: %.1f TFLOP/s\n", flops / ms / 1e9);
    dmma<<<blocks, 256>>>(10, o);
    cudaEventRecord(a); dmma<<<blocks, 256>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * (256 / 32);
    printf("DMMA m8n8k4: %.1f TFLOP/s  err %s\n", flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
