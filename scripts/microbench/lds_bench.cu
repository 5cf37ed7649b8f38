// Microbenchmark: shared-memory load bandwidth per SM on B200 (the DAS
// gather's binding resource).  Every SM runs one CTA of W warps that stream
// conflict-free LDS.64 (or LDS.128) loads over a 64 KB buffer -- the access
// shape of das2_kernel's tap gather (each half-warp reads one 128-byte row)
// -- and reports bytes per SM clock and GB/s over all SMs.  The clock is the
// SM clock read with clock64() inside the kernel; GB/s uses CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bench lds_bench.cu
//   ./lds_bench            -> one JSON line per (width, warps)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VEC>
__global__ void __launch_bounds__(1024, 1) lds_kernel(int iters, float* out, long long* clk) {
  extern __shared__ float4 sm[];  // 64 KB
  const int n4 = 4096;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc = 0.f;
  const long long t0 = clock64();
  if (VEC == 2) {
    const float2* s2 = reinterpret_cast<const float2*>(sm);
    // half-warp h reads row (warp, it, h): 16 lanes x 8 B = one 128-byte row
    int base = (warp * 37) & 511;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int row = (base + u * 2 + (lane >> 4)) & 511;
        const float2 v = s2[row * 16 + (lane & 15)];
        acc += v.x * v.y;
      }
      base = (base + 32) & 511;
    }
  } else {
    int base = (warp * 37) & 127;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int row = (base + u) & 127;  // a warp reads one 512-byte row
        const float4 v = sm[row * 32 + lane];
        acc += v.x * v.w;
      }
      base = (base + 16) & 127;
    }
  }
  const long long t1 = clock64();
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  long long* clk;
  cudaMalloc(&out, 4);
  cudaMalloc(&clk, sizeof(long long) * sms);
  const int iters = 20000;
  for (int vec : {2, 4}) {
    for (int warps : {8, 16, 24, 32}) {
      void* fn = vec == 2 ? (void*)lds_kernel<2> : (void*)lds_kernel<4>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      void* args[] = {(void*)&iters, (void*)&out, (void*)&clk};
      cudaLaunchKernel(fn, dim3(sms), dim3(32 * warps), args, 65536, 0);  // warm-up
      cudaEventRecord(a);
      cudaLaunchKernel(fn, dim3(sms), dim3(32 * warps), args, 65536, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      long long hc[1024];
      cudaMemcpy(hc, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
      long long cmax = 0;
      for (int i = 0; i < sms; ++i) cmax = hc[i] > cmax ? hc[i] : cmax;
      const double bytes_sm = (double)warps * 32 * iters * 16 * (vec * 4);
      const double gbs = bytes_sm * sms / (ms * 1e-3) / 1e9;
      printf("{\"lds\": \"LDS.%d\", \"warps\": %d, \"bytes_per_clk_sm\": %.2f, \"GBs\": %.1f, "
             "\"ms\": %.3f, \"sm_mhz_effective\": %.0f, \"sms\": %d, \"err\": \"%s\"}\n",
             vec * 32, warps, bytes_sm / (double)cmax, gbs, ms, (double)cmax / (ms * 1e3), sms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
