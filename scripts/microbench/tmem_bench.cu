// Microbenchmark: TMEM ld/st throughput (tcgen05.ld/st 32x32b.x32) per SM,
// alone and together with a shared-memory LDS.64 stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) bench(int iters, int mode, float* out) {
  __shared__ uint32_t slot;
  __shared__ float2 sm[4096];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_float2(i, 1);
  if (warp == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int q = warp & 3;
  const uint32_t col = (uint32_t)((warp >> 2) * 128);
  const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + col;
  float acc = 0.f;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = 0;
  for (int it = 0; it < iters; ++it) {
    if (mode & 1) {
#pragma unroll
      for (int c = 0; c < 128; c += 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) + 1.0f);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
            ::"r"(taddr + c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
              "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
              "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
              "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (mode & 2) {
#pragma unroll 16
      for (int k = 0; k < 64; ++k) {
        float2 v = sm[((it * 64 + k) * 32 + lane) & 4095];
        acc += v.x * v.y;
      }
    }
  }
  for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int mode = 1; mode <= 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      bench<<<sms, warps * 32>>>(10, mode, out);
      cudaEventRecord(a);
      bench<<<sms, warps * 32>>>(iters, mode, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double clk = 1.965e9 * ms / 1e3;
      double tm_bytes = (mode & 1) ? (double)warps * 32 * 128 * 4 * 2 * iters : 0;  // ld+st
      double sm_bytes = (mode & 2) ? (double)warps * 32 * 64 * 8 * iters : 0;
      printf("mode %d warps %2d: %.3f ms  TMEM %.1f B/clk/SM  SMEM %.1f B/clk/SM  err=%s\n", mode, warps, ms,
             tm_bytes / clk, sm_bytes / clk, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
