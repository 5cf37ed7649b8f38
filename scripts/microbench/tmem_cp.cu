#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}

__global__ void cp_test(uint32_t lbo, uint32_t sbo, uint32_t* out) {
  __shared__ __align__(1024) uint32_t buf[4096];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  if (threadIdx.x == 0) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  if (warp == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint64_t d = sdesc((uint32_t)__cvta_generic_to_shared(buf), lbo, sbo);
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem), "l"(d));
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
  }
  {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(b) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(tmem + ((uint32_t)(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 8; ++c) out[(32 * warp + lane) * 8 + c] = r[c];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

// throughput of tcgen05.ld.32x32b.x4 (16 B per lane), 8 in flight per wait
__global__ void __launch_bounds__(512, 1) ld_bench(int iters, float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t col = (uint32_t)(((it * 8 + k) * 4 + warp * 16) & 511);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[4 * k]), "=r"(r[4 * k + 1]), "=r"(r[4 * k + 2]), "=r"(r[4 * k + 3])
                   : "r"(tmem + col));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; ++k) acc += __uint_as_float(r[k]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 8 * 4);
  uint32_t h[128 * 8];
  for (auto lbsb : {std::pair<int,int>{128, 256}, std::pair<int,int>{2048, 128}}) {
    cp_test<<<1, 128>>>(lbsb.first, lbsb.second, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("LBO %d SBO %d err %s\n", lbsb.first, lbsb.second, cudaGetErrorString(e));
    for (int lane : {0, 1, 2, 7, 8, 9, 16, 127}) {
      printf("  lane %3d:", lane);
      for (int c = 0; c < 8; ++c) printf(" %5u", h[lane * 8 + c]);
      printf("\n");
    }
  }
  float* o;
  cudaMalloc(&o, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int warps : {4, 8, 16}) {
    ld_bench<<<sms, warps * 32>>>(10, o);
    cudaEventRecord(a);
    ld_bench<<<sms, warps * 32>>>(20000, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)warps * 32 * 16 * 8 * 20000;
    printf("ld.x4 warps %2d: %.1f B/clk/SM  err %s\n", warps, bytes / (1.965e9 * ms / 1e3),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
