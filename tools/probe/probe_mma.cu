// tcgen05.mma throughput probe (1 CTA per SM, operands resident in smem).
// Reports ns per MMA instruction and the implied operand bytes/cycle.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int M, int N>
__global__ void k(int iters, long long* out, int chains, int issuers) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  long long t0 = clock64();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < issuers) {
    const uint32_t a = sa(base) + w * 16384, b = sa(base + 65536);
    for (int i = 0; i < iters / issuers; ++i) {
      const int kk = i & 3;
      const uint32_t d = tm + (uint32_t)(((w * chains + i % chains) * N) & 255);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                   :: "r"(d), "l"(desc(a + (i & 15) * 4096 + kk * 32)), "l"(desc(b + kk * 32)), "r"(idesc), "r"(1));
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar)));
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" :: "r"(sa(&bar)));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
}
template <int M, int N>
void run(const char* name, int chains, int issuers = 1) {
  long long* d; cudaMalloc(&d, 8);
  auto kern = k<M, N>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 20000;
  kern<<<148, 128, 200 * 1024>>>(100, d, chains, issuers); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<148, 128, 200 * 1024>>>(iters, d, chains, issuers); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double cpm = (double)cyc / iters;
  printf("%-34s issuers %d chains %d: %7.2f cycles/MMA  %6.1f ns/MMA  A %5d B + B %5d B -> A-bytes/cycle %6.1f   err=%s\n", name, issuers, chains, cpm,
         ms * 1e6 / iters, M * 32, N * 32, M * 32 / cpm, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<128, 16>("SS M128 N16", 1, 1); run<128, 16>("SS M128 N16", 1, 2); run<128, 16>("SS M128 N16", 1, 4);
  run<128, 64>("SS M128 N64", 1, 2); run<128, 256>("SS M128 N256", 1, 1); run<128, 256>("SS M128 N256", 1, 2);
  return 0;
}
