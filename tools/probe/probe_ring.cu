// Cost of the smem mbarrier ring handshake (no data): producer warp arrives
// full[s]; `nc` consumer warps wait full[s] (and xfull[s] from a second
// producer warp when `twoprod`) and arrive on empty[s] (count nc).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph, int spin) {
  if (spin) {
    asm volatile("{ .reg .pred q; W%=: mbarrier.test_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W%=; }" ::"r"(sa(b)), "r"(ph) : "memory");
  } else {
    asm volatile("{ .reg .pred q; W%=: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W%=; }" ::"r"(sa(b)), "r"(ph) : "memory");
  }
}
template <int S>
__global__ void ring(int units, int nc, int twoprod, int spin, long long* out) {
  __shared__ uint64_t full[S], xfull[S], empty[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&xfull[s], 1); init(&empty[s], nc); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (lane == 0) {
    if (w == 0 || (w == 1 && twoprod)) {
      uint64_t* f = w == 0 ? full : xfull;
      for (int u = 0; u < units; ++u) {
        const int s = u % S;
        wait(&empty[s], ((u / S) & 1) ^ 1, spin);
        arrive(&f[s]);
      }
    } else if (w >= 2 && w < 2 + nc) {
      for (int u = 0; u < units; ++u) {
        const int s = u % S;
        wait(&full[s], (u / S) & 1, spin);
        if (twoprod) wait(&xfull[s], (u / S) & 1, spin);
        arrive(&empty[s]);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  long long* out; cudaMalloc(&out, 8 * 148);
  long long h[148];
  for (int spin = 0; spin < 2; ++spin)
    for (int nc : {1, 4})
      for (int two : {0, 1}) {
        const int units = 20000;
        ring<11><<<148, 320>>>(units, nc, two, spin, out);
        cudaDeviceSynchronize();
        ring<11><<<148, 320>>>(units, nc, two, spin, out);
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%s consumers=%d two_producers=%d: %.1f cycles/unit\n", spin ? "test_wait spin" : "try_wait     ", nc, two,
               (double)h[0] / units);
      }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
