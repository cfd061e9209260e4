// Streaming-engine probe for decode_gv.cu: one producer warp bulk-copies 16 KB units of a
// contiguous per-CTA region through an NST-slot shared-memory ring; W consumer warps take the
// units round-robin (or in blocks of BU consecutive units) and run the mma.sync m16n8k16 GEMV
// over each (or only wait / release).  Prints GB/s for each variant at the full grid.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr int UNIT = 16384;

// MODE 0: wait + release only; 1: mma over the unit
template <int W, int MODE>
__global__ void k_probe(const char* __restrict__ p, size_t bytes, int nst, int bu, float* out) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = (uint64_t*)(sm + nst * UNIT);
  uint64_t* empty = full + 16;
  int* seq = (int*)(empty + 16);
  const size_t per = (bytes / gridDim.x) / UNIT * UNIT;
  const char* base = p + per * blockIdx.x;
  const int nu = (int)(per / UNIT);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
      seq[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == W) {
    if (lane == 0) {
      for (int i = 0; i < nu; ++i) {
        const int s = i % nst;
        if (i >= nst) while (!try_wait(sa(&empty[s]), ((i / nst) - 1) & 1)) {}
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(UNIT));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sm + s * UNIT)), "l"(base + (size_t)i * UNIT), "r"(UNIT), "r"(sa(&full[s])));
      }
    }
    return;
  }
  float c[4] = {0, 0, 0, 0};
  const int mrow = (lane & 7) + 8 * ((lane >> 3) & 1), mchunk = lane >> 4;
  // units in blocks of bu consecutive units; block j -> warp j % W
  for (int j = warp; j * bu < nu; j += W) {
    for (int u = j * bu; u < min(nu, (j + 1) * bu); ++u) {
      const int s = u % nst;
      while (((volatile int*)seq)[s] < u / nst) {}
      while (!try_wait(sa(&full[s]), (u / nst) & 1)) {}
      if (MODE == 1) {
        const uint32_t st = sa(sm + s * UNIT) + mrow * 1024;
        for (int kb = 0; kb < 32; kb += 4) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(st + (((2 * (kb + t) + mchunk) ^ (mrow & 7)) * 16), a0, a1, a2, a3);
            mma(c, a0, a1, a2, a3, lane, lane + 1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        ((volatile int*)seq)[s] = u / nst + 1;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
      }
    }
  }
  if (c[0] == 1234.5f) out[0] = c[1];
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int i = 0; i < 5; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main() {
  size_t bytes = (size_t)2 << 30;
  char* p; float* out; CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&out, 4)); CK(cudaMemset(p, 1, bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define RUN(W, MODE, NST, BU, G) { auto k = k_probe<W, MODE>; int sm = NST * UNIT + 1024; \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
    float ms = timeit([&] { k<<<G, (W + 1) * 32, sm>>>(p, bytes, NST, BU, out); }); CK(cudaGetLastError()); \
    printf("W %d %s nst %2d block-units %2d grid %3d: %7.1f GB/s\n", W, MODE ? "mma " : "wait", NST, BU, G, bytes / ms / 1e6); }
  RUN(8, 0, 10, 1, sms) RUN(8, 1, 10, 1, sms) RUN(8, 1, 10, 4, sms) RUN(8, 1, 12, 4, sms)
  RUN(4, 1, 10, 1, sms) RUN(4, 1, 10, 4, sms) RUN(8, 1, 13, 1, sms)
  RUN(8, 0, 10, 1, 64) RUN(8, 1, 10, 1, 64) RUN(8, 1, 10, 4, 64) RUN(8, 1, 13, 1, 64)
  return 0;
}
