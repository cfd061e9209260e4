// Read-bandwidth probe on B200: how fast can a kernel stream weights?
//  (1) LDG.128 grid-stride read, (2) cp.async.bulk 1D contiguous 16 KB chunks
//  into a smem ring (per-CTA contiguous region), (3) same bulk copies but
//  strided like a [128 rows x 128 B] box of an 8 KB-pitch matrix.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void rd_ldg(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK, int STAGES, bool STRIDED>
__global__ void rd_bulk(const char* __restrict__ p, size_t bytes, uint32_t* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  size_t per = (bytes / gridDim.x) / CHUNK * CHUNK;
  const char* base = p + per * blockIdx.x;
  int nchunks = (int)(per / CHUNK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int i) {
    int s = i % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[s])), "r"(CHUNK));
    if (!STRIDED) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(sm + s * CHUNK)), "l"(base + (size_t)i * CHUNK), "r"(CHUNK), "r"(sa(&bar[s])));
    } else {
      // CHUNK/128 pieces of 128 B at 8 KB pitch (like a 128-row TMA box of an 8 KB-pitch matrix)
      const char* tile = p + (((size_t)blockIdx.x * 977 + i) % (bytes / (CHUNK * 64))) * (CHUNK * 64) + (i % 64) * 128;
      for (int r = 0; r < CHUNK / 128; ++r)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(sm + s * CHUNK + r * 128)), "l"(tile + (size_t)r * 8192), "r"(128), "r"(sa(&bar[s])));
    }
  };
  for (int i = 0; i < STAGES && i < nchunks; ++i) issue(i);
  for (int i = 0; i < nchunks; ++i) {
    int s = i % STAGES; uint32_t ph = (i / STAGES) & 1;
    asm volatile("{ .reg .pred q; W%=: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W%=; }" :: "r"(sa(&bar[s])), "r"(ph));
    if (i + STAGES < nchunks) issue(i + STAGES);
  }
  if (sm[0] == 123 && out) out[0] = 1;
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int i = 0; i < 5; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main() {
  size_t bytes = (size_t)4 << 30;
  char* p; uint32_t* out; CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&out, 4)); CK(cudaMemset(p, 1, bytes));
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    float ms = timeit([&] { rd_ldg<<<g, 256>>>((const uint4*)p, bytes / 16, out); });
    printf("LDG.128 x8 unroll grid %5d: %7.1f GB/s\n", g, bytes / ms / 1e6);
  }
#define BULK(C, S, ST, G) { auto k = rd_bulk<C, S, ST>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C * S); \
    float ms = timeit([&] { k<<<G, 32, C * S>>>(p, bytes, out); }); CK(cudaGetLastError()); \
    printf("bulk %s chunk %6d stages %2d grid %4d (%3d KB in flight/CTA): %7.1f GB/s\n", ST ? "strided" : "contig ", C, S, G, C * S / 1024, bytes / ms / 1e6); }
  BULK(16384, 5, false, 148) BULK(16384, 8, false, 148) BULK(16384, 12, false, 148) BULK(32768, 6, false, 148)
  BULK(16384, 5, false, 296) BULK(16384, 6, false, 296)
  BULK(16384, 5, true, 148) BULK(16384, 8, true, 148) BULK(16384, 12, true, 148)
  // per-SM streaming rate at partial grids (the persistent forward's 10-stage ring)
  BULK(16384, 10, false, 16) BULK(16384, 10, false, 32) BULK(16384, 10, false, 84) BULK(16384, 10, false, 148)
  BULK(32768, 6, false, 16) BULK(65536, 3, false, 16)
  BULK(16384, 11, false, 148) BULK(16384, 11, false, 64) BULK(16384, 11, false, 32)
  return 0;
}
