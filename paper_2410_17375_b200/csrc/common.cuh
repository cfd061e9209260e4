// common.cuh -- device helpers shared by every AMUSD kernel (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define AMUSD_DEV __device__ __forceinline__

namespace amusd {

// ---------------------------------------------------------- host helpers
// Per-DEVICE host caches: one process may drive models on several GPUs (split pair),
// so nothing device-specific is cached process-wide.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
// SM count of the current device.
inline int device_sms() {
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (!n[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    n[dev] = v;
  }
  return n[dev];
}
// Dynamic shared-memory opt-in of one kernel, applied once per device (largest size seen).
struct SmemOptIn {
  int bytes[kMaxDevices] = {};
  template <class K>
  cudaError_t ensure(K kern, int want) {
    const int dev = current_device();
    if (want <= bytes[dev]) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
    if (e == cudaSuccess) bytes[dev] = want;
    return e;
  }
};


// ---- memory ordering for the mailbox (single writer per field) -------------
// Writers store payload, then st.release the counter/epoch; readers
// ld.acquire the counter, then read payload.  .sys scope so the same code is
// correct for a peer GPU's HBM mapped over NVLink.
AMUSD_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
AMUSD_DEV void st_release(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
AMUSD_DEV int ld_volatile(const int* p) { return *(volatile const int*)p; }

AMUSD_DEV long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- PDL (programmatic dependent launch) -----------------------------------
AMUSD_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
AMUSD_DEV void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

// ---- splitmix64 (models.py:50-55) -------------------------------------------
AMUSD_DEV uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kAgreeSalt = 0xD1B54A32D192ED03ull;     // models.py:46
constexpr uint64_t kDisagreeSalt = 0x8CB92BA72F3D8DD7ull;  // models.py:47

// models.py:256-261
AMUSD_DEV int chain_draw(uint64_t h, int vocab, int eos, int exclude_eos) {
  if (!exclude_eos) return (int)(h % (uint64_t)vocab);
  int r = (int)(h % (uint64_t)(vocab - 1));
  return r + (r >= eos ? 1 : 0);
}
// models.py:306-314 (sorted exclusion remap)
AMUSD_DEV int different_token(uint64_t h, int agreed, int vocab, int eos, int exclude_eos) {
  int a = agreed, b = eos;
  int nskip = 1;
  if (exclude_eos && eos != agreed) { nskip = 2; if (b < a) { int t = a; a = b; b = t; } }
  int d = (int)(mix64(h ^ kDisagreeSalt) % (uint64_t)(vocab - nskip));
  if (d >= a) ++d;
  if (nskip == 2 && d >= b) ++d;
  return d;
}
// models.py:300-304
AMUSD_DEV int coin_token(uint64_t h, int agreed, uint64_t thr, int vocab, int eos, int exclude_eos) {
  if (mix64(h ^ kAgreeSalt) < thr) return agreed;
  return different_token(h, agreed, vocab, eos, exclude_eos);
}

// ---- first-index argmax packing --------------------------------------------
// key = orderable(value) << 32 | ~index : max(key) = max value, smallest index.
AMUSD_DEV unsigned long long argmax_key(float v, int idx) {
  unsigned int b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (unsigned long long)(0xFFFFFFFFu - (unsigned int)idx);
}
AMUSD_DEV int argmax_key_index(unsigned long long k) { return (int)(0xFFFFFFFFu - (unsigned int)(k & 0xFFFFFFFFu)); }
AMUSD_DEV float argmax_key_value(unsigned long long k) {
  unsigned int b = (unsigned int)(k >> 32);
  b = (b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b;
  return __uint_as_float(b);
}
AMUSD_DEV unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

AMUSD_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
AMUSD_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- QKV group-block layout ----------------------------------------------------
// Output column n of the blocked QKV projection -> row of the natural [q|k|v]
// weight: block g = [q heads g*G..g*G+G-1 | k head g | v head g], (G+2)*hd wide.
__host__ __device__ inline int qkv_group_row(int n, int H, int KV, int hd) {
  const int G = H / KV, bw = (G + 2) * hd;
  const int g = n / bw, w = n - g * bw;
  if (w < G * hd) return g * G * hd + w;
  if (w < (G + 1) * hd) return H * hd + g * hd + (w - G * hd);
  return (H + KV) * hd + g * hd + (w - (G + 1) * hd);
}

// ---- element loads -----------------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kVec = 4;  // elements per 16-byte load
  AMUSD_DEV static float to_f(float v) { return v; }
  AMUSD_DEV static float from_f(float v) { return v; }
  AMUSD_DEV static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  AMUSD_DEV static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  AMUSD_DEV static __nv_bfloat16 from_f(float v) { return __float2bfloat16(v); }
  AMUSD_DEV static void unpack(const uint4& u, float* f) {
    const unsigned int w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};

// Streaming 128-bit weight load: read-only, no L1 allocation.
AMUSD_DEV uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

}  // namespace amusd
