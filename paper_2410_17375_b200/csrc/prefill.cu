// prefill.cu -- compute-bound prompt prefill: init_state of a long prompt
// (models.py:109-118) as dense tcgen05 GEMMs plus a causal attention over the prompt.
//
// The decode forward streams every weight byte once per <= 16 token rows (HBM-bound by
// design).  A 4096-token prompt through it re-streams the weights 256 times.  Here every
// projection is ONE GEMM over all prompt tokens:
//
//   C[token][n] = sum_k X[token][k] * W[n][k]
//
// with the weight tile as the M=128 operand (the decode path's tile-contiguous SW128 16 KB
// units, one bulk copy each) and 256 tokens as the N operand (TMA, SWIZZLE_128B) of
// tcgen05.mma.cta_group::1.kind::f16 M128 N256 K16, fp32 accumulators in TMEM (two 256-
// column buffers: the epilogue of one tile overlaps the MMAs of the next).  Work items are
// (weight tile, token tile) pairs in weight-tile-major order, so the CTAs working at any
// moment share a few weight tiles through L2 and each weight byte comes from HBM about once.
//
// Per layer: RMSNorm (bf16(h*g), per-token scale) -> QKV GEMM (scaled) -> RoPE + bf16 K/V into
// the cache -> causal attention -> O GEMM (+= residual) -> RMSNorm -> gate/up GEMM (SiLU*up)
// -> down GEMM (+= residual).  The last layer stops after its K/V: the pending-token scheme
// leaves the last prompt token for the first decode step, which predicts from it.
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "gemm_tc.h"
#include "prefill.h"
#include "tc_ptx.cuh"

namespace amusd {
namespace pf {

using namespace amusd::tc;

constexpr int kStages = 4;
constexpr int kWB = 16384;            // weight unit: 128 rows x 64 K bf16
constexpr int kXB = TN * BK * 2;      // token tile: 256 rows x 64 K bf16 (32 KB)
constexpr int kThreads = 192;         // w0 producer, w1 MMA issuer, w2..w5 epilogue
constexpr int kTmemCols = 2 * TN;     // two accumulator buffers of 256 columns
constexpr int kXchgPad = 33;
constexpr int kSmem = 1024 + kStages * (kWB + kXB) + 64 * kXchgPad * 4 + 256;
// D f32, A/B bf16 K-major, N = 256, M = 128
constexpr uint32_t kIdescPf = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) |
                              ((uint32_t)(BM >> 4) << 24);

AMUSD_DEV void umma_pf(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescPf), "r"(accumulate));
}

__global__ void __launch_bounds__(kThreads, 1) k_pf_gemm(const __grid_constant__ CUtensorMap mx, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sW = smem;
  uint8_t* sX = smem + kStages * kWB;
  float* xchg = (float*)(sX + kStages * kXB);
  uint64_t* bars = (uint64_t*)(xchg + 64 * kXchgPad);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(smem_u32(&full[s]), 1); mbar_init(smem_u32(&empty[s]), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(smem_u32(&tfull[b]), 1); mbar_init(smem_u32(&tempty[b]), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntt = (a.M + TN - 1) / TN;
  const int total = a.ntiles * ntt;
  if (warp == 0) {
    if (lane == 0) {  // ===== producer: weight unit (bulk) + token tile (TMA) per stage
      const uint64_t pol_w = policy_evict_last();  // re-read by the other token tiles of this weight tile
      const uint64_t pol_x = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (int i = blockIdx.x; i < total; i += gridDim.x) {
        const int wt = i / ntt, tt = i - wt * ntt;
        const uint8_t* src = a.wt + (size_t)wt * a.kb * kWB;
        for (int u = 0; u < a.kb; ++u) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1u);
          mbar_expect_tx(smem_u32(&full[s]), kWB + kXB);
          bulk_load(smem_u32(sW + s * kWB), src + (size_t)u * kWB, kWB, smem_u32(&full[s]), pol_w);
          tma_load_2d(smem_u32(sX + s * kXB), &mx, u * BK, tt * TN, smem_u32(&full[s]), pol_x);
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      int s = 0, n = 0;
      uint32_t ph = 0;
      for (int i = blockIdx.x; i < total; i += gridDim.x, ++n) {
        const int b = n & 1;
        mbar_wait(smem_u32(&tempty[b]), ((n >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * TN);
        for (int u = 0; u < a.kb; ++u) {
          mbar_wait(smem_u32(&full[s]), ph);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_pf(d, umma_desc(smem_u32(sW + s * kWB) + kk * 32), umma_desc(smem_u32(sX + s * kXB) + kk * 32),
                    (u | kk) ? 1u : 0u);
          umma_commit(smem_u32(&empty[s]));
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
        umma_commit(smem_u32(&tfull[b]));
      }
    }
  } else {
    // ===== epilogue: thread = weight row nl of the tile, 32 tokens per TMEM load
    const int q = warp & 3, nl = q * 32 + lane;
    int n = 0;
    for (int i = blockIdx.x; i < total; i += gridDim.x, ++n) {
      const int b = n & 1;
      const int wt = i / ntt, tt = i - wt * ntt;
      mbar_wait(smem_u32(&tfull[b]), (n >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < TN / 32; ++c) {
        const int tok0 = tt * TN + c * 32;
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TN + c * 32), v);
        if (c == TN / 32 - 1) {  // the buffer is free for the next tile's MMAs
          tc_fence_before();
          mbar_arrive(smem_u32(&tempty[b]));
        }
        if (tok0 >= a.M) continue;  // (uniform across the 128 epilogue threads)
        const int nt = min(32, a.M - tok0);
        if (a.epi == kEpStoreScaled) {
          const int col = wt * BM + nl;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nt) a.out[(size_t)(tok0 + j) * a.ldo + col] = v[j] * a.inv[tok0 + j];
        } else if (a.epi == kEpResid) {
          const int col = wt * BM + nl;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < nt) {
              float* p = a.out + (size_t)(tok0 + j) * a.ldo + col;
              *p += v[j];
            }
          }
        } else {  // gate/up: rows 0..63 gate, 64..127 up of features [64 wt, 64 wt + 64)
          if (nl >= 64)
#pragma unroll
            for (int j = 0; j < 32; ++j) xchg[(nl - 64) * kXchgPad + j] = v[j];
          named_bar(1, 128);
          if (nl < 64) {
            const int f = wt * 64 + nl;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (j < nt) {
                const float iv = a.inv[tok0 + j];
                const float g = v[j] * iv, up = xchg[nl * kXchgPad + j] * iv;
                a.out_b[(size_t)(tok0 + j) * a.ldo + f] = __float2bfloat16((g / (1.f + expf(-g))) * up);
              }
            }
          }
          named_bar(1, 128);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

cudaError_t launch_gemm(const CUtensorMap& mx, const GemmArgs& a, cudaStream_t st) {
  static SmemOptIn opt;
  if (cudaError_t e = opt.ensure(k_pf_gemm, kSmem)) return e;
  const int items = a.ntiles * ((a.M + TN - 1) / TN);
  const int grid = std::max(1, std::min(items, device_sms()));
  k_pf_gemm<<<grid, kThreads, kSmem, st>>>(mx, a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ SIMT kernels
__global__ void k_pf_embed(const int* tok, const __nv_bfloat16* emb, float* h, int d) {
  const int t = blockIdx.x;
  const __nv_bfloat16* e = emb + (size_t)tok[t] * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) h[(size_t)t * d + i] = __bfloat162float(e[i]);
}

// x = bf16(h * g), inv = rsqrt(mean(h^2) + eps) (applied after the GEMM, like the decode path)
__global__ void k_pf_norm(const float* h, const __nv_bfloat16* g, __nv_bfloat16* x, float* inv, int d, float eps) {
  const int t = blockIdx.x;
  const float* hr = h + (size_t)t * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = hr[i];
    ss += v * v;
    x[(size_t)t * d + i] = __float2bfloat16(v * __bfloat162float(g[i]));
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    inv[t] = rsqrtf(tot / (float)d + eps);
  }
}

// Group-blocked QKV columns: group g = [q of G heads | k | v], (G + 2) hd wide.
__global__ void k_pf_rope_kv(float* qkv, const float* cos, const float* sin, __nv_bfloat16* kc, __nv_bfloat16* vc,
                             int H, int KV, int hd, int S) {
  const int t = blockIdx.x, G = H / KV, half = hd / 2, ncols = (H + 2 * KV) * hd;
  float* row = qkv + (size_t)t * ncols;
  const float* cs = cos + (size_t)t * half;
  const float* sn = sin + (size_t)t * half;
  // q and k halves: (G + 1) heads per group rotate, v copies
  for (int i = threadIdx.x; i < KV * (G + 1) * half; i += blockDim.x) {
    const int g = i / ((G + 1) * half), r = i - g * (G + 1) * half, j = r / half, e = r - j * half;
    float* p = row + (size_t)g * (G + 2) * hd + j * hd;
    const float x0 = p[e], x1 = p[e + half];
    const float r0 = x0 * cs[e] - x1 * sn[e], r1 = x1 * cs[e] + x0 * sn[e];
    if (j < G) {
      p[e] = r0;
      p[e + half] = r1;
    } else {  // the K head: rounded to bf16 exactly as the decode steps read it back
      __nv_bfloat16* k = kc + ((size_t)g * S + t) * hd;
      k[e] = __float2bfloat16(r0);
      k[e + half] = __float2bfloat16(r1);
    }
  }
  for (int i = threadIdx.x; i < KV * hd; i += blockDim.x) {
    const int g = i / hd, e = i - g * hd;
    vc[((size_t)g * S + t) * hd + e] = __float2bfloat16(row[(size_t)g * (G + 2) * hd + (G + 1) * hd + e]);
  }
}

// Causal attention, one block per (32-query tile, KV group): the G query heads of the group
// share every K / V chunk staged in shared memory.  Two threads per (query, head), each owning
// half of the head dims; online softmax per 32-key chunk.
constexpr int kKC = 32;
template <int G>
constexpr int qt_of() { return 128 / G; }  // queries per block: 2 x 128 = 256 threads for every G
template <int HD, int G>
__global__ void __launch_bounds__(256) k_pf_attn(const float* qkv, const __nv_bfloat16* kc,
                                                         const __nv_bfloat16* vc, __nv_bfloat16* out, int M, int KV,
                                                         int S, float scale) {
  constexpr int HH = HD / 2, kQT = qt_of<G>();
  __shared__ __align__(16) __nv_bfloat16 ks[kKC][HD];
  __shared__ __align__(16) __nv_bfloat16 vs[kKC][HD];
  const int g = blockIdx.y, q0 = blockIdx.x * kQT;
  const int tid = threadIdx.x, pair = tid >> 1, hf = tid & 1;
  const int qi = pair / G, j = pair - qi * G;   // query in the tile, head in the group
  const int qp = q0 + qi;                        // its position
  const int H = KV * G, ncols = (H + 2 * KV) * HD;
  float qv[HH], acc[HH];
  const float* qsrc = qkv + (size_t)min(qp, M - 1) * ncols + (size_t)g * (G + 2) * HD + j * HD + hf * HH;
#pragma unroll
  for (int e = 0; e < HH; ++e) { qv[e] = qsrc[e] * scale; acc[e] = 0.f; }
  float m = -INFINITY, l = 0.f;
  const int kend = min(q0 + kQT, M);   // keys [0, kend) cover every query of the tile
  const __nv_bfloat16* kg = kc + (size_t)g * S * HD;
  const __nv_bfloat16* vg = vc + (size_t)g * S * HD;
  for (int k0 = 0; k0 < kend; k0 += kKC) {
    __syncthreads();
    for (int i = tid; i < kKC * HD / 8; i += blockDim.x) {
      const int r = i / (HD / 8), c = i - r * (HD / 8);
      uint4 kz = make_uint4(0, 0, 0, 0), vz = kz;
      if (k0 + r < kend) {
        kz = *(const uint4*)(kg + (size_t)(k0 + r) * HD + c * 8);
        vz = *(const uint4*)(vg + (size_t)(k0 + r) * HD + c * 8);
      }
      *(uint4*)&ks[r][c * 8] = kz;
      *(uint4*)&vs[r][c * 8] = vz;
    }
    __syncthreads();
    float s[kKC];
    float cm = -INFINITY;
#pragma unroll
    for (int r = 0; r < kKC; ++r) {
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < HH; e += 2) {
        const float2 kv2 = __bfloat1622float2(*(const __nv_bfloat162*)&ks[r][hf * HH + e]);
        dot = fmaf(qv[e], kv2.x, dot);
        dot = fmaf(qv[e + 1], kv2.y, dot);
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      s[r] = (k0 + r <= qp && qp < M) ? dot : -INFINITY;
      cm = fmaxf(cm, s[r]);
    }
    const float mn = fmaxf(m, cm);
    if (mn == -INFINITY) continue;  // (uniform per pair; rows past M only)
    const float corr = expf(m - mn);
    l *= corr;
#pragma unroll
    for (int e = 0; e < HH; ++e) acc[e] *= corr;
#pragma unroll
    for (int r = 0; r < kKC; ++r) {
      const float p = expf(s[r] - mn);
      l += p;
#pragma unroll
      for (int e = 0; e < HH; e += 2) {
        const float2 vv = __bfloat1622float2(*(const __nv_bfloat162*)&vs[r][hf * HH + e]);
        acc[e] = fmaf(p, vv.x, acc[e]);
        acc[e + 1] = fmaf(p, vv.y, acc[e + 1]);
      }
    }
    m = mn;
  }
  if (qp < M) {
    __nv_bfloat16* o = out + (size_t)qp * H * HD + (size_t)(g * G + j) * HD + hf * HH;
    const float il = 1.f / l;
#pragma unroll
    for (int e = 0; e < HH; e += 2) *(__nv_bfloat162*)(o + e) = __floats2bfloat162_rn(acc[e] * il, acc[e + 1] * il);
  }
}

cudaError_t launch_embed(const int* tok, const __nv_bfloat16* emb, float* h, int M, int d, cudaStream_t st) {
  k_pf_embed<<<M, 256, 0, st>>>(tok, emb, h, d);
  return cudaGetLastError();
}
cudaError_t launch_norm(const float* h, const __nv_bfloat16* g, __nv_bfloat16* x, float* inv, int M, int d, float eps,
                        cudaStream_t st) {
  k_pf_norm<<<M, 256, 0, st>>>(h, g, x, inv, d, eps);
  return cudaGetLastError();
}
cudaError_t launch_rope_kv(float* qkv, const float* cos, const float* sin, __nv_bfloat16* kc, __nv_bfloat16* vc,
                           int M, int H, int KV, int hd, int S, cudaStream_t st) {
  k_pf_rope_kv<<<M, 256, 0, st>>>(qkv, cos, sin, kc, vc, H, KV, hd, S);
  return cudaGetLastError();
}
cudaError_t launch_attention(const float* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc, __nv_bfloat16* out,
                             int M, int H, int KV, int hd, int S, float scale, cudaStream_t st) {
  const int G = H / KV;
#define AMUSD_PF_ATTN(HD_, G_) \
  if (hd == HD_ && G == G_) { \
    const dim3 grid((M + qt_of<G_>() - 1) / qt_of<G_>(), KV); \
    k_pf_attn<HD_, G_><<<grid, 256, 0, st>>>(qkv, kc, vc, out, M, KV, S, scale); \
    return cudaGetLastError(); \
  }
  AMUSD_PF_ATTN(64, 2) AMUSD_PF_ATTN(64, 4) AMUSD_PF_ATTN(64, 8)
  AMUSD_PF_ATTN(128, 2) AMUSD_PF_ATTN(128, 4) AMUSD_PF_ATTN(128, 8)
#undef AMUSD_PF_ATTN
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ workspace
static size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

size_t work_bytes(int mx, int d, int H, int KV, int hd, int ffn) {
  const size_t ncols = (size_t)(H + 2 * KV) * hd, xw = std::max(d, H * hd);
  return a256((size_t)mx * d * 4) + a256((size_t)mx * 4) + a256((size_t)mx * xw * 2) + a256((size_t)mx * ncols * 4) +
         a256((size_t)mx * ffn * 2) + a256((size_t)mx * 4) + 256;
}

void carve(Work* w, void* base, int mx, int d, int H, int KV, int hd, int ffn) {
  const size_t ncols = (size_t)(H + 2 * KV) * hd, xw = std::max(d, H * hd);
  char* p = (char*)(((uintptr_t)base + 255) & ~(uintptr_t)255);
  w->max_tokens = mx;
  w->h = (float*)p; p += a256((size_t)mx * d * 4);
  w->inv = (float*)p; p += a256((size_t)mx * 4);
  w->x = (__nv_bfloat16*)p; p += a256((size_t)mx * xw * 2);
  w->qkv = (float*)p; p += a256((size_t)mx * ncols * 4);
  w->act = (__nv_bfloat16*)p; p += a256((size_t)mx * ffn * 2);
  w->tok = (int*)p;
}

bool make_maps(Work* w, int d, int hh, int ffn) {
  return tc::make_map(&w->map_x_d, w->x, w->max_tokens, d, TN) && tc::make_map(&w->map_x_hh, w->x, w->max_tokens, hh, TN) &&
         make_map(&w->map_act, w->act, w->max_tokens, ffn, TN);
}

}  // namespace pf
}  // namespace amusd
