// gemm_tc.cu -- tcgen05/TMA small-M GEMM for the verify forward.
//
// Y[r][n] = epi( sum_k X[r][k] * W[n][k] )  for r < 16 window rows, n < N.
// Swap-AB: the weight tile is the M=128 operand (A, K-major, SWIZZLE_128B via
// TMA), the 16 token rows are the N=16 operand (B), the fp32 accumulator
// lives in TMEM (128 lanes x 16 columns, double-buffered).  One elected
// thread issues tcgen05.mma.cta_group::1.kind::f16 (M128 N16 K16).
//
// Work split: persistent stream-K.  The (tile, k-block) units of the whole
// GEMM are cut into gridDim.x contiguous ranges (one CTA per SM), so every SM
// streams the same number of weight bytes whatever the matrix shape.  A tile
// shared by several CTAs is finished by its last-arriving contributor, which
// sums the partials in contributor order -- deterministic and independent of
// the number of valid rows (batch invariance, see transformer.cu).
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM alloc + MMA issuer,
// w2..w5 epilogue (TMEM lane quarter = warp % 4).
#include <cuda.h>

#include "common.cuh"
#include "gemm_tc.h"
#include "internal.h"
#include "tc_ptx.cuh"

namespace amusd {
namespace tc {

// Tile geometry (swap-AB): the weight tile is the M=128 operand, the <=16
// token rows the N=16 operand.  Measured on B200 (tools/probe/probe_mma.cu):
// one issuing thread sustains only ~1 tcgen05.mma per ~150 cycles (issue-side
// cost), while the tensor core executes an M128 N16 K16 MMA far faster; the 4
// K-slices of each stage are therefore issued by 4 different warps, each into
// its own TMEM accumulator chain (summed in fixed order by the epilogue:
// deterministic and batch-invariant).
constexpr int STAGES = 5;         // ~96 KB smem: two CTAs per SM (PDL prefetch overlap)
constexpr int kThreads = 32 * (1 + NACC + 4);  // w0 TMA, w1..w4 MMA issuers, w5..w8 epilogue
constexpr int kTmemCols = 2 * NACC * BN;  // double-buffered: 128 columns
constexpr int smem_bytes() { return STAGES * (kWBytes + kXBytes) + 1024 + 4096 + 512; }

// ------------------------------------------------------------ stream-K map
struct Split {
  long long U;  // total units
  int G, kb;
  AMUSD_DEV long long start(int g) const { return U * g / G; }
  AMUSD_DEV int owner(long long u) const {  // CTA whose range holds unit u
    int g = (int)((u * G) / U);
    while (g + 1 < G && start(g + 1) <= u) ++g;
    while (g > 0 && start(g) > u) --g;
    return g;
  }
};

// ------------------------------------------------------------ epilogues
// Executed by the 4 epilogue warps: thread holds tile row nl (its TMEM lane)
// and the 16 token columns v[0..15].
AMUSD_DEV void final_epilogue(const TcArgs& a, int t, int nl, float* v, int rows, const float* inv, float* xchg,
                              unsigned long long* kx, int q, int lane) {
  if (a.epi == kTcStoreScaled) {
    const int n = t * BM + nl;
#pragma unroll
    for (int r = 0; r < BN; ++r)
      if (r < rows) a.out[(size_t)r * a.ldo + n] = v[r] * inv[r];
  } else if (a.epi == kTcResid) {
    const int n = t * BM + nl;
    const float gn = a.xnext ? __bfloat162float(a.gnext[n]) : 0.f;
    float* sq = xchg;  // [4][BN]
#pragma unroll
    for (int r = 0; r < BN; ++r) {
      float hn = 0.f;
      if (r < rows) {
        hn = a.out[(size_t)r * a.ldo + n] + v[r];
        a.out[(size_t)r * a.ldo + n] = hn;
        if (a.xnext) a.xnext[(size_t)r * a.ldo + n] = __float2bfloat16(hn * gn);
      }
      if (a.xnext) {
        const float s2 = warp_sum(hn * hn);
        if (lane == 0) sq[q * BN + r] = s2;
      }
    }
    if (a.xnext) {
      named_bar(1, 128);
      if (q == 0 && lane < BN) {  // fixed order over the 4 lane quarters
        const float tot = sq[0 * BN + lane] + sq[1 * BN + lane] + sq[2 * BN + lane] + sq[3 * BN + lane];
        a.ssp[(size_t)lane * a.ssp_tiles + t] = lane < rows ? tot : 0.f;
      }
      named_bar(1, 128);
    }
  } else if (a.epi == kTcGateUp) {
    // lanes 0..63: gate rows, 64..127: up rows of the same 64 features
    if (nl >= 64) {
#pragma unroll
      for (int r = 0; r < BN; ++r) xchg[(nl - 64) * BN + r] = v[r];
    }
    named_bar(1, 128);
    if (nl < 64) {
      const int f = t * 64 + nl;
#pragma unroll
      for (int r = 0; r < BN; ++r) {
        if (r < rows) {
          const float g = v[r] * inv[r], u = xchg[nl * BN + r] * inv[r];
          a.out_b[(size_t)r * a.ldo + f] = __float2bfloat16((g / (1.f + expf(-g))) * u);
        }
      }
    }
    named_bar(1, 128);
  } else {  // argmax over the tile's rows, per token row
    const int n = t * BM + nl;
    const bool valid_n = n < a.N && !(a.exclude_eos && n == a.eos);
#pragma unroll
    for (int r = 0; r < BN; ++r) {
      if (a.logits && n < a.N && r < rows) a.logits[(size_t)r * a.N + n] = v[r] * inv[r];
      unsigned long long key = (valid_n && r < rows) ? argmax_key(v[r] * inv[r], n) : 0ull;
      key = warp_max_u64(key);
      if (lane == 0) kx[q * BN + r] = key;
    }
    named_bar(1, 128);
    if (q == 0 && lane < BN && lane < rows) {
      unsigned long long b = kx[lane];
      for (int w = 1; w < 4; ++w) b = kx[w * BN + lane] > b ? kx[w * BN + lane] : b;
      a.part[(size_t)lane * a.ntiles + t] = b;
    }
    named_bar(1, 128);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_gemm_tc(const __grid_constant__ CUtensorMap mapX, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * kWBytes;
  float* xchg = (float*)(sX + STAGES * kXBytes);                     // 4 KB
  uint64_t* bars = (uint64_t*)((uint8_t*)xchg + 4096);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);
  int* flag = (int*)(tmem_slot + 1);
  __shared__ unsigned long long kx[4 * BN];
  __shared__ float s_inv[BN];

  pdl_launch();  // the next kernel may launch now; it prefetches only weights before its own wait
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Split sp{(long long)a.ntiles * a.kb, (int)gridDim.x, a.kb};
  const long long u0 = sp.start(blockIdx.x), u1 = sp.start(blockIdx.x + 1);
  const int nunits = (int)(u1 - u0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(smem_u32(&full[s]), 1); mbar_init(smem_u32(&empty[s]), NACC); }
    for (int i = 0; i < 2; ++i) { mbar_init(smem_u32(&tfull[i]), NACC); mbar_init(smem_u32(&tempty[i]), 128); }
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

  if (warp == 0) {
    // ===== producer: weights by contiguous bulk copies, tokens by TMA =====
    if (lane == 0 && nunits > 0) {
      const uint64_t pol_w = policy_evict_first();   // weights stream once
      const uint64_t pol_x = policy_evict_last();    // tokens are re-read by every CTA
      const int pre = min(nunits, STAGES);
      // Weights do not depend on the previous kernel: issue them before the
      // grid-dependency wait (PDL), token rows after it.
      for (int i = 0; i < pre; ++i) {
        const uint32_t fb = smem_u32(&full[i]);
        mbar_expect_tx(fb, kWBytes + kXBytes);
        bulk_load(smem_u32(sW + i * kWBytes), a.wt + (size_t)(u0 + i) * kWBytes, kWBytes, fb, pol_w);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(smem_u32(sX + i * kXBytes), &mapX, (int)((u0 + i) % a.kb) * BK, 0, smem_u32(&full[i]), pol_x);
      const int upto = a.ctl->active ? nunits : pre;  // inactive step: drain the prefetch only
      for (int i = pre; i < upto; ++i) {
        const int s = i % STAGES;
        mbar_wait(smem_u32(&empty[s]), ((i / STAGES) & 1) ^ 1);
        const uint32_t fb = smem_u32(&full[s]);
        mbar_expect_tx(fb, kWBytes + kXBytes);
        bulk_load(smem_u32(sW + s * kWBytes), a.wt + (size_t)(u0 + i) * kWBytes, kWBytes, fb, pol_w);
        tma_load_2d(smem_u32(sX + s * kXBytes), &mapX, (int)((u0 + i) % a.kb) * BK, 0, fb, pol_x);
      }
    }
  } else if (warp <= NACC) {
    // ===== MMA issuers: warp w issues K-slice kk = w-1 of every stage =====
    const int kk = warp - 1;
    pdl_wait();
    if (lane == 0 && !a.ctl->active) {  // inactive step: consume the prefetched stages, no MMA
      for (int i = 0; i < min(nunits, STAGES); ++i) {
        mbar_wait(smem_u32(&full[i]), 0);
      }
    } else if (lane == 0) {
      int seg = -1;
      for (int i = 0; i < nunits; ++i) {
        const long long u = u0 + i;
        const int b = (int)(u % a.kb);
        const bool first = (i == 0) || b == 0;
        const bool last = (i == nunits - 1) || b == a.kb - 1;
        if (first) {
          ++seg;
          mbar_wait(smem_u32(&tempty[seg & 1]), ((seg >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const int s = i % STAGES;
        mbar_wait(smem_u32(&full[s]), (i / STAGES) & 1);
        tc_fence_after();
        const uint32_t aw = smem_u32(sW + s * kWBytes), ax = smem_u32(sX + s * kXBytes);
        const uint32_t d = tmem + (uint32_t)(((seg & 1) * NACC + kk) * BN);
        umma(d, umma_desc(aw + kk * 32), umma_desc(ax + kk * 32), first ? 0u : 1u);
        umma_commit(smem_u32(&empty[s]));
        if (last) umma_commit(smem_u32(&tfull[seg & 1]));
      }
    }
  } else {
    // ===== epilogue warps =====
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int nl = q * 32 + lane;     // tile row held by this thread
    const int et = threadIdx.x - 32 * (1 + NACC);  // 0..127
    pdl_wait();
    const int rows = a.ctl->rows;
    if (et < BN) {
      float iv = 1.f;
      if (a.ssp_in) {  // inv_rms from the producer's per-tile sums, fixed tile order
        float tot = 0.f;
        for (int j = 0; j < a.ssp_tiles; ++j) tot += a.ssp_in[(size_t)et * a.ssp_tiles + j];
        iv = rsqrtf(tot / a.norm_dim + a.eps);
      } else if (a.inv) {
        iv = a.inv[et];
      }
      s_inv[et] = iv;
    }
    named_bar(1, 128);
    float inv[BN];
#pragma unroll
    for (int r = 0; r < BN; ++r) inv[r] = s_inv[r];
    int seg = -1;
    long long u = a.ctl->active ? u0 : u1;
    while (u < u1) {
      const int t = (int)(u / a.kb);
      const long long tile_end = (long long)(t + 1) * a.kb;
      const long long seg_end = tile_end < u1 ? tile_end : u1;
      const bool whole = (u == (long long)t * a.kb) && seg_end == tile_end;
      ++seg;
      mbar_wait(smem_u32(&tfull[seg & 1]), (seg >> 1) & 1);
      tc_fence_after();
      float v[BN];
      {
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((seg & 1) * NACC * BN);
        float w[BN];
        tmem_ld16(base, v);
#pragma unroll
        for (int c = 1; c < NACC; ++c) {  // fixed chain order
          tmem_ld16(base + c * BN, w);
#pragma unroll
          for (int r = 0; r < BN; ++r) v[r] += w[r];
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty[seg & 1]));
      if (whole) {
        final_epilogue(a, t, nl, v, rows, inv, xchg, kx, q, lane);
      } else {
        // partial tile: slot 0 = this CTA's first tile, 1 = its last tile
        const int slot = (u == u0) ? 0 : 1;
        float4* dst = (float4*)(a.ws + (((size_t)blockIdx.x * 2 + slot) * BM + nl) * BN);
#pragma unroll
        for (int j = 0; j < BN / 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __threadfence();
        named_bar(1, 128);
        const int g_first = sp.owner((long long)t * a.kb), g_last = sp.owner(tile_end - 1);
        if (et == 0) {
          const int old = atomicAdd(&a.counters[t], 1);
          *flag = (old == g_last - g_first);
          if (*flag) a.counters[t] = 0;  // re-arm for the next launch
        }
        named_bar(1, 128);
        if (*flag) {
          __threadfence();
          float acc[BN];
#pragma unroll
          for (int r = 0; r < BN; ++r) acc[r] = 0.f;
          for (int g = g_first; g <= g_last; ++g) {  // fixed contributor order: deterministic
            const int gs = (sp.start(g) >= (long long)t * a.kb) ? 0 : 1;  // range begins inside t: its first tile
            const float4* src = (const float4*)(a.ws + (((size_t)g * 2 + gs) * BM + nl) * BN);
#pragma unroll
            for (int j = 0; j < BN / 4; ++j) {
              const float4 p = __ldcg(src + j);
              acc[4 * j] += p.x; acc[4 * j + 1] += p.y; acc[4 * j + 2] += p.z; acc[4 * j + 3] += p.w;
            }
          }
          final_epilogue(a, t, nl, acc, rows, inv, xchg, kx, q, lane);
        }
        named_bar(1, 128);
      }
      u = seg_end;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

// --------------------------------------------------- weight re-layout
// dst unit (t, b) = 128 rows x 64 cols at byte (t*kb + b)*16384; row i, col j
// at i*128 + (((j>>3) ^ (i&7)) << 4) + (j&7)*2 -- the SWIZZLE_128B K-major
// layout the UMMA descriptor expects, so a plain bulk copy lands it ready.
// Gate/up pair (src2 != null): tile t = gate rows 64t.. (lanes 0-63) then up
// rows 64t.. (lanes 64-127), matching the fused SiLU*mul epilogue.
__global__ void k_tile_weights(const __nv_bfloat16* __restrict__ src, const __nv_bfloat16* __restrict__ src2,
                               __nv_bfloat16* __restrict__ dst, int N, int K, int qkv_H, int qkv_KV, int qkv_hd) {
  const int kb = K / BK;
  const size_t total = (size_t)(src2 ? 2 * N : N) * K;
  for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < total; o += (size_t)gridDim.x * blockDim.x) {
    const size_t unit = o / (BM * BK);
    const int within = (int)(o % (BM * BK));
    const int i = within / BK, jj = within % BK;  // destination row, swizzled column slot
    const int chunk = (jj >> 3) ^ (i & 7);
    const int j = chunk * 8 + (jj & 7);           // logical column inside the unit
    const int t = (int)(unit / kb), b = (int)(unit % kb);
    const int k = b * BK + j;
    const __nv_bfloat16* s;
    int n;
    if (src2) { n = t * (BM / 2) + (i & (BM / 2 - 1)); s = i < BM / 2 ? src : src2; }
    else { n = t * BM + i; s = src; }
    if (qkv_H) {  // QKV rows in group blocks [q(G heads) | k | v] per KV head (qkv_group_row)
      n = qkv_group_row(n, qkv_H, qkv_KV, qkv_hd);
    }
    dst[o] = s[(size_t)n * K + k];
  }
}

size_t tiled_bytes(int N, int K) { return (size_t)N * K * 2; }

cudaError_t launch_tile_weights(const void* src, const void* src2, void* dst, int N, int K, cudaStream_t st,
                               int qkv_H, int qkv_KV, int qkv_hd) {
  k_tile_weights<<<148 * 8, 256, 0, st>>>((const __nv_bfloat16*)src, (const __nv_bfloat16*)src2,
                                          (__nv_bfloat16*)dst, N, K, qkv_H, qkv_KV, qkv_hd);
  return cudaGetLastError();
}

// ------------------------------------------------- embedding (TC path)
// h[r] = E[tok_r]; xb[r] = bf16(h * g_attn0); ssp[r][t] = sum over the
// 128-wide chunk t of h^2 (same tiling as the residual epilogues).
__global__ void k_embed_tc(const StepCtl* ctl, const __nv_bfloat16* __restrict__ emb, float* __restrict__ h,
                           const __nv_bfloat16* __restrict__ g, __nv_bfloat16* __restrict__ xb, float* __restrict__ ssp,
                           int d) {
  pdl_wait();
  pdl_launch();
  const int r = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool live = ctl->active && r < ctl->rows;
  const __nv_bfloat16* src = emb + (size_t)(live ? ctl->tok[r] : 0) * d;
  for (int t = warp; t < d / BM; t += blockDim.x >> 5) {
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < BM / 32; ++e) {
      const int k = t * BM + e * 32 + lane;
      const float x = live ? __bfloat162float(src[k]) : 0.f;
      h[(size_t)r * d + k] = x;
      xb[(size_t)r * d + k] = __float2bfloat16(x * __bfloat162float(g[k]));
      ss += x * x;
    }
    ss = warp_sum(ss);
    if (lane == 0) ssp[(size_t)r * (d / BM) + t] = ss;
  }
}

cudaError_t launch_embed_tc(const StepCtl* ctl, const void* emb, float* h, const void* g, void* xb, float* ssp, int d,
                            cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(KMAX);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_embed_tc, ctl, (const __nv_bfloat16*)emb, h, (const __nv_bfloat16*)g,
                            (__nv_bfloat16*)xb, ssp, d);
}

// ------------------------------------------------------ RMSNorm prep
// xb[r][k] = bf16(h[r][k] * g[k]); inv[r] = rsqrt(mean(h[r]^2) + eps).
// Rows >= `rows` are written as zeros so the MMA sees finite inputs.
__global__ void k_prep_norm(const StepCtl* ctl, const float* __restrict__ h, const __nv_bfloat16* __restrict__ g,
                            __nv_bfloat16* __restrict__ xb, float* __restrict__ inv, int d, float eps) {
  pdl_wait();
  const int r = blockIdx.x;
  const bool live = ctl->active && r < ctl->rows;
  __shared__ float red[32];
  float ss = 0.f;
  for (int k = threadIdx.x * 4; k < d; k += blockDim.x * 4) {
    float4 x = live ? *(const float4*)(h + (size_t)r * d + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
    __nv_bfloat162 lo = __floats2bfloat162_rn(x.x * __bfloat162float(g[k]), x.y * __bfloat162float(g[k + 1]));
    __nv_bfloat162 hi = __floats2bfloat162_rn(x.z * __bfloat162float(g[k + 2]), x.w * __bfloat162float(g[k + 3]));
    *(__nv_bfloat162*)(xb + (size_t)r * d + k) = lo;
    *(__nv_bfloat162*)(xb + (size_t)r * d + k + 2) = hi;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    inv[r] = live ? rsqrtf(t / (float)d + eps) : 0.f;
  }
  pdl_launch();
}

// ----------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, int rows, int cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int tc_grid(int ntiles, int kb) {
  const int g_num_sms = device_sms();
  static int cap = -1;
  if (cap < 0) {  // AMUSD_TC_GRID: leave SMs to a co-located draft (scheduling knob)
    const char* e = getenv("AMUSD_TC_GRID");
    cap = e ? atoi(e) : 0;
  }
  const int sms = cap > 0 && cap < g_num_sms ? cap : g_num_sms;
  const long long U = (long long)ntiles * kb;
  return (int)(U < sms ? U : sms);
}

cudaError_t launch_gemm_tc(const CUtensorMap& mx, const TcArgs& a, cudaStream_t st, bool pdl) {
  static SmemOptIn opt;  // per device
  if (cudaError_t e = opt.ensure(k_gemm_tc, smem_bytes())) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tc_grid(a.ntiles, a.kb));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_gemm_tc, mx, a);
}

cudaError_t launch_prep_norm(const StepCtl* ctl, const float* h, const void* g, void* xb, float* inv, int d, float eps,
                             cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(KMAX);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_prep_norm, ctl, h, (const __nv_bfloat16*)g, (__nv_bfloat16*)xb, inv, d, eps);
}

}  // namespace tc
}  // namespace amusd
