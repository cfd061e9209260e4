// transformer.cu -- SIMT forward kernels of the Llama-style draft/verify
// decoders (replaces MockModel._predict/_extend, models.py:171-185, for real
// models; SURVEY.md section 2.1 kernels K2/K4).
//
// One forward processes `rows` (<= KMAX) tokens at absolute positions
// pos0..pos0+rows-1 read from a device StepCtl, so the same captured graph
// serves any window size.  Every row is computed with a fixed reduction
// order that does not depend on `rows` or on the other rows: the verify
// model is batch-invariant, which is what makes AMUSD/sync output identical
// to AR output on the GPU (engines.py:1-17).
//
// Per layer: gemv(QKV, RMSNorm fused) -> attention (RoPE + KV append fused)
//            -> gemv(O, +residual) -> gemv(gate/up, RMSNorm + SiLU*mul fused)
//            -> gemv(down, +residual).
// RMSNorm is applied as  norm(x) W^T = rsqrt(mean(x^2)+eps) * ((x*g) W^T):
// the sum of squares is accumulated while x is staged, the scale lands in the
// epilogue -- no separate normalisation kernel (oracle/ref_decoder.py uses
// the same evaluation order).
#include "common.cuh"
#include "internal.h"
#include "transformer.h"

namespace amusd {

// ----------------------------------------------------------------- embed
template <typename WT>
__global__ void k_embed(const StepCtl* __restrict__ ctl, const WT* __restrict__ emb, float* __restrict__ h,
                        int d) {
  pdl_wait();
  pdl_launch();
  if (!ctl->active) return;
  const int r = blockIdx.x;
  if (r >= ctl->rows) return;
  const WT* src = emb + (size_t)ctl->tok[r] * d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) h[(size_t)r * d + k] = Elem<WT>::to_f(src[k]);
}

// ------------------------------------------------------------------ gemv
// out[r][n] = epi( sum_k W[n][k] * xs[r][k] ), xs = x (* gamma), with
// optional RMSNorm scale rsqrt(mean(x^2)+eps) applied after the sum.
// CTA = 8 warps, warp w owns rows n = (blockIdx.x*8 + w)*RPW + i.
constexpr int kGemvThreads = 256;

template <int NR, typename WT, int EPI, int RPW>
__global__ void __launch_bounds__(kGemvThreads) k_gemv(GemvArgs a) {
  extern __shared__ float xs[];  // [NR][kc]
  __shared__ float s_ss[NR][kGemvThreads / 32];
  __shared__ unsigned long long s_best[NR][kGemvThreads / 32];
  constexpr int VEC = Elem<WT>::kVec;
  constexpr int U = (VEC == 8) ? 4 : 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_base = (blockIdx.x * (kGemvThreads / 32) + warp) * RPW;

  // Weights do not depend on the previous kernel: warm L2 with this CTA's
  // slice before waiting on the producer of x (PDL overlap).
  {
    const size_t row_bytes = (size_t)a.K * sizeof(WT);
    for (int i = 0; i < RPW; ++i) {
      const int n = n_base + i;
      if (n < a.N) {
        const char* p = (const char*)a.W + (size_t)n * row_bytes;
        for (size_t off = (size_t)lane * 128; off < row_bytes; off += 32 * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
        if (EPI == kEpiGateUp) {
          const char* p2 = (const char*)a.W2 + (size_t)n * row_bytes;
          for (size_t off = (size_t)lane * 128; off < row_bytes; off += 32 * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p2 + off));
        }
      }
    }
  }
  pdl_wait();
  pdl_launch();
  if (!a.ctl->active) return;
  const int rows = a.ctl->rows;

  float acc[RPW][NR];
  float acc2[RPW][NR];  // gate/up second matrix
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int r = 0; r < NR; ++r) { acc[i][r] = 0.f; acc2[i][r] = 0.f; }
  float ss[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) ss[r] = 0.f;

  const WT* gam = (const WT*)a.gamma;
  for (int kc0 = 0; kc0 < a.K; kc0 += a.kc) {
    const int kl = min(a.kc, a.K - kc0);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      for (int k = threadIdx.x * 4; k < kl; k += kGemvThreads * 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < rows) {
          v = *(const float4*)(a.x + (size_t)r * a.ldx + kc0 + k);
          if (gam) {
            ss[r] += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
            v.x *= Elem<WT>::to_f(gam[kc0 + k]);
            v.y *= Elem<WT>::to_f(gam[kc0 + k + 1]);
            v.z *= Elem<WT>::to_f(gam[kc0 + k + 2]);
            v.w *= Elem<WT>::to_f(gam[kc0 + k + 3]);
          }
        }
        *(float4*)(xs + r * kl + k) = v;
      }
    }
    __syncthreads();
    for (int kb = 0; kb < kl; kb += 32 * VEC * U) {
      uint4 wv[RPW][U], wv2[RPW][U];
#pragma unroll
      for (int i = 0; i < RPW; ++i)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = kb + (u * 32 + lane) * VEC;
          const int n = n_base + i;
          const bool ok = (k < kl) && (n < a.N);
          wv[i][u] = ok ? ld_stream((const WT*)a.W + (size_t)n * a.K + kc0 + k) : make_uint4(0, 0, 0, 0);
          if (EPI == kEpiGateUp)
            wv2[i][u] = ok ? ld_stream((const WT*)a.W2 + (size_t)n * a.K + kc0 + k) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + (u * 32 + lane) * VEC;
        if (k >= kl) break;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          float wf[VEC], wf2[VEC];
          Elem<WT>::unpack(wv[i][u], wf);
          if (EPI == kEpiGateUp) Elem<WT>::unpack(wv2[i][u], wf2);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            if (r < rows) {
              const float4* xp = (const float4*)(xs + r * kl + k);
#pragma unroll
              for (int e4 = 0; e4 < VEC / 4; ++e4) {
                const float4 xv = xp[e4];
                acc[i][r] = fmaf(wf[4 * e4 + 0], xv.x, acc[i][r]);
                acc[i][r] = fmaf(wf[4 * e4 + 1], xv.y, acc[i][r]);
                acc[i][r] = fmaf(wf[4 * e4 + 2], xv.z, acc[i][r]);
                acc[i][r] = fmaf(wf[4 * e4 + 3], xv.w, acc[i][r]);
                if (EPI == kEpiGateUp) {
                  acc2[i][r] = fmaf(wf2[4 * e4 + 0], xv.x, acc2[i][r]);
                  acc2[i][r] = fmaf(wf2[4 * e4 + 1], xv.y, acc2[i][r]);
                  acc2[i][r] = fmaf(wf2[4 * e4 + 2], xv.z, acc2[i][r]);
                  acc2[i][r] = fmaf(wf2[4 * e4 + 3], xv.w, acc2[i][r]);
                }
              }
            }
          }
        }
      }
    }
  }

  // RMSNorm scale per row (every CTA computes the same value, same order).
  float inv[NR];
  if (gam) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float v = warp_sum(ss[r]);
      if (lane == 0) s_ss[r][warp] = v;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float t = 0.f;
      for (int w = 0; w < kGemvThreads / 32; ++w) t += s_ss[r][w];
      inv[r] = rsqrtf(t / (float)a.K + a.eps);
    }
  } else {
#pragma unroll
    for (int r = 0; r < NR; ++r) inv[r] = 1.f;
  }

  unsigned long long best[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) best[r] = 0ull;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int n = n_base + i;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float v = warp_sum(acc[i][r]) * inv[r];
      float v2 = 0.f;
      if (EPI == kEpiGateUp) v2 = warp_sum(acc2[i][r]) * inv[r];
      if (n < a.N && r < rows) {
        if (EPI == kEpiStore) {
          if (lane == 0) a.out[(size_t)r * a.ldo + n] = v;
        } else if (EPI == kEpiResid) {
          if (lane == 0) a.out[(size_t)r * a.ldo + n] += v;
        } else if (EPI == kEpiGateUp) {
          if (lane == 0) a.out[(size_t)r * a.ldo + n] = (v / (1.f + expf(-v))) * v2;
        } else {  // argmax
          if (a.logits && lane == 0) a.logits[(size_t)r * a.N + n] = v;
          if (!(a.exclude_eos && n == a.eos)) {
            const unsigned long long key = argmax_key(v, n);
            best[r] = key > best[r] ? key : best[r];
          }
        }
      }
    }
  }
  if (EPI == kEpiArgmax) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (lane == 0) s_best[r][warp] = best[r];
    __syncthreads();
    if (threadIdx.x < NR && (int)threadIdx.x < rows) {
      unsigned long long b = 0ull;
      for (int w = 0; w < kGemvThreads / 32; ++w) b = s_best[threadIdx.x][w] > b ? s_best[threadIdx.x][w] : b;
      a.part[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = b;
    }
  }
}

// Final argmax over the per-CTA partials; writes ctl->preds[r].
__global__ void k_argmax_final(StepCtl* ctl, const unsigned long long* __restrict__ part, int nparts) {
  pdl_wait();
  pdl_launch();
  if (!ctl->active) return;
  const int r = blockIdx.x;
  if (r >= ctl->rows) return;
  unsigned long long b = 0ull;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    const unsigned long long v = part[(size_t)r * nparts + i];
    b = v > b ? v : b;
  }
  b = warp_max_u64(b);
  __shared__ unsigned long long sb[32];
  if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = sb[w] > m ? sb[w] : m;
    ctl->preds[r] = argmax_key_index(m);
  }
}

// ------------------------------------------------------------- attention
// Decode/verify attention, one CTA per (KV head g, window row r, position
// split).  The GROUP query heads sharing KV head g are processed together so
// K/V are read once.  Row r (position p = pos0 + r) attends [0, p]; keys and
// values of this step's rows come from the QKV buffer (RoPE applied here,
// rounded to the cache dtype so they equal what a later step reads back from
// the cache); the CTA owning position p appends row r's K/V to the cache.
// Positions are split in chunks of kAttnChunk; a row with several chunks is
// finished by the last-arriving chunk CTA, which merges the (max, sum, acc)
// partials in chunk order -- deterministic, and the chunking depends on the
// position only (never on the number of rows): batch invariant.
constexpr int kAttnChunk = 256;

template <typename WT, int HD, int GROUP>
__global__ void __launch_bounds__(128) k_attention(AttnArgs a) {
  constexpr int DPL = HD / 32;  // dims per lane
  __shared__ float qs[GROUP][HD];
  __shared__ float kn[KMAX][HD];
  __shared__ float vn[KMAX][HD];
  __shared__ float sc[GROUP][kAttnChunk];
  __shared__ float red[4][GROUP][HD];
  __shared__ float stat[2][GROUP];
  __shared__ int s_last;
  const int g = blockIdx.x, r = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  pdl_launch();
  if (!a.ctl->active) return;
  const int rows = a.ctl->rows, pos0 = a.ctl->pos0;
  if (r >= rows) return;
  const int p = pos0 + r;
  const int nsplit = (p + kAttnChunk) / kAttnChunk;  // chunks covering [0, p]
  if (split >= nsplit) return;
  const int lo = split * kAttnChunk, hi = min(p + 1, lo + kAttnChunk);
  const int half = HD / 2, ncols = (a.H + 2 * a.KV) * HD;
  // column offsets of this group's q / k / v (natural [q|k|v] or group-blocked layout)
  const int qoff = a.blocked ? g * (GROUP + 2) * HD : g * GROUP * HD;
  const int koff = a.blocked ? qoff + GROUP * HD : (a.H + g) * HD;
  const int voff = a.blocked ? qoff + (GROUP + 1) * HD : (a.H + a.KV + g) * HD;
  // rotated queries of the group
  for (int i = threadIdx.x; i < GROUP * half; i += blockDim.x) {
    const int j = i / half, e = i - j * half;
    const float* q = a.qkv + (size_t)r * ncols + qoff + j * HD;
    const float c = a.cos[(size_t)p * half + e], s = a.sin[(size_t)p * half + e];
    qs[j][e] = q[e] * c - q[e + half] * s;
    qs[j][e + half] = q[e + half] * c + q[e] * s;
  }
  // this step's keys/values for rows 0..r, only if the chunk reaches pos0
  const int jmax = hi > pos0 ? min(r, hi - 1 - pos0) : -1;
  for (int i = threadIdx.x; i < (jmax + 1) * half; i += blockDim.x) {
    const int j = i / half, e = i - j * half;
    const int pj = pos0 + j;
    const float* kr = a.qkv + (size_t)j * ncols + koff;
    const float c = a.cos[(size_t)pj * half + e], s = a.sin[(size_t)pj * half + e];
    kn[j][e] = Elem<WT>::to_f(Elem<WT>::from_f(kr[e] * c - kr[e + half] * s));
    kn[j][e + half] = Elem<WT>::to_f(Elem<WT>::from_f(kr[e + half] * c + kr[e] * s));
  }
  for (int i = threadIdx.x; i < (jmax + 1) * HD; i += blockDim.x) {
    const int j = i / HD, e = i - j * HD;
    vn[j][e] = Elem<WT>::to_f(Elem<WT>::from_f(a.qkv[(size_t)j * ncols + voff + e]));
  }
  __syncthreads();
  WT* kc = (WT*)a.kc + (size_t)g * a.S * HD;
  WT* vc = (WT*)a.vc + (size_t)g * a.S * HD;
  if (p >= lo && p < hi) {  // KV append for row r (pending-token scheme)
    for (int e = threadIdx.x; e < HD; e += blockDim.x) {
      kc[(size_t)p * HD + e] = Elem<WT>::from_f(kn[r][e]);
      vc[(size_t)p * HD + e] = Elem<WT>::from_f(vn[r][e]);
    }
  }
  // scores: warp w takes positions lo+w, lo+w+4, ...; lane holds DPL dims
  float qreg[GROUP][DPL];
#pragma unroll
  for (int j = 0; j < GROUP; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) qreg[j][e] = qs[j][lane * DPL + e];
  for (int t = lo + warp; t < hi; t += 4) {
    float kv[DPL];
    if (t < pos0) {
      const WT* kt = kc + (size_t)t * HD + lane * DPL;
#pragma unroll
      for (int e = 0; e < DPL; ++e) kv[e] = Elem<WT>::to_f(kt[e]);
    } else {
#pragma unroll
      for (int e = 0; e < DPL; ++e) kv[e] = kn[t - pos0][lane * DPL + e];
    }
#pragma unroll
    for (int j = 0; j < GROUP; ++j) {
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) d = fmaf(qreg[j][e], kv[e], d);
      d = warp_sum(d);
      if (lane == 0) sc[j][t - lo] = d * a.scale;
    }
  }
  __syncthreads();
  // per-head max and exp-sum over this chunk (one warp per head, fixed order)
  for (int j = warp; j < GROUP; j += 4) {
    float m = -INFINITY;
    for (int t = lane; t < hi - lo; t += 32) m = fmaxf(m, sc[j][t]);
    m = warp_max(m);
    float l = 0.f;
    for (int t = lane; t < hi - lo; t += 32) {
      const float e = expf(sc[j][t] - m);
      sc[j][t] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) { stat[0][j] = m; stat[1][j] = l; }
  }
  __syncthreads();
  // unnormalised output: warp w takes positions lo+w, lo+w+4, ...
  float acc[GROUP][DPL];
#pragma unroll
  for (int j = 0; j < GROUP; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[j][e] = 0.f;
  for (int t = lo + warp; t < hi; t += 4) {
    float vv[DPL];
    if (t < pos0) {
      const WT* vt = vc + (size_t)t * HD + lane * DPL;
#pragma unroll
      for (int e = 0; e < DPL; ++e) vv[e] = Elem<WT>::to_f(vt[e]);
    } else {
#pragma unroll
      for (int e = 0; e < DPL; ++e) vv[e] = vn[t - pos0][lane * DPL + e];
    }
#pragma unroll
    for (int j = 0; j < GROUP; ++j) {
      const float pj = sc[j][t - lo];
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(pj, vv[e], acc[j][e]);
    }
  }
#pragma unroll
  for (int j = 0; j < GROUP; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) red[warp][j][lane * DPL + e] = acc[j][e];
  __syncthreads();
  auto emit = [&](int j, int e, float o) {
    const size_t idx = (size_t)r * a.ldo + (g * GROUP + j) * HD + e;
    if (a.out_b) ((__nv_bfloat16*)a.out_b)[idx] = __float2bfloat16(o);
    else a.out[idx] = o;
  };
  if (nsplit == 1) {
    for (int i = threadIdx.x; i < GROUP * HD; i += blockDim.x) {
      const int j = i / HD, e = i - j * HD;
      const float o = red[0][j][e] + red[1][j][e] + red[2][j][e] + red[3][j][e];
      emit(j, e, o / stat[1][j]);
    }
    return;
  }
  // multi-chunk row: park the partial, the last chunk CTA merges in chunk order
  float* ws = a.ws + (((size_t)g * KMAX + r) * a.max_splits + split) * GROUP * (HD + 2);
  for (int i = threadIdx.x; i < GROUP * HD; i += blockDim.x) {
    const int j = i / HD, e = i - j * HD;
    ws[j * (HD + 2) + e] = red[0][j][e] + red[1][j][e] + red[2][j][e] + red[3][j][e];
  }
  if (threadIdx.x < GROUP) {
    ws[threadIdx.x * (HD + 2) + HD] = stat[0][threadIdx.x];
    ws[threadIdx.x * (HD + 2) + HD + 1] = stat[1][threadIdx.x];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* cnt = a.counters + g * KMAX + r;
    const int old = atomicAdd(cnt, 1);
    s_last = (old == nsplit - 1);
    if (s_last) *cnt = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = a.ws + ((size_t)g * KMAX + r) * a.max_splits * GROUP * (HD + 2);
  for (int i = threadIdx.x; i < GROUP * HD; i += blockDim.x) {
    const int j = i / HD, e = i - j * HD;
    float M = -INFINITY;
    for (int s2 = 0; s2 < nsplit; ++s2) M = fmaxf(M, __ldcg(base + ((size_t)s2 * GROUP + j) * (HD + 2) + HD));
    float L = 0.f, O = 0.f;
    for (int s2 = 0; s2 < nsplit; ++s2) {
      const float* w = base + ((size_t)s2 * GROUP + j) * (HD + 2);
      const float f = expf(__ldcg(w + HD) - M);
      L += __ldcg(w + HD + 1) * f;
      O += __ldcg(w + e) * f;
    }
    emit(j, e, O / L);
  }
}

int attn_max_splits(int max_seq) { return (max_seq + kAttnChunk - 1) / kAttnChunk; }

// ----------------------------------------------------------- launchers
template <typename F, typename... Args>
static cudaError_t launch_pdl(F kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int NR, typename WT, int EPI, int RPW>
static cudaError_t gemv_launch(const GemvArgs& a, cudaStream_t st, bool pdl) {
  constexpr int rows_per_cta = (kGemvThreads / 32) * RPW;
  const int grid = (a.N + rows_per_cta - 1) / rows_per_cta;
  const size_t smem = (size_t)NR * a.kc * sizeof(float);
  auto kern = k_gemv<NR, WT, EPI, RPW>;
  static SmemOptIn opt;  // per device
  if (cudaError_t e = opt.ensure(kern, 96 * 1024)) return e;
  return launch_pdl(kern, dim3(grid), dim3(kGemvThreads), smem, st, pdl, a);
}

int gemv_grid(int N, int rpw) { return (N + (kGemvThreads / 32) * rpw - 1) / ((kGemvThreads / 32) * rpw); }

template <int NR, typename WT>
static cudaError_t gemv_dispatch(int epi, const GemvArgs& a, cudaStream_t st, bool pdl) {
  switch (epi) {
    case kEpiStore: return gemv_launch<NR, WT, kEpiStore, 2>(a, st, pdl);
    case kEpiResid: return gemv_launch<NR, WT, kEpiResid, 2>(a, st, pdl);
    case kEpiGateUp: return gemv_launch<NR, WT, kEpiGateUp, 1>(a, st, pdl);
    default: return gemv_launch<NR, WT, kEpiArgmax, 2>(a, st, pdl);
  }
}

cudaError_t launch_gemv(int nr, int dtype, int epi, const GemvArgs& a, cudaStream_t st, bool pdl) {
  if (dtype == AMUSD_BF16) {
    return nr <= 2 ? gemv_dispatch<2, __nv_bfloat16>(epi, a, st, pdl) : gemv_dispatch<KMAX, __nv_bfloat16>(epi, a, st, pdl);
  }
  return nr <= 2 ? gemv_dispatch<2, float>(epi, a, st, pdl) : gemv_dispatch<KMAX, float>(epi, a, st, pdl);
}

int gemv_kc(int nr, int K) {
  const int cap = nr <= 2 ? 8192 : 1024;
  return K < cap ? K : cap;
}

cudaError_t launch_embed(int dtype, const StepCtl* ctl, const void* emb, float* h, int d, cudaStream_t st, bool pdl) {
  if (dtype == AMUSD_BF16)
    return launch_pdl(k_embed<__nv_bfloat16>, dim3(KMAX), dim3(256), 0, st, pdl, ctl, (const __nv_bfloat16*)emb, h, d);
  return launch_pdl(k_embed<float>, dim3(KMAX), dim3(256), 0, st, pdl, ctl, (const float*)emb, h, d);
}

template <typename WT>
static cudaError_t attention_dispatch(const AttnArgs& a, cudaStream_t st, bool pdl) {
  const dim3 grid(a.KV, KMAX, attn_max_splits(a.S));
  const int group = a.H / a.KV;
#define AMUSD_ATTN(HD_, G_) \
  if (a.hd == HD_ && group == G_) return launch_pdl(k_attention<WT, HD_, G_>, grid, dim3(128), 0, st, pdl, a);
  AMUSD_ATTN(64, 2) AMUSD_ATTN(64, 4) AMUSD_ATTN(64, 8) AMUSD_ATTN(128, 2) AMUSD_ATTN(128, 4) AMUSD_ATTN(128, 8)
#undef AMUSD_ATTN
  return cudaErrorInvalidValue;
}

cudaError_t launch_attention(int dtype, const AttnArgs& a, cudaStream_t st, bool pdl) {
  if (dtype == AMUSD_BF16) return attention_dispatch<__nv_bfloat16>(a, st, pdl);
  return attention_dispatch<float>(a, st, pdl);
}

cudaError_t launch_argmax_final(StepCtl* ctl, const unsigned long long* part, int nparts, cudaStream_t st, bool pdl) {
  return launch_pdl(k_argmax_final, dim3(KMAX), dim3(256), 0, st, pdl, ctl, part, nparts);
}

}  // namespace amusd
