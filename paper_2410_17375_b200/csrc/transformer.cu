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
  if (!ctl->active) return;
  const int r = blockIdx.x;
  if (r >= ctl->rows) return;
  const WT* src = emb + (size_t)ctl->tok[r] * d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) h[(size_t)r * d + k] = Elem<WT>::to_f(src[k]);
  pdl_launch();
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
  pdl_launch();

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
  pdl_launch();
}

// ------------------------------------------------------------- attention
// Grid (H, KMAX).  CTA (h, r) attends row r (position p = pos0 + r) over
// positions [0, p].  Keys/values of this step's rows come straight from the
// QKV buffer (RoPE applied here, rounded to the cache dtype so the result is
// identical to reading them back from the cache in a later step); the CTA of
// the first head of each KV group also appends row r's K/V to the cache.
template <typename WT>
__global__ void __launch_bounds__(128) k_attention(AttnArgs a) {
  extern __shared__ float sm[];
  const int h = blockIdx.x, r = blockIdx.y;
  const int hd = a.hd, half = hd >> 1;
  const int group = a.H / a.KV, g = h / group;
  float* qs = sm;                 // [hd]
  float* kn = qs + hd;            // [KMAX][hd] this step's rotated keys
  float* vn = kn + KMAX * hd;     // [KMAX][hd]
  float* sc = vn + KMAX * hd;     // [S] scores
  __shared__ float red[32];
  pdl_wait();
  if (!a.ctl->active) return;
  const int rows = a.ctl->rows, pos0 = a.ctl->pos0;
  if (r >= rows) return;
  const int p = pos0 + r;
  const int ncols = (a.H + 2 * a.KV) * hd;
  // rotate q (row r, head h) and the step's keys/values of group g
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float c = a.cos[(size_t)p * half + i], s = a.sin[(size_t)p * half + i];
    const float* q = a.qkv + (size_t)r * ncols + h * hd;
    const float x1 = q[i], x2 = q[i + half];
    qs[i] = x1 * c - x2 * s;
    qs[i + half] = x2 * c + x1 * s;
  }
  for (int j = 0; j <= r; ++j) {
    const int pj = pos0 + j;
    const float* kr = a.qkv + (size_t)j * ncols + (a.H + g) * hd;
    const float* vr = a.qkv + (size_t)j * ncols + (a.H + a.KV + g) * hd;
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
      const float c = a.cos[(size_t)pj * half + i], s = a.sin[(size_t)pj * half + i];
      const float x1 = kr[i], x2 = kr[i + half];
      kn[j * hd + i] = Elem<WT>::to_f(Elem<WT>::from_f(x1 * c - x2 * s));
      kn[j * hd + i + half] = Elem<WT>::to_f(Elem<WT>::from_f(x2 * c + x1 * s));
    }
    for (int i = threadIdx.x; i < hd; i += blockDim.x) vn[j * hd + i] = Elem<WT>::to_f(Elem<WT>::from_f(vr[i]));
  }
  __syncthreads();
  WT* kc = (WT*)a.kc + (size_t)g * a.S * hd;
  WT* vc = (WT*)a.vc + (size_t)g * a.S * hd;
  if (h % group == 0) {  // append row r's K/V (KV-cache write, pending-token scheme)
    for (int i = threadIdx.x; i < hd; i += blockDim.x) {
      kc[(size_t)p * hd + i] = Elem<WT>::from_f(kn[r * hd + i]);
      vc[(size_t)p * hd + i] = Elem<WT>::from_f(vn[r * hd + i]);
    }
  }
  // scores
  float mx = -INFINITY;
  for (int t = threadIdx.x; t <= p; t += blockDim.x) {
    float dot = 0.f;
    if (t < pos0) {
      const WT* kt = kc + (size_t)t * hd;
      for (int i = 0; i < hd; i += Elem<WT>::kVec) {
        float f[Elem<WT>::kVec];
        Elem<WT>::unpack(*(const uint4*)(kt + i), f);
#pragma unroll
        for (int e = 0; e < Elem<WT>::kVec; ++e) dot = fmaf(qs[i + e], f[e], dot);
      }
    } else {
      const float* kt = kn + (t - pos0) * hd;
      for (int i = 0; i < hd; ++i) dot = fmaf(qs[i], kt[i], dot);
    }
    dot *= a.scale;
    sc[t] = dot;
    mx = fmaxf(mx, dot);
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int t = threadIdx.x; t <= p; t += blockDim.x) {
    const float e = expf(sc[t] - mx);
    sc[t] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
  const float inv = 1.f / sum;
  for (int i = threadIdx.x; i < hd; i += blockDim.x) {
    float o = 0.f;
    for (int t = 0; t < pos0 && t <= p; ++t) o = fmaf(sc[t], Elem<WT>::to_f(vc[(size_t)t * hd + i]), o);
    for (int t = pos0; t <= p; ++t) o = fmaf(sc[t], vn[(t - pos0) * hd + i], o);
    a.out[(size_t)r * a.ldo + h * hd + i] = o * inv;
  }
  pdl_launch();
}

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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
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

cudaError_t launch_attention(int dtype, const AttnArgs& a, cudaStream_t st, bool pdl) {
  const size_t smem = (size_t)(a.hd + 2 * KMAX * a.hd + a.S) * sizeof(float);
  if (dtype == AMUSD_BF16) {
    auto k = k_attention<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return launch_pdl(k, dim3(a.H, KMAX), dim3(128), smem, st, pdl, a);
  }
  auto k = k_attention<float>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  return launch_pdl(k, dim3(a.H, KMAX), dim3(128), smem, st, pdl, a);
}

cudaError_t launch_argmax_final(StepCtl* ctl, const unsigned long long* part, int nparts, cudaStream_t st, bool pdl) {
  return launch_pdl(k_argmax_final, dim3(KMAX), dim3(256), 0, st, pdl, ctl, part, nparts);
}

}  // namespace amusd
