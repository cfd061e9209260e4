// prefill.h -- compute-bound prompt prefill (init_state, models.py:109-118).
//
// The decode forward (forward_tc.cu) streams every weight once per <= 16 token rows, so
// a 4096-token prompt through it re-reads the weights 256 times.  The prefill instead runs
// the prompt as dense GEMMs -- weights (the same tile-contiguous SW128 units) as the M=128
// operand, 256 tokens as the N operand of tcgen05.mma M128 N256 K16 -- plus a causal
// attention over the prompt, and writes the KV cache the decode steps continue from.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {
namespace pf {

constexpr int TN = 256;  // tokens per GEMM tile (MMA N)

enum { kEpStoreScaled = 0, kEpResid = 1, kEpGateUp = 2 };

struct GemmArgs {
  const uint8_t* wt;      // tiled weights of this GEMM (16 KB units, [tile][kb])
  int ntiles, kb;         // 128-row weight tiles, K / 64
  int M;                  // tokens
  int epi;
  float* out;             // StoreScaled: [M][ldo] fp32; Resid: h [M][ldo] (+=)
  __nv_bfloat16* out_b;   // GateUp: [M][ldo] bf16 activation
  int ldo;
  const float* inv;       // [M] RMSNorm scale of the input rows (StoreScaled / GateUp)
};

// Per-model prefill workspace (caller memory; amusd_prefill_bytes).
struct Work {
  int max_tokens;
  float* h;               // [max][d] residual stream
  float* inv;             // [max]
  __nv_bfloat16* x;       // [max][max(d, H hd)] normed GEMM input / attention output
  float* qkv;             // [max][(H + 2 KV) hd] (group-blocked columns)
  __nv_bfloat16* act;     // [max][ffn]
  int* tok;               // [max] prompt tokens
  CUtensorMap map_x_d, map_x_hh, map_act;  // TMA maps (box 64 x TN, SW128)
};

size_t work_bytes(int max_tokens, int d, int H, int KV, int hd, int ffn);
void carve(Work* w, void* base, int max_tokens, int d, int H, int KV, int hd, int ffn);
bool make_maps(Work* w, int d, int hh, int ffn);

cudaError_t launch_gemm(const CUtensorMap& mx, const GemmArgs& a, cudaStream_t st);
cudaError_t launch_embed(const int* tok, const __nv_bfloat16* emb, float* h, int M, int d, cudaStream_t st);
cudaError_t launch_norm(const float* h, const __nv_bfloat16* g, __nv_bfloat16* x, float* inv, int M, int d, float eps,
                        cudaStream_t st);
// RoPE on q / k of positions [0, M), K / V rounded to bf16 into the layer's cache (the decode
// steps read them back from there), q rotated in place (fp32).
cudaError_t launch_rope_kv(float* qkv, const float* cos, const float* sin, __nv_bfloat16* kc, __nv_bfloat16* vc,
                           int M, int H, int KV, int hd, int S, cudaStream_t st);
// Causal attention of positions [0, M) over the cached bf16 K / V, output bf16 [M][H hd].
cudaError_t launch_attention(const float* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc, __nv_bfloat16* out,
                             int M, int H, int KV, int hd, int S, float scale, cudaStream_t st);

}  // namespace pf
}  // namespace amusd
