// transformer.h -- launch interface of the SIMT forward kernels.
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {

enum { kEpiStore = 0, kEpiResid = 1, kEpiGateUp = 2, kEpiArgmax = 3 };

struct GemvArgs {
  const StepCtl* ctl;
  const float* x;          // [KMAX][ldx] fp32 activations
  int ldx;
  const void* gamma;       // RMSNorm weight [K] (model dtype) or nullptr
  const void* W;           // [N][K]
  const void* W2;          // [N][K] up-projection (gate/up epilogue)
  int N, K, kc;            // kc: K-chunk staged in shared memory
  float eps;
  float* out;              // store / residual / activation output
  int ldo;
  unsigned long long* part;  // argmax partials [KMAX][grid]
  float* logits;             // optional fp32 logits [KMAX][N] (debug/parity)
  int eos, exclude_eos;
};

struct AttnArgs {
  const StepCtl* ctl;
  const float* qkv;        // [KMAX][(H+2KV)*hd] fp32, un-rotated
  void* kc;                // this layer's K cache [KV][S][hd]
  void* vc;                // this layer's V cache [KV][S][hd]
  const float* cos;        // [S][hd/2]
  const float* sin;
  float* out;              // [KMAX][ldo] fp32 (SIMT path)
  void* out_b;             // [KMAX][ldo] bf16 (tensor-core path) -- used when non-null
  int ldo;
  int H, KV, hd, S;
  float scale;
  float* ws;               // split partials [KV][KMAX][max_splits][group][hd+2]
  int* counters;           // [KV][KMAX] arrival counters (self re-arming)
  int max_splits;
  int blocked;             // qkv in group-blocked layout (tensor-core models, qkv_group_row)
};

int attn_max_splits(int max_seq);

int gemv_kc(int nr, int K);
int gemv_grid(int N, int rpw);
cudaError_t launch_gemv(int nr, int dtype, int epi, const GemvArgs& a, cudaStream_t st, bool pdl);
cudaError_t launch_embed(int dtype, const StepCtl* ctl, const void* emb, float* h, int d, cudaStream_t st, bool pdl);
cudaError_t launch_attention(int dtype, const AttnArgs& a, cudaStream_t st, bool pdl);
cudaError_t launch_argmax_final(StepCtl* ctl, const unsigned long long* part, int nparts, cudaStream_t st, bool pdl);

}  // namespace amusd
