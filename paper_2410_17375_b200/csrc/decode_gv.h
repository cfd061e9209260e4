// decode_gv.h -- persistent SIMT decode forward for few-row forwards: the draft model's
// next_token + advance (models.py:120-131), north-star subsystem (1): fused RMSNorm + GEMV
// phases over the row-major bf16 weights with 128-bit loads and warp-shuffle reductions,
// KV-cache attention, fused argmax.  ONE launch per forward.
//
// Why a second persistent forward next to forward_tc.cu's tcgen05 one: a 1-row forward is a
// GEMV.  Its rows are partitioned STATICALLY over the CTAs (every phase, every layer), so a
// producer warp knows every weight byte its CTA will read for the whole forward and streams
// them through the shared-memory ring without ever waiting on a dependency; only the
// consumers wait (one grid barrier per phase).  The work-queue kernel's per-item machinery
// (grab, TMEM hand-off, split-K publish/merge) is what held the 1B draft at ~0.43 of HBM
// roofline.
//
// Co-residency: the grid barrier needs every CTA resident.  Launches use grid <= the SMs the
// caller reserves for the model (all SMs alone, the draft share when co-located) and each CTA
// leaves room on its SM for the 1-CTA protocol kernels that may spin beside it (registers
// capped, 2 KB of shared memory left free).  Every wait is bounded (trap, never a hang).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {
namespace gv {

constexpr int kMaxLayers = AMUSD_MAX_LAYERS;
constexpr int kDbgEvents = 2 * (5 * kMaxLayers + 1) + 2;

struct GvArgs {
  // GEMV weights tiled by tile_weights (decode layout): per layer [qkv | o | gate-up | down],
  // LM head after the last layer
  const uint8_t* wt;
  long long wt_layer_bytes, wt_off_o, wt_off_gu, wt_off_down;
  const uint8_t* wt_lm;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* lm;        // LM head [vocab][d] (== embed when tied)
  const __nv_bfloat16* norms;     // packed RMSNorm weights [2L+1][d]: attn(l) 2l, mlp(l) 2l+1, final 2L
  const float* cos;               // RoPE tables [S][hd/2]
  const float* sin;
  StepCtl* ctl;
  char* kcache;                   // [L][KV][S][hd] bf16
  char* vcache;
  long long kv_layer_bytes;
  // scratch (model-owned, HBM)
  float* h;                       // [KMAX][d] residual stream
  __nv_bfloat16* xa;              // [KMAX][d] bf16(h * g): QKV / LM-head input
  __nv_bfloat16* xb;              // [KMAX][d] gate/up input
  float* qkv;                     // [KMAX][(H+2KV)hd] natural [q | k | v] order, RMSNorm scale applied
  __nv_bfloat16* attn_b;          // [KMAX][H hd] attention output (O input)
  __nv_bfloat16* act_b;           // [KMAX][ffn] SiLU(gate) * up (down input)
  float* ss;                      // [grid][KMAX] per-CTA sums of squares of the residual rows it owns
  float* attn_ws;                 // [KV][nsplit][KMAX][G][hd + 2] attention split partials (m, l, o)
  int* sync;                      // counters (sync_ints), self-resetting
  unsigned long long* best;       // [KMAX] argmax keys, self-resetting
  float* logits;                  // optional [KMAX][vocab]
  // draft cut (co-located / split AMUSD draft, else null): see FwArgs::ab_req
  const int* ab_req;
  const int* ab_done;
  int* cuts;                      // cut counter (amusd_run_info.draft_cuts)
  int d, H, KV, hd, ffn, vocab, L, S, eos, exclude_eos;
  float eps, scale;
  int stages;                     // weight ring stages (16 KB each)
  int l2_ahead;                   // L2 prefetch distance in units (0 = off)
  long long* dbg;                 // optional per-CTA phase timeline [grid][kDbgEvents] (perf analysis)
  int debug;                      // perf-isolation bits (AMUSD_GV_DEBUG): 1 no weights, 2 no grid waits
  int max_splits;                 // attention splits the workspace holds
};

// Shapes the kernel takes: GEMV K a multiple of 64 (<= 16384), output rows in 16-row blocks,
// head_dim 64 or 128, at most 8 query heads per KV head.
bool supported(int d, int H, int KV, int hd, int ffn, int vocab);
size_t sync_ints(int KV);
size_t ss_floats();
int attn_splits(int S);
size_t attn_ws_floats(int KV, int G, int hd, int S);
int max_stages(int d, int H, int KV, int hd, int ffn);
// Decode weight layout: bytes of one layer and the kind offsets inside it; total incl. LM head.
struct Layout {
  long long layer_bytes, off_o, off_gu, off_down, lm_off, total;
};
Layout layout(int d, int H, int KV, int hd, int ffn, int vocab, int L);
// Tile one GEMM kind of one layer (row-major [N][K] bf16; gate/up: two [ffn][d] sources) into
// its decode units at dst.
cudaError_t tile_weights(const void* src, const void* src2, int N, int K, void* dst, cudaStream_t st);
cudaError_t launch(const GvArgs& a, int grid, cudaStream_t st);

}  // namespace gv
}  // namespace amusd
