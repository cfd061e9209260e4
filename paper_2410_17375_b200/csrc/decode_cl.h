// decode_cl.h -- cluster decode forward: the draft model's next_token + advance
// (models.py:120-131) with two grid-wide dependencies per layer instead of five.
//
// Why: the 1-row forward is a chain of dependent phases (QKV -> attention -> O -> gate/up ->
// down); every grid-wide hand-off costs ~1.5-5 us on B200, which is what
// holds the 1B draft near 0.43 of the HBM roofline in both other persistent designs.  Here:
//
//   phase A  one thread-block CLUSTER of 8 CTAs per KV head group: QKV rows of the group,
//            cluster barrier (DSMEM), attention of the group over all positions split across
//            the 8 CTAs, cluster barrier, every CTA merges the 8 partials from its peers' shared
//            memory, then its slice of the O projection restricted to the group's head columns
//            -> int64 fixed-point red.add into the residual accumulator (split-K over groups);
//   grid barrier;
//   phase B  every CTA: gate/up of its 16-feature blocks -> SiLU*up -> the down projection of
//            exactly those features (down^T slabs, K = 16 per block) -> int64 red.add;
//   grid barrier; every CTA rebuilds h = h + O + down itself (fixed order: deterministic).
//
// Integer accumulators commute, so the result is independent of arrival order.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {
namespace cl {

constexpr int kCluster = 8;   // CTAs per cluster (portable size)
constexpr int kMaxRows = 8;   // activation rows per forward (the MMA's N)

struct ClArgs {
  // weights in the cluster-decode layout (tile_layer / tile_lm): per layer
  // [qkv by group | o by group | gate/up by 16-feature block | down^T by 16-feature block]
  const uint8_t* wt;
  long long layer_bytes, off_o, off_gu, off_dn;
  const uint8_t* wt_lm;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* norms;     // packed [2L+1][d]: attn(l) 2l, mlp(l) 2l+1, final 2L
  const float* cos;
  const float* sin;
  StepCtl* ctl;
  char* kcache;                   // [L][KV][S][hd] bf16
  char* vcache;
  long long kv_layer_bytes;
  float* h;                       // [2][kMaxRows][d] residual stream at layer entry (parity)
  unsigned long long* acc;        // [2 kinds: O, down][2 parity][kMaxRows][d] int64 (2^-32)
  int* sync;                      // counters (sync_ints), self-resetting
  unsigned long long* best;       // [KMAX]
  float* logits;                  // optional [KMAX][vocab]
  const int* ab_req;              // draft cut (see FwArgs::ab_req)
  const int* ab_done;
  int* cuts;
  int d, H, KV, hd, ffn, vocab, L, S, eos, exclude_eos;
  float eps, scale;
  int stages;
  int l2_ahead;                   // L2 prefetch distance in units (0 = off)
  int debug;
  long long* dbg;                 // optional per-CTA timeline [grid][kDbgPerLayer * L] (perf analysis)
};
constexpr int kDbgPerLayer = 12;

struct Layout {
  long long layer_bytes, off_o, off_gu, off_dn, lm_off, total;
};
bool supported(int d, int H, int KV, int hd, int ffn, int vocab);
Layout layout(int d, int H, int KV, int hd, int ffn, int vocab, int L);
// Tile one layer (row-major bf16 weights) / the LM head into the layout above.
cudaError_t tile_layer(const void* wqkv, const void* wo, const void* wgate, const void* wup, const void* wdown,
                       int d, int H, int KV, int hd, int ffn, void* dst, cudaStream_t st);
cudaError_t tile_lm(const void* lm, int vocab, int d, void* dst, cudaStream_t st);
size_t sync_ints();
size_t h_bytes(int d);
size_t acc_bytes(int d);
int max_stages(int d, int H, int KV, int hd);
// Largest grid (a multiple of 8) whose clusters can all be resident at once (<= want).
int grid_for(const ClArgs& a, int want);
cudaError_t launch(const ClArgs& a, int grid, cudaStream_t st);

}  // namespace cl
}  // namespace amusd
