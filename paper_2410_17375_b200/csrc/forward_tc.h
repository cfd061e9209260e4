// forward_tc.h -- persistent tcgen05 decoder forward: ONE launch per model
// forward (draft next_token+advance, models.py:120-131; verify
// verify_tokens+advance, models.py:151-169), replacing 1 + 5L + 2 kernels.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {
namespace fw {

// Phase kinds.  Phase p: 0 = embedding; 1 + 5l + k = layer l, k in
// {QKV, ATTN, O, GU, DOWN}; 1 + 5L = LM head.  Every phase depends on p-1.
enum { kKQkv = 0, kKAttn = 1, kKO = 2, kKGu = 3, kKDown = 4, kKEmbed = 5, kKLm = 6 };
// GEMM epilogues
enum { kEpStoreScaled = 0, kEpResid = 1, kEpGateUp = 2, kEpArgmax = 3 };
// GEMM kinds in FwArgs::g[]
enum { kGQkv = 0, kGO = 1, kGGu = 2, kGDown = 3, kGLm = 4, kNumGemm = 5 };

// One GEMM of the layer (identical shape in every layer; per-layer pointers
// are base + layer * stride).  Lives in the kernel parameters (constant
// bank): the persistent kernel never reads its schedule from global memory.
struct GemmKind {
  const uint8_t* wt;            // tile-contiguous SW128 weights (16 KB per unit), layer 0
  long long wt_stride;          // bytes between layers
  float* out;                   // StoreScaled / Resid output (fp32)
  __nv_bfloat16* out_b;         // GateUp output (bf16)
  __nv_bfloat16* xnext;         // Resid: next GEMM input bf16(h * gnext)
  const __nv_bfloat16* gnext;   // Resid: next RMSNorm weight, layer 0
  float* ssp_in;                // RMSNorm sums of this GEMM's input rows (StoreScaled / GateUp / Argmax)
  float* ssp_out;               // Resid: RMSNorm sums of the next GEMM's input
  long long ws_off;             // this kind's int64 split-K accumulator region (elements into FwArgs::ws)
  int cnt_off;                  // this kind's tile counters (ints into FwArgs::tile_cnt)
  int gnext_stride;             // elements between layers
  int epi, map;                 // epilogue, X map (0 xa, 1 attn, 2 act, 3 xb)
  int ntiles, kb, kc, nchunks, nitems;  // 128-row tiles, 64-wide K units per tile, units per item, items per tile
  int N, ldo;
  // Tensor parallelism (row-parallel O / down): this rank holds a K slice; every chunk red.adds
  // its int64 partial into EVERY rank's accumulator (peer memory) and bumps every rank's tile
  // count, so each rank's merger reads the exact all-rank sum -- the allreduce fused into the
  // split-K merge, bit-identical to the unsharded forward's sum over the same chunks.
  int xr;                       // 1: cross-rank reduce over FwArgs::peer_*
  int nchunks_total;            // chunks per tile over all ranks (== nchunks when xr == 0)
};

constexpr int kMaxTp = 8;       // tensor-parallel ranks of one verify model

struct FwArgs {
  GemmKind g[kNumGemm];
  int L;                        // layers
  int attn_max;                 // attention items per layer for 16 rows at max_seq (sizing only)
  StepCtl* ctl;
  int* sched;                   // 128-byte lines: [0] next item, [1] exit count, [2 + p] done count of phase p (self-resetting)
  // model
  const __nv_bfloat16* embed;
  const __nv_bfloat16* norms;   // packed RMSNorm weights [2L+1][d]: attn(l) at 2l, mlp(l) at 2l+1, final at 2L
  float* h;                     // [16][d] residual stream
  __nv_bfloat16* xa;            // [16][d] bf16(h * g): input of QKV / LM head (written by embed / down)
  float* ssp;                   // [16][d/128] per-tile sum of squares of h (pairs with xa)
  __nv_bfloat16* xb;            // [16][d] input of gate-up (written by O): double buffer of xa
  float* sspb;                  // pairs with xb
  long long* tflag;             // per-tile completion stamps of QKV / O / GU / DOWN (one 128-byte line each)
  int tflag_tiles;              // tiles per kind region
  int* agrp;                    // [L][KV] attention items finished per head group (self-resetting)
  float* qkv;                   // [16][(H+2KV)hd], group-blocked (qkv_group_row)
  __nv_bfloat16* attn_b;        // [16][H hd]
  char* kcache;                 // [L][KV][S][hd] bf16
  char* vcache;
  long long kv_layer_bytes;
  float* ws;                    // split-K partials [ntiles*nchunks][128][16]
  int* tile_cnt;                // split-K arrival counters, one 128-byte line per tile (self-resetting)
  float* attn_ws;               // attention split partials
  int* attn_cnt;
  const float* cos;
  const float* sin;
  unsigned long long* best;     // [16] argmax keys (self-resetting)
  float* logits;                // optional [16][V]
  int d, H, KV, hd, S, max_splits, vocab, eos, exclude_eos;
  float scale, eps;
  int stages;
  int prefetch_items;           // L2 prefetch distance in work items (0 = off)
  int prefetch_next;            // DOWN items prefetch the next layer's QKV + O weights into L2
  size_t qo_bytes;              // QKV + O tiled weight bytes of one layer (contiguous)
  int inflight;                 // max unlanded weight units per CTA (0 = ring depth)
  int debug;                    // perf-isolation bits (AMUSD_FW_DEBUG), 0 in production
  // Fused gate/up -> down (AMUSD_FW_FUSE, small models): every gate/up item is a whole tile (64
  // features); after its SiLU*up epilogue the same CTA streams the down weights of exactly those
  // 64 features (one 16 KB unit per output tile), multiplies them by the fresh act tile and
  // red.adds the int64 partials into the down accumulators.  The down phase shrinks to one
  // weight-less item per output tile that waits for all gate/up contributions and runs the
  // residual epilogue: one dependent GEMM phase less per layer.
  int fuse;
  int fine;                     // AMUSD_FW_FINE: bit (1 << consumer kind) = per-tile dependencies for
                                // that kind; 0 = phase-level everywhere (default)
  // Draft cut (co-located / split AMUSD draft only, else null): once the verifier has raised
  // a rollback request (*ab_req != ctl->rb_ack_local) or completion (*ab_done), this forward's
  // token will be discarded (k_draft_end), so the grab counter is moved past the item list.
  // Grabs are in index order and every wait targets lower indices, so the grabbed prefix
  // drains normally; launch_cut_cleanup re-arms the split state a cut tile/row left behind.
  const int* ab_req;
  const int* ab_done;
  long long* dbg;               // optional per-item timeline [item][8] (perf analysis), null in production
  int dbg_items;
  // Tensor parallelism (tp > 1): this rank's LM-head rows are global vocab ids
  // [vocab_off, vocab_off + N); the argmax keys go to every rank's `best` and the LM items of all
  // ranks are counted in every rank's lm counter (sched line 2, int 4) before a rank finalizes.
  int tp;
  int vocab_off;
  int lm_items_total;           // LM-head items over all ranks
  unsigned long long* peer_ws[kMaxTp];    // every rank's split-K accumulators (self included), rank order
  int* peer_cnt[kMaxTp];                  // every rank's split-K tile counters
  unsigned long long* peer_best[kMaxTp];  // every rank's argmax keys
  int* peer_sched[kMaxTp];                // every rank's schedule block (its LM arrival counter: lm_counter)
};

__host__ __device__ inline int num_phases(int L) { return 2 + 5 * L; }
constexpr int kCounterInts = 32;  // ints per schedule counter (one 128-byte line)
int attn_items_max(int KV, int S);
int attn_splits(int S);  // position splits of the persistent forward's attention (64-position chunks)
int max_positions();     // longest context (max_seq) the persistent forward's split merge supports

// Host: fill the GEMM kinds of a model (tiled weights laid out per layer as
// [qkv | o | gate-up | down], LM head after the last layer).
struct ModelView {
  int d, H, KV, hd, ffn, vocab, L, S;
  // tensor parallelism: the unsharded model's heads / kv heads / ffn (0 = not sharded); the
  // shard's kinds take the unsharded model's chunking so that every chunk partial -- and hence
  // the int64 all-rank sum -- is the unsharded forward's
  int tp, H_full, KV_full, ffn_full;
  const uint8_t* wt_layer0;     // tiled weights of layer 0 (qkv first)
  long long wt_layer_bytes;
  const uint8_t* wt_lm;
  const __nv_bfloat16* norms;   // packed [2L+1][d]
  float* h;
  float* qkv;
  __nv_bfloat16* xa;
  __nv_bfloat16* xb;
  float* ssp;
  float* sspb;
  __nv_bfloat16* act_b;
  int fuse;                     // 1: gate/up -> down fused (FwArgs::fuse); build_kinds clears it where unsupported
};
// ws_floats: int64 accumulator regions of all kinds (in float units); cnt_ints: tile counters;
// max_tiles: largest producer tile count (flag region size).
// grid > 0: kinds for a launch on `grid` (< all) SMs (larger items, see forward_tc.cu); the
// accumulator / counter needs never exceed the grid = 0 build's.
// Returns false when a tensor-parallel shard cannot take the unsharded chunking (a rank's K slice
// is not a whole number of chunks).
bool build_kinds(const ModelView& m, int units_per_item, FwArgs* a, size_t* ws_floats, int* cnt_ints, int* max_tiles,
                 int grid = 0);

cudaError_t launch_forward(const FwArgs& a, const CUtensorMap& m_xa, const CUtensorMap& m_attn,
                           const CUtensorMap& m_act, const CUtensorMap& m_xb, int grid, int stages, cudaStream_t st);
// After a forward launched with ab_req: if it was cut (flag in the schedule), zero the split-K
// accumulators / counters, attention counters and argmax keys (one CTA; a no-op otherwise).
cudaError_t launch_cut_cleanup(int* sched, const StepCtl* ctl, float* ws, size_t ws_floats, int* tile_cnt,
                               size_t cnt_ints, int* attn_cnt, size_t attn_cnt_ints, unsigned long long* best,
                               cudaStream_t st);
// Draft cuts counted by the cleanup (sched line 2, int 2).
inline int* cut_counter(int* sched) { return sched + 2 * kCounterInts + 2; }
// LM-head items of all tensor-parallel ranks that reached this rank (sched line 2, int 4).
__host__ __device__ inline int* lm_counter(int* sched) { return sched + 2 * kCounterInts + 4; }
// schedule counters: grab, exit, epoch (+ cut flag), then one per phase (kCounterInts each)
inline size_t sched_ints(int L) { return (size_t)(3 + num_phases(L)) * kCounterInts; }
int forward_smem_bytes(int stages, int hd, int group);

}  // namespace fw
}  // namespace amusd
