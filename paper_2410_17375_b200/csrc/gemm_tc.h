// gemm_tc.h -- tcgen05 GEMM interface (verify/prefill forwards, bf16).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {
namespace tc {

enum { kTcStoreScaled = 0, kTcResid = 1, kTcGateUp = 2, kTcArgmax = 3 };

struct TcArgs {
  const StepCtl* ctl;
  const uint8_t* wt;     // weights pre-tiled: [ntiles][kb][128 rows][128 B], SW128-swizzled (16 KB per unit)
  int epi;
  int ntiles;            // 128-row weight tiles (gate/up: 64 features per tile)
  int kb;                // K / 64
  int N;                 // output features (argmax guard)
  const float* inv;      // per-row RMSNorm scale or nullptr
  float* out;            // fp32 output (store / residual)
  __nv_bfloat16* out_b;  // bf16 output (gate/up activation)
  int ldo;
  unsigned long long* part;  // argmax partials [16][ntiles]
  float* logits;             // optional fp32 logits [16][N] (parity/debug)
  int eos, exclude_eos;
  // RMSNorm fusion: residual epilogues emit the next GEMM's bf16 input and
  // per-tile sums of squares; consumers turn them into inv_rms per row.
  __nv_bfloat16* xnext;        // [16][ldo] bf16(h_new * gnext) or nullptr
  const __nv_bfloat16* gnext;  // next RMSNorm weight [ldo]
  float* ssp;                  // [16][ssp_tiles] partial sum of h_new^2 (written by residual epilogues)
  const float* ssp_in;         // same buffer read by consumers (nullptr: no norm)
  int ssp_tiles;               // d / 128
  float norm_dim, eps;
  float* ws;             // stream-K partials [grid][2][128][16]
  int* counters;         // per-tile arrival counters (zeroed once, self re-arming)
  int debug;             // perf-isolation knobs (AMUSD_TC_DEBUG), 0 in production
};

bool make_map(CUtensorMap* m, const void* ptr, int rows, int cols, int box_rows);
// Re-layout a row-major bf16 [N][K] matrix (or a gate/up pair) into the
// tile-contiguous SW128 layout read by the GEMM (one 16 KB bulk copy per unit).
size_t tiled_bytes(int N, int K);
// qkv_H > 0: the QKV weight rows are re-ordered into per-KV-head group blocks
// [q of the G heads | k | v] (qkv_group_row), so a head group's outputs are
// produced by consecutive 128-row tiles.
cudaError_t launch_tile_weights(const void* src, const void* src2, void* dst, int N, int K, cudaStream_t st,
                                int qkv_H = 0, int qkv_KV = 0, int qkv_hd = 0);
int tc_grid(int ntiles, int kb);
cudaError_t launch_gemm_tc(const CUtensorMap& mx, const TcArgs& a, cudaStream_t st, bool pdl);
cudaError_t launch_embed_tc(const StepCtl* ctl, const void* emb, float* h, const void* g, void* xb, float* ssp,
                            int d, cudaStream_t st, bool pdl);
cudaError_t launch_prep_norm(const StepCtl* ctl, const float* h, const void* g, void* xb, float* inv, int d, float eps,
                             cudaStream_t st, bool pdl);

}  // namespace tc
}  // namespace amusd
