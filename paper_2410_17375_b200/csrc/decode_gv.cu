// decode_gv.cu -- persistent decode forward for few-row forwards (see decode_gv.h): the
// draft model's next_token + advance (reference plug-in models.py:120-131), ONE launch per
// forward.
//
// Phases per layer: QKV (GEMV, RMSNorm scale in the epilogue) | attention (RoPE, KV append,
// 128-position splits merged by the last split) | O (GEMV + residual) | gate/up (GEMV,
// SiLU(gate)*up) | down (GEMV + residual); then the LM head with a fused first-index argmax.
//
// GEMV: the weights are re-laid-out once (amusd_model_set_decode) as 16 KB units of 16 rows x
// 512 K (16-byte chunks XOR-swizzled by row: conflict-free ldmatrix), 16-row blocks of
// consecutive units.  Blocks are partitioned statically over the CTAs, so the units a CTA
// streams are known for the whole forward: warp 8 (the producer) bulk-copies them through a
// ring of shared-memory stages and never waits on a dependency -- HBM keeps streaming through
// the grid barriers between phases.  Warps 0-7 take the CTA's blocks round-robin and run
// mma.sync m16n8k16 (bf16 in, fp32 accumulate) with the 16 weight rows as A and the <= 8 live
// activation rows (bf16 in shared memory) as B: ~8x fewer instructions than FMA GEMVs and no
// cross-lane reductions -- every accumulator lane holds finished (row, activation-row) sums.
//
// Numerics (as forward_tc.cu, so the bf16-faithful oracle describes both): GEMV inputs are
// bf16 (bf16(h*g) for normed inputs, the attention output, SiLU*up); accumulation fp32; the
// RMSNorm factor rsqrt(mean(h^2)+eps) scales the GEMV output; K/V are rounded to bf16 before
// use.  Every sum has a fixed order, and a row's arithmetic does not depend on how many rows
// the forward carries (batch invariance: MMA columns are independent).
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "decode_gv.h"
#include "tc_ptx.cuh"

namespace amusd {
namespace gv {

using bf16 = __nv_bfloat16;
using tc::bulk_load;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::named_bar;
using tc::policy_evict_first;
using tc::smem_u32;

constexpr int kCW = 8;                   // consumer warps
constexpr int kCT = kCW * 32;            // consumer threads
constexpr int kThreads = kCT + 32;       // + producer warp
constexpr int kMB = 16;                  // weight rows per block (MMA M)
constexpr int kKW = 512;                 // K per unit
constexpr int kStage = kMB * kKW * 2;    // ring stage bytes (one unit)
constexpr int kChunk = 128;              // attention positions per split
constexpr int kPad = 32;                 // ints per counter line
constexpr int kMaxStages = 16;
constexpr int kMaxGrid = 256;
constexpr int kMaxG = 8;
constexpr int kSsBlk = 8;                // residual blocks per CTA whose h^2 sums stay in shared memory
constexpr int kSmemBudget = 232448 - 2048;  // leave room for 1-CTA protocol kernels on the SM
constexpr long long kWaitNs = 4ll * 1000 * 1000 * 1000;

// sync block lines
constexpr int kSyncBar = 0;              // grid-barrier arrivals (monotone within a launch)
constexpr int kSyncExit = 1 * kPad;      // CTAs done
constexpr int kSyncLm = 2 * kPad;        // LM-head arrivals
constexpr int kSyncCut = 3 * kPad;       // 1: some CTA cut this forward
constexpr int kSyncAttn = 4 * kPad;      // + g * kPad: attention splits finished for kv head g

enum { kQkv = 0, kO = 1, kGu = 2, kDown = 3, kLm = 4 };

struct alignas(16) Aux {
  unsigned long long full[kMaxStages];
  unsigned long long empty[kMaxStages];
  int seq[kMaxStages];     // times each ring slot was consumed (orders a slot's reuse across warps)
  float scale[KMAX];
  unsigned long long key[KMAX];
  float ml[4][kMaxG][2];
  float part[kCW][32][4];  // per-warp MMA partials of a K-split block
  float ssb[kSsBlk][KMAX];  // residual phases: sum of h^2 per (owned block, activation row)
  int cut;
  int go;
  int consumed;
  int issued;
  int last;
};

// Shared memory after the ring: the GEMV input rows (bf16, rows padded by 16 bytes: the B
// fragment loads of 8 rows hit 8 distinct bank groups) or, in the attention phase, the
// queries and scores.
__host__ __device__ inline int xs_pitch(int K) { return K * 2 + 16; }
// Attention scratch in the union: ks, vs [kChunk][HD + 8] bf16 (16-byte row padding: the
// score threads' row reads spread over the bank groups) | qs [4][G][HD] f32 | sc [4][G][kChunk] f32.
__host__ __device__ inline int attn_pitch(int hd) { return hd * 2 + 16; }
__host__ __device__ inline int attn_bytes(int G, int hd) {
  return 2 * kChunk * attn_pitch(hd) + 4 * G * hd * 4 + 4 * G * kChunk * 4;
}

__host__ __device__ inline int union_bytes(int d, int H, int KV, int hd, int ffn) {
  const int kmax = d > H * hd ? (d > ffn ? d : ffn) : (H * hd > ffn ? H * hd : ffn);
  const int xs = 2 * xs_pitch(kmax), at = attn_bytes(H / KV, hd);
  return ((xs > at ? xs : at) + 127) / 128 * 128;
}

// ------------------------------------------------------------------ helpers
AMUSD_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
AMUSD_DEV bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok;
}
AMUSD_DEV void mbar_wait_b(uint32_t a, uint32_t parity) {
  if (mbar_try(a, parity)) return;
  const long long t0 = globaltimer();
  for (int it = 1; !mbar_try(a, parity); ++it)
    if ((it & 63) == 0 && globaltimer() - t0 > kWaitNs) __trap();
}
struct F8 {
  float v[8];
};
AMUSD_DEV F8 unpack8(const uint4& u) {
  F8 f;
  f.v[0] = __uint_as_float(u.x << 16); f.v[1] = __uint_as_float(u.x & 0xFFFF0000u);
  f.v[2] = __uint_as_float(u.y << 16); f.v[3] = __uint_as_float(u.y & 0xFFFF0000u);
  f.v[4] = __uint_as_float(u.z << 16); f.v[5] = __uint_as_float(u.z & 0xFFFF0000u);
  f.v[6] = __uint_as_float(u.w << 16); f.v[7] = __uint_as_float(u.w & 0xFFFF0000u);
  return f;
}
AMUSD_DEV float bfr(float v) { return __bfloat162float(__float2bfloat16(v)); }

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }

// Warp reduce-scatter of V lane-partials (V a power of two <= 32): returns the warp total of
// value index (lane >> (5 - log2 V)).  V - 1 + 5 - log2 V shuffles instead of 5 V.
template <int V>
AMUSD_DEV float reduce_scatter(float (&v)[V], int lane) {
  constexpr int LV = ilog2(V);
#pragma unroll
  for (int st = 0; st < LV; ++st) {
    const int half = V >> (st + 1);
    const int o = 16 >> st;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  float s = v[0];
#pragma unroll
  for (int o = 16 >> LV; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
AMUSD_DEV uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
AMUSD_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
AMUSD_DEV void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------------ GEMV schedule
// Phase of the static schedule: this CTA's 16-row blocks [b0, b1), nk units (K / 512) each.
// Gate/up blocks are 8 gate rows then the 8 up rows of the same 8 features.
struct WPhase {
  const uint8_t* w;   // first unit of block 0 of this kind and layer
  int K, nk, b0, b1;
};
AMUSD_DEV WPhase wphase_of(const GvArgs& a, int kind, int l) {
  WPhase p;
  int N;
  const uint8_t* lw = a.wt + (size_t)l * a.wt_layer_bytes;  // (kind kLm: unused)
  switch (kind) {
    case kQkv: p.w = lw; p.K = a.d; N = (a.H + 2 * a.KV) * a.hd; break;
    case kO: p.w = lw + a.wt_off_o; p.K = a.H * a.hd; N = a.d; break;
    case kGu: p.w = lw + a.wt_off_gu; p.K = a.d; N = 2 * a.ffn; break;
    case kDown: p.w = lw + a.wt_off_down; p.K = a.ffn; N = a.d; break;
    default: p.w = a.wt_lm; p.K = a.d; N = a.vocab; break;
  }
  const int nb = N / kMB, G = gridDim.x, c = blockIdx.x;
  p.b0 = (int)((long long)nb * c / G);
  p.b1 = (int)((long long)nb * (c + 1) / G);
  p.nk = (p.K + kKW - 1) / kKW;
  return p;
}
// Unit q of a block: K columns [512 q, 512 q + kw), kw = min(512, K - 512 q) (a multiple of 64).
AMUSD_DEV int unit_kw(int K, int q) { return min(kKW, K - q * kKW); }
AMUSD_DEV size_t unit_off(int K, int b, int q) { return (size_t)b * kMB * K * 2 + (size_t)q * kMB * kKW * 2; }
// Activation rows per pass: the MMA's N = 8, or what the shared-memory copy holds for this K.
AMUSD_DEV int pass_rows(const GvArgs& a, int K) {
  return min(8, union_bytes(a.d, a.H, a.KV, a.hd, a.ffn) / xs_pitch(K));
}

// ------------------------------------------------------------------ producer
// Position in the CTA's static unit schedule (layers x {QKV, O, gate/up, down} x passes x
// blocks x units, then the LM head).
struct Cursor {
  int l, kind, ps, b, q, npass;
  WPhase p;
  bool done;
};
AMUSD_DEV void cursor_phase(const GvArgs& a, Cursor& c, int R, int xs_bytes) {
  for (;;) {
    if (c.l > a.L || (c.l == a.L && c.kind > 0)) { c.done = true; return; }
    c.p = wphase_of(a, c.l == a.L ? kLm : c.kind, c.l == a.L ? 0 : c.l);
    c.npass = (R + pass_rows(a, c.p.K) - 1) / pass_rows(a, c.p.K);
    c.ps = 0; c.b = c.p.b0; c.q = 0;
    if (c.p.b1 > c.p.b0) return;
    if (++c.kind == 4) { c.kind = 0; ++c.l; }
  }
}
AMUSD_DEV void cursor_init(const GvArgs& a, Cursor& c, int R, int xs_bytes) {
  c.l = 0; c.kind = 0; c.done = false;
  cursor_phase(a, c, R, xs_bytes);
}
AMUSD_DEV void cursor_next(const GvArgs& a, Cursor& c, int R, int xs_bytes) {
  if (++c.q < c.p.nk) return;
  c.q = 0;
  if (++c.b < c.p.b1) return;
  c.b = c.p.b0;
  if (++c.ps < c.npass) return;
  if (++c.kind == 4 || c.l == a.L) { c.kind = 0; ++c.l; }
  cursor_phase(a, c, R, xs_bytes);
}

// Streams every weight unit of this CTA's static schedule, in consumption order.  Optionally
// (a.l2_ahead = D > 0) prefetches unit i + D into L2 when unit i enters the ring: HBM keeps
// streaming D units ahead while the consumers sit in a grid barrier or the attention phase
// with the ring full.  Stops early only when the consumers have cut the forward (ax->cut);
// the issued stages are drained at exit.
AMUSD_DEV void producer(const GvArgs& a, Aux* ax, uint8_t* ring, int R, int xs_bytes) {
  const uint64_t pol = policy_evict_first(), pol_keep = tc::policy_evict_last();
  volatile int* cut = &ax->cut;
  Cursor c, f;
  cursor_init(a, c, R, xs_bytes);
  if (a.debug & 1) { ax->issued = 0; return; }  // perf isolation: no weight traffic
  const int D = a.l2_ahead;
  if (D > 0) {  // prefetch cursor D units ahead of the ring's
    cursor_init(a, f, R, xs_bytes);
    for (int j = 0; j < D && !f.done; ++j) {
      if (j >= a.stages) {
        const int ub = kMB * unit_kw(f.p.K, f.q) * 2;
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(f.p.w + unit_off(f.p.K, f.b, f.q)),
                     "r"(ub), "l"(pol_keep) : "memory");
      }
      cursor_next(a, f, R, xs_bytes);
    }
  }
  int i = 0;
  for (; !c.done; cursor_next(a, c, R, xs_bytes), ++i) {
    const int slot = i % a.stages;
    if (i >= a.stages) {
      const uint32_t bar = smem_u32(&ax->empty[slot]), par = ((i / a.stages) - 1) & 1;
      const long long t0 = globaltimer();
      while (!mbar_try(bar, par)) {
        if (*cut) { ax->issued = i; return; }
        if (globaltimer() - t0 > kWaitNs) __trap();
      }
    }
    if (*cut) { ax->issued = i; return; }
    const int ub = kMB * unit_kw(c.p.K, c.q) * 2;
    const uint32_t full = smem_u32(&ax->full[slot]);
    mbar_expect_tx(full, ub);
    bulk_load(smem_u32(ring + (size_t)slot * kStage), c.p.w + unit_off(c.p.K, c.b, c.q), ub, full, pol);
    if (D > 0 && !f.done) {
      const int fb = kMB * unit_kw(f.p.K, f.q) * 2;
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(f.p.w + unit_off(f.p.K, f.b, f.q)),
                   "r"(fb), "l"(pol_keep) : "memory");
      cursor_next(a, f, R, xs_bytes);
    }
  }
  ax->issued = i;
}

// ------------------------------------------------------------------ consumer state
struct Cons {
  int ct, warp, lane;
  int R, pos0;
  int stage;     // ring stages of the CTA's schedule before this phase
  int bar;       // grid barriers passed
  int blk;       // 16-row blocks of the CTA's schedule before this phase (warp rotation)
  long long* dbg;  // this CTA's timeline row (null: off)
  int ev;
};

// Residual rows this CTA owns: the 16-row blocks of the O / down partition.
AMUSD_DEV void own_rows(int d, int& n0, int& n1) {
  const int nb = d / kMB;
  n0 = kMB * (int)((long long)nb * blockIdx.x / gridDim.x);
  n1 = kMB * (int)((long long)nb * (blockIdx.x + 1) / gridDim.x);
}

// Grid barrier b complete (every CTA arrived b+1 times).  Thread 0 polls; the decision (go
// or cut) is broadcast through shared memory so every consumer takes the same branch.
AMUSD_DEV bool grid_wait(const GvArgs& a, Aux* ax, Cons& cs) {
  const int target = (cs.bar + 1) * (int)gridDim.x;
  ++cs.bar;
  if (cs.ct == 0) {
    int go = 1;
    const int ack = a.ab_req ? ld_volatile(&a.ctl->rb_ack_local) : 0;
    const long long t0 = globaltimer();
    for (int it = 0;; ++it) {
      if ((a.debug & 2) || ld_acquire_gpu(a.sync + kSyncBar) >= target) break;
      if (a.ab_req && ((ld_volatile(a.ab_req) ^ ack) | ld_volatile(a.ab_done))) { go = 0; break; }
      if ((it & 63) == 63 && globaltimer() - t0 > kWaitNs) __trap();
    }
    if (!go) *(volatile int*)&ax->cut = 1;
    ax->go = go;
    if (cs.dbg) cs.dbg[cs.ev] = globaltimer();
  }
  ++cs.ev;
  named_bar(1, kCT);
  return ax->go != 0;
}
// This CTA's writes of the phase are done (all consumers passed the barrier before): release.
AMUSD_DEV void grid_arrive(const GvArgs& a, Cons& cs) {
  named_bar(1, kCT);
  if (cs.ct == 0) {
    if (cs.dbg) cs.dbg[cs.ev] = globaltimer();
    // release (cumulative over the CTA's writes ordered before it by the barrier above)
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.sync + kSyncBar) : "memory");
  }
  ++cs.ev;
}

// Layer-0 input straight from the embedding rows (no embedding phase): every CTA computes the
// factor of each row itself and writes the residual rows it owns.
AMUSD_DEV void embed_prologue(const GvArgs& a, Aux* ax, const Cons& cs) {
  for (int r = cs.warp; r < cs.R; r += kCW) {
    const bf16* e = a.embed + (size_t)a.ctl->tok[r] * a.d;
    float s = 0.f;
    for (int k = cs.lane * 8; k < a.d; k += 256) {
      const F8 f = unpack8(__ldg((const uint4*)(e + k)));
#pragma unroll
      for (int j = 0; j < 8; ++j) s = fmaf(f.v[j], f.v[j], s);
    }
    s = warp_sum(s);
    if (cs.lane == 0) ax->scale[r] = 1.0f / sqrtf(s / (float)a.d + a.eps);
  }
  int n0, n1;
  own_rows(a.d, n0, n1);
  for (int i = cs.ct; i < cs.R * (n1 - n0); i += kCT) {
    const int r = i / (n1 - n0), n = n0 + i % (n1 - n0);
    a.h[(size_t)r * a.d + n] = __bfloat162float(a.embed[(size_t)a.ctl->tok[r] * a.d + n]);
  }
  named_bar(1, kCT);
}

// 8 activations of row `row` at k (bf16).  src == null: layer-0 input bf16(E[tok] * g0).
AMUSD_DEV uint4 x_global(const GvArgs& a, const bf16* src, const bf16* gamma, int K, int row, int k) {
  if (src) return __ldcg((const uint4*)(src + (size_t)row * K + k));
  const F8 e = unpack8(__ldg((const uint4*)(a.embed + (size_t)a.ctl->tok[row] * a.d + k)));
  const F8 g = unpack8(__ldg((const uint4*)(gamma + k)));
  __nv_bfloat162 b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(e.v[2 * j] * g.v[2 * j], e.v[2 * j + 1] * g.v[2 * j + 1]);
  return *(const uint4*)b;
}

// Phase start: activation rows r0 .. r0 + nrows - 1 of the GEMV input into shared memory.
AMUSD_DEV void fill_xs(const GvArgs& a, Aux* ax, uint8_t* xs, int r0, int nrows, const bf16* src, const bf16* gamma,
                       int K, bool scales, const Cons& cs) {
  // the RMSNorm factors (per-CTA sums of squares of the previous residual phase) are fetched in
  // the same round trip as the activations: issue both, then reduce
  float ssv[(kMaxGrid + 31) / 32];
  const int G = gridDim.x;
  const bool sc = scales && cs.warp < cs.R;
  if (sc) {
#pragma unroll
    for (int j = 0; j < (kMaxGrid + 31) / 32; ++j) {
      const int c = cs.lane + 32 * j;
      ssv[j] = c < G ? __ldcg(a.ss + (size_t)c * KMAX + cs.warp) : 0.f;
    }
  }
  const int n8 = K / 8;
  for (int i = cs.ct; i < nrows * n8; i += kCT) {
    const int r = i / n8, k = (i % n8) * 8;
    *(uint4*)(xs + (size_t)r * xs_pitch(K) + k * 2) = x_global(a, src, gamma, K, r0 + r, k);
  }
  if (scales) {
    for (int r = cs.warp; r < cs.R; r += kCW) {
      float s = 0.f;
      if (r == cs.warp) {
#pragma unroll
        for (int j = 0; j < (kMaxGrid + 31) / 32; ++j) s += ssv[j];
      } else {  // > 8 live rows: the extra rows in a second round trip
        for (int c = cs.lane; c < G; c += 32) s += __ldcg(a.ss + (size_t)c * KMAX + r);
      }
      s = warp_sum(s);
      if (cs.lane == 0) ax->scale[r] = 1.0f / sqrtf(s / (float)a.d + a.eps);
    }
  }
  named_bar(1, kCT);
}

// One warp, one 16-row block over its units q0, q0 + qstep, ... < nk: mma.sync m16n8k16 with
// the 16 weight rows as A (ldmatrix from the swizzled unit) and the <= 8 activation rows of
// the pass as B (bf16 in shared memory; rows >= nx read as zero).  C in the MMA accumulator
// layout: c[e] = (block row g + 8 (e >> 1), activation row r0 + 2 q + (e & 1)), g = lane / 4,
// q = lane % 4.  Four independent MMA chains (k-block mod 4), summed in fixed order.
AMUSD_DEV void block_mma(const GvArgs& a, Aux* ax, uint32_t ring_s, uint32_t xs_s, int K, int nk, int i0, int q0,
                         int qstep, int nx, float (&c)[4], const Cons& cs) {
  const int lane = cs.lane, g = lane >> 2, q = lane & 3;
  const int pitch = xs_pitch(K);
  // ldmatrix x4 row addresses: matrix j = lane/8 -> rows (lane&7) + 8*(j&1), 16-byte chunk (j>>1)
  const int mrow = (lane & 7) + 8 * ((lane >> 3) & 1), mchunk = lane >> 4, msw = mrow & 7;
  const bool bx = g < nx;
  const uint32_t xrow = xs_s + (uint32_t)(g * pitch + q * 4);
  float acc[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  for (int u = q0; u < nk; u += qstep) {
    const int i = i0 + u, slot = i % a.stages, kw = unit_kw(K, u);
    if (!(a.debug & 1)) {  // the slot's previous stage (another warp's) must be consumed first: only
       // then is its full barrier one phase behind and the parity wait unambiguous
      const volatile int* sq = &ax->seq[slot];
      if (*sq < i / a.stages) {
        const long long t0 = globaltimer();
        for (int it = 1; *sq < i / a.stages; ++it) {
          __nanosleep(64);
          if ((it & 255) == 0 && globaltimer() - t0 > kWaitNs) __trap();
        }
      }
      mbar_wait_b(smem_u32(&ax->full[slot]), (i / a.stages) & 1);
    }
    const uint32_t st = ring_s + slot * kStage + (uint32_t)(mrow * kw * 2);
    const uint32_t xk = xrow + (uint32_t)(u * kKW * 2);
    for (int kb = 0; kb < kw / 16; kb += 4) {  // kw is a multiple of 64
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(st + (uint32_t)(((2 * (kb + t) + mchunk) ^ msw) * 16), a0, a1, a2, a3);
        const uint32_t b0 = bx ? lds32(xk + (kb + t) * 32) : 0u;
        const uint32_t b1 = bx ? lds32(xk + (kb + t) * 32 + 16) : 0u;
        mma_bf16(acc[t], a0, a1, a2, a3, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0 && !(a.debug & 1)) {
      *(volatile int*)&ax->seq[slot] = i / a.stages + 1;
      mbar_arrive(smem_u32(&ax->empty[slot]));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) c[e] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
}

// Fused epilogue of one block: this lane's (row, activation row) sums c[0..3].
AMUSD_DEV void block_epilogue(const GvArgs& a, Aux* ax, int kind, int l, int b, int r0, const float (&c)[4],
                              const float (&hpre)[4], const Cons& cs) {
  const int g = cs.lane >> 2, q = cs.lane & 3;
  unsigned long long best[2] = {0ull, 0ull};
  float sq[2] = {0.f, 0.f};  // residual phases: this lane's sum of h^2 per activation row (rows g, g + 8)
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int row = g + 8 * (e >> 1), r = r0 + 2 * q + (e & 1);
    if (r >= cs.R) continue;
    const float acc = c[e];
    switch (kind) {
      case kQkv: {
        const int ncols = (a.H + 2 * a.KV) * a.hd;
        a.qkv[(size_t)r * ncols + b * kMB + row] = acc * ax->scale[r];
        break;
      }
      case kO:
      case kDown: {
        const int n = b * kMB + row;
        const float hn = hpre[e] + acc;
        sq[e & 1] = fmaf(hn, hn, sq[e & 1]);
        a.h[(size_t)r * a.d + n] = hn;
        const bf16* gam = a.norms + (size_t)(kind == kO ? 2 * l + 1 : 2 * l + 2) * a.d;
        bf16* xn = kind == kO ? a.xb : a.xa;
        xn[(size_t)r * a.d + n] = __float2bfloat16(hn * __bfloat162float(gam[n]));
        break;
      }
      case kGu: {
        if (e < 2) {  // gate rows 0-7 with their up rows 8-15 (c[e + 2])
          const float gg = acc * ax->scale[r], uu = c[e + 2] * ax->scale[r];
          a.act_b[(size_t)r * a.ffn + b * 8 + row] = __float2bfloat16((gg / (1.f + expf(-gg))) * uu);
        }
        break;
      }
      default: {
        const int n = b * kMB + row;
        const float v = acc * ax->scale[r];
        if (a.logits) a.logits[(size_t)r * a.vocab + n] = v;
        const unsigned long long k = (a.exclude_eos && n == a.eos) ? 0ull : argmax_key(v, n);
        best[e & 1] = k > best[e & 1] ? k : best[e & 1];
        break;
      }
    }
  }
  if (kind == kO || kind == kDown) {  // block's sum of squares per activation row, fixed shuffle tree
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v = sq[h];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      const int r = r0 + 2 * q + h;
      if (g == 0 && r < cs.R) ax->ssb[b % kSsBlk][r] = v;
    }
  }
  if (kind == kLm) {  // max over the lanes holding the same activation row, one smem atomic
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      unsigned long long k = best[h];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, k, o);
        k = w > k ? w : k;
      }
      const int r = r0 + 2 * q + h;
      if (g == 0 && r < cs.R && k) atomicMax(&ax->key[r], k);
    }
  }
}

// One GEMV phase: passes of up to 8 activation rows (one pass for the draft's 1-2 rows; more
// rows than shared memory holds: several passes, each re-streaming the phase's units).
__device__ __noinline__ void gemv_phase(const GvArgs& a, Aux* ax, uint8_t* ring, uint8_t* xs, int kind, int l,
                                        const bf16* src, const bf16* gamma, bool scales, Cons& cs) {
  const WPhase p = wphase_of(a, kind, l);
  const int nb = p.b1 - p.b0;
  const bool resid = kind == kO || kind == kDown;
  long long* pm = (cs.dbg && cs.ct == 0) ? cs.dbg + (size_t)(gridDim.x - blockIdx.x) * kDbgEvents +
                                               ((size_t)blockIdx.x * (kCW + 1) + kCW) * 24 + kind * 4 : nullptr;
  long long tp0 = clock64();
  const uint32_t ring_s = smem_u32(ring), xs_s = smem_u32(xs);
  const int cap = pass_rows(a, p.K), npass = (cs.R + cap - 1) / cap;
  // few blocks (QKV, O, down): S warps split each block's units (K), partials reduced in
  // shared memory in fixed order; many blocks (gate/up, LM head): one warp per block
  int S = 1;
  if (nb > 0 && nb < kCW) {
    int p2 = 1;
    while (p2 < nb) p2 <<= 1;
    S = min(p.nk, kCW / p2);
  }
  const int groups = kCW / S, js = cs.warp / S, qs = cs.warp % S;
  for (int ps = 0; ps < npass; ++ps) {
    const int r0 = ps * cap, nx = min(cap, cs.R - r0);
    fill_xs(a, ax, xs, r0, nx, src, gamma, p.K, scales && ps == 0, cs);
    if (pm) { const long long t = clock64(); pm[0] += t - tp0; tp0 = t; }
    for (int j = js; j < nb; j += groups) {
      const int b = p.b0 + j;
      const long long c0 = clock64();
      float hpre[4] = {0.f, 0.f, 0.f, 0.f};
      if (resid && qs == 0) {
        const int g = cs.lane >> 2, q = cs.lane & 3;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = r0 + 2 * q + (e & 1);
          if (r < cs.R) hpre[e] = __ldcg(a.h + (size_t)r * a.d + b * kMB + g + 8 * (e >> 1));
        }
      }
      float c[4];
      block_mma(a, ax, ring_s, xs_s, p.K, p.nk, cs.stage + j * p.nk, qs, S, nx, c, cs);
      const long long c1 = clock64();
      if (S == 1) {
        block_epilogue(a, ax, kind, l, b, r0, c, hpre, cs);
      } else {
        float* pp = &ax->part[cs.warp][cs.lane][0];
        pp[0] = c[0]; pp[1] = c[1]; pp[2] = c[2]; pp[3] = c[3];
        named_bar(2, kCT);  // all consumers: exactly one round when S > 1
        if (qs == 0) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = ax->part[js * S][cs.lane][e];
            for (int t = 1; t < S; ++t) v += ax->part[js * S + t][cs.lane][e];
            c[e] = v;
          }
          block_epilogue(a, ax, kind, l, b, r0, c, hpre, cs);
        }
      }
      if (cs.dbg && cs.lane == 0) {  // per-warp cycle sums: blocks, mma (incl. waits), epilogue, units
        long long* w = cs.dbg + (size_t)(gridDim.x - blockIdx.x) * kDbgEvents +
                       ((size_t)blockIdx.x * (kCW + 1) + cs.warp) * 24 + kind * 4;
        w[0] += 1; w[1] += c1 - c0; w[2] += clock64() - c1; w[3] += (p.nk - qs + S - 1) / S;
      }
    }
    if (S > 1 && js >= nb) named_bar(2, kCT);  // idle warps join the partial-sum barrier
    cs.stage += nb * p.nk;
    cs.blk += nb;
    named_bar(1, kCT);  // every epilogue write of the pass done, xs free
    if (pm) { const long long t = clock64(); pm[1] += t - tp0; pm[3] += 1; tp0 = t; }
  }
}

// Sum of squares of the residual rows this CTA owns, for the next RMSNorm: the blocks' sums the
// epilogues left in shared memory, added in block order (no re-read of h).
AMUSD_DEV void publish_ss(const GvArgs& a, Aux* ax, const Cons& cs) {
  int n0, n1;
  own_rows(a.d, n0, n1);
  const int b0 = n0 / kMB, nb = (n1 - n0) / kMB;
  for (int r = cs.ct; r < cs.R; r += kCT) {
    float s = 0.f;
    if (nb <= kSsBlk) {
      for (int j = 0; j < nb; ++j) s += ax->ssb[(b0 + j) % kSsBlk][r];
    } else {
      for (int n = n0; n < n1; ++n) {
        const float v = __ldcg(a.h + (size_t)r * a.d + n);
        s = fmaf(v, v, s);
      }
    }
    a.ss[(size_t)blockIdx.x * KMAX + r] = s;
  }
}

// ------------------------------------------------------------------ attention
// Item (kv head g, split s): positions [s*128, min(P, s*128+128)) of every live row.  The item
// owning a position appends this step's K (RoPE) / V there, rounded to bf16 as later steps
// read them; scores, softmax statistics and P.V per (row, query head of the group); one
// split is final, several are merged by the last-arriving split in split order.
AMUSD_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
AMUSD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
AMUSD_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


// Cached K/V rows [lo, hi) of one kv head into shared memory (cp.async, one round trip).
template <int HD>
AMUSD_DEV void attn_stage(uint32_t ks, uint32_t vs, const bf16* kg, const bf16* vg, int lo, int hi, int ct) {
  constexpr int NC = HD / 8;
  const int n = (hi - lo) * NC;
  for (int i = ct; i < 2 * n; i += kCT) {
    const int which = i >= n, r = which ? i - n : i, t = r / NC, c = r % NC;
    cp_async16((which ? vs : ks) + (uint32_t)(t * attn_pitch(HD) + c * 16), (which ? vg : kg) + (size_t)(lo + t) * HD + c * 8);
  }
  cp_async_commit();
}

// Item (kv head g, split s): positions [s*128, min(P, s*128+128)) of every live row.  The
// cached rows of the CTA's first item are staged BEFORE the grid barrier (they do not depend
// on this step), so after the QKV phase completes one round trip (queries + this step's K/V)
// remains.  The item owning a position appends this step's K (RoPE) / V, rounded to bf16 as
// later steps read them; scores, softmax statistics and P.V per (row, query head of the
// group); one split is final, several are merged by the last-arriving split in split order.
// Returns the barrier's go (false: the forward was cut).
template <int HD>
__device__ __noinline__ bool attn_phase(const GvArgs& a, Aux* ax, uint8_t* un, int layer, Cons& cs) {
  const int G = a.H / a.KV, half = HD / 2, ncols = (a.H + 2 * a.KV) * HD, ct = cs.ct;
  const int P = cs.pos0 + cs.R, nsplit = (P + kChunk - 1) / kChunk, items = a.KV * nsplit;
  constexpr int PITCH = HD + 8;  // bf16 elements per staged row
  bf16* ksp = (bf16*)un;
  bf16* vsp = ksp + kChunk * PITCH;
  const uint32_t ks = smem_u32(ksp), vs = smem_u32(vsp);
  float* qs = (float*)(un + 2 * kChunk * attn_pitch(HD));
  float* sc = qs + 4 * G * HD;
  bf16* kl = (bf16*)(a.kcache + (size_t)layer * a.kv_layer_bytes);
  bf16* vl = (bf16*)(a.vcache + (size_t)layer * a.kv_layer_bytes);
  if ((int)blockIdx.x < items) {
    const int g = blockIdx.x / nsplit, s = blockIdx.x % nsplit, lo = s * kChunk;
    const int hc = min(min(P, lo + kChunk), cs.pos0);
    if (hc > lo) attn_stage<HD>(ks, vs, kl + (size_t)g * a.S * HD, vl + (size_t)g * a.S * HD, lo, hc, ct);
  }
  if (!grid_wait(a, ax, cs)) {
    cp_async_wait_all();
    return false;
  }
  long long* tl = (cs.dbg && ct == 0) ? cs.dbg + (size_t)(gridDim.x - blockIdx.x) * kDbgEvents +
                                            ((size_t)blockIdx.x * (kCW + 1)) * 24 + 20 : nullptr;
  auto mark = [&](int k) { if (tl && k < 4) tl[k] += clock64(); };
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int g = it / nsplit, s = it % nsplit;
    const int lo = s * kChunk, hi = min(P, lo + kChunk);
    bf16* kg = kl + (size_t)g * a.S * HD;
    bf16* vg = vl + (size_t)g * a.S * HD;
    if (tl) { const long long t = clock64(); tl[0] -= t; tl[1] -= t; tl[2] -= t; tl[3] -= t; }
    if (it != (int)blockIdx.x) {
      const int hc = min(hi, cs.pos0);
      if (hc > lo) attn_stage<HD>(ks, vs, kg, vg, lo, hc, ct);
    }
    // 1) this step's K/V rows in [lo, hi): to the cache and to the staged rows
    const int j0 = max(lo, cs.pos0) - cs.pos0, j1 = hi - cs.pos0;
    for (int i = ct; i < (j1 - j0) * half; i += kCT) {
      const int j = j0 + i / half, e = i % half, p = cs.pos0 + j;
      const float* kr = a.qkv + (size_t)j * ncols + (a.H + g) * HD;
      const float* vr = a.qkv + (size_t)j * ncols + (a.H + a.KV + g) * HD;
      const float x0 = __ldcg(kr + e), x1 = __ldcg(kr + e + half);
      const float v0 = __ldcg(vr + e), v1 = __ldcg(vr + e + half);
      const float c = a.cos[(size_t)p * half + e], sn = a.sin[(size_t)p * half + e];
      const bf16 k0 = __float2bfloat16(x0 * c - x1 * sn), k1 = __float2bfloat16(x1 * c + x0 * sn);
      const bf16 w0 = __float2bfloat16(v0), w1 = __float2bfloat16(v1);
      kg[(size_t)p * HD + e] = k0;
      kg[(size_t)p * HD + e + half] = k1;
      vg[(size_t)p * HD + e] = w0;
      vg[(size_t)p * HD + e + half] = w1;
      bf16* kd = ksp + (p - lo) * PITCH;
      bf16* vd = vsp + (p - lo) * PITCH;
      kd[e] = k0; kd[e + half] = k1; vd[e] = w0; vd[e + half] = w1;
    }
    for (int rg0 = 0; rg0 < cs.R; rg0 += 4) {
      const int nrg = min(4, cs.R - rg0);
      // 2) RoPE'd queries of the group's heads: qs[(rr*G + jh)*HD + e]
      for (int i = ct; i < nrg * G * half; i += kCT) {
        const int rr = i / (G * half), rem = i % (G * half), jh = rem / half, e = rem % half;
        const int p = cs.pos0 + rg0 + rr;
        const float* q = a.qkv + (size_t)(rg0 + rr) * ncols + (g * G + jh) * HD;
        const float x0 = __ldcg(q + e), x1 = __ldcg(q + e + half);
        const float c = a.cos[(size_t)p * half + e], sn = a.sin[(size_t)p * half + e];
        qs[(rr * G + jh) * HD + e] = x0 * c - x1 * sn;
        qs[(rr * G + jh) * HD + e + half] = x1 * c + x0 * sn;
      }
      cp_async_wait_all();
      named_bar(1, kCT);
      mark(0);
      // 3) scores: thread = (position, query head) pair (a quad of lanes shares the K row)
      for (int pr = ct; pr < (hi - lo) * G; pr += kCT) {
        const int pi = pr / G, jh = pr % G, t = lo + pi;
        const uint4* kr = (const uint4*)(ksp + pi * PITCH);
        float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) {
          const F8 f8 = unpack8(kr[c]);
          const float* f = f8.v;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            if (rr < nrg) {
              const float4* q4 = (const float4*)(qs + (rr * G + jh) * HD + c * 8);
              const float4 qa = q4[0], qb = q4[1];
              float d = dot[rr];
              d = fmaf(qa.x, f[0], d); d = fmaf(qa.y, f[1], d); d = fmaf(qa.z, f[2], d); d = fmaf(qa.w, f[3], d);
              d = fmaf(qb.x, f[4], d); d = fmaf(qb.y, f[5], d); d = fmaf(qb.z, f[6], d); d = fmaf(qb.w, f[7], d);
              dot[rr] = d;
            }
          }
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
          if (rr < nrg) sc[(rr * G + jh) * kChunk + pi] = t <= cs.pos0 + rg0 + rr ? dot[rr] * a.scale : -INFINITY;
      }
      for (int i = ct; i < G * kChunk; i += kCT) {  // positions past the chunk's end
        const int jh = i / kChunk, pi = i % kChunk;
        if (pi >= hi - lo)
          for (int rr = 0; rr < nrg; ++rr) sc[(rr * G + jh) * kChunk + pi] = -INFINITY;
      }
      named_bar(1, kCT);
      mark(1);
      // 4) softmax statistics per (row, head): one warp per pair
      for (int pr = cs.warp; pr < nrg * G; pr += kCW) {
        float* row = sc + pr * kChunk;
        float x[kChunk / 32];
        float m = -INFINITY;
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) {
          x[u] = row[cs.lane + 32 * u];
          m = fmaxf(m, x[u]);
        }
        m = warp_max(m);
        float l = 0.f;
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) {
          const float e = m == -INFINITY ? 0.f : expf(x[u] - m);
          row[cs.lane + 32 * u] = e;
          l += e;
        }
        l = warp_sum(l);
        if (cs.lane == 0) { ax->ml[pr / G][pr % G][0] = m; ax->ml[pr / G][pr % G][1] = l; }
      }
      named_bar(1, kCT);
      mark(2);
      // 5) P.V: thread = (head, dim), positions in order
      for (int i = ct; i < G * HD; i += kCT) {
        const int jh = i / HD, e = i % HD;
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        const bf16* vp = vsp + e;
#pragma unroll 8
        for (int t = 0; t < hi - lo; ++t) {
          const float vv = __bfloat162float(vp[t * PITCH]);
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
            if (rr < nrg) o[rr] = fmaf(sc[(rr * G + jh) * kChunk + t], vv, o[rr]);
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          if (rr >= nrg) continue;
          const int r = rg0 + rr;
          const float m = ax->ml[rr][jh][0], l = ax->ml[rr][jh][1];
          if (nsplit == 1) {
            a.attn_b[(size_t)r * a.H * HD + (g * G + jh) * HD + e] = __float2bfloat16(o[rr] / l);
          } else {
            float* w = a.attn_ws + ((((size_t)g * a.max_splits + s) * KMAX + r) * G + jh) * (HD + 2);
            w[2 + e] = o[rr];
            if (e == 0) { w[0] = m; w[1] = l; }
          }
        }
      }
      named_bar(1, kCT);  // qs / sc / staged rows reuse
      mark(3);
    }
    if (nsplit > 1) {
      if (ct == 0) {
        __threadfence();
        const int old = atomicAdd(a.sync + kSyncAttn + g * kPad, 1);
        ax->last = old == nsplit - 1;
        if (ax->last) {
          __threadfence();
          a.sync[kSyncAttn + g * kPad] = 0;
        }
      }
      named_bar(1, kCT);
      if (ax->last) {  // merge every live row's splits in split order
        for (int i = ct; i < cs.R * G * HD; i += kCT) {
          const int r = i / (G * HD), rem = i % (G * HD), jh = rem / HD, e = rem % HD;
          const int ns = (cs.pos0 + r) / kChunk + 1;  // splits holding positions <= pos0 + r
          const float* w0 = a.attn_ws + ((((size_t)g * a.max_splits) * KMAX + r) * G + jh) * (HD + 2);
          const size_t sstride = (size_t)KMAX * G * (HD + 2);
          float M = -INFINITY;
          for (int q = 0; q < ns; ++q) M = fmaxf(M, __ldcg(w0 + q * sstride));
          float L = 0.f, O = 0.f;
          for (int q = 0; q < ns; ++q) {
            const float wq = expf(__ldcg(w0 + q * sstride) - M);
            L = fmaf(wq, __ldcg(w0 + q * sstride + 1), L);
            O = fmaf(wq, __ldcg(w0 + q * sstride + 2 + e), O);
          }
          a.attn_b[(size_t)r * a.H * HD + (g * G + jh) * HD + e] = __float2bfloat16(O / L);
        }
      }
      named_bar(1, kCT);
    }
  }
  return true;
}

// ------------------------------------------------------------------ kernel
template <int HD>
__global__ void __launch_bounds__(kThreads, 1) k_decode(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  StepCtl* ctl = a.ctl;
  if (!ctl->active) return;
  uint8_t* ring = smem;
  const int G = a.H / a.KV;
  uint8_t* un = smem + (size_t)a.stages * kStage;        // GEMV input rows | attention scratch
  uint8_t* xs = un;
  const int ub = union_bytes(a.d, a.H, a.KV, a.hd, a.ffn);
  Aux* ax = (Aux*)(un + ub);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(smem_u32(&ax->full[i]), 1);
      mbar_init(smem_u32(&ax->empty[i]), 1);
      ax->seq[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ax->cut = 0;
    ax->consumed = 0;
    ax->issued = 0;
  }
  if (tid < KMAX) ax->key[tid] = 0ull;
  __syncthreads();
  if (warp == kCW) {
    if ((tid & 31) == 0) producer(a, ax, ring, min(max(ctl->rows, 1), KMAX), ub);
    __syncwarp();
  } else {
    Cons cs;
    cs.ct = tid; cs.warp = warp; cs.lane = tid & 31;
    cs.R = min(max(ctl->rows, 1), KMAX); cs.pos0 = ctl->pos0;
    cs.stage = 0; cs.bar = 0; cs.blk = 0; cs.ev = 1;
    cs.dbg = a.dbg ? a.dbg + (size_t)blockIdx.x * kDbgEvents : nullptr;
    if (cs.dbg && tid == 0) cs.dbg[0] = globaltimer();
    bool ok = true;
    embed_prologue(a, ax, cs);
    for (int l = 0; l < a.L && ok; ++l) {
      const bf16* gamma_attn = a.norms + (size_t)(2 * l) * a.d;
      if (l > 0 && !(ok = grid_wait(a, ax, cs))) break;
      gemv_phase(a, ax, ring, xs, kQkv, l, l == 0 ? nullptr : a.xa, gamma_attn, l > 0, cs);
      grid_arrive(a, cs);
      if (!(ok = attn_phase<HD>(a, ax, un, l, cs))) break;
      grid_arrive(a, cs);
      if (!(ok = grid_wait(a, ax, cs))) break;
      gemv_phase(a, ax, ring, xs, kO, l, a.attn_b, nullptr, false, cs);
      publish_ss(a, ax, cs);
      grid_arrive(a, cs);
      if (!(ok = grid_wait(a, ax, cs))) break;
      gemv_phase(a, ax, ring, xs, kGu, l, a.xb, nullptr, true, cs);
      grid_arrive(a, cs);
      if (!(ok = grid_wait(a, ax, cs))) break;
      gemv_phase(a, ax, ring, xs, kDown, l, a.act_b, nullptr, false, cs);
      publish_ss(a, ax, cs);
      grid_arrive(a, cs);
    }
    if (ok && (ok = grid_wait(a, ax, cs))) {
      gemv_phase(a, ax, ring, xs, kLm, 0, a.xa, nullptr, true, cs);
      if (cs.ct == 0) {
        for (int r = 0; r < cs.R; ++r) atomicMax(a.best + r, ax->key[r]);
        __threadfence();
        if (atomicAdd(a.sync + kSyncLm, 1) == (int)gridDim.x - 1) {
          __threadfence();
          for (int r = 0; r < cs.R; ++r) ctl->preds[r] = argmax_key_index(atomicExch(a.best + r, 0ull));
          a.sync[kSyncLm] = 0;
        }
      }
    }
    if (cs.ct == 0) ax->consumed = cs.stage;
  }
  __syncthreads();
  // drain bulk copies a cut left in flight (none otherwise) before the CTA's smem is released
  if (warp == kCW && (tid & 31) == 0) {
    for (int i = ax->consumed; i < ax->issued; ++i)
      mbar_wait_b(smem_u32(&ax->full[i % a.stages]), (i / a.stages) & 1);
  }
  __syncthreads();
  if (tid == 0) {
    if (ax->cut) atomicExch(a.sync + kSyncCut, 1);
    __threadfence();
    if (atomicAdd(a.sync + kSyncExit, 1) == (int)gridDim.x - 1) {
      __threadfence();
      a.sync[kSyncBar] = 0;
      if (atomicExch(a.sync + kSyncCut, 0)) {  // re-arm what a cut forward left behind
        a.sync[kSyncLm] = 0;
        for (int g = 0; g < a.KV; ++g) a.sync[kSyncAttn + g * kPad] = 0;
        for (int r = 0; r < KMAX; ++r) a.best[r] = 0ull;
        if (a.cuts) *a.cuts += 1;
      }
      a.sync[kSyncExit] = 0;
    }
  }
}

// ------------------------------------------------------------------ host
bool supported(int d, int H, int KV, int hd, int ffn, int vocab) {
  auto ok_k = [](int K) { return K % 64 == 0 && K <= 16384; };
  if (!(hd == 64 || hd == 128) || KV <= 0 || H % KV || H / KV > kMaxG) return false;
  if (!ok_k(d) || !ok_k(H * hd) || !ok_k(ffn)) return false;
  return ((H + 2 * KV) * hd) % kMB == 0 && d % kMB == 0 && ffn % 8 == 0 && vocab % kMB == 0 &&
         max_stages(d, H, KV, hd, ffn) >= 4;
}
Layout layout(int d, int H, int KV, int hd, int ffn, int vocab, int L) {
  Layout t;
  t.off_o = 2ll * (H + 2 * KV) * hd * d;
  t.off_gu = t.off_o + 2ll * d * H * hd;
  t.off_down = t.off_gu + 4ll * ffn * d;
  t.layer_bytes = t.off_down + 2ll * d * ffn;
  t.lm_off = t.layer_bytes * L;
  t.total = t.lm_off + 2ll * vocab * d;
  return t;
}

// One 16-byte destination chunk per thread: block b, unit q, row n, physical chunk pc holds
// logical chunk pc ^ (n & 7) of the row (the swizzle ldmatrix reads conflict-free).
__global__ void k_tile_gv(const uint4* __restrict__ src, const uint4* __restrict__ src2, int N, int K,
                          uint4* __restrict__ dst) {
  const long long nchunks = (long long)N * K / 8;
  for (long long ci = blockIdx.x * (long long)blockDim.x + threadIdx.x; ci < nchunks;
       ci += (long long)gridDim.x * blockDim.x) {
    const long long per_block = 2ll * K;  // 16 rows x K / 8 chunks
    const int b = (int)(ci / per_block);
    const int rem = (int)(ci - (long long)b * per_block);
    const int q = rem / (kMB * kKW / 8);
    const int kw = min(kKW, K - q * kKW);
    const int pc_all = rem - q * (kMB * kKW / 8);
    const int n = pc_all / (kw / 8), pc = pc_all % (kw / 8);
    const int c = pc ^ (n & 7);
    const int col = q * kKW + c * 8;
    const uint4* s;
    long long row;
    if (src2) {  // gate/up block: 8 gate rows then the 8 up rows of features 8b .. 8b+7
      s = n < 8 ? src : src2;
      row = (long long)b * 8 + (n & 7);
    } else {
      s = src;
      row = (long long)b * kMB + n;
    }
    dst[ci] = s[(row * K + col) / 8];
  }
}
cudaError_t tile_weights(const void* src, const void* src2, int N, int K, void* dst, cudaStream_t st) {
  k_tile_gv<<<148 * 8, 256, 0, st>>>((const uint4*)src, (const uint4*)src2, N, K, (uint4*)dst);
  return cudaGetLastError();
}
size_t sync_ints(int KV) { return (size_t)(4 + KV) * kPad; }
size_t ss_floats() { return (size_t)kMaxGrid * KMAX; }
int attn_splits(int S) { return (S + kChunk - 1) / kChunk; }
size_t attn_ws_floats(int KV, int G, int hd, int S) { return (size_t)KV * attn_splits(S) * KMAX * G * (hd + 2); }
static int tail_bytes(const GvArgs& a) { return union_bytes(a.d, a.H, a.KV, a.hd, a.ffn) + (int)sizeof(Aux); }
int max_stages(int d, int H, int KV, int hd, int ffn) {
  return std::min(kMaxStages, (kSmemBudget - union_bytes(d, H, KV, hd, ffn) - (int)sizeof(Aux)) / kStage);
}

cudaError_t launch(const GvArgs& a, int grid, cudaStream_t st) {
  if (grid <= 0 || grid > kMaxGrid || a.stages < 2 || a.stages > max_stages(a.d, a.H, a.KV, a.hd, a.ffn))
    return cudaErrorInvalidValue;
  const int smem = a.stages * kStage + tail_bytes(a);
  static SmemOptIn opt64, opt128;  // per device
  if (a.hd == 64) {
    if (cudaError_t e = opt64.ensure(k_decode<64>, smem)) return e;
    k_decode<64><<<grid, kThreads, smem, st>>>(a);
  } else {
    if (cudaError_t e = opt128.ensure(k_decode<128>, smem)) return e;
    k_decode<128><<<grid, kThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace gv
}  // namespace amusd
