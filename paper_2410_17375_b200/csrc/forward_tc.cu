// forward_tc.cu -- persistent tcgen05 decoder forward (SURVEY.md K2 + K4).
//
// One launch runs a whole forward of the Llama-style model over <= 16 token
// rows (the draft's pending token, the verify window).  The forward is a list
// of phases -- embed, then per layer QKV GEMM / attention / O GEMM / gate-up
// GEMM / down GEMM, then the LM-head GEMM with the greedy argmax -- cut into
// work items that CTAs grab from one global counter in phase order.
//
// Why a work queue rather than one kernel per GEMM: a decode forward is a
// stream of 2.5 GB (1B) / 15 GB (8B) of weights with a dependency every few
// tens of MB.  Weights never depend on activations, so a CTA that grabbed an
// item of phase p+1 streams that item's weights into its shared-memory ring
// right away and waits for phase p only before loading the activation tile
// (X) and issuing the MMAs.  HBM stays busy across the layer's dependency
// chain instead of draining at every kernel boundary.  Items are grabbed in
// global order, so every item a CTA waits on was grabbed by a CTA that is
// already running: forward progress never needs co-residency, and a draft
// forward and a verify forward can share the GPU (co-located AMUSD).
//
// Warp roles (320 threads):
//   w0      scheduler + weight producer (1-D bulk copies, 16 KB per unit)
//   w1      activation loader: waits for the dependency, then X tiles by TMA
//   w2..w5  tcgen05.mma issuers: warp w issues K-slice w-2 of every unit into
//           its own TMEM accumulator chain (issue-rate bound)
//   w6..w9  epilogue (TMEM -> registers -> fused epilogue) and the SIMT items
//           (embedding, attention)
// The roles follow the same item sequence through a 4-deep shared-memory
// queue; weight/X stages and the TMEM double buffer are mbarrier rings.
//
// Determinism / batch invariance: split-K partials of a tile are summed by
// the last-arriving item in fixed chunk order, attention splits merge in
// split order, the argmax is an order-independent max over (value, ~index)
// keys.  Nothing depends on the number of valid rows, so a row's logits are
// the same whatever the verify window size (AMUSD tokens == AR tokens).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "forward_tc.h"
#include "internal.h"
#include "tc_ptx.cuh"

namespace amusd {
namespace fw {

using namespace amusd::tc;

constexpr int kQ = 4;                  // item queue depth
// Units (16 KB weight tile + 2 KB token tile) per ring stage: one full/empty handshake and one
// commit per stage.  The handshake (~200 cycles, tools/probe/probe_ring.cu) plus the MMA issue
// per 16 KB capped a CTA at ~45 GB/s with 1 unit per stage; a bare bulk-copy ring streams
// ~200 GB/s per SM (tools/probe/probe_bw.cu).
constexpr int kUPS = 2;
constexpr int kStageW = kUPS * kWBytes;
constexpr int kStageX = kUPS * kXBytes;
constexpr int kThreads = 320;
constexpr int kWarpX = 1, kWarpMma0 = 2, kWarpEpi0 = 6;
constexpr int kTbuf = 4;                 // TMEM accumulator buffers (MMA may run 3 items ahead of the epilogue)
constexpr int kTmemCols = kTbuf * NACC * BN;  // 256
constexpr int kMaxMerge = 128;         // max position splits of one row (8192 positions)
constexpr int kCutIndex = 1 << 28;     // grab counter value after a draft cut (> any item count)
constexpr int kAttnChunk = 64;         // positions per attention split (K/V chunk staged in smem; 2 threads each)
constexpr long long kWaitNs = 4ll * 1000 * 1000 * 1000;  // dependency waits trap after 4 s
// Every schedule counter owns a 128-byte line (grab counter, exit counter, one
// per phase, one per split-K tile): 148 CTAs poll and bump them concurrently.
constexpr int kPad = kCounterInts;
#ifndef AMUSD_POLL_NS
#define AMUSD_POLL_NS 100
#endif
constexpr unsigned a_poll_ns = AMUSD_POLL_NS;  // dependency-poll back-off (ns)
constexpr unsigned kSuspendNs = 20000;  // mbarrier try_wait suspend-time hint

// ------------------------------------------------------------ memory model
AMUSD_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
AMUSD_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// One round trip: release (this CTA's writes ordered before, via the preceding CTA barrier)
// + acquire (the other contributors' writes visible after).
AMUSD_DEV int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
AMUSD_DEV void red_add_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
AMUSD_DEV void red_add_relaxed(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// System scope (tensor-parallel peers write these words over NVLink).
AMUSD_DEV int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
AMUSD_DEV void red_add_sys(int* p, int v) {
  asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
AMUSD_DEV void red_add_u64_sys(unsigned long long* p, long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
AMUSD_DEV void wait_count_sys(const int* p, int target) {
  if (ld_acquire_sys(p) >= target) return;
  const long long t0 = globaltimer();
  for (;;) {
    __nanosleep(a_poll_ns);
    if (ld_acquire_sys(p) >= target) return;
    if (globaltimer() - t0 > kWaitNs) __trap();
  }
}

AMUSD_DEV void wait_count(const int* p, int target) {
  if (ld_acquire_gpu(p) >= target) return;
  const long long t0 = globaltimer();
  for (;;) {
    __nanosleep(a_poll_ns);  // back off: many CTAs poll the same line
    if (ld_acquire_gpu(p) >= target) return;
    if (globaltimer() - t0 > kWaitNs) __trap();
  }
}

// mbarrier wait with a wall-clock bound: a scheduling bug traps the kernel
// (the host sees a launch error) instead of hanging the GPU.
AMUSD_DEV void mbar_wait_t(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  if (ok) return;
  const long long t0 = globaltimer();
  for (int it = 0;; ++it) {
    // suspend-time hint: the waiting warp sleeps (wakes as soon as the phase completes)
    // instead of re-issuing, leaving the SMSP's issue slots to the epilogue warp
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(kSuspendNs)
        : "memory");
    if (ok) return;
    if ((it & 15) == 15 && globaltimer() - t0 > kWaitNs) __trap();
  }
}

// Optional per-item timeline (tools/fw_timeline.py): slot 0 item|cta<<20|phase<<32,
// 1 grabbed, 2 weights issued, 3 X dependency met, 4 MMA done, 5 epilogue done.
AMUSD_DEV void dbg_mark(const FwArgs& a, int item, int slot, long long v) {
  if (a.dbg && item < a.dbg_items) a.dbg[(size_t)item * 8 + slot] = v;
}

// Bulk L2 prefetch of a contiguous weight range (no shared memory involved).
AMUSD_DEV void prefetch_l2(const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(policy)
               : "memory");
}

AMUSD_DEV long long ld_acquire_gpu64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
AMUSD_DEV void st_release_gpu64(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Wait until every flag in [t0, t1) of a producer kind carries at least `stamp`:
// all flags are loaded at once (one round trip when they are already set),
// then only the missing ones are polled.
AMUSD_DEV void wait_tiles(const long long* flags, int t0, int t1, long long stamp) {
  constexpr int kBatch = 16;
  for (int b0 = t0; b0 < t1; b0 += kBatch) {
    long long v[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
      v[i] = b0 + i < t1 ? ld_acquire_gpu64(flags + (size_t)(b0 + i) * (kCounterInts / 2)) : stamp;
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      if (v[i] >= stamp) continue;
      const long long* f = flags + (size_t)(b0 + i) * (kCounterInts / 2);
      const long long t_start = globaltimer();
      for (;;) {
        __nanosleep(a_poll_ns);
        if (ld_acquire_gpu64(f) >= stamp) break;
        if (globaltimer() - t_start > kWaitNs) __trap();
      }
    }
  }
}

// Ring cursor: stage index + phase parity, advanced incrementally (no division).
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  AMUSD_DEV void next(int S) {
    if (++s == S) { s = 0; ph ^= 1u; }
  }
};

// ------------------------------------------------------------ item layout
// All schedule arithmetic comes from the kernel parameters (constant bank):
// no role ever reads the schedule from global memory (the acquire polls
// invalidate L1, which would turn every such read into an L2 round trip).
struct Lay {
  int A;       // attention items per layer (dynamic: rows x KV x splits)
  int PL;      // items per layer
  int total;   // items this launch
  int rows, pos0;
  int pre[5];  // first item of each layer phase relative to the layer's first item
};

AMUSD_DEV int nsplit_of(int p) { return p / kAttnChunk + 1; }

AMUSD_DEV int kind_of(int p, int L) { return p == 0 ? kKEmbed : (p == 1 + 5 * L ? kKLm : (p - 1) % 5); }
AMUSD_DEV int layer_of(int p) { return p == 0 ? 0 : (p - 1) / 5; }
AMUSD_DEV int gemm_of(int kind) {
  return kind == kKQkv ? kGQkv : kind == kKO ? kGO : kind == kKGu ? kGGu : kind == kKDown ? kGDown : kGLm;
}
AMUSD_DEV bool is_gemm(int kind) { return kind != kKAttn && kind != kKEmbed; }
// Per-tile (fine) dependencies for consumer `kind` (AMUSD_FW_FINE bit 1 << kind).
AMUSD_DEV bool fine_for(const FwArgs& a, int kind) { return (a.fine >> kind) & 1; }

// item index -> (phase, index within the phase)
AMUSD_DEV int2 locate(const FwArgs& a, const Lay& L, int i) {
  if (i < KMAX) return make_int2(0, i);
  int r = i - KMAX;
  const int l = r / L.PL;
  if (l >= a.L) return make_int2(1 + 5 * a.L, r - a.L * L.PL);
  r -= l * L.PL;
  // select chain, not L.pre[k]: a dynamically indexed array would live in local memory,
  // and every acquire poll invalidates L1 (CCTL.IVALL) -> an L2 round trip per lookup
  const int k = r >= L.pre[4] ? 4 : r >= L.pre[3] ? 3 : r >= L.pre[2] ? 2 : r >= L.pre[1] ? 1 : 0;
  const int base = k == 4 ? L.pre[4] : k == 3 ? L.pre[3] : k == 2 ? L.pre[2] : k == 1 ? L.pre[1] : 0;
  return make_int2(1 + 5 * l + k, r - base);
}
AMUSD_DEV int phase_first(const FwArgs& a, const Lay& L, int p) {
  if (p == 0) return 0;
  const int l = layer_of(p), k = p == 1 + 5 * a.L ? 0 : (p - 1) % 5;
  const int off = k == 4 ? L.pre[4] : k == 3 ? L.pre[3] : k == 2 ? L.pre[2] : k == 1 ? L.pre[1] : 0;
  return KMAX + l * L.PL + off;
}
AMUSD_DEV int phase_count(const FwArgs& a, const Lay& L, int p) {
  const int kind = kind_of(p, a.L);
  return kind == kKEmbed ? KMAX : kind == kKAttn ? L.A : a.g[gemm_of(kind)].nitems;
}

// A GEMM kind resolved for one layer.
struct GemmRes {
  const uint8_t* wt;
  const __nv_bfloat16* gnext;
  int epi, map, kb, kc, nchunks, nitems, ntiles;
};
AMUSD_DEV GemmRes resolve(const FwArgs& a, int gk, int layer) {
  const GemmKind& g = a.g[gk];
  GemmRes r;
  r.wt = g.wt + (size_t)layer * g.wt_stride;
  r.gnext = g.gnext ? g.gnext + (size_t)layer * g.gnext_stride : nullptr;
  r.epi = g.epi; r.map = g.map; r.kb = g.kb; r.kc = g.kc; r.nchunks = g.nchunks; r.nitems = g.nitems;
  r.ntiles = g.ntiles;
  return r;
}

// ------------------------------------------------------------ epilogues
// 4-byte asynchronous global -> shared copy (L2 only: the data was written by other CTAs)
AMUSD_DEV void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
AMUSD_DEV void cp_async_wait_all() { asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory"); }

// Per-item epilogue temporaries: alias the attention K/V staging buffers (both belong to the
// epilogue warps, which run one item at a time; the attention mbarrier stays outside).
struct EpiTmp {
  float xchg[64 * BN];                // gate/up exchange
  unsigned long long kx[4 * BN];      // argmax per lane-quarter
  float sq[4 * BN];                   // residual sum-of-squares per lane-quarter
  float hs[BN][BM];                   // residual epilogue: the tile's h rows, prefetched (cp.async)
  __nv_bfloat16 gs[BM];               // ... and the tile's slice of the next RMSNorm weight
};
// Epilogue state that persists across items (the RMSNorm scale of the current phase).
struct EpiSmem {
  float inv[BN];
  int inv_phase;
};

// Final epilogue of one 128-row tile; thread holds tile row nl, v[r] for the
// 16 token rows.  Activations written here are read by other CTAs of the same
// launch: all loads/stores bypass L1 (.cg).
// Residual epilogue inputs of tile t: this thread's h column for every live row -> et->hs
// (asynchronous; consumed by tile_epilogue after cp_async_wait_all, by the same thread).
// The caller waits (cp_async_wait_all) before the CTA barrier that precedes tile_epilogue.
AMUSD_DEV void resid_prefetch(const GemmKind& ph, const __nv_bfloat16* gnext, int t, int nl, int rows, EpiTmp* et) {
  const int n = t * BM + nl;
  for (int r = 0; r < rows; ++r) cp_async4(&et->hs[r][nl], ph.out + (size_t)r * ph.ldo + n);
  if (nl < BM / 8)  // 16 threads x 16 bytes: the tile's 128 norm weights
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&et->gs[nl * 8])),
                 "l"(gnext + t * BM + nl * 8) : "memory");
}

template <bool TP>
AMUSD_DEV void tile_epilogue(const FwArgs& a, const GemmKind& ph, const __nv_bfloat16* gnext, int t, int nl,
                             const float (&v)[BN], int rows, EpiSmem* es, EpiTmp* et, int q, int lane) {
  const float* inv = es->inv;
  if (ph.epi == kEpStoreScaled) {
    const int n = t * BM + nl;
#pragma unroll
    for (int r = 0; r < BN; ++r)
      if (r < rows) __stcg(ph.out + (size_t)r * ph.ldo + n, v[r] * inv[r]);
  } else if (ph.epi == kEpResid) {  // h rows and norm weights prefetched by resid_prefetch
    const int n = t * BM + nl;
    const float gn = __bfloat162float(et->gs[nl]);
    // live rows only (`rows` is uniform across the launch): the shuffle trees of the 16-row
    // tile cost ~1.2 us on the merger's critical path
#pragma unroll
    for (int r = 0; r < BN; ++r) {
      if (r < rows) {
        const float hn = et->hs[r][nl] + v[r];
        __stcg(ph.out + (size_t)r * ph.ldo + n, hn);
        ph.xnext[(size_t)r * ph.ldo + n] = __float2bfloat16(hn * gn);
        const float s2 = warp_sum(hn * hn);
        if (lane == 0) et->sq[q * BN + r] = s2;
      }
    }
    named_bar(1, 128);
    if (q == 0 && lane < BN) {  // fixed order over the 4 lane quarters
      const float tot = et->sq[0 * BN + lane] + et->sq[1 * BN + lane] + et->sq[2 * BN + lane] + et->sq[3 * BN + lane];
      __stcg(ph.ssp_out + (size_t)lane * (a.d / BM) + t, lane < rows ? tot : 0.f);
    }
  } else if (ph.epi == kEpGateUp) {
    // lanes 0..63: gate rows, 64..127: up rows of the same 64 features
    if (nl >= 64) {
#pragma unroll
      for (int r = 0; r < BN; ++r) et->xchg[(nl - 64) * BN + r] = v[r];
    }
    named_bar(1, 128);
    if (nl < 64) {
      const int f = t * 64 + nl;
#pragma unroll
      for (int r = 0; r < BN; ++r) {
        if (r < rows) {
          const float g = v[r] * inv[r], u = et->xchg[nl * BN + r] * inv[r];
          ph.out_b[(size_t)r * ph.ldo + f] = __float2bfloat16((g / (1.f + expf(-g))) * u);
        }
      }
    }
  } else {  // LM head: per-row argmax over the tile, merged by atomicMax (order independent)
    const int n = t * BM + nl, ng = a.vocab_off + n;  // ng: global vocab id (tensor-parallel shard offset)
    const bool valid_n = n < ph.N && !(a.exclude_eos && ng == a.eos);
#pragma unroll
    for (int r = 0; r < BN; ++r) {
      if (r < rows) {  // live rows only (uniform)
        if (a.logits && n < ph.N) a.logits[(size_t)r * ph.N + n] = v[r] * inv[r];
        unsigned long long key = valid_n ? argmax_key(v[r] * inv[r], ng) : 0ull;
        key = warp_max_u64(key);
        if (lane == 0) et->kx[q * BN + r] = key;
      }
    }
    named_bar(1, 128);
    if (q == 0 && lane < BN && lane < rows) {
      unsigned long long b = et->kx[lane];
      for (int w = 1; w < 4; ++w) b = et->kx[w * BN + lane] > b ? et->kx[w * BN + lane] : b;
      if (TP && a.tp > 1) {  // every rank's keys (order-independent max: the all-rank argmax everywhere)
        for (int p = 0; p < a.tp; ++p) atomicMax_system(a.peer_best[p] + lane, b);
      } else {
        atomicMax(a.best + lane, b);
      }
    }
  }
}

// ------------------------------------------------------------ SIMT items
// Embedding of row r: h = E[tok], xa = bf16(h * g0), ssp per 128-wide tile.
// Thread tid owns 16-byte vectors tid, tid+128, ...; a 128-wide tile is 16
// consecutive vectors, reduced over 16 lanes (fixed shuffle tree).
AMUSD_DEV void embed_item(const FwArgs& a, int r, int rows, int tid) {
  const bool live = r < rows;
  const uint4* src = (const uint4*)(a.embed + (size_t)(live ? a.ctl->tok[r] : 0) * a.d);
  const uint4* gam = (const uint4*)a.norms;  // attention RMSNorm of layer 0
  constexpr int kMaxVec = 8;  // d <= 8192
  const int nv = a.d / 8;
  uint4 x[kMaxVec], gv[kMaxVec];
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int q = tid + 128 * k;
    if (q < nv) { x[k] = live ? src[q] : make_uint4(0, 0, 0, 0); gv[k] = gam[q]; }
  }
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int q = tid + 128 * k;
    if (q >= nv) break;
    float f[8], g[8];
    Elem<__nv_bfloat16>::unpack(x[k], f);
    Elem<__nv_bfloat16>::unpack(gv[k], g);
    float4* hp = (float4*)(a.h + (size_t)r * a.d + q * 8);
    __stcg(hp, make_float4(f[0], f[1], f[2], f[3]));
    __stcg(hp + 1, make_float4(f[4], f[5], f[6], f[7]));
    uint4 o;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(f[0] * g[0], f[1] * g[1]), t1 = __floats2bfloat162_rn(f[2] * g[2], f[3] * g[3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(f[4] * g[4], f[5] * g[5]), t3 = __floats2bfloat162_rn(f[6] * g[6], f[7] * g[7]);
    o.x = *(uint32_t*)&t0; o.y = *(uint32_t*)&t1; o.z = *(uint32_t*)&t2; o.w = *(uint32_t*)&t3;
    *(uint4*)(a.xa + (size_t)r * a.d + q * 8) = o;
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
    ss += __shfl_xor_sync(0xffffffffu, ss, 8);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    if ((tid & 15) == 0) __stcg(a.ssp + (size_t)r * (a.d / BM) + q / 16, ss);
  }
}

// Attention scratch layout (epilogue warps only).
template <int HD, int G>
struct AttnSmem {
  __nv_bfloat16 kb[kAttnChunk][HD];   // cached K rows of the chunk (bulk copy); red[4][G][HD] aliases it after P.V
  __nv_bfloat16 vb[kAttnChunk][HD];   // cached V rows of the chunk (bulk copy)
  float qs[G * HD];                   // rotated queries, float4 chunks [G][lo/hi][HD/8] (attn_qidx)
  __nv_bfloat16 kn[KMAX][HD];         // this step's rotated K rows (bf16, exactly as the cache holds them)
  __nv_bfloat16 vn[KMAX][HD];         // ... and V rows
  float sc[kAttnChunk][G];            // scores -> probabilities (position-major: one vector load per position)
  float stat[2][G];
  float wred[4][G];
  int last;
  uint64_t bar;                       // K/V bulk-copy completion
};

// Rotated-query layout: dims [8c, 8c+4) of head j at float4 (2j)*NC + c, [8c+4, 8c+8) at (2j+1)*NC + c.
template <int HD>
AMUSD_DEV int attn_qidx(int j, int e) {
  constexpr int NC = HD / 8;
  return ((2 * j + ((e >> 2) & 1)) * NC + (e >> 3)) * 4 + (e & 3);
}
template <int G, int NC>
AMUSD_DEV void attn_dot8(float (&dot)[G], const float (&f)[8], const float4* qv, int c) {
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float4 qa = qv[2 * j * NC + c], qb = qv[(2 * j + 1) * NC + c];
    dot[j] = fmaf(f[0], qa.x, dot[j]); dot[j] = fmaf(f[1], qa.y, dot[j]);
    dot[j] = fmaf(f[2], qa.z, dot[j]); dot[j] = fmaf(f[3], qa.w, dot[j]);
    dot[j] = fmaf(f[4], qb.x, dot[j]); dot[j] = fmaf(f[5], qb.y, dot[j]);
    dot[j] = fmaf(f[6], qb.z, dot[j]); dot[j] = fmaf(f[7], qb.w, dot[j]);
  }
}
// DPL consecutive bf16 of a cached V row (one 4- or 8-byte load)
template <int DPL>
AMUSD_DEV void attn_vrow(const __nv_bfloat16* v, float (&f)[DPL]) {
  static_assert(DPL == 2 || DPL == 4, "DPL");
  if constexpr (DPL == 4) {
    const uint2 u = *(const uint2*)v;
    const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)&u.x), b = __bfloat1622float2(*(const __nv_bfloat162*)&u.y);
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
  } else {
    const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)v);
    f[0] = a.x; f[1] = a.y;
  }
}
// the G probabilities of one position (vector loads)
template <int G>
AMUSD_DEV void attn_prow(const float* s, float (&p)[G]) {
  if constexpr (G % 4 == 0) {
#pragma unroll
    for (int j = 0; j < G; j += 4) {
      const float4 x = *(const float4*)(s + j);
      p[j] = x.x; p[j + 1] = x.y; p[j + 2] = x.z; p[j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < G; j += 2) {
      const float2 x = *(const float2*)(s + j);
      p[j] = x.x; p[j + 1] = x.y;
    }
  }
}

// Issue the bulk copies of the cached K/V rows [lo, min(hi, pos0)) of head g
// (they do not depend on this step): called before the QKV dependency wait.
template <int HD, int G>
AMUSD_DEV bool attn_prefetch(const FwArgs& a, AttnSmem<HD, G>* sm, int layer, int g, int lo, int hi, int pos0) {
  const int tc = min(hi, pos0);
  if (tc <= lo) return false;
  const uint32_t bytes = (uint32_t)(tc - lo) * HD * 2;
  const size_t off = ((size_t)g * a.S + lo) * HD * 2;
  const char* kc = a.kcache + layer * a.kv_layer_bytes + off;
  const char* vc = a.vcache + layer * a.kv_layer_bytes + off;
  const uint32_t b = smem_u32(&sm->bar);
  mbar_expect_tx(b, 2 * bytes);
  const uint64_t pol = policy_evict_first();
  bulk_load(smem_u32(&sm->kb[0][0]), kc, bytes, b, pol);
  bulk_load(smem_u32(&sm->vb[0][0]), vc, bytes, b, pol);
  return true;
}

// Decode/verify attention for (KV head g, window row r, position split): the
// GROUP query heads of g together (K/V read once).  RoPE applied here; this
// step's K/V rounded to bf16 exactly as a later step reads them from the
// cache; the item owning position p appends row r's K/V; multi-split rows are
// merged in split order by the last-arriving split.  Cached K/V come from
// shared memory (staged before the dependency wait), so after the QKV phase
// completes only the query rows cost a round trip.
template <int HD, int G>
AMUSD_DEV void attn_item(const FwArgs& a, AttnSmem<HD, G>* sm, bool staged, uint32_t bar_par, int layer, int g, int r,
                         int split, int pos0, int tid, int dbg_item = -1) {
  constexpr int DPL = HD / 32, NC = HD / 8;
  const int wi = tid >> 5, lane = tid & 31;
  float(*red)[G][HD] = (float(*)[G][HD])&sm->kb[0][0];
  static_assert(4 * G * HD * 4 <= kAttnChunk * HD * 2, "red alias");
  const int p = pos0 + r;
  const int nsplit = nsplit_of(p);
  const int lo = split * kAttnChunk, hi = min(p + 1, lo + kAttnChunk);
  const int half = HD / 2, ncols = (a.H + 2 * a.KV) * HD;
  const float* qkv = a.qkv;
  const int qoff = g * (G + 2) * HD, koff = qoff + G * HD, voff = koff + HD;  // group-blocked q|k|v
  // ---- gather: q rows of the group, this step's K/V window rows; RoPE; one L2 round
  // trip (every load of a batch issued before any use)
  const int jmax = hi > pos0 ? min(r, hi - 1 - pos0) : -1;
  const int nq = G * half, nk = (jmax + 1) * half, ntot = nq + nk + (jmax + 1) * HD;
  for (int b = tid; b < ntot; b += 128 * 4) {
    float x0[4], x1[4], cs[4], sn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = b + 128 * u;
      x1[u] = cs[u] = sn[u] = 0.f;
      if (i < nq) {
        const int j = i / half, e = i - j * half;
        const float* q = qkv + (size_t)r * ncols + qoff + j * HD + e;
        x0[u] = __ldcg(q);
        x1[u] = __ldcg(q + half);
        cs[u] = a.cos[(size_t)p * half + e];
        sn[u] = a.sin[(size_t)p * half + e];
      } else if (i < nq + nk) {
        const int i2 = i - nq, j = i2 / half, e = i2 - j * half;
        const float* k = qkv + (size_t)j * ncols + koff + e;
        x0[u] = __ldcg(k);
        x1[u] = __ldcg(k + half);
        cs[u] = a.cos[(size_t)(pos0 + j) * half + e];
        sn[u] = a.sin[(size_t)(pos0 + j) * half + e];
      } else if (i < ntot) {
        const int i2 = i - nq - nk, j = i2 / HD, e = i2 - j * HD;
        x0[u] = __ldcg(qkv + (size_t)j * ncols + voff + e);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = b + 128 * u;
      const float r0 = x0[u] * cs[u] - x1[u] * sn[u], r1 = x1[u] * cs[u] + x0[u] * sn[u];
      if (i < nq) {
        const int j = i / half, e = i - j * half;
        sm->qs[attn_qidx<HD>(j, e)] = r0;
        sm->qs[attn_qidx<HD>(j, e + half)] = r1;
      } else if (i < nq + nk) {
        const int i2 = i - nq, j = i2 / half, e = i2 - j * half;
        sm->kn[j][e] = __float2bfloat16(r0);
        sm->kn[j][e + half] = __float2bfloat16(r1);
      } else if (i < ntot) {
        const int i2 = i - nq - nk, j = i2 / HD, e = i2 - j * HD;
        sm->vn[j][e] = __float2bfloat16(x0[u]);
      }
    }
  }
  if (staged) mbar_wait_t(smem_u32(&sm->bar), bar_par);
  named_bar(1, 128);
  if (a.dbg && tid == 0 && dbg_item >= 0) dbg_mark(a, dbg_item, 6, globaltimer());  // inputs ready
  if (p >= lo && p < hi) {  // KV append for row r (pending-token scheme)
    __nv_bfloat16* kc = (__nv_bfloat16*)(a.kcache + layer * a.kv_layer_bytes) + ((size_t)g * a.S + p) * HD;
    __nv_bfloat16* vc = (__nv_bfloat16*)(a.vcache + layer * a.kv_layer_bytes) + ((size_t)g * a.S + p) * HD;
    for (int e = tid; e < HD; e += 128) {
      kc[e] = sm->kn[r][e];
      vc[e] = sm->vn[r][e];
    }
  }
  // ---- scores: a thread pair per position (kAttnChunk == 64, 128 threads), each thread one
  // half of the head dims, then one shuffle.  Chunk order rotated so the 8 threads of a
  // quarter-warp read 8 distinct 16-byte bank groups of their K rows and the warp reads few
  // distinct query chunks.  Cached and window keys use the SAME order (batch invariance: a
  // position's score must not depend on whether it is in the cache or the window).
  const float4* qv = (const float4*)sm->qs;
  constexpr int NH = NC / 2;  // 16-byte chunks per half row
  const int pi = tid >> 1, hf = tid & 1;
  float mloc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) mloc[j] = -INFINITY;
  {
    const int t = lo + pi;
    float dot[G];
#pragma unroll
    for (int j = 0; j < G; ++j) dot[j] = 0.f;
    if (t < hi) {
      const uint4* kt = (const uint4*)(t < pos0 ? &sm->kb[t - lo][0] : &sm->kn[t - pos0][0]);
#pragma unroll 4
      for (int cc = 0; cc < NH; ++cc) {
        const int c = hf * NH + ((HD == 128 ? cc + (tid & 7) : cc + pi) & (NH - 1));
        float f[8];
        Elem<__nv_bfloat16>::unpack(kt[c], f);
        attn_dot8<G, NC>(dot, f, qv, c);
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) dot[j] += __shfl_xor_sync(0xffffffffu, dot[j], 1);
    if (t < hi) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const float sv = dot[j] * a.scale;
        if (hf == 0) sm->sc[t - lo][j] = sv;
        mloc[j] = sv;
      }
    }
  }
  if (a.dbg && tid == 0 && dbg_item >= 0) dbg_mark(a, dbg_item, 2, globaltimer());  // scores done
  // ---- softmax statistics per head (fixed reduction tree)
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float m = warp_max(mloc[j]);
    if (lane == 0) sm->wred[wi][j] = m;
  }
  named_bar(1, 128);
  float mj[G], lloc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    mj[j] = fmaxf(fmaxf(sm->wred[0][j], sm->wred[1][j]), fmaxf(sm->wred[2][j], sm->wred[3][j]));
    lloc[j] = 0.f;
  }
  if (tid < kAttnChunk && lo + tid < hi) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float e = expf(sm->sc[tid][j] - mj[j]);
      sm->sc[tid][j] = e;
      lloc[j] = e;
    }
  }
  named_bar(1, 128);  // wred reuse
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float l = warp_sum(lloc[j]);
    if (lane == 0) sm->wred[wi][j] = l;
  }
  named_bar(1, 128);
  if (wi == 0) {  // one warp records the per-head stats (mj[] stays in registers: constant indices)
#pragma unroll
    for (int j = 0; j < G; ++j)
      if (lane == j) {
        sm->stat[0][j] = mj[j];
        sm->stat[1][j] = (sm->wred[0][j] + sm->wred[1][j]) + (sm->wred[2][j] + sm->wred[3][j]);
      }
  }
  // ---- unnormalised P.V from shared memory: warp w takes positions lo+w, lo+w+4, ...
  // (cached rows, then window rows: increasing t, the same order at every batch size)
  float acc[G][DPL];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[j][e] = 0.f;
  const int tce = min(hi, pos0);
  int t = lo + wi;
  for (; t + 12 < tce; t += 16) {  // 4 positions' loads in flight
    float vv[4][DPL], pp[4][G];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      attn_vrow<DPL>(&sm->vb[t + 4 * u - lo][lane * DPL], vv[u]);
      attn_prow<G>(sm->sc[t + 4 * u - lo], pp[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < G; ++j)
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(pp[u][j], vv[u][e], acc[j][e]);
  }
  for (; t < tce; t += 4) {
    float vv[DPL], pp[G];
    attn_vrow<DPL>(&sm->vb[t - lo][lane * DPL], vv);
    attn_prow<G>(sm->sc[t - lo], pp);
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(pp[j], vv[e], acc[j][e]);
  }
  for (; t < hi; t += 4) {
    float vv[DPL], pp[G];
    attn_vrow<DPL>(&sm->vn[t - pos0][lane * DPL], vv);
    attn_prow<G>(sm->sc[t - lo], pp);
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(pp[j], vv[e], acc[j][e]);
  }
  named_bar(1, 128);  // everyone is done with kb before red overwrites it
  if (a.dbg && tid == 0 && dbg_item >= 0) dbg_mark(a, dbg_item, 7, globaltimer());  // P.V done
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) red[wi][j][lane * DPL + e] = acc[j][e];
  named_bar(1, 128);
  __nv_bfloat16* out = a.attn_b;
  const int ldo = a.H * HD;
  if (nsplit == 1) {
    for (int i = tid; i < G * HD; i += 128) {
      const int j = i / HD, e = i - j * HD;
      const float o = red[0][j][e] + red[1][j][e] + red[2][j][e] + red[3][j][e];
      out[(size_t)r * ldo + (g * G + j) * HD + e] = __float2bfloat16(o / sm->stat[1][j]);
    }
    return;
  }
  // The row's last split (grabbed after its other splits) merges; the others publish and go.
  int* cnt = a.attn_cnt + (g * KMAX + r) * kPad;
  if (split != nsplit - 1) {
    float* ws = a.attn_ws + (((size_t)g * KMAX + r) * a.max_splits + split) * G * (HD + 2);
    for (int i = tid; i < G * HD; i += 128) {
      const int j = i / HD, e = i - j * HD;
      __stcg(ws + j * (HD + 2) + e, red[0][j][e] + red[1][j][e] + red[2][j][e] + red[3][j][e]);
    }
    if (tid < G) {
      __stcg(ws + tid * (HD + 2) + HD, sm->stat[0][tid]);
      __stcg(ws + tid * (HD + 2) + HD + 1, sm->stat[1][tid]);
    }
    named_bar(1, 128);
    if (tid == 0) red_add_release(cnt, 1);
    return;
  }
  if (tid == 0) {
    wait_count(cnt, nsplit - 1);
    *cnt = 0;
  }
  named_bar(1, 128);
  // Merge in ONE round trip: the first 8 remote splits' o values (registers) and every split's
  // (m, l) (shared memory; this split's own from its stats) are issued together; then
  // M = max m, weights w_s = exp(m_s - M), L = sum l_s w_s in split order, O = sum o_s w_s in
  // split order (further batches of 8 splits: one more round trip each).  Deterministic and
  // position-only (batch invariant).
  const float* base = a.attn_ws + ((size_t)g * KMAX + r) * a.max_splits * G * (HD + 2);
  // [kMaxMerge][G] m (then the weights) and l, in the V staging buffer (dead after P.V)
  float* wts = (float*)&sm->vb[0][0];
  float* mlv = wts + kMaxMerge * G;
  static_assert(2 * kMaxMerge * G * 4 <= kAttnChunk * HD * 2, "merge scratch alias");
  constexpr int II = G * HD / 128;
  const int nrem = nsplit - 1;
  float o[II][8];
#pragma unroll
  for (int ii = 0; ii < II; ++ii) {
    const int i = tid + 128 * ii, j = i / HD, e = i - j * HD;
#pragma unroll
    for (int u = 0; u < 8; ++u) o[ii][u] = u < nrem ? __ldcg(base + ((size_t)u * G + j) * (HD + 2) + e) : 0.f;
  }
  for (int i = tid; i < nsplit * G; i += 128) {
    const int sp = i / G, j = i - sp * G;
    float m, l;
    if (sp < nsplit - 1) {
      const float* w = base + ((size_t)sp * G + j) * (HD + 2);
      m = __ldcg(w + HD);
      l = __ldcg(w + HD + 1);
    } else {
      m = sm->stat[0][j];
      l = sm->stat[1][j];
    }
    wts[i] = m;
    mlv[i] = l;
  }
  named_bar(1, 128);
  if (tid < G) {
    float M = -INFINITY;
    for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, wts[sp * G + tid]);
    float Ls = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float w = expf(wts[sp * G + tid] - M);
      wts[sp * G + tid] = w;
      Ls += mlv[sp * G + tid] * w;
    }
    sm->stat[1][tid] = Ls;  // (own stat no longer needed)
  }
  named_bar(1, 128);
  float O[II];
#pragma unroll
  for (int ii = 0; ii < II; ++ii) O[ii] = 0.f;
  for (int b0 = 0; b0 < nrem; b0 += 8) {  // remote splits in batches of 8 (the first already loaded)
    if (b0 > 0) {
#pragma unroll
      for (int ii = 0; ii < II; ++ii) {
        const int i = tid + 128 * ii, j = i / HD, e = i - j * HD;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          o[ii][u] = b0 + u < nrem ? __ldcg(base + ((size_t)(b0 + u) * G + j) * (HD + 2) + e) : 0.f;
      }
    }
#pragma unroll
    for (int ii = 0; ii < II; ++ii) {
      const int j = (tid + 128 * ii) / HD;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + u < nrem) O[ii] = fmaf(o[ii][u], wts[(b0 + u) * G + j], O[ii]);
    }
  }
#pragma unroll
  for (int ii = 0; ii < II; ++ii) {  // own split last, then normalise
    const int i = tid + 128 * ii, j = i / HD, e = i - j * HD;
    const float own = red[0][j][e] + red[1][j][e] + red[2][j][e] + red[3][j][e];
    O[ii] = fmaf(own, wts[(nsplit - 1) * G + j], O[ii]);
    out[(size_t)r * ldo + (g * G + j) * HD + e] = __float2bfloat16(O[ii] / sm->stat[1][j]);
  }
}

// ------------------------------------------------------------ the kernel
template <int HD, int G>
constexpr int attn_scratch_bytes() {
  return ((int)sizeof(AttnSmem<HD, G>) + 127) & ~127;
}
constexpr int epi_bytes() { return ((int)sizeof(EpiSmem) + 127) & ~127; }

// TP: a tensor-parallel shard's instance (cross-rank split-K reduce, all-rank argmax).  The
// unsharded instance compiles those branches out: as runtime checks in the split-K path they
// cost 8% (8B) / 17% (1B) of the forward.
template <int HD, int G, int MINB, bool TP, bool FUSE>
__global__ void __launch_bounds__(kThreads, MINB)
    k_forward(const __grid_constant__ CUtensorMap m_xa, const __grid_constant__ CUtensorMap m_attn,
              const __grid_constant__ CUtensorMap m_act, const __grid_constant__ CUtensorMap m_xb,
              const __grid_constant__ FwArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = a.stages;
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * kStageW;
  uint8_t* scratch = sX + S * kStageX;  // attention scratch / epilogue exchange (epilogue warps only)
  constexpr int kAttnBytes = attn_scratch_bytes<HD, G>();
  constexpr int kScratch = kAttnBytes + epi_bytes();
  uint64_t* bars = (uint64_t*)(scratch + kScratch);
  uint64_t* wfull = bars;
  uint64_t* xfull = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = tfull + kTbuf;
  uint64_t* qfull = tempty + kTbuf;
  uint64_t* qempty = qfull + kQ;
  int2* queue = (int2*)(qempty + kQ);
  uint32_t* tmem_slot = (uint32_t*)(queue + kQ);
  int* s_lay = (int*)(tmem_slot + 1);  // A, rows, pos0, active, epoch

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // FUSE: [0] act tile written (epilogue -> X loader), [1] down-slab MMAs done (MMA -> epilogue),
  // [2] down-slab accumulators free (epilogue -> MMA)
  __shared__ uint64_t s_fb[3];
  constexpr uint32_t kCols = FUSE ? 512 : kTmemCols;  // FUSE: 16 down-slab accumulators after the 256
  if (threadIdx.x == 0) {
    const StepCtl* c = a.ctl;
    const int active = c->active;
    const int rows = active ? c->rows : 0, pos0 = c->pos0;
    int A = 0;
    for (int r = 0; r < rows; ++r) A += a.KV * nsplit_of(pos0 + r);
    s_lay[0] = A;
    s_lay[1] = rows;
    s_lay[2] = pos0;
    s_lay[3] = active;
    s_lay[4] = ld_volatile(a.sched + 2 * kPad);  // launch epoch (bumped by the last CTA of each launch)
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&wfull[s]), 1);
      mbar_init(smem_u32(&xfull[s]), 1);
      mbar_init(smem_u32(&empty[s]), NACC);
    }
    for (int i = 0; i < kTbuf; ++i) { mbar_init(smem_u32(&tfull[i]), NACC); mbar_init(smem_u32(&tempty[i]), 128); }
    for (int i = 0; i < kQ; ++i) { mbar_init(smem_u32(&qfull[i]), 1); mbar_init(smem_u32(&qempty[i]), 1 + NACC + 1); }
    mbar_init(smem_u32(&((AttnSmem<HD, G>*)scratch)->bar), 1);
    if (FUSE) {
      mbar_init(smem_u32(&s_fb[0]), 1);
      mbar_init(smem_u32(&s_fb[1]), NACC);
      mbar_init(smem_u32(&s_fb[2]), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!s_lay[3]) return;  // inactive step: nothing grabbed, nothing to reset
  // The launch layout lives in shared memory: as a long-lived register struct it spills to
  // local memory, and every acquire poll on the SM invalidates L1 (CCTL.IVALL), turning each
  // reload into an L2 round trip.
  __shared__ Lay s_L;
  __shared__ int s_epi_done;  // items the epilogue warps have finished (producer: lazy attention grabs)
  if (threadIdx.x == 0) {
    s_epi_done = 0;
    s_L.A = s_lay[0]; s_L.rows = s_lay[1]; s_L.pos0 = s_lay[2];
    s_L.pre[0] = 0;
    s_L.pre[1] = a.g[kGQkv].nitems;
    s_L.pre[2] = s_L.pre[1] + s_L.A;
    s_L.pre[3] = s_L.pre[2] + a.g[kGO].nitems;
    s_L.pre[4] = s_L.pre[3] + a.g[kGGu].nitems;
    s_L.PL = s_L.pre[4] + a.g[kGDown].nitems;
    s_L.total = KMAX + a.L * s_L.PL + a.g[kGLm].nitems;
  }
  const Lay& L = s_L;
  if (warp == kWarpMma0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int* done = a.sched + 3 * kPad;  // done count of phase p at done[p * kPad]
  // Per-tile completion stamps: epoch * 2^16 + layer + 1 (monotonic: never reset).
  const long long epoch_base = (long long)s_lay[4] << 16;
  auto stamp = [&](int layer) { return epoch_base + layer + 1; };
  auto flags_of = [&](int gk) { return a.tflag + (size_t)gk * a.tflag_tiles * (kPad / 2); };

  if (warp == 0) {
    // ===== scheduler + weight producer =====
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once
      int n = 0;
      long long gu = 0;
      Ring rg, rl;  // rg: stage being filled; rl: stage `inflight` units behind (outstanding cap)
      // Optional L2 prefetch stream (AMUSD_FW_L2_MB): the grabber of item i prefetches item i + ahead.
      const uint64_t pol_keep = policy_evict_last();
      const int ahead = a.prefetch_items;
      const int inflight = a.inflight > 0 ? min(a.inflight, S) : S;
      auto prefetch_item = [&](int k) {
        if (k >= L.total) return;
        const int2 pj = locate(a, L, k);
        const int kind = kind_of(pj.x, a.L);
        if (!is_gemm(kind)) return;
        const GemmRes g = resolve(a, gemm_of(kind), layer_of(pj.x));
        const int c = pj.y / g.ntiles, t = pj.y - c * g.ntiles;
        prefetch_l2(g.wt + ((size_t)t * g.kb + (size_t)c * g.kc) * kWBytes, (uint32_t)g.kc * kWBytes, pol_keep);
      };
      if (a.prefetch_next) {  // layer 0's QKV + O slice of this CTA
        const size_t span = a.qo_bytes;
        const size_t lo = span * blockIdx.x / gridDim.x & ~(size_t)15, hi = span * (blockIdx.x + 1) / gridDim.x & ~(size_t)15;
        if (hi > lo) prefetch_l2(a.g[kGQkv].wt + lo, (uint32_t)(hi - lo), pol_keep);
      }
      if (ahead > 0)  // the first `ahead` items have no earlier grabber: spread them over the CTAs
        for (int k = blockIdx.x; k < ahead; k += gridDim.x) prefetch_item(k);
      // draft cut probe: loaded with each grab, consumed at the next (never blocks the stream)
      const int ab_ack = a.ab_req ? ld_volatile(&a.ctl->rb_ack_local) : 0;
      auto ab_probe = [&]() { return a.ab_req ? (ld_volatile(a.ab_req) ^ ab_ack) | ld_volatile(a.ab_done) : 0; };
      bool cut = false;
      int ab_next = ab_probe();
      int i_next = atomicAdd(a.sched, 1);  // grab counter: sched[0]; exit counter: sched[kPad]
      // Attention items go to drained CTAs: grabbed eagerly behind a GEMM still in flight, an
      // attention item (and its row's split merge) would wait for that GEMM's whole epilogue.
      auto attn_at = [&](int k) { return k < L.total && kind_of(locate(a, L, k).x, a.L) == kKAttn; };
      for (;;) {
        // the grab of the following item is in flight while this one streams (GEMM items)
        // (only QKV and attention items can be followed by an attention grab: the others
        // grab eagerly, without the peek's round trip)
        const int i = i_next;
        if (ab_next && !cut) {  // cut: no item beyond the grabbed prefix is handed out
          cut = true;
          atomicMax(a.sched, kCutIndex);
          atomicExch(a.sched + 2 * kPad + 1, 1);  // launch_cut_cleanup flag
        }
        bool have_next = false;
        if (i < L.total) {
          const int k = kind_of(locate(a, L, i).x, a.L);
          if (k != kKQkv && k != kKAttn) {
            i_next = atomicAdd(a.sched, 1);
            if (!cut) ab_next = ab_probe();
            have_next = true;
          }
        }
        if (ahead > 0 && i < L.total) prefetch_item(i + ahead);
        const int slot = n % kQ;
        mbar_wait_t(smem_u32(&qempty[slot]), ((n / kQ) & 1) ^ 1);
        if (i >= L.total) {
          queue[slot] = make_int2(-1, 0);
          mbar_arrive(smem_u32(&qfull[slot]));
          break;
        }
        const int2 pj = locate(a, L, i);
        dbg_mark(a, i, 0, (long long)i | ((long long)blockIdx.x << 20) | ((long long)pj.x << 32));
        dbg_mark(a, i, 1, globaltimer());
        queue[slot] = pj;
        mbar_arrive(smem_u32(&qfull[slot]));
        ++n;
        const int kind = kind_of(pj.x, a.L);
        if (kind == kKDown && a.prefetch_next && layer_of(pj.x) + 1 < a.L) {
          // Move the next layer's QKV + O weights (the latency-bound part of its chain) to L2
          // while this bandwidth-bound phase streams: down item j prefetches slice j.
          const size_t span = a.qo_bytes, nslices = (size_t)a.g[kGDown].nitems;
          const size_t lo = span * pj.y / nslices & ~(size_t)15, hi = span * (pj.y + 1) / nslices & ~(size_t)15;
          if (hi > lo)
            prefetch_l2(a.g[kGQkv].wt + (size_t)(layer_of(pj.x) + 1) * a.g[kGQkv].wt_stride + lo, (uint32_t)(hi - lo),
                        pol_keep);
        }
        if (is_gemm(kind) && !(FUSE && kind == kKDown)) {  // (FUSE: down items carry no weights)
          const GemmRes g = resolve(a, gemm_of(kind), layer_of(pj.x));
          const int c = pj.y / g.ntiles, t = pj.y - c * g.ntiles;  // chunk-major item order
          const uint8_t* src = g.wt + ((size_t)t * g.kb + (size_t)c * g.kc) * kWBytes;
          for (int u = 0; u < g.kc; u += kUPS, ++gu, rg.next(S)) {  // (kc % kUPS == 0: build_kinds)
            const int s = rg.s;
            mbar_wait_t(smem_u32(&empty[s]), rg.ph ^ 1u);
            // Optional outstanding-load cap (AMUSD_FW_INFLIGHT): at most `inflight` unlanded stages.
            if (inflight < S && gu >= inflight) {
              mbar_wait_t(smem_u32(&wfull[rl.s]), rl.ph);
              rl.next(S);
            }
            if (a.debug & 8) {  // perf isolation: no weight traffic
              mbar_arrive(smem_u32(&wfull[s]));
              continue;
            }
            mbar_expect_tx(smem_u32(&wfull[s]), kStageW);
#pragma unroll
            for (int uu = 0; uu < kUPS; ++uu) {
              const uint32_t dst = smem_u32(sW + s * kStageW + uu * kWBytes);
              const uint8_t* from = src + (size_t)(u + uu) * kWBytes;
              if (a.debug & 16)  // perf knob: no L2 eviction hint on the weight stream
                bulk_load_nohint(dst, from, kWBytes, smem_u32(&wfull[s]));
              else
                bulk_load(dst, from, kWBytes, smem_u32(&wfull[s]), pol_w);
            }
          }
          if (FUSE && kind == kKGu && c == g.nchunks - 1) {
            // the tile's merging chunk: the down weights of its 64 features, unit (output tile o,
            // K unit t) of every output tile (the down layout is tile-major, 64-wide K units)
            const GemmRes gd = resolve(a, kGDown, layer_of(pj.x));
            const int nt = a.g[kGDown].ntiles;
            for (int o = 0; o < nt; o += kUPS, ++gu, rg.next(S)) {
              const int s = rg.s;
              mbar_wait_t(smem_u32(&empty[s]), rg.ph ^ 1u);
              if (inflight < S && gu >= inflight) {
                mbar_wait_t(smem_u32(&wfull[rl.s]), rl.ph);
                rl.next(S);
              }
              if (a.debug & 8) {
                mbar_arrive(smem_u32(&wfull[s]));
                continue;
              }
              mbar_expect_tx(smem_u32(&wfull[s]), kStageW);
#pragma unroll
              for (int uu = 0; uu < kUPS; ++uu)
                bulk_load(smem_u32(sW + s * kStageW + uu * kWBytes), gd.wt + ((size_t)(o + uu) * gd.kb + t) * kWBytes,
                          kWBytes, smem_u32(&wfull[s]), pol_w);
            }
          }
          dbg_mark(a, i, 2, globaltimer());
        }
        if (!have_next) {  // peek; an attention item waits until this CTA's pipeline has drained
          for (;;) {
            if (!attn_at(ld_volatile(a.sched))) break;
            if (atomicAdd(&s_epi_done, 0) >= n) break;  // (shared atomics: a race-free flag)
            __nanosleep(64);
          }
          i_next = atomicAdd(a.sched, 1);
          if (!cut) ab_next = ab_probe();
        }
      }
    }
  } else if (warp == kWarpX) {
    // ===== activation loader: dependency wait, then X tiles by TMA =====
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_last();  // X is re-read by every CTA of the phase
      int n = 0, dep_ok = -1, fz = 0;
      Ring rg;
      for (;;) {
        const int slot = n % kQ;
        mbar_wait_t(smem_u32(&qfull[slot]), (n / kQ) & 1);
        const int2 it = queue[slot];
        mbar_arrive(smem_u32(&qempty[slot]));
        ++n;
        if (it.x < 0) break;
        const int kind = kind_of(it.x, a.L);
        if (!is_gemm(kind) || (FUSE && kind == kKDown)) continue;
        const GemmKind& g = a.g[gemm_of(kind)];
        const int c = it.y / g.ntiles, kc = g.kc, layer = layer_of(it.x);
        const int prod = it.x - 1;  // producer phase
        if (!(a.debug & 2) && prod > dep_ok) {  // debug bit 1: ignore GEMM dependencies (timing only)
          // Fine-grained: wait only for the producer tiles covering this item's K range --
          // unless the whole producer phase is already known (or now seen) complete.
          const int k0 = c * kc * BK, k1 = k0 + kc * BK;  // input columns [k0, k1)
          if (!fine_for(a, kind)) {  // phase-level dependency (default, measured faster)
            wait_count(done + prod * kPad, phase_count(a, L, prod));
            dep_ok = prod;
          } else if (ld_acquire_gpu(done + prod * kPad) >= phase_count(a, L, prod)) {
            dep_ok = prod;
          } else if (kind == kKQkv && layer == 0) {
            wait_count(done, KMAX);  // embedding rows
          } else if (kind == kKQkv || kind == kKLm) {  // xa <- down(layer-1) tiles (128 columns each)
            wait_tiles(flags_of(kGDown), k0 / BM, (k1 + BM - 1) / BM, stamp(kind == kKLm ? a.L - 1 : layer - 1));
          } else if (kind == kKO) {  // attn_b columns -> heads -> head groups of this layer
            const int g0 = k0 / a.hd / (a.H / a.KV), g1 = ((k1 + a.hd - 1) / a.hd + a.H / a.KV - 1) / (a.H / a.KV);
            const int per_group = L.A / a.KV;
            for (int gg = g0; gg < g1; ++gg) wait_count(a.agrp + ((size_t)layer * a.KV + gg) * kPad, per_group);
          } else if (kind == kKGu) {  // xb <- O(layer) tiles
            wait_tiles(flags_of(kGO), k0 / BM, (k1 + BM - 1) / BM, stamp(layer));
          } else {  // down: act features [k0, k1) <- gate/up tiles of 64 features
            wait_tiles(flags_of(kGGu), k0 / 64, (k1 + 63) / 64, stamp(layer));
          }
          fence_proxy_async();
        }
        if (a.dbg) dbg_mark(a, phase_first(a, L, it.x) + it.y, 3, globaltimer());
        const CUtensorMap* map = g.map == 0 ? &m_xa : (g.map == 1 ? &m_attn : (g.map == 2 ? &m_act : &m_xb));
        for (int u = 0; u < kc; u += kUPS, rg.next(S)) {
          const int s = rg.s;
          mbar_wait_t(smem_u32(&empty[s]), rg.ph ^ 1u);
          if (a.debug & 4) {  // perf isolation: no activation traffic
            mbar_arrive(smem_u32(&xfull[s]));
            continue;
          }
          mbar_expect_tx(smem_u32(&xfull[s]), kStageX);
#pragma unroll
          for (int uu = 0; uu < kUPS; ++uu)
            tma_load_2d(smem_u32(sX + s * kStageX + uu * kXBytes), map, (c * kc + u + uu) * BK, 0,
                        smem_u32(&xfull[s]), pol_x);
        }
        if (FUSE && kind == kKGu && c == g.nchunks - 1) {  // the act tile of these 64 features, once written
          mbar_wait_t(smem_u32(&s_fb[0]), fz & 1);
          ++fz;
          fence_proxy_async();
          const int nt = a.g[kGDown].ntiles;
          for (int o = 0; o < nt; o += kUPS, rg.next(S)) {
            const int s = rg.s;
            mbar_wait_t(smem_u32(&empty[s]), rg.ph ^ 1u);
            mbar_expect_tx(smem_u32(&xfull[s]), kStageX);
#pragma unroll
            for (int uu = 0; uu < kUPS; ++uu)
              tma_load_2d(smem_u32(sX + s * kStageX + uu * kXBytes), &m_act, (it.y - c * g.ntiles) * BK, 0,
                          smem_u32(&xfull[s]), pol_x);
          }
        }
      }
    }
  } else if (warp < kWarpEpi0) {
    // ===== MMA issuers: warp w issues K-slice kk of every unit =====
    if (lane == 0) {
      const int kk = warp - kWarpMma0;
      int n = 0, seg = 0, fz = 0;
      Ring rg;
      for (;;) {
        const int slot = n % kQ;
        mbar_wait_t(smem_u32(&qfull[slot]), (n / kQ) & 1);
        const int2 it = queue[slot];
        mbar_arrive(smem_u32(&qempty[slot]));
        ++n;
        if (it.x < 0) break;
        const bool nomma = a.debug & 1;
        const int kind = kind_of(it.x, a.L);
        if (!is_gemm(kind) || (FUSE && kind == kKDown)) continue;
        const int kc = a.g[gemm_of(kind)].kc;
        const int b = seg % kTbuf;
        mbar_wait_t(smem_u32(&tempty[b]), ((seg / kTbuf) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((b * NACC + kk) * BN);
        for (int u = 0; u < kc; u += kUPS, rg.next(S)) {
          const int s = rg.s;
          const uint32_t par = rg.ph;
          mbar_wait_t(smem_u32(&wfull[s]), par);
          mbar_wait_t(smem_u32(&xfull[s]), par);
          tc_fence_after();
          if (nomma) {  // perf isolation: consume the stage without an MMA
            mbar_arrive(smem_u32(&empty[s]));
            continue;
          }
#pragma unroll
          for (int uu = 0; uu < kUPS; ++uu)
            umma(d, umma_desc(smem_u32(sW + s * kStageW + uu * kWBytes) + kk * 32),
                 umma_desc(smem_u32(sX + s * kStageX + uu * kXBytes) + kk * 32), (u + uu) > 0 ? 1u : 0u);
          umma_commit(smem_u32(&empty[s]));  // one commit per stage
        }
        if (nomma) mbar_arrive(smem_u32(&tfull[b]));
        else umma_commit(smem_u32(&tfull[b]));
        ++seg;
        if (FUSE && kind == kKGu && it.y / a.g[kGGu].ntiles == a.g[kGGu].nchunks - 1) {
          // down slab (the tile's merging chunk): unit o (output tile o, K = this tile's 64 features) into its own
          // accumulator (columns 256 + 16 o); warp kk issues the units o = kk mod 4, all 4 K16 steps
          mbar_wait_t(smem_u32(&s_fb[2]), (fz & 1) ^ 1);
          ++fz;
          tc_fence_after();
          const int nt = a.g[kGDown].ntiles;
          for (int o = 0; o < nt; o += kUPS, rg.next(S)) {
            const int s = rg.s;
            const uint32_t par = rg.ph;
            mbar_wait_t(smem_u32(&wfull[s]), par);
            mbar_wait_t(smem_u32(&xfull[s]), par);
            tc_fence_after();
#pragma unroll
            for (int uu = 0; uu < kUPS; ++uu) {
              if (((o + uu) & (NACC - 1)) != kk || nomma) continue;
              const uint32_t d2 = tmem + (uint32_t)(kTmemCols + (o + uu) * BN);
#pragma unroll
              for (int ks = 0; ks < BK / 16; ++ks)
                umma(d2, umma_desc(smem_u32(sW + s * kStageW + uu * kWBytes) + ks * 32),
                     umma_desc(smem_u32(sX + s * kStageX + uu * kXBytes) + ks * 32), ks > 0 ? 1u : 0u);
            }
            umma_commit(smem_u32(&empty[s]));
          }
          umma_commit(smem_u32(&s_fb[1]));
        }
      }
    }
  } else {
    // ===== epilogue + SIMT items (128 threads) =====
    const int tid = threadIdx.x - 32 * kWarpEpi0;
    const int q = warp & 3;        // TMEM lane quarter this warp may access
    const int nl = q * 32 + lane;  // tile row held by this thread
    EpiSmem* es = (EpiSmem*)(scratch + kAttnBytes);  // never aliased by the attention scratch
    EpiTmp* et = (EpiTmp*)&((AttnSmem<HD, G>*)scratch)->kb[0][0];  // per item: aliases the K/V staging
    static_assert(sizeof(EpiTmp) <= 2 * sizeof(((AttnSmem<HD, G>*)nullptr)->kb), "EpiTmp alias");
    using AS = AttnSmem<HD, G>;
    static_assert(offsetof(AS, vb) == sizeof(((AS*)nullptr)->kb), "kb|vb contiguous");
    if (tid == 0) es->inv_phase = -1;
    int n = 0, seg = 0, attn_dep_ok = -1, ez = 0;
    uint32_t attn_par = 0;
    for (;;) {
      const int slot = n % kQ;
      mbar_wait_t(smem_u32(&qfull[slot]), (n / kQ) & 1);
      const int2 it = queue[slot];
      named_bar(1, 128);
      if (tid == 0) mbar_arrive(smem_u32(&qempty[slot]));
      ++n;
      if (it.x < 0) break;
      const int p = it.x, j = it.y;
      const int kind = kind_of(p, a.L), layer = layer_of(p);
      bool wrote = true, lm_last_check = false;
      if (FUSE && kind == kKDown) {
        // down tile j: every gate/up tile has red.added its 64 features' partial; merge and run
        // the residual epilogue (h, the next norm input, its sums of squares)
        const GemmKind& g = a.g[kGDown];
        const __nv_bfloat16* gnext = g.gnext + (size_t)layer * g.gnext_stride;
        // Every gate/up item of THIS layer contributes to every down tile, so the dependency is
        // the gate/up phase count (per layer; a shared per-tile counter would let a later layer's
        // merge item, grabbed early, fire on this layer's contributions).  Nothing of the layer
        // is read before it: h's writer, the O phase, may still be running when this is grabbed.
        if (tid == 0) {
          wait_count(done + (p - 1) * kPad, a.g[kGGu].nitems);
          if (a.dbg) dbg_mark(a, phase_first(a, L, p) + j, 6, globaltimer());
        }
        named_bar(1, 128);
        resid_prefetch(g, gnext, j, nl, L.rows, et);
        cp_async_wait_all();
        named_bar(1, 128);
        unsigned long long* acc64 = (unsigned long long*)a.ws + (size_t)g.ws_off + (size_t)j * BN * BM + nl;
        long long s64[BN];
        float acc[BN];
#pragma unroll
        for (int r = 0; r < BN; ++r) s64[r] = r < L.rows ? (long long)__ldcg(acc64 + r * BM) : 0ll;
#pragma unroll
        for (int r = 0; r < BN; ++r) {
          acc[r] = (float)((double)s64[r] * (1.0 / 4294967296.0));
          if (r < L.rows) __stcg(acc64 + r * BM, 0ull);
        }
        tile_epilogue<TP>(a, g, gnext, j, nl, acc, L.rows, es, et, q, lane);
      } else if (is_gemm(kind)) {
        const GemmKind& g = a.g[gemm_of(kind)];
        const int b = seg % kTbuf;
        mbar_wait_t(smem_u32(&tfull[b]), (seg / kTbuf) & 1);
        tc_fence_after();
        if (a.dbg && tid == 0) dbg_mark(a, phase_first(a, L, p) + j, 4, globaltimer());
        float v[BN];
        {
          const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NACC * BN);
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
        mbar_arrive(smem_u32(&tempty[b]));
        ++seg;
        const int epi = g.epi, nchunks = g.nchunks;
        // RMSNorm scale of the phase's input rows (once per phase per CTA).  Only the merging
        // item scales (the scale is linear and applies to the exact sum): contributors skip
        // this round trip and publish at once.
        const bool need_inv = epi == kEpStoreScaled || epi == kEpGateUp || epi == kEpArgmax;
        const bool final_item = nchunks <= 1 || j / g.ntiles == nchunks - 1;
        if (need_inv && final_item && es->inv_phase != p) {
          // the RMSNorm scale needs the whole input row: wait for the full producer phase
          // (the MMA above only needed the tiles of its K range)
          if (fine_for(a, kind)) {  // (phase-level mode: the MMA already waited for the whole phase)
            if (tid == 0) {
              const int prod = p - 1;  // O(l) for gate/up; down(l-1) for QKV(l); down(L-1) for the LM head
              wait_count(done + prod * kPad, phase_count(a, L, prod));
            }
            named_bar(1, 128);
          }
          // 8 threads per row, each a strided slice of the row's tile sums; fixed shuffle tree
          const float* ssp_in = g.ssp_in;
          const int nt = a.d / BM, rr = tid >> 3, part = tid & 7;
          float tot = 0.f;
          {  // all loads first (one round trip), then the fixed-order sum; d <= 8192 -> <= 8 per thread
            float vals[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int k = part + 8 * u;
              vals[u] = k < nt ? __ldcg(ssp_in + (size_t)rr * nt + k) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) tot += vals[u];
          }
          tot += __shfl_xor_sync(0xffffffffu, tot, 1);
          tot += __shfl_xor_sync(0xffffffffu, tot, 2);
          tot += __shfl_xor_sync(0xffffffffu, tot, 4);
          named_bar(1, 128);
          if (part == 0) es->inv[rr] = rsqrtf(tot / (float)a.d + a.eps);
          named_bar(1, 128);
          if (tid == 0) es->inv_phase = p;
        }
        // Chunk-major order: item j = c * ntiles + t.  Every tile's chunk 0 is grabbed before
        // any chunk 1, ..., so a tile's merging (last) chunk comes a full round after the
        // chunks it waits for.
        const int cj = j / g.ntiles, t = j - cj * g.ntiles;
        bool final = true;
        float acc[BN];
        if (nchunks > 1 || (TP && g.xr)) {
          // Split-K in exact int64 fixed point (2^-32): the red.adds commute, so the merged
          // tile is bit-identical whatever the chunks' arrival order (deterministic, batch
          // invariant) and no partial ever needs a merge round trip.  Layout [tile][row][128].
          const size_t off = (size_t)g.ws_off + (size_t)t * BN * BM + nl;
          unsigned long long* acc64 = (unsigned long long*)a.ws + off;
          // live rows only: dead rows' accumulators are never added, read or re-armed
#pragma unroll
          for (int r = 0; r < BN; ++r) {
            if (r < L.rows) {
              const long long fx = __float2ll_rn(v[r] * 4294967296.0f);
              if (TP && g.xr) {  // tensor parallel: into every rank's accumulator (the fused allreduce)
                for (int pr = 0; pr < a.tp; ++pr) red_add_u64_sys(a.peer_ws[pr] + off + r * BM, fx);
              } else {
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc64 + r * BM), "l"(fx) : "memory");
              }
            }
          }
          named_bar(1, 128);
          // The tile's last chunk (grabbed after its other chunks) merges; the others publish
          // with a fire-and-forget release and move on -- no round trip in their epilogue.
          // Tensor parallel: every chunk (mergers included) bumps every rank's tile count after
          // a system-scope fence; each rank's local last chunk merges once all ranks' chunks
          // have arrived.
          final = cj == nchunks - 1;
          if (TP && g.xr && tid == 0) {
            __threadfence_system();
            for (int pr = 0; pr < a.tp; ++pr) red_add_sys(a.peer_cnt[pr] + g.cnt_off + t * kPad, 1);
          }
          if (!final) {
            if (tid == 0 && !(TP && g.xr)) {
              if (a.debug & 32) red_add_relaxed(a.tile_cnt + g.cnt_off + t * kPad, 1);  // timing experiment only
              else red_add_release(a.tile_cnt + g.cnt_off + t * kPad, 1);
            }
          } else {
            // the residual rows and the next norm weight are final since earlier phases:
            // fetch them while the chunk count is awaited
            const __nv_bfloat16* gnext = g.gnext ? g.gnext + (size_t)layer * g.gnext_stride : nullptr;
            if (epi == kEpResid) {
              resid_prefetch(g, gnext, t, nl, L.rows, et);
              cp_async_wait_all();  // (lands while tid 0 awaits the count; others wait at the barrier)
            }
            if (tid == 0) {
              if (TP && g.xr) wait_count_sys(a.tile_cnt + g.cnt_off + t * kPad, g.nchunks_total);
              else wait_count(a.tile_cnt + g.cnt_off + t * kPad, nchunks - 1);
              a.tile_cnt[g.cnt_off + t * kPad] = 0;  // re-arm for the next phase / launch
              if (a.dbg) dbg_mark(a, phase_first(a, L, p) + j, 6, globaltimer());
            }
            named_bar(1, 128);
            long long s64[BN];
#pragma unroll
            for (int r = 0; r < BN; ++r) s64[r] = r < L.rows ? (long long)__ldcg(acc64 + r * BM) : 0ll;
#pragma unroll
            for (int r = 0; r < BN; ++r) {
              acc[r] = (float)((double)s64[r] * (1.0 / 4294967296.0));
              if (r < L.rows) __stcg(acc64 + r * BM, 0ull);  // re-arm (next use is a later phase)
            }
          }
        } else {
          if (epi == kEpResid) {
            resid_prefetch(g, g.gnext + (size_t)layer * g.gnext_stride, t, nl, L.rows, et);
            cp_async_wait_all();
            named_bar(1, 128);
          }
#pragma unroll
          for (int r = 0; r < BN; ++r) acc[r] = v[r];
        }
        if (final) {
          const __nv_bfloat16* gnext = g.gnext ? g.gnext + (size_t)layer * g.gnext_stride : nullptr;
          tile_epilogue<TP>(a, g, gnext, t, nl, acc, L.rows, es, et, q, lane);
        }
        if (FUSE && kind == kKGu && final) {
          // hand the act tile (global, written above) to the X loader, then fold the down-slab
          // products of these 64 features into the down tiles' int64 accumulators.  The TMA reads
          // through L2: the act stores must be performed at gpu scope first (a CTA-scope hand-off
          // alone may leave them in the SM's write path)
          __threadfence();
          fence_proxy_async();
          named_bar(1, 128);
          if (tid == 0) mbar_arrive(smem_u32(&s_fb[0]));
          mbar_wait_t(smem_u32(&s_fb[1]), ez & 1);
          ++ez;
          tc_fence_after();
          const GemmKind& gd = a.g[kGDown];
          unsigned long long* accd = (unsigned long long*)a.ws + (size_t)gd.ws_off + nl;
          for (int o = 0; o < gd.ntiles; ++o) {
            float w[BN];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(kTmemCols + o * BN), w);
#pragma unroll
            for (int r = 0; r < BN; ++r)
              if (r < L.rows) {
                const long long fx = __float2ll_rn(w[r] * 4294967296.0f);
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(accd + (size_t)o * BN * BM + r * BM),
                             "l"(fx) : "memory");
              }
          }
          tc_fence_before();
          mbar_arrive(smem_u32(&s_fb[2]));  // (the item's publish below releases the red.adds)
        }
        wrote = final;
        lm_last_check = epi == kEpArgmax;
      } else if (kind == kKEmbed) {
        embed_item(a, j, L.rows, tid);
      } else {  // attention
        int r = 0, rem = j;
        for (;;) {
          const int cnt = a.KV * nsplit_of(L.pos0 + r);
          if (rem < cnt) break;
          rem -= cnt;
          ++r;
        }
        const int gh = rem % a.KV, split = rem / a.KV;
        const int lo = split * kAttnChunk, hi = min(L.pos0 + r + 1, lo + kAttnChunk);
        AttnSmem<HD, G>* asm_ = (AttnSmem<HD, G>*)scratch;
        // the cached K/V rows do not depend on this step: stage them before the wait
        bool staged = false;
        if (tid == 0) {
          staged = attn_prefetch<HD, G>(a, asm_, layer, gh, lo, hi, L.pos0);
          asm_->last = staged;
        }
        if (tid == 0) {
          if (fine_for(a, kKAttn)) {  // this head group's QKV tiles only (group-blocked: consecutive tiles)
            const int tpg = (G + 2) * HD / BM;
            wait_tiles(flags_of(kGQkv), gh * tpg, (gh + 1) * tpg, stamp(layer));
          } else if (p - 1 > attn_dep_ok) {
            wait_count(done + (p - 1) * kPad, phase_count(a, L, p - 1));
          }
        }
        attn_dep_ok = p - 1;
        named_bar(1, 128);
        staged = asm_->last;
        if (a.dbg && tid == 0) dbg_mark(a, phase_first(a, L, p) + j, 3, globaltimer());
        attn_item<HD, G>(a, asm_, staged, attn_par, layer, gh, r, split, L.pos0, tid, phase_first(a, L, p) + j);
        if (a.dbg && tid == 0) dbg_mark(a, phase_first(a, L, p) + j, 4, globaltimer());
        if (staged) attn_par ^= 1u;
      }
      // publish: this item's writes are visible (generic and async proxy) before the count
      // (CTA barrier, then one release by thread 0: the cooperative-groups grid-sync pattern).
      // (attention items: slot 2 = scores done, 6 = inputs ready, 7 = P.V done -- set in attn_item)
      if (a.dbg && tid == 0 && kind != kKAttn) dbg_mark(a, phase_first(a, L, p) + j, 7, globaltimer());
      if (wrote) fence_proxy_async();
      named_bar(1, 128);
      if (tid == 0) {
        if (a.dbg) dbg_mark(a, phase_first(a, L, p) + j, 5, globaltimer());
        if (lm_last_check) {
          if (TP && a.tp > 1) {  // this item's keys reached every rank: count it everywhere
            __threadfence_system();
            for (int pr = 0; pr < a.tp; ++pr) red_add_sys(lm_counter(a.peer_sched[pr]), 1);
          }
          const int old = atom_add_acq_rel(done + p * kPad, 1);
          if (old == a.g[kGLm].nitems - 1) {  // last LM-head item: final argmax per row
            if (TP && a.tp > 1) {  // ... once every rank's LM items have merged their keys here
              wait_count_sys(lm_counter(a.sched), a.lm_items_total);
              *lm_counter(a.sched) = 0;
            }
            for (int r = 0; r < L.rows; ++r) {
              const unsigned long long k = atomicExch(a.best + r, 0ull);
              a.ctl->preds[r] = argmax_key_index(k);
            }
          }
        } else if (wrote) {
          if (!fine_for(a, kind_of(p + 1, a.L))) {  // the consumer phase waits phase-level
          } else if (is_gemm(kind)) {  // tile final: stamp it for the fine-grained consumers
            const int gk = gemm_of(kind);
            const int t = j % a.g[gk].ntiles;
            st_release_gpu64(flags_of(gk) + (size_t)t * (kPad / 2), stamp(layer));
          } else if (kind == kKAttn) {
            int r = 0, rem = j;
            for (;;) {
              const int cnt = a.KV * nsplit_of(L.pos0 + r);
              if (rem < cnt) break;
              rem -= cnt;
              ++r;
            }
            red_add_release(a.agrp + ((size_t)layer * a.KV + rem % a.KV) * kPad, 1);
          }
          red_add_release(done + p * kPad, 1);
        } else {
          // non-final split-K item: its partial was released by the tile count; the consumers'
          // acquire of the phase count reaches the final items' releases through the RMW chain
          red_add_relaxed(done + p * kPad, 1);
        }
        atomicExch(&s_epi_done, n);  // item n done (the producer's lazy attention grab)
      }
    }
  }
  __syncthreads();
  if (warp == kWarpMma0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(a.sched + kPad, 1);
    if (old == (int)gridDim.x - 1) {  // last CTA out: re-arm the schedule for the next launch
      a.sched[0] = 0;
      a.sched[kPad] = 0;
      for (int i = 0; i < num_phases(a.L); ++i) done[i * kPad] = 0;
      for (int i = 0; i < a.L * a.KV; ++i) a.agrp[(size_t)i * kPad] = 0;
      a.sched[2 * kPad] = s_lay[4] + 1;  // next launch's epoch (tile stamps stay monotonic)
      __threadfence();
    }
  }
}

// Re-arm the split-K state a draft cut left behind (a no-op when the forward was not cut).
// Only the live rows of the int64 accumulators were ever added (k_forward adds rows < rows), so
// only those are cleared; the work is spread over kCleanCtas CTAs and the last one out clears
// the flag and counts the cut (sched layout: [2*kPad] epoch, +1 cut flag, +2 cuts, +3 exit count).
constexpr int kCleanCtas = 16;
__global__ void __launch_bounds__(512) k_cut_cleanup(int* sched, const StepCtl* ctl, unsigned long long* ws,
                                                     size_t ws_blocks, int* tile_cnt, size_t cnt_ints, int* attn_cnt,
                                                     size_t attn_cnt_ints, unsigned long long* best) {
  int* flag = sched + 2 * kPad + 1;
  if (ld_volatile(flag) == 0) return;  // not cut: nothing to re-arm
  const int rows = max(1, min(KMAX, ctl->rows));
  const size_t per_block = (size_t)rows * BM;  // live rows of one [16][128] tile block
  const size_t n = ws_blocks * per_block;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    ws[(i / per_block) * (BN * BM) + i % per_block] = 0ull;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt_ints; i += (size_t)gridDim.x * blockDim.x)
    tile_cnt[i] = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < attn_cnt_ints; i += (size_t)gridDim.x * blockDim.x)
    attn_cnt[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < KMAX) best[threadIdx.x] = 0ull;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sched + 2 * kPad + 3, 1) == (int)gridDim.x - 1) {
      sched[2 * kPad + 3] = 0;
      sched[2 * kPad + 2] += 1;  // cuts so far (amusd_run_info.draft_cuts)
      *flag = 0;
    }
  }
}

cudaError_t launch_cut_cleanup(int* sched, const StepCtl* ctl, float* ws, size_t ws_floats, int* tile_cnt,
                               size_t cnt_ints, int* attn_cnt, size_t attn_cnt_ints, unsigned long long* best,
                               cudaStream_t st) {
  static_assert(BN == KMAX, "accumulator blocks are [KMAX rows][BM]");
  k_cut_cleanup<<<kCleanCtas, 512, 0, st>>>(sched, ctl, (unsigned long long*)ws, ws_floats / 2 / (BN * BM), tile_cnt,
                                            cnt_ints, attn_cnt, attn_cnt_ints, best);
  return cudaGetLastError();
}

// ------------------------------------------------------------ host side
int attn_items_max(int KV, int S) { return KV * KMAX * attn_splits(S); }
int attn_splits(int S) { return (S + kAttnChunk - 1) / kAttnChunk; }
int max_positions() { return kMaxMerge * kAttnChunk; }

static int num_sms_host() { return device_sms(); }

// Units per item: the largest divisor of kb that is <= target and a whole number of ring
// stages (kb is even for every supported shape: tc_shapes_ok).
static int pick_kc(int kb, int target) {
  int best = kUPS;
  for (int k = kUPS; k <= kb; k += kUPS)
    if (kb % k == 0 && k <= std::max(target, kUPS)) best = k;
  return best;
}

// Units (16 KB) per work item of each GEMM kind; AMUSD_FW_UNITS_{QKV,O,GU,DOWN,LM} override.
static int kind_units(const char* name, int dflt) {
  char key[64];
  snprintf(key, sizeof(key), "AMUSD_FW_UNITS_%s", name);
  const char* e = getenv(key);
  return (e && *e) ? atoi(e) : dflt;
}

bool build_kinds(const ModelView& m, int units_per_item, FwArgs* a, size_t* ws_floats, int* cnt_ints, int* max_tiles,
                 int grid) {
  const int ncols = (m.H + 2 * m.KV) * m.hd, hh = m.H * m.hd;
  // Tensor-parallel shard: the unsharded model's chunking (dry run of the full view)
  int kc_full[kNumGemm] = {0, 0, 0, 0, 0}, kb_full[kNumGemm] = {0, 0, 0, 0, 0};
  if (m.tp > 1) {
    ModelView f = m;
    f.tp = 0; f.H = m.H_full; f.KV = m.KV_full; f.ffn = m.ffn_full;
    FwArgs fa{};
    size_t w0;
    int c0, t0;
    build_kinds(f, units_per_item, &fa, &w0, &c0, &t0, 0);
    for (int k = 0; k < kNumGemm; ++k) { kc_full[k] = fa.g[k].kc; kb_full[k] = fa.g[k].kb; }
  }
  bool ok = true;
  int gk_next = 0;  // GEMM kind index of the next kind() call (construction order below)
  const long long b_qkv = (long long)ncols * m.d * 2, b_o = (long long)m.d * hh * 2, b_gu = 2ll * m.ffn * m.d * 2;
  long long ws = 0;  // int64 elements
  int cnt = 0, mt = 0;
  auto kind = [&](int epi, int map, int ntiles, int K, int N, int ldo, const uint8_t* wt, long long stride,
                  const char* name) {
    GemmKind g{};
    g.epi = epi; g.map = map; g.ntiles = ntiles; g.kb = K / BK;
    // QKV / O sit on the latency-bound part of the layer chain: half-size items; the LM head
    // takes whole-K items (no split-K merge before the argmax) -- both measured best
    const bool chain = name[0] == 'Q' || (name[0] == 'O' && name[1] == 0);
    const bool lm = name[0] == 'L';
    int dflt = chain ? std::max(1, units_per_item / 2) : (lm ? 64 : units_per_item);
    // small models (the 1B draft): O with fewer than half an item per SM takes quarter-size
    // items (1B, 148 SMs: 0.872 -> 0.853 ms); on a partial grid (co-located AMUSD draft) both
    // chain kinds do (1B, 64 SMs, with gate/up doubled below: 1.081 -> 0.947 ms)
    if (chain && units_per_item == 16) {
      const int q = std::max(1, units_per_item / 4);
      const bool few = 2 * ntiles * (g.kb / pick_kc(g.kb, dflt)) < num_sms_host();
      if (grid > 0 || (few && name[0] == 'O')) dflt = q;
    }
    if (!chain && !lm && units_per_item == 16) {
      // gate/up and down: the largest of 32 / 16 / 8 units that still gives >= 1.5 items per
      // SM (measured: 8B down 32, 1B down 8, gate/up 32 / 16 within noise)
      const int sms = num_sms_host();
      dflt = 8;
      for (int u : {32, 16})
        if (2 * ntiles * (g.kb / pick_kc(g.kb, u)) >= 3 * sms) { dflt = u; break; }
    }
    const int want = kind_units(name, dflt);
    g.kc = pick_kc(g.kb, want);
    // A forward on a partial grid (co-located AMUSD draft) streams through fewer SMs: items
    // twice as large (fewer grabs and split-K merges) while every CTA still gets one -- measured
    // 1.30 -> 1.23 ms (1B, 64 SMs; 8B on 84 SMs 5.26 -> 5.03 ms, but the verify may not use it:
    // the chunking changes the fp32 partials, and AMUSD must equal AR bit for bit).
    // Env overrides are exact.
    if (grid > 0 && want == dflt && !lm && !chain) {
      const int kc2 = pick_kc(g.kb, 2 * want);
      if (kc2 > g.kc && ntiles * (g.kb / kc2) >= grid) g.kc = kc2;
    }
    const int gk = gk_next++;
    if (m.tp > 1) {  // the unsharded chunking; O / down reduce across the ranks
      g.kc = kc_full[gk];
      if (g.kb % g.kc) ok = false;
      g.xr = gk == kGO || gk == kGDown;
    }
    g.nchunks = g.kb / g.kc;
    g.nitems = ntiles * g.nchunks;
    g.nchunks_total = g.xr ? kb_full[gk] / g.kc : g.nchunks;
    g.N = N; g.ldo = ldo; g.wt = wt; g.wt_stride = stride;
    if (epi != kEpArgmax) mt = std::max(mt, ntiles);
    return g;
  };
  // every kind owns its accumulators / counters (consecutive phases overlap under the
  // fine-grained dependencies).  O and down first: their tile counts (d / 128) are the same on
  // every tensor-parallel rank, so their regions sit at the same offsets in every rank's
  // workspace -- the peers' red.adds target them.
  // Fused gate/up -> down (FwArgs::fuse): small models only -- the 16-column accumulators of
  // every down output tile must fit the 256 spare TMEM columns, and only the hd 64 instances
  // are compiled with it.
  const bool fuse = m.fuse && m.tp <= 1 && m.hd == 64 && (m.H / m.KV == 2 || m.H / m.KV == 4) &&
                    (m.d / BM) % kUPS == 0 && (m.d / BM) * BN <= 256;
  auto place_ws = [&](GemmKind& g) {
    g.ws_off = ws;
    g.cnt_off = cnt;
    if (g.nchunks > 1 || g.xr || (fuse && &g == &a->g[kGDown])) ws += (long long)g.ntiles * BM * BN;
    cnt += g.ntiles * kCounterInts;
  };
  const uint8_t* w0 = m.wt_layer0;
  a->g[kGQkv] = kind(kEpStoreScaled, 0, ncols / BM, m.d, ncols, ncols, w0, m.wt_layer_bytes, "QKV");
  a->g[kGQkv].out = m.qkv;
  a->g[kGQkv].ssp_in = m.ssp;
  a->g[kGO] = kind(kEpResid, 1, m.d / BM, hh, m.d, m.d, w0 + b_qkv, m.wt_layer_bytes, "O");
  a->g[kGO].out = m.h; a->g[kGO].xnext = m.xb; a->g[kGO].ssp_out = m.sspb;  // -> gate/up (double buffer)
  a->g[kGO].gnext = m.norms + m.d;          // mlp RMSNorm of layer l at 2l+1
  a->g[kGO].gnext_stride = 2 * m.d;
  a->g[kGGu] = kind(kEpGateUp, 3, m.ffn / 64, m.d, m.ffn, m.ffn, w0 + b_qkv + b_o, m.wt_layer_bytes, "GU");
  a->g[kGGu].out_b = m.act_b;
  a->g[kGGu].ssp_in = m.sspb;
  a->g[kGDown] = kind(kEpResid, 2, m.d / BM, m.ffn, m.d, m.d, w0 + b_qkv + b_o + b_gu, m.wt_layer_bytes, "DOWN");
  a->g[kGDown].out = m.h; a->g[kGDown].xnext = m.xa; a->g[kGDown].ssp_out = m.ssp;  // -> next QKV / LM head
  a->g[kGDown].gnext = m.norms + 2 * m.d;   // attention RMSNorm of layer l+1 at 2l+2 (final norm at 2L)
  a->g[kGDown].gnext_stride = 2 * m.d;
  a->g[kGLm] = kind(kEpArgmax, 0, m.vocab / BM, m.d, m.vocab, m.vocab, m.wt_lm, 0, "LM");
  a->fuse = fuse;
  if (fuse) {  // down: one weight-less merge item per output tile (gate/up keeps its chunking;
               // its merging chunks carry the down slabs)
    GemmKind& g = a->g[kGDown];
    g.kc = g.kb; g.nchunks = 1; g.nitems = g.ntiles; g.nchunks_total = 1;
  }
  if (m.tp > 1) {
    for (int k : {kGO, kGDown, kGQkv, kGGu, kGLm}) place_ws(a->g[k]);
  } else {  // unsharded: construction order
    for (int k : {kGQkv, kGO, kGGu, kGDown, kGLm}) place_ws(a->g[k]);
  }
  a->g[kGLm].ssp_in = m.ssp;
  a->L = m.L;
  a->attn_max = attn_items_max(m.KV, m.S);
  a->qo_bytes = (size_t)(b_qkv + b_o);
  a->tflag_tiles = mt;
  *ws_floats = (size_t)std::max(ws, 1ll) * 2;
  *cnt_ints = std::max(cnt, 1);
  *max_tiles = mt;
  return ok;
}

template <int HD, int G>
static constexpr int scratch_bytes() {
  return attn_scratch_bytes<HD, G>() + epi_bytes();
}

int forward_smem_bytes(int stages, int hd, int group) {
  int sc = 0;
#define AMUSD_SC(HD_, G_) \
  if (hd == HD_ && group == G_) sc = scratch_bytes<HD_, G_>();
  AMUSD_SC(64, 2) AMUSD_SC(64, 4) AMUSD_SC(64, 8) AMUSD_SC(128, 2) AMUSD_SC(128, 4) AMUSD_SC(128, 8)
#undef AMUSD_SC
  if (!sc) return 0;
  const int ctl = (3 * stages + 2 * kTbuf + 2 * kQ) * 8 + kQ * 8 + 4 + 5 * 4;
  return 1024 + stages * (kStageW + kStageX) + sc + ((ctl + 127) & ~127);
}

template <int HD, int G, int MINB, bool TP, bool FUSE = false>
static cudaError_t launch_m(const FwArgs& a, const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                            const CUtensorMap& m3, int grid, int stages, cudaStream_t st) {
  const int smem = forward_smem_bytes(stages, HD, G);
  static SmemOptIn opt;  // per device (one process may hold models on two GPUs)
  if (cudaError_t e = opt.ensure(k_forward<HD, G, MINB, TP, FUSE>, smem)) return e;
  FwArgs b = a;
  b.stages = stages;
  k_forward<HD, G, MINB, TP, FUSE><<<grid, kThreads, smem, st>>>(m0, m1, m2, m3, b);
  return cudaGetLastError();
}

// Rings small enough for two CTAs per SM (co-located draft + verify forwards)
// take the register-capped instance so that two CTAs fit the register file too.
template <int HD, int G>
static cudaError_t launch_t(const FwArgs& a, const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                            const CUtensorMap& m3, int grid, int stages, cudaStream_t st) {
  if (a.tp > 1) return launch_m<HD, G, 1, true>(a, m0, m1, m2, m3, grid, stages, st);
  if constexpr (HD == 64 && (G == 2 || G == 4)) {
    if (a.fuse) return launch_m<HD, G, 1, false, true>(a, m0, m1, m2, m3, grid, stages, st);  // 512 TMEM columns
  }
  if (forward_smem_bytes(stages, HD, G) <= 232448 / 2 - 1024)
    return launch_m<HD, G, 2, false>(a, m0, m1, m2, m3, grid, stages, st);
  return launch_m<HD, G, 1, false>(a, m0, m1, m2, m3, grid, stages, st);
}

cudaError_t launch_forward(const FwArgs& a, const CUtensorMap& m_xa, const CUtensorMap& m_attn,
                           const CUtensorMap& m_act, const CUtensorMap& m_xb, int grid, int stages, cudaStream_t st) {
  const int G = a.H / a.KV;
#define AMUSD_FW(HD_, G_) \
  if (a.hd == HD_ && G == G_) return launch_t<HD_, G_>(a, m_xa, m_attn, m_act, m_xb, grid, stages, st);
  AMUSD_FW(64, 2) AMUSD_FW(64, 4) AMUSD_FW(64, 8) AMUSD_FW(128, 2) AMUSD_FW(128, 4) AMUSD_FW(128, 8)
#undef AMUSD_FW
  return cudaErrorInvalidValue;
}

}  // namespace fw
}  // namespace amusd
