// decode_cl.cu -- cluster decode forward (see decode_cl.h): two grid-wide dependencies per
// layer.  The draft model's next_token + advance (reference plug-in models.py:120-131).
//
// GEMV tiles: 16 weight rows x 512 K units (16-byte chunks XOR-swizzled by row, ldmatrix
// conflict-free) through mma.sync m16n8k16 with the <= 8 live activation rows as N; the down
// projection as 16 x 16 tiles of W_down^T per 16-feature block.  A producer warp streams the
// CTA's static unit schedule through a shared-memory ring and never waits on a dependency.
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "decode_cl.h"
#include "tc_ptx.cuh"

namespace amusd {
namespace cl {

using bf16 = __nv_bfloat16;
using tc::bulk_load;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::named_bar;
using tc::policy_evict_first;
using tc::smem_u32;

constexpr int kCW = 8;                   // consumer warps
constexpr int kCT = kCW * 32;
constexpr int kThreads = kCT + 32;       // + producer warp
constexpr int kMB = 16;                  // rows per block (MMA M)
constexpr int kKW = 512;                 // K per unit
constexpr int kStage = kMB * kKW * 2;    // 16 KB
constexpr int kTiles = kStage / 512;     // down^T 16 x 16 tiles per unit (32)
constexpr int kChunk = 64;               // attention positions per staged sub-chunk
constexpr int kPad = 32;
constexpr int kMaxStages = 16;
constexpr int kMaxG = 8;
constexpr int kMaxD = 2048;              // down accumulators in registers: d / 16 / 8 warps <= 16 tiles
constexpr int kSmemBudget = 232448 - 2048;
constexpr long long kWaitNs = 4ll * 1000 * 1000 * 1000;
constexpr float kFix = 4294967296.0f;    // int64 fixed point 2^32

constexpr int kSyncBar = 0, kSyncExit = kPad, kSyncLm = 2 * kPad, kSyncCut = 3 * kPad;

enum { kQkv = 0, kO = 1, kGu = 2, kDn = 3, kLm = 4 };

struct alignas(16) Aux {
  unsigned long long full[kMaxStages];
  unsigned long long empty[kMaxStages];
  int rel[kMaxStages];          // release weight per slot (8 per full consumption)
  float scale[kMaxRows];
  unsigned long long key[kMaxRows];
  float part[kCW][32][4];       // K-split MMA partials
  float ml[kMaxRows][kMaxG][2]; // attention running max / sum per (row, head)
  float fsc[kMaxRows * kMaxG];  // online-softmax rescale of the running o per (row, head)
  unsigned long long clbar;     // cluster hand-off barrier: one arrival per cluster CTA per use
  int cut, go, consumed, issued;
};

// shared-memory layout after the ring (offsets in bytes, host + device)
struct Smem {
  int xs, osb, qkvs, parts, acts, gus, att, aux, total;
};
__host__ __device__ inline int al128(int v) { return (v + 127) / 128 * 128; }
__host__ __device__ inline int xs_pitch(int K) { return K * 2 + 16; }
__host__ __device__ inline Smem smem_layout(int stages, int d, int H, int KV, int hd) {
  const int G = H / KV, NG = (G + 2) * hd;
  Smem s;
  int o = stages * kStage;
  s.xs = o;   o += al128(kMaxRows * xs_pitch(d));                 // x rows (QKV, GU, LM input)
  s.osb = o;  o += al128(kMaxRows * xs_pitch(G * hd));            // merged attention output (O input)
  s.qkvs = o; o += al128(((NG / kMB + kCluster - 1) / kCluster) * kMB * kMaxRows * 4);  // this CTA's QKV rows
  s.parts = o; o += al128(kMaxRows * G * (hd + 2) * 4);           // attention partial (peers read it)
  s.acts = o; o += al128(8 * kMB * kMaxRows * 2);                  // act per owned feature block (<= 8)
  s.gus = o;  o += al128(16 * kMB * kMaxRows * 4);                 // gate/up row-block results (<= 16)
  s.att = o;  o += al128(kMaxRows * G * hd * 4 + 2 * kMaxRows * hd * 2 + 2 * kChunk * (hd + 8) * 2 +
                         kMaxRows * G * kChunk * 4 + kMaxRows * G * hd * 4);  // q, k/v new, staged K/V, scores, o
  s.aux = o;  o += al128((int)sizeof(Aux));
  s.total = o;
  return s;
}

// ------------------------------------------------------------------ PTX helpers
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
AMUSD_DEV void mbar_arrive_n(uint32_t a, int n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(n) : "memory");
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
AMUSD_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
AMUSD_DEV void cp_async_wait_all() { asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory"); }
AMUSD_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
AMUSD_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared address of the same variable in cluster CTA `rank`
AMUSD_DEV uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
AMUSD_DEV float ld_dsmem(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
// Cluster hand-off among the CONSUMER warps (the producer warp keeps streaming, so the hardware
// cluster barrier, which counts every thread, cannot be used): after the consumers' CTA barrier,
// thread 0 releases at cluster scope and arrives on every peer's barrier; then it waits for the
// use's 8 arrivals on its own barrier (acquire), and the CTA barrier passes the result on.
AMUSD_DEV void cluster_handoff(unsigned long long* bar, int use, int ct) {
  named_bar(1, kCT);
  if (ct == 0) {
    const uint32_t b = smem_u32(bar);
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
#pragma unroll
    for (int c = 0; c < kCluster; ++c)
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(b, c)) : "memory");
    const uint32_t par = use & 1;
    const long long t0 = globaltimer();
    for (int it = 0;; ++it) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(b), "r"(par)
          : "memory");
      if (ok) break;
      if ((it & 63) == 63 && globaltimer() - t0 > kWaitNs) __trap();
    }
  }
  named_bar(1, kCT);
}
AMUSD_DEV void red_add_u64(unsigned long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
AMUSD_DEV float fix2f(unsigned long long v) { return __ll2float_rn((long long)v) * (1.0f / kFix); }

// ------------------------------------------------------------------ schedule
AMUSD_DEV int part(int n, int i, int parts) { return (int)((long long)n * i / parts); }
AMUSD_DEV int unit_kw(int K, int q) { return min(kKW, K - q * kKW); }
AMUSD_DEV int nunits(int K) { return (K + kKW - 1) / kKW; }
// byte offset of unit q inside a 16-row block of width K
AMUSD_DEV size_t unit_off(int K, int q) { return (size_t)q * kMB * kKW * 2; }

struct Dims {
  int G, NG, nbq, nbo, nfb, ndt, ndn, nbl, nkd, nko;
};
AMUSD_DEV Dims dims_of(const ClArgs& a) {
  Dims m;
  m.G = a.H / a.KV; m.NG = (m.G + 2) * a.hd; m.nbq = m.NG / kMB; m.nbo = a.d / kMB; m.nfb = a.ffn / kMB;
  m.ndt = a.d / kMB; m.ndn = (m.ndt + kTiles - 1) / kTiles; m.nbl = a.vocab / kMB;
  m.nkd = nunits(a.d); m.nko = nunits(m.G * a.hd);
  return m;
}
// This CTA's ranges.
struct Ranges {
  bool grp;               // this cluster owns a KV group (phase A)
  int g, crank;
  int qb0, qb1, ob0, ob1; // QKV / O blocks of the group (cluster-local partition)
  int fb0, fb1;           // feature blocks (grid partition)
  int lb0, lb1;           // LM blocks
  int own0, own1;         // residual rows this CTA owns (grid partition of d, for h / acc upkeep)
};
AMUSD_DEV Ranges ranges_of(const ClArgs& a, const Dims& m) {
  Ranges r;
  const int cid = blockIdx.x / kCluster;
  r.crank = (int)cluster_rank();
  r.grp = cid < a.KV;
  r.g = cid;
  r.qb0 = part(m.nbq, r.crank, kCluster); r.qb1 = part(m.nbq, r.crank + 1, kCluster);
  r.ob0 = part(m.nbo, r.crank, kCluster); r.ob1 = part(m.nbo, r.crank + 1, kCluster);
  const int G = gridDim.x, b = blockIdx.x;
  r.fb0 = part(m.nfb, b, G); r.fb1 = part(m.nfb, b + 1, G);
  r.lb0 = part(m.nbl, b, G); r.lb1 = part(m.nbl, b + 1, G);
  r.own0 = part(a.d, b, G); r.own1 = part(a.d, b + 1, G);
  return r;
}
AMUSD_DEV const uint8_t* qkv_block(const ClArgs& a, const Dims& m, int l, int g, int j) {
  return a.wt + (size_t)l * a.layer_bytes + ((size_t)g * m.nbq + j) * kMB * a.d * 2;
}
AMUSD_DEV const uint8_t* o_block(const ClArgs& a, const Dims& m, int l, int g, int b) {
  return a.wt + (size_t)l * a.layer_bytes + a.off_o + ((size_t)g * m.nbo + b) * kMB * m.G * a.hd * 2;
}
AMUSD_DEV const uint8_t* gu_block(const ClArgs& a, int l, int fb, int half) {
  return a.wt + (size_t)l * a.layer_bytes + a.off_gu + ((size_t)fb * 2 + half) * kMB * a.d * 2;
}
AMUSD_DEV const uint8_t* dn_unit(const ClArgs& a, const Dims& m, int l, int fb, int u) {
  return a.wt + (size_t)l * a.layer_bytes + a.off_dn + (size_t)fb * m.ndt * 512 + (size_t)u * kStage;
}
AMUSD_DEV int dn_bytes(const Dims& m, int u) { return min(kTiles, m.ndt - u * kTiles) * 512; }
AMUSD_DEV const uint8_t* lm_block(const ClArgs& a, int b) { return a.wt_lm + (size_t)b * kMB * a.d * 2; }

// ------------------------------------------------------------------ producer
AMUSD_DEV bool produce(const ClArgs& a, Aux* ax, uint8_t* ring, int& i, const uint8_t* src, int bytes, uint64_t pol) {
  volatile int* cut = &ax->cut;
  const int slot = i % a.stages;
  if (i >= a.stages) {
    const uint32_t bar = smem_u32(&ax->empty[slot]), par = ((i / a.stages) - 1) & 1;
    const long long t0 = globaltimer();
    while (!mbar_try(bar, par)) {
      if (*cut) return false;
      if (globaltimer() - t0 > kWaitNs) __trap();
    }
  }
  if (*cut) return false;
  const uint32_t full = smem_u32(&ax->full[slot]);
  mbar_expect_tx(full, bytes);
  bulk_load(smem_u32(ring + (size_t)slot * kStage), src, bytes, full, pol);
  ++i;
  return true;
}
AMUSD_DEV void producer(const ClArgs& a, Aux* ax, uint8_t* ring) {
  const uint64_t pol = policy_evict_first();
  const Dims m = dims_of(a);
  const Ranges rg = ranges_of(a, m);
  int i = 0;
#define PROD(src, bytes) \
  if (!produce(a, ax, ring, i, (src), (bytes), pol)) { ax->issued = i; return; }
  for (int l = 0; l < a.L; ++l) {
    if (rg.grp) {
      for (int j = rg.qb0; j < rg.qb1; ++j)
        for (int q = 0; q < m.nkd; ++q) PROD(qkv_block(a, m, l, rg.g, j) + unit_off(a.d, q), kMB * unit_kw(a.d, q) * 2)
      for (int b = rg.ob0; b < rg.ob1; ++b)
        for (int q = 0; q < m.nko; ++q)
          PROD(o_block(a, m, l, rg.g, b) + unit_off(m.G * a.hd, q), kMB * unit_kw(m.G * a.hd, q) * 2)
    }
    for (int fb = rg.fb0; fb < rg.fb1; ++fb)
      for (int half = 0; half < 2; ++half)
        for (int q = 0; q < m.nkd; ++q) PROD(gu_block(a, l, fb, half) + unit_off(a.d, q), kMB * unit_kw(a.d, q) * 2)
    for (int fb = rg.fb0; fb < rg.fb1; ++fb)
      for (int u = 0; u < m.ndn; ++u) PROD(dn_unit(a, m, l, fb, u), dn_bytes(m, u))
  }
  for (int b = rg.lb0; b < rg.lb1; ++b)
    for (int q = 0; q < m.nkd; ++q) PROD(lm_block(a, b) + unit_off(a.d, q), kMB * unit_kw(a.d, q) * 2)
#undef PROD
  ax->issued = i;
}

// ------------------------------------------------------------------ consumers
struct Cons {
  int ct, warp, lane, R, pos0;
  int stage, bar, clu;
};

AMUSD_DEV void unit_wait(const ClArgs& a, Aux* ax, int i) {
  const int slot = i % a.stages;
  const volatile int* rel = &ax->rel[slot];
  if (*rel < kCW * (i / a.stages)) {  // the slot's previous use fully released: the parity wait is unambiguous
    const long long t0 = globaltimer();
    for (int it = 1; *rel < kCW * (i / a.stages); ++it) {
      __nanosleep(64);
      if ((it & 255) == 0 && globaltimer() - t0 > kWaitNs) __trap();
    }
  }
  mbar_wait_b(smem_u32(&ax->full[slot]), (i / a.stages) & 1);
}
// release weight w (kCW = the whole consumption by one warp; 1 = one of kCW warps)
AMUSD_DEV void unit_release(const ClArgs& a, Aux* ax, int i, int w, int lane) {
  __syncwarp();
  if (lane == 0) {
    const int slot = i % a.stages;
    atomicAdd(&ax->rel[slot], w);
    mbar_arrive_n(smem_u32(&ax->empty[slot]), w);
  }
}

AMUSD_DEV bool grid_wait(const ClArgs& a, Aux* ax, Cons& cs) {
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
  }
  named_bar(1, kCT);
  return ax->go != 0;
}
AMUSD_DEV void grid_arrive(const ClArgs& a, const Cons& cs) {
  named_bar(1, kCT);
  if (cs.ct == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.sync + kSyncBar) : "memory");
}

// MMA over one 16-row block's units q0, q0 + qstep, ... (B = activation rows in shared memory at
// xb, pitch bytes per row, nx live rows).  c: (rows g, g + 8) x (activation rows 2q, 2q + 1).
AMUSD_DEV void block_mma(const ClArgs& a, Aux* ax, uint32_t ring_s, uint32_t xb, int pitch, int K, int nk, int i0,
                         int q0, int qstep, int nx, float (&c)[4], int lane) {
  const int g = lane >> 2, q = lane & 3;
  const int mrow = (lane & 7) + 8 * ((lane >> 3) & 1), mchunk = lane >> 4, msw = mrow & 7;
  const bool bx = g < nx;
  const uint32_t xrow = xb + (uint32_t)(g * pitch + q * 4);
  float acc[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  for (int u = q0; u < nk; u += qstep) {
    const int i = i0 + u, slot = i % a.stages, kw = unit_kw(K, u);
    unit_wait(a, ax, i);
    const uint32_t st = ring_s + slot * kStage + (uint32_t)(mrow * kw * 2);
    const uint32_t xk = xrow + (uint32_t)(u * kKW * 2);
    for (int kb = 0; kb < kw / 16; kb += 4) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(st + (uint32_t)(((2 * (kb + t) + mchunk) ^ msw) * 16), a0, a1, a2, a3);
        const uint32_t b0 = bx ? lds32(xk + (kb + t) * 32) : 0u;
        const uint32_t b1 = bx ? lds32(xk + (kb + t) * 32 + 16) : 0u;
        mma_bf16(acc[t], a0, a1, a2, a3, b0, b1);
      }
    }
    unit_release(a, ax, i, kCW, lane);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) c[e] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
}

// Blocks [b0, b1) of width K, nk units each (starting at stage cs.stage), spread over the warps
// (K-split S for few blocks); epi(b, c) runs on the finishing warp with the full sums.
template <class Epi>
AMUSD_DEV void gemv_blocks(const ClArgs& a, Aux* ax, uint32_t ring_s, uint32_t xb, int pitch, int K, int nb, int nk,
                           int nx, Cons& cs, Epi epi) {
  int S = 1;
  if (nb > 0 && nb < kCW) {
    int p2 = 1;
    while (p2 < nb) p2 <<= 1;
    S = min(nk, kCW / p2);
  }
  const int groups = kCW / S, js = cs.warp / S, qs = cs.warp % S;
  for (int j = js; j < nb; j += groups) {
    float c[4];
    block_mma(a, ax, ring_s, xb, pitch, K, nk, cs.stage + j * nk, qs, S, nx, c, cs.lane);
    if (S == 1) {
      epi(j, c);
    } else {
      float* pp = &ax->part[cs.warp][cs.lane][0];
      pp[0] = c[0]; pp[1] = c[1]; pp[2] = c[2]; pp[3] = c[3];
      named_bar(2, kCT);
      if (qs == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = ax->part[js * S][cs.lane][e];
          for (int t = 1; t < S; ++t) v += ax->part[js * S + t][cs.lane][e];
          c[e] = v;
        }
        epi(j, c);
      }
    }
  }
  if (S > 1 && js >= nb) named_bar(2, kCT);
  cs.stage += nb * nk;
  named_bar(1, kCT);
}

// Residual rows of every activation row at a phase entry, rebuilt from the layer-entry residual
// and the integer accumulators in fixed order (every CTA gets bit-identical values):
//   stage 0: h = h_in (+ O)      stage 1: h = h_in + O + down
// Writes x = bf16(h * gamma) rows into xs (pitch(d)) and the RMSNorm factors; owners store h
// (the next layer's h_in) when `store` is set.
AMUSD_DEV void build_x(const ClArgs& a, Aux* ax, uint8_t* xs, const float* hin, const unsigned long long* ao,
                       const unsigned long long* ad, const bf16* gamma, float* hout, int own0, int own1,
                       const Cons& cs) {
  const int d = a.d, R = cs.R;
  float* red = &ax->part[0][0][0];  // [kCW][kMaxRows] partial sums of squares (reuses the MMA partials)
  float ss[kMaxRows];
#pragma unroll
  for (int r = 0; r < kMaxRows; ++r) ss[r] = 0.f;
  for (int k = cs.ct * 8; k < d; k += kCT * 8) {
    float gm[8];
    {
      const uint4 gu = __ldg((const uint4*)(gamma + k));
      const __nv_bfloat162* g2 = (const __nv_bfloat162*)&gu;
#pragma unroll
      for (int j = 0; j < 4; ++j) { const float2 f = __bfloat1622float2(g2[j]); gm[2 * j] = f.x; gm[2 * j + 1] = f.y; }
    }
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r) {
      if (r >= R) continue;
      const size_t o = (size_t)r * d + k;
      // every load of the row issued before any use (one round trip; no aliasing with the stores)
      float h[8];
      if (hin) {
        const float4 h0 = __ldcg((const float4*)(hin + o)), h1 = __ldcg((const float4*)(hin + o) + 1);
        h[0] = h0.x; h[1] = h0.y; h[2] = h0.z; h[3] = h0.w; h[4] = h1.x; h[5] = h1.y; h[6] = h1.z; h[7] = h1.w;
      } else {
        const uint4 e = __ldg((const uint4*)(a.embed + (size_t)a.ctl->tok[r] * d + k));
        const __nv_bfloat162* e2 = (const __nv_bfloat162*)&e;
#pragma unroll
        for (int j = 0; j < 4; ++j) { const float2 f = __bfloat1622float2(e2[j]); h[2 * j] = f.x; h[2 * j + 1] = f.y; }
      }
      ulonglong2 va[4], vd[4];
      if (ao) {
#pragma unroll
        for (int j = 0; j < 4; ++j) va[j] = __ldcg((const ulonglong2*)(ao + o) + j);
      }
      if (ad) {
#pragma unroll
        for (int j = 0; j < 4; ++j) vd[j] = __ldcg((const ulonglong2*)(ad + o) + j);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v = h[j];
        if (ao) v += fix2f((j & 1) ? va[j >> 1].y : va[j >> 1].x);
        if (ad) v += fix2f((j & 1) ? vd[j >> 1].y : vd[j >> 1].x);
        h[j] = v;
        ss[r] = fmaf(v, v, ss[r]);
      }
      if (hout && k >= own0 && k + 8 <= own1) {
        *(float4*)(hout + o) = make_float4(h[0], h[1], h[2], h[3]);
        *((float4*)(hout + o) + 1) = make_float4(h[4], h[5], h[6], h[7]);
      } else if (hout) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (k + j >= own0 && k + j < own1) hout[o + j] = h[j];
      }
      __nv_bfloat162 b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(h[2 * j] * gm[2 * j], h[2 * j + 1] * gm[2 * j + 1]);
      *(uint4*)(xs + (size_t)r * xs_pitch(d) + k * 2) = *(const uint4*)b;
    }
  }
#pragma unroll
  for (int r = 0; r < kMaxRows; ++r) {
    if (r >= R) continue;
    const float s = warp_sum(ss[r]);
    if (cs.lane == 0) red[cs.warp * kMaxRows + r] = s;
  }
  named_bar(1, kCT);
  if (cs.ct < R) {
    float s = 0.f;
    for (int w = 0; w < kCW; ++w) s += red[w * kMaxRows + cs.ct];
    ax->scale[cs.ct] = 1.0f / sqrtf(s / (float)d + a.eps);
  }
  named_bar(1, kCT);
}

// ------------------------------------------------------------------ phase A: attention of the group
template <int HD>
AMUSD_DEV void attention(const ClArgs& a, Aux* ax, const Dims& m, const Ranges& rg, uint8_t* sm, const Smem& L,
                         int layer, const Cons& cs) {
  const int G = m.G, half = HD / 2, R = cs.R, ct = cs.ct, crank = rg.crank, g = rg.g;
  float* qg = (float*)(sm + L.att);                              // [R][G][HD] roped queries
  bf16* kn = (bf16*)(qg + kMaxRows * G * HD);                    // [R][HD] this step's K (roped, bf16)
  bf16* vn = kn + kMaxRows * HD;                                 // [R][HD]
  bf16* kst = vn + kMaxRows * HD;                                // [kChunk][HD + 8] staged cached K
  bf16* vst = kst + kChunk * (HD + 8);
  float* sc = (float*)(vst + kChunk * (HD + 8));                 // [R][G][kChunk]
  float* oacc = sc + kMaxRows * G * kChunk;                      // [R][G][HD]
  float* parts = (float*)(sm + L.parts);                         // [R][G][HD + 2] -> peers
  const uint32_t qkvs_s = smem_u32(sm + L.qkvs);
  // 1) gather the group's q / k / v rows from the cluster's CTAs (DSMEM), RoPE, bf16 K/V
  for (int i = ct; i < R * (G + 1) * half; i += kCT) {
    const int r = i / ((G + 1) * half), rem = i % ((G + 1) * half), jh = rem / half, e = rem % half;
    // row of the group's [q (G heads) | k] block rows: head jh, dims e and e + half
    float x[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int row = jh * HD + e + w * half, blk = row / kMB;
      int owner = 0;
      while (part(m.nbq, owner + 1, kCluster) <= blk) ++owner;
      const int lrow = (blk - part(m.nbq, owner, kCluster)) * kMB + row % kMB;
      x[w] = ld_dsmem(mapa(qkvs_s + (uint32_t)((lrow * kMaxRows + r) * 4), owner));
    }
    const int p = cs.pos0 + r;
    const float c = a.cos[(size_t)p * half + e], s = a.sin[(size_t)p * half + e];
    const float r0 = x[0] * c - x[1] * s, r1 = x[1] * c + x[0] * s;
    if (jh < G) {
      qg[(r * G + jh) * HD + e] = r0;
      qg[(r * G + jh) * HD + e + half] = r1;
    } else {
      kn[r * HD + e] = __float2bfloat16(r0);
      kn[r * HD + e + half] = __float2bfloat16(r1);
    }
  }
  for (int i = ct; i < R * HD; i += kCT) {  // V rows
    const int r = i / HD, e = i % HD, row = (G + 1) * HD + e, blk = row / kMB;
    int owner = 0;
    while (part(m.nbq, owner + 1, kCluster) <= blk) ++owner;
    const int lrow = (blk - part(m.nbq, owner, kCluster)) * kMB + row % kMB;
    vn[r * HD + e] = __float2bfloat16(ld_dsmem(mapa(qkvs_s + (uint32_t)((lrow * kMaxRows + r) * 4), owner)));
  }
  named_bar(1, kCT);
  bf16* kl = (bf16*)(a.kcache + (size_t)layer * a.kv_layer_bytes) + (size_t)g * a.S * HD;
  bf16* vl = (bf16*)(a.vcache + (size_t)layer * a.kv_layer_bytes) + (size_t)g * a.S * HD;
  if (crank == 0) {  // KV append (pending-token scheme): this step's rows at positions pos0 + r
    for (int i = ct; i < R * HD; i += kCT) {
      const int r = i / HD, e = i % HD;
      kl[(size_t)(cs.pos0 + r) * HD + e] = kn[r * HD + e];
      vl[(size_t)(cs.pos0 + r) * HD + e] = vn[r * HD + e];
    }
  }
  // 2) this CTA's positions [p0, p1): cached ones staged in sub-chunks, this step's from kn / vn;
  //    online softmax per (row, head)
  // positions in 64-position chunks dealt round-robin to the cluster's CTAs: a position's
  // chunk, its CTA and the summation order depend on the position only (batch invariance)
  const int P = cs.pos0 + R;
  for (int i = ct; i < R * G; i += kCT) { ax->ml[i / G][i % G][0] = -INFINITY; ax->ml[i / G][i % G][1] = 0.f; }
  for (int i = ct; i < R * G * HD; i += kCT) oacc[i] = 0.f;
  named_bar(1, kCT);
  for (int c0 = crank * kChunk; c0 < P; c0 += kCluster * kChunk) {
    const int c1 = min(P, c0 + kChunk), cc = min(c1, cs.pos0);  // cached part [c0, cc)
    for (int i = ct; i < (cc - c0) * (HD / 8) * 2; i += kCT) {
      const int which = i >= (cc - c0) * (HD / 8), ii = which ? i - (cc - c0) * (HD / 8) : i;
      const int t = ii / (HD / 8), ch = ii % (HD / 8);
      cp_async16(smem_u32((which ? vst : kst) + t * (HD + 8) + ch * 8), (which ? vl : kl) + (size_t)(c0 + t) * HD + ch * 8);
    }
    cp_async_wait_all();
    for (int i = ct; i < (c1 - max(c0, cs.pos0)) * HD; i += kCT) {  // this step's rows into the chunk
      const int t = max(c0, cs.pos0) + i / HD - c0, e = i % HD;
      kst[t * (HD + 8) + e] = kn[(c0 + t - cs.pos0) * HD + e];
      vst[t * (HD + 8) + e] = vn[(c0 + t - cs.pos0) * HD + e];
    }
    named_bar(1, kCT);
    // scores: thread = (position, head); rows in a loop
    for (int pr = ct; pr < kChunk * G; pr += kCT) {
      const int ti = pr / G, jh = pr % G, t = c0 + ti;
      for (int r = 0; r < R; ++r) {
        float dot = -INFINITY;
        if (t < c1 && t <= cs.pos0 + r) {
          const bf16* kr = kst + ti * (HD + 8);
          const float* qr = qg + (r * G + jh) * HD;
          float s = 0.f;
#pragma unroll 8
          for (int e = 0; e < HD; e += 2) {
            const float2 kf = __bfloat1622float2(*(const __nv_bfloat162*)(kr + e));
            s = fmaf(qr[e], kf.x, s);
            s = fmaf(qr[e + 1], kf.y, s);
          }
          dot = s * a.scale;
        }
        sc[(r * G + jh) * kChunk + ti] = dot;
      }
    }
    named_bar(1, kCT);
    // online softmax update per (row, head): one warp per pair
    for (int pr = cs.warp; pr < R * G; pr += kCW) {
      float* row = sc + pr * kChunk;
      float x0 = row[cs.lane], x1 = row[cs.lane + 32];
      float mc = warp_max(fmaxf(x0, x1));
      const float mo = ax->ml[pr / G][pr % G][0], mn = fmaxf(mo, mc);
      const float e0 = mn == -INFINITY ? 0.f : expf(x0 - mn), e1 = mn == -INFINITY ? 0.f : expf(x1 - mn);
      row[cs.lane] = e0;
      row[cs.lane + 32] = e1;
      const float ls = warp_sum(e0 + e1);
      __syncwarp();
      if (cs.lane == 0) {
        const float f = mo == -INFINITY ? 0.f : expf(mo - mn);
        ax->ml[pr / G][pr % G][0] = mn;
        ax->ml[pr / G][pr % G][1] = ax->ml[pr / G][pr % G][1] * f + ls;
        ax->fsc[pr] = f;
      }
    }
    named_bar(1, kCT);
    // P.V with the running rescale: thread = (head, dim), rows in a loop
    for (int i = ct; i < G * HD; i += kCT) {
      const int jh = i / HD, e = i % HD;
      for (int r = 0; r < R; ++r) {
        const int pr = r * G + jh;
        float o = oacc[pr * HD + e] * ax->fsc[pr];
        const float* pp = sc + pr * kChunk;
        for (int t = 0; t < c1 - c0; ++t) o = fmaf(pp[t], __bfloat162float(vst[t * (HD + 8) + e]), o);
        oacc[pr * HD + e] = o;
      }
    }
    named_bar(1, kCT);
  }
  for (int i = ct; i < R * G * (HD + 2); i += kCT) {  // partial (m, l, o) for the peers
    const int pr = i / (HD + 2), e = i % (HD + 2);
    parts[i] = e == 0 ? ax->ml[pr / G][pr % G][0] : e == 1 ? ax->ml[pr / G][pr % G][1] : oacc[pr * HD + e - 2];
  }
}

// Every CTA merges the 8 partials of its cluster (split order) into the O input (bf16).
template <int HD>
AMUSD_DEV void merge(const ClArgs& a, const Dims& m, uint8_t* sm, const Smem& L, const Cons& cs) {
  const int G = m.G, R = cs.R;
  const uint32_t parts_s = smem_u32(sm + L.parts);
  bf16* osb = (bf16*)(sm + L.osb);
  for (int i = cs.ct; i < R * G * HD; i += kCT) {
    const int pr = i / HD, e = i % HD, r = pr / G, jh = pr % G;
    const uint32_t off = (uint32_t)(pr * (HD + 2) * 4);
    float mc[kCluster], lc[kCluster], oc[kCluster];
#pragma unroll
    for (int c = 0; c < kCluster; ++c) {
      const uint32_t base = mapa(parts_s + off, c);
      mc[c] = ld_dsmem(base);
      lc[c] = ld_dsmem(base + 4);
      oc[c] = ld_dsmem(base + 8 + e * 4);
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < kCluster; ++c) M = fmaxf(M, mc[c]);
    float Ls = 0.f, O = 0.f;
#pragma unroll
    for (int c = 0; c < kCluster; ++c) {
      const float w = mc[c] == -INFINITY ? 0.f : expf(mc[c] - M);
      Ls = fmaf(w, lc[c], Ls);
      O = fmaf(w, oc[c], O);
    }
    osb[(size_t)r * (xs_pitch(G * HD) / 2) + jh * HD + e] = __float2bfloat16(O / Ls);
  }
  named_bar(1, kCT);
}

// ------------------------------------------------------------------ the kernel
template <int HD>
__global__ void __launch_bounds__(kThreads, 1) k_decode_cl(const __grid_constant__ ClArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  StepCtl* ctl = a.ctl;
  if (!ctl->active) return;
  if (ctl->rows > kMaxRows) __trap();  // host-driven forwards are chunked to kMaxRows rows
  const Smem L = smem_layout(a.stages, a.d, a.H, a.KV, a.hd);
  uint8_t* ring = smem;
  Aux* ax = (Aux*)(smem + L.aux);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(smem_u32(&ax->full[i]), 1);
      mbar_init(smem_u32(&ax->empty[i]), kCW);
      ax->rel[i] = 0;
    }
    mbar_init(smem_u32(&ax->clbar), kCluster);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ax->cut = 0; ax->consumed = 0; ax->issued = 0;
  }
  if (tid < kMaxRows) ax->key[tid] = 0ull;
  __syncthreads();
  cluster_sync();  // every peer's barriers initialised before any DSMEM traffic
  if (warp == kCW) {
    if ((tid & 31) == 0) producer(a, ax, ring);
    __syncwarp();
  } else {
    const Dims m = dims_of(a);
    const Ranges rg = ranges_of(a, m);
    Cons cs;
    cs.ct = tid; cs.warp = warp; cs.lane = tid & 31;
    cs.R = min(max(ctl->rows, 1), kMaxRows); cs.pos0 = ctl->pos0;
    cs.stage = 0; cs.bar = 0; cs.clu = 0;
    const uint32_t ring_s = smem_u32(ring);
    uint8_t* xs = smem + L.xs;
    const uint32_t xs_s = smem_u32(xs), osb_s = smem_u32(smem + L.osb);
    const int d = a.d, R = cs.R;
    const size_t dkr = (size_t)kMaxRows * d;  // one [kMaxRows][d] plane
    float* qkvs = (float*)(smem + L.qkvs);
    float* gus = (float*)(smem + L.gus);
    bf16* acts = (bf16*)(smem + L.acts);
    bool ok = true;
    long long* dbg = (a.dbg && cs.ct == 0) ? a.dbg + (size_t)blockIdx.x * kDbgPerLayer * a.L : nullptr;
#define MARK(k) \
  if (dbg) dbg[l * kDbgPerLayer + (k)] = globaltimer();
    for (int l = 0; l < a.L && ok; ++l) {
      const int par = l & 1, pp = par ^ 1;
      unsigned long long* ao = a.acc + (size_t)(0 * 2 + par) * dkr;   // O accumulator of this layer
      unsigned long long* ad = a.acc + (size_t)(1 * 2 + par) * dkr;   // down accumulator of this layer
      const unsigned long long* aop = a.acc + (size_t)(0 * 2 + pp) * dkr;
      const unsigned long long* adp = a.acc + (size_t)(1 * 2 + pp) * dkr;
      // ---- phase A entry: h_in(l) (from h_in(l-1) + O + down of layer l-1), x for QKV
      if (l > 0 && !(ok = grid_wait(a, ax, cs))) break;
      MARK(0)
      build_x(a, ax, xs, l > 0 ? a.h + (size_t)pp * dkr : nullptr, l > 0 ? aop : nullptr, l > 0 ? adp : nullptr,
              a.norms + (size_t)(2 * l) * d, a.h + (size_t)par * dkr, rg.own0, rg.own1, cs);
      MARK(1)
      if (rg.grp) {
        // QKV rows of the group -> this CTA's qkv rows (scaled by the RMSNorm factor)
        gemv_blocks(a, ax, ring_s, xs_s, xs_pitch(d), d, rg.qb1 - rg.qb0, m.nkd, R, cs, [&](int j, const float(&c)[4]) {
          const int g8 = cs.lane >> 2, q = cs.lane & 3;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int row = j * kMB + g8 + 8 * (e >> 1), r = 2 * q + (e & 1);
            if (r < R) qkvs[row * kMaxRows + r] = c[e] * ax->scale[r];
          }
        });
        MARK(2)
        cluster_handoff(&ax->clbar, cs.clu++, cs.ct);   // every CTA's QKV rows ready
        MARK(3)
        attention<HD>(a, ax, m, rg, smem, L, l, cs);
        MARK(4)
        cluster_handoff(&ax->clbar, cs.clu++, cs.ct);   // every CTA's attention partial ready
        merge<HD>(a, m, smem, L, cs);
        MARK(5)
        // O slice of the group: red.add into the layer's O accumulator
        gemv_blocks(a, ax, ring_s, osb_s, xs_pitch(m.G * HD), m.G * HD, rg.ob1 - rg.ob0, m.nko, R, cs,
                    [&](int j, const float(&c)[4]) {
          const int g8 = cs.lane >> 2, q = cs.lane & 3, b = rg.ob0 + j;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = b * kMB + g8 + 8 * (e >> 1), r = 2 * q + (e & 1);
            if (r < R) red_add_u64(ao + (size_t)r * d + n, (long long)__float2ll_rn(c[e] * kFix));
          }
        });
      }
      MARK(6)
      grid_arrive(a, cs);
      // ---- phase B: gate/up -> SiLU*up -> down (K = the CTA's features)
      if (!(ok = grid_wait(a, ax, cs))) break;
      MARK(7)
      // re-arm the previous layer's accumulators (every CTA has rebuilt h_in(l) from them)
      for (int i = rg.own0 + cs.ct; i < rg.own1; i += kCT)
        for (int r = 0; r < kMaxRows; ++r) {
          a.acc[(size_t)(0 * 2 + pp) * dkr + (size_t)r * d + i] = 0ull;
          a.acc[(size_t)(1 * 2 + pp) * dkr + (size_t)r * d + i] = 0ull;
        }
      build_x(a, ax, xs, a.h + (size_t)par * dkr, ao, nullptr, a.norms + (size_t)(2 * l + 1) * d, nullptr, 0, 0, cs);
      MARK(8)
      const int nfb = rg.fb1 - rg.fb0;
      gemv_blocks(a, ax, ring_s, xs_s, xs_pitch(d), d, 2 * nfb, m.nkd, R, cs, [&](int j, const float(&c)[4]) {
        const int g8 = cs.lane >> 2, q = cs.lane & 3;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = g8 + 8 * (e >> 1), r = 2 * q + (e & 1);
          if (r < R) gus[(j * kMB + row) * kMaxRows + r] = c[e] * ax->scale[r];
        }
      });
      for (int i = cs.ct; i < nfb * kMB * kMaxRows; i += kCT) {  // act = SiLU(gate) * up, bf16 (zero for dead rows)
        const int f = i / kMaxRows, r = i % kMaxRows, fb = f / kMB, k = f % kMB;
        float v = 0.f;
        if (r < R) {
          const float gg = gus[((2 * fb) * kMB + k) * kMaxRows + r], uu = gus[((2 * fb + 1) * kMB + k) * kMaxRows + r];
          v = (gg / (1.f + expf(-gg))) * uu;
        }
        acts[(fb * kMaxRows + r) * kMB + k] = __float2bfloat16(v);
      }
      named_bar(1, kCT);
      MARK(9)
      {  // down^T tiles: every warp takes 4 tiles of every unit; accumulators over the CTA's blocks
        float dacc[4][4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int t = 0; t < 4; ++t) dacc[u][t][0] = dacc[u][t][1] = dacc[u][t][2] = dacc[u][t][3] = 0.f;
        const int g8 = cs.lane >> 2, q = cs.lane & 3;
        const int mrow = (cs.lane & 7) + 8 * ((cs.lane >> 3) & 1), mchunk = cs.lane >> 4;
        for (int fb = 0; fb < nfb; ++fb) {
          // B = act of this block: [16 features] x [rows]: b0 = act[row g][k = 2q, 2q + 1], b1 = ... + 8
          const uint32_t ab = smem_u32(acts + (fb * kMaxRows + g8) * kMB);
          const uint32_t b0 = g8 < R ? lds32(ab + q * 4) : 0u, b1 = g8 < R ? lds32(ab + 16 + q * 4) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (u >= m.ndn) break;
            const int i = cs.stage + fb * m.ndn + u;
            unit_wait(a, ax, i);
            const uint32_t st = ring_s + (i % a.stages) * kStage;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int tile = cs.warp * 4 + t;
              if (u * kTiles + tile < m.ndt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4(st + tile * 512 + mrow * 32 + mchunk * 16, a0, a1, a2, a3);
                mma_bf16(dacc[u][t], a0, a1, a2, a3, b0, b1);
              }
            }
            unit_release(a, ax, i, 1, cs.lane);
          }
        }
        cs.stage += nfb * m.ndn;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (u >= m.ndn) break;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int rb = u * kTiles + cs.warp * 4 + t;
            if (rb >= m.ndt || nfb == 0) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int n = rb * kMB + g8 + 8 * (e >> 1), r = 2 * q + (e & 1);
              if (r < R) red_add_u64(ad + (size_t)r * d + n, (long long)__float2ll_rn(dacc[u][t][e] * kFix));
            }
          }
        }
      }
      MARK(10)
      grid_arrive(a, cs);
    }
#undef MARK
    if (ok && (ok = grid_wait(a, ax, cs))) {
      const int lp = (a.L - 1) & 1;
      build_x(a, ax, xs, a.h + (size_t)lp * dkr, a.acc + (size_t)(0 * 2 + lp) * dkr,
              a.acc + (size_t)(1 * 2 + lp) * dkr, a.norms + (size_t)(2 * a.L) * d, nullptr, 0, 0, cs);
      // zero the last layer's accumulators after every CTA read them: done by the next launch's
      // owners is not possible (parity), so the LM arrival counter orders it (below)
      gemv_blocks(a, ax, ring_s, xs_s, xs_pitch(d), d, rg.lb1 - rg.lb0, m.nkd, R, cs, [&](int j, const float(&c)[4]) {
        const int g8 = cs.lane >> 2, q = cs.lane & 3, b = rg.lb0 + j;
        unsigned long long best[2] = {0ull, 0ull};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n = b * kMB + g8 + 8 * (e >> 1), r = 2 * q + (e & 1);
          if (r >= R) continue;
          const float v = c[e] * ax->scale[r];
          if (a.logits) a.logits[(size_t)r * a.vocab + n] = v;
          const unsigned long long k = (a.exclude_eos && n == a.eos) ? 0ull : argmax_key(v, n);
          best[e & 1] = k > best[e & 1] ? k : best[e & 1];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          unsigned long long k = best[h];
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            const unsigned long long w = __shfl_xor_sync(0xffffffffu, k, o);
            k = w > k ? w : k;
          }
          const int r = 2 * q + h;
          if (g8 == 0 && r < R && k) atomicMax(&ax->key[r], k);
        }
      });
      if (cs.ct == 0) {
        for (int r = 0; r < R; ++r) atomicMax(a.best + r, ax->key[r]);
        __threadfence();
        if (atomicAdd(a.sync + kSyncLm, 1) == (int)gridDim.x - 1) {
          __threadfence();
          for (int r = 0; r < R; ++r) ctl->preds[r] = argmax_key_index(atomicExch(a.best + r, 0ull));
          a.sync[kSyncLm] = 0;
        }
      }
    }
    if (cs.ct == 0) ax->consumed = cs.stage;
  }
  __syncthreads();
  if (warp == kCW && (tid & 31) == 0) {  // drain the copies a cut left in flight
    for (int i = ax->consumed; i < ax->issued; ++i) mbar_wait_b(smem_u32(&ax->full[i % a.stages]), (i / a.stages) & 1);
  }
  __syncthreads();
  cluster_sync();  // no peer reads this CTA's shared memory any more
  if (tid == 0) {
    if (ax->cut) atomicExch(a.sync + kSyncCut, 1);
    __threadfence();
    if (atomicAdd(a.sync + kSyncExit, 1) == (int)gridDim.x - 1) {
      __threadfence();
      a.sync[kSyncBar] = 0;
      if (atomicExch(a.sync + kSyncCut, 0)) {
        a.sync[kSyncLm] = 0;
        for (int r = 0; r < KMAX; ++r) a.best[r] = 0ull;
        if (a.cuts) *a.cuts += 1;
      }
      a.sync[kSyncExit] = 0;
    }
  }
}

// Zero the accumulators (both kinds, both parities): after every launch the last layer's pair
// and, after a cut, any partially added one.  A separate tiny kernel keeps the forward simple.
__global__ void k_zero_acc(unsigned long long* acc, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc[i] = 0ull;
}

// ------------------------------------------------------------------ host
bool supported(int d, int H, int KV, int hd, int ffn, int vocab) {
  if (!(hd == 64 || hd == 128) || KV <= 0 || H % KV || H / KV > kMaxG) return false;
  const int G = H / KV;
  if (d % 64 || d > kMaxD || (G * hd) % 64 || ffn % kMB || vocab % kMB || ((G + 2) * hd) % kMB) return false;
  if (ffn / kMB < 1) return false;
  return max_stages(d, H, KV, hd) >= 4;
}
Layout layout(int d, int H, int KV, int hd, int ffn, int vocab, int L) {
  Layout t;
  const long long ncols = (long long)(H + 2 * KV) * hd;
  t.off_o = 2ll * ncols * d;
  t.off_gu = t.off_o + 2ll * d * H * hd;
  t.off_dn = t.off_gu + 4ll * ffn * d;
  t.layer_bytes = t.off_dn + 2ll * ffn * d;
  t.lm_off = t.layer_bytes * L;
  t.total = t.lm_off + 2ll * vocab * d;
  return t;
}

// Row-block units: one 16-byte destination chunk per thread.  Source row of block-row n given
// by `mode`: 0 QKV (group blocks), 1 O (output rows, the group's head columns), 2 gate/up,
// 3 plain rows (LM head).
__global__ void k_tile_rows(const uint4* __restrict__ s0, const uint4* __restrict__ s1, int mode, int nblocks, int K,
                            int ldk, int H, int KV, int hd, int d, uint4* __restrict__ dst) {
  const int G = H / KV, NG = (G + 2) * hd, nbq = NG / kMB, nbo = d / kMB;
  const long long per_block = 2ll * K;  // 16 rows x K / 8 chunks
  const long long nchunks = (long long)nblocks * per_block;
  for (long long ci = blockIdx.x * (long long)blockDim.x + threadIdx.x; ci < nchunks; ci += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(ci / per_block);
    const int rem = (int)(ci - (long long)b * per_block);
    const int q = rem / (kMB * kKW / 8);
    const int kw = min(kKW, K - q * kKW);
    const int pc_all = rem - q * (kMB * kKW / 8);
    const int n = pc_all / (kw / 8), pc = pc_all % (kw / 8);
    const int col = q * kKW + (pc ^ (n & 7)) * 8;
    const uint4* s = s0;
    long long srow, scol = col;
    if (mode == 0) {  // group g = b / nbq, row rr of [q (G heads) | k | v]
      const int g = b / nbq, rr = (b % nbq) * kMB + n;
      srow = rr < G * hd ? (long long)g * G * hd + rr
           : rr < (G + 1) * hd ? (long long)H * hd + g * hd + (rr - G * hd)
                               : (long long)(H + KV) * hd + g * hd + (rr - (G + 1) * hd);
    } else if (mode == 1) {  // O: block (g, ob): output rows ob*16 + n, columns of group g's heads
      const int g = b / nbo, ob = b % nbo;
      srow = (long long)ob * kMB + n;
      scol = (long long)g * G * hd + col;
    } else if (mode == 2) {  // gate/up: block = 2 fb + half
      s = (b & 1) ? s1 : s0;
      srow = (long long)(b >> 1) * kMB + n;
    } else {
      srow = (long long)b * kMB + n;
    }
    dst[ci] = s[(srow * ldk + scol) / 8];
  }
}
// down^T: feature block fb, tile rb: rows rb*16 + n (output rows), features fb*16 + k; 16 x 16
// bf16, row n at n * 32 bytes.
__global__ void k_tile_down(const __nv_bfloat16* __restrict__ wd, int d, int ffn, __nv_bfloat16* __restrict__ dst) {
  const long long n_el = (long long)d * ffn;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_el; i += (long long)gridDim.x * blockDim.x) {
    const int ndt = d / kMB;
    const long long fb = i / ((long long)ndt * 256);
    const int rem = (int)(i - fb * ndt * 256), rb = rem / 256, n = (rem % 256) / 16, k = rem % 16;
    dst[i] = wd[((long long)rb * kMB + n) * ffn + fb * kMB + k];
  }
}

cudaError_t tile_layer(const void* wqkv, const void* wo, const void* wgate, const void* wup, const void* wdown,
                       int d, int H, int KV, int hd, int ffn, void* dst, cudaStream_t st) {
  const int G = H / KV, NG = (G + 2) * hd;
  const Layout t = layout(d, H, KV, hd, ffn, 16, 1);
  uint8_t* o = (uint8_t*)dst;
  const dim3 grid(148 * 8), blk(256);
  k_tile_rows<<<grid, blk, 0, st>>>((const uint4*)wqkv, nullptr, 0, KV * (NG / kMB), d, d, H, KV, hd, d, (uint4*)o);
  k_tile_rows<<<grid, blk, 0, st>>>((const uint4*)wo, nullptr, 1, KV * (d / kMB), G * hd, H * hd, H, KV, hd, d,
                                    (uint4*)(o + t.off_o));
  k_tile_rows<<<grid, blk, 0, st>>>((const uint4*)wgate, (const uint4*)wup, 2, 2 * (ffn / kMB), d, d, H, KV, hd, d,
                                    (uint4*)(o + t.off_gu));
  k_tile_down<<<grid, blk, 0, st>>>((const __nv_bfloat16*)wdown, d, ffn, (__nv_bfloat16*)(o + t.off_dn));
  return cudaGetLastError();
}
cudaError_t tile_lm(const void* lm, int vocab, int d, void* dst, cudaStream_t st) {
  k_tile_rows<<<148 * 8, 256, 0, st>>>((const uint4*)lm, nullptr, 3, vocab / kMB, d, d, 1, 1, 64, d, (uint4*)dst);
  return cudaGetLastError();
}
size_t sync_ints() { return (size_t)4 * kPad; }
size_t h_bytes(int d) { return (size_t)2 * kMaxRows * d * 4; }
size_t acc_bytes(int d) { return (size_t)4 * kMaxRows * d * 8; }
int max_stages(int d, int H, int KV, int hd) {
  const Smem s0 = smem_layout(0, d, H, KV, hd);
  return std::min(kMaxStages, (kSmemBudget - s0.total) / kStage);
}

template <int HD>
static cudaError_t launch_t(const ClArgs& a, int grid, cudaStream_t st, bool query, int* max_clusters) {
  const int smem = smem_layout(a.stages, a.d, a.H, a.KV, a.hd).total;
  static SmemOptIn opt;
  if (cudaError_t e = opt.ensure(k_decode_cl<HD>, smem)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (query) return cudaOccupancyMaxActiveClusters(max_clusters, k_decode_cl<HD>, &cfg);
  if (cudaError_t e = cudaLaunchKernelEx(&cfg, k_decode_cl<HD>, a)) return e;
  // re-arm the accumulators for the next launch (the last layer's pair, and any a cut left)
  k_zero_acc<<<64, 256, 0, st>>>(a.acc, acc_bytes(a.d) / 8);
  return cudaGetLastError();
}

int grid_for(const ClArgs& a, int want) {
  int mc = 0;
  const cudaError_t e = a.hd == 64 ? launch_t<64>(a, kCluster, 0, true, &mc) : launch_t<128>(a, kCluster, 0, true, &mc);
  if (e != cudaSuccess || mc <= 0) return 0;
  const int g = std::min(want / kCluster, mc) * kCluster;
  // per-CTA buffers hold <= 8 feature blocks (gate/up results, act)
  return g >= a.KV * kCluster && (a.ffn / kMB + g - 1) / g <= 8 ? g : 0;
}

cudaError_t launch(const ClArgs& a, int grid, cudaStream_t st) {
  if (grid <= 0 || grid % kCluster || grid / kCluster < a.KV || a.stages < 2 ||
      a.stages > max_stages(a.d, a.H, a.KV, a.hd))
    return cudaErrorInvalidValue;
  return a.hd == 64 ? launch_t<64>(a, grid, st, false, nullptr) : launch_t<128>(a, grid, st, false, nullptr);
}

}  // namespace cl
}  // namespace amusd
