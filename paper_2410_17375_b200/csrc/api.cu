// api.cu -- the extern "C" boundary declared in include/amusd.h.
//
// Host side of the path: model handles (MockModel, models.py:85-200),
// sessions (SharedDecodeState + executor, coordination.py:114-275,
// engines.py:409-561) and the CUDA-graph construction that turns each engine
// into a device-driven WHILE loop.  No device allocation happens here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/amusd.h"
#include "common.cuh"
#include "decode_cl.h"
#include "decode_gv.h"
#include "internal.h"
#include "protocol.h"
#include "transformer.h"
#include "gemm_tc.h"
#include "forward_tc.h"
#include "prefill.h"

using namespace amusd;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                          \
  do {                                                                                       \
    cudaError_t e__ = (x);                                                                   \
    if (e__ != cudaSuccess)                                                                  \
      return fail(AMUSD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e__));        \
  } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? (T*)(base + off) : nullptr;
    off += sizeof(T) * count;
    return p;
  }
};

}  // namespace

// ------------------------------------------------------------------- model
struct amusd_model {
  int kind = 0;  // 0 transformer, 1 hash chain
  int vocab = 0, eos = 0, exclude_eos = 0, max_seq = 0;
  // device state
  SeqHdr* seq = nullptr;
  int* tok = nullptr;
  StepCtl* api_ctl = nullptr;
  // host mirror of the sequence (parity API)
  int prompt_len = 0, len = 0, kv_len = 0;
  bool pred_valid = false;
  int pred = 0;
  bool dirty = false;  // device loops advanced the state since the last sync
  std::vector<int> htok;
  // hash chain
  unsigned long long seed = 0;
  unsigned long long* chain = nullptr;
  bool agree = false, agree_always = false;
  unsigned long long agree_thr = 0;
  // scripted model (models.py:317-346): device script table, 0 = none
  int* script = nullptr;
  int script_len = 0, eos_position = 0;
  // transformer
  amusd_tf_config cfg{};
  amusd_tf_weights w{};
  void *kc = nullptr, *vc = nullptr;
  float *h = nullptr, *qkv = nullptr, *attn = nullptr, *act = nullptr, *logits = nullptr;
  float* attn_ws = nullptr;
  int* attn_cnt = nullptr;
  unsigned long long* part = nullptr;
  int lm_grid = 0;
  size_t kv_layer_elems = 0;
  int last_rows = 0;
  // tensor-core (tcgen05) path for 16-row forwards
  bool tc = false;
  __nv_bfloat16 *xa_b = nullptr, *attn_b = nullptr, *act_b = nullptr;
  float* inv = nullptr;
  float* ssp = nullptr;
  float* tc_ws = nullptr;
  int* tc_cnt = nullptr;
  // weights re-laid-out as tile-contiguous SW128 16 KB units (one bulk copy each)
  std::vector<const uint8_t*> wt_qkv, wt_o, wt_gu, wt_d;
  const uint8_t* wt_lm = nullptr;
  uint8_t* tiled = nullptr;
  CUtensorMap map_xa{}, map_attn{}, map_act{}, map_xb{};
  // persistent forward (forward_tc.cu): phase table + self-resetting schedule
  fw::FwArgs fw_args{};           // schedule (GEMM kinds) + model pointers, built at create
  bool fw_ready = false;
  __nv_bfloat16* fw_norms = nullptr;  // packed RMSNorm weights [2L+1][d]
  float* fw_attn_ws = nullptr;        // attention split partials (128-position chunks)
  __nv_bfloat16* fw_xb = nullptr;     // gate/up input (double buffer of xa_b)
  float* fw_sspb = nullptr;
  long long* fw_tflag = nullptr;      // per-tile completion stamps
  int* fw_agrp = nullptr;             // attention items finished per (layer, head group)
  int* fw_attn_cnt = nullptr;
  int* fw_sched = nullptr;
  unsigned long long* fw_best = nullptr;
  float* fw_ws = nullptr;
  int* fw_tile_cnt = nullptr;
  int fw_grid = 0, fw_stages = 0;  // launch shape (set per engine at graph capture)
  fw::ModelView fw_view{};          // persistent-forward model view (kinds rebuilt per grid)
  fw::GemmKind fw_kinds_part[fw::kNumGemm];  // kinds for a partial-grid launch ...
  int fw_part_grid = 0;             // ... built for this many SMs (0 = none yet)
  bool fw_part_ok = false;          // draft role only: split-K chunking changes the fp32 partials,
                                    // so the verify keeps one chunking in every engine (AR parity)
  const int* fw_ab_req = nullptr;   // draft cut words (set while capturing the AMUSD draft loop)
  const int* fw_ab_done = nullptr;
  size_t fw_ws_floats = 0, fw_cnt_ints = 0, fw_attn_cnt_ints = 0;  // cut cleanup extents
  int grid_override = 0;            // amusd_model_set_grid: SMs of amusd_time_forward launches (0 = all)
  int max_grid = 0;                 // amusd_model_set_max_grid: cap of every persistent launch (0 = all SMs)
  int path = AMUSD_PATH_PERSISTENT;
  // persistent SIMT decode forward (decode_gv.cu, AMUSD_PATH_DECODE): counters, per-CTA sums
  // of squares, attention split partials
  bool gv_ok = false;
  // cluster decode forward (decode_cl.cu, AMUSD_PATH_CLUSTER)
  bool cl_ok = false;
  const uint8_t* cl_wt = nullptr;  // cluster-decode weight layout (amusd_model_set_cluster, caller-owned)
  float* cl_h = nullptr;
  unsigned long long* cl_acc = nullptr;
  int* cl_sync = nullptr;
  const uint8_t* gv_wt = nullptr;  // decode-layout weights (amusd_model_set_decode, caller-owned)
  int* gv_sync = nullptr;
  float* gv_ss = nullptr;
  float* gv_attn_ws = nullptr;
  bool row_major = true;  // row-major layer weights still valid (amusd_model_release_row_major)
  long long* fw_dbg = nullptr;  // optional per-item timeline (amusd_model_set_timeline)
  int fw_dbg_items = 0;
  // compute-bound prompt prefill (prefill.cu), caller workspace (amusd_model_set_prefill)
  pf::Work pf{};
  bool pf_ready = false;
  // tensor-parallel shard (amusd_tf_create_shard): tp.tp_size == 0 when not sharded
  amusd_tp_shard tp{};
  bool tp_connected = false;
};

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}
// AMUSD_FW=0 selects the per-kernel tcgen05 path (A/B comparisons only).
static bool fw_enabled() {
  static int v = -1;
  if (v < 0) v = env_int("AMUSD_FW", 1) != 0;
  return v;
}
static int fw_units() {
  static int v = -1;
  if (v < 0) v = std::max(1, env_int("AMUSD_FW_UNITS", 16));
  return v;
}
// AMUSD_FW_FUSE: gate/up -> down fused in the persistent forward where the shape allows it
// (read when a model is created; forward_tc.h FwArgs::fuse).
static int fw_fuse() { return env_int("AMUSD_FW_FUSE", 0); }
static int num_sms() { return device_sms(); }
// SMs of this model's persistent launches outside co-located AMUSD (amusd_model_set_max_grid).
static int model_sms(const amusd_model* m) { return m->max_grid > 0 ? std::min(m->max_grid, num_sms()) : num_sms(); }
// Deepest weight ring that fits `per_sm` CTAs on one SM (227 KB smem per SM).
static int fw_max_stages(const amusd_tf_config& c, int per_sm) {
  const int group = c.n_heads / c.n_kv_heads;
  const int budget = (per_sm == 1 ? 232448 : 233472 / per_sm - 1024);
  int s = 2;
  while (s < 16 && fw::forward_smem_bytes(s + 1, c.head_dim, group) <= budget) ++s;
  return s;
}

static bool tc_shapes_ok(const amusd_tf_config* c) {
  const int ncols = (c->n_heads + 2 * c->n_kv_heads) * c->head_dim;
  // tcgen05 tiles: 128 weight rows (64 gate + 64 up features) x 64 K per unit
  // and a QKV group block [q(G heads) | k | v] spans whole 128-row tiles
  const int G = c->n_kv_heads ? c->n_heads / c->n_kv_heads : 0;
  return c->dtype == AMUSD_BF16 && c->use_tensor_cores && c->d_model % 128 == 0 && ncols % 128 == 0 &&
         c->ffn % 128 == 0 && c->vocab % 128 == 0 && (c->n_heads * c->head_dim) % 128 == 0 &&
         ((G + 2) * c->head_dim) % 128 == 0;
}

// Split-K workspace sizes of a config (dry run of build_kinds without pointers).
static void view_shard(fw::ModelView* v, const amusd_tp_shard* sh) {
  if (!sh || sh->tp_size < 2) return;
  v->tp = sh->tp_size; v->H_full = sh->n_heads_full; v->KV_full = sh->n_kv_heads_full; v->ffn_full = sh->ffn_full;
}
static bool fw_sizes(const amusd_tf_config* c, const amusd_tp_shard* sh, size_t* ws_floats, int* cnt_ints,
                     int* max_tiles) {
  fw::ModelView v{};
  v.d = c->d_model; v.H = c->n_heads; v.KV = c->n_kv_heads; v.hd = c->head_dim; v.ffn = c->ffn; v.vocab = c->vocab;
  v.L = c->n_layers; v.S = c->max_seq;
  v.fuse = fw_fuse();
  view_shard(&v, sh);
  fw::FwArgs a{};
  return fw::build_kinds(v, fw_units(), &a, ws_floats, cnt_ints, max_tiles);
}

static size_t tf_carve(const amusd_tf_config* c, void* base, amusd_model* m, const amusd_tp_shard* sh = nullptr) {
  Carver cv(base);
  const size_t wsz = c->dtype == AMUSD_BF16 ? 2 : 4;
  const int ncols = (c->n_heads + 2 * c->n_kv_heads) * c->head_dim;
  const size_t kv = (size_t)c->n_layers * c->n_kv_heads * c->max_seq * c->head_dim;
  const int lm_grid = gemv_grid(c->vocab, 2);
  SeqHdr* seq = cv.take<SeqHdr>(1);
  int* tok = cv.take<int>(c->max_seq + 1);
  StepCtl* ctl = cv.take<StepCtl>(1);
  char* kc = cv.take<char>(kv * wsz);
  char* vc = cv.take<char>(kv * wsz);
  float* h = cv.take<float>((size_t)KMAX * c->d_model);
  float* qkv = cv.take<float>((size_t)KMAX * ncols);
  float* attn = cv.take<float>((size_t)KMAX * c->n_heads * c->head_dim);
  float* act = cv.take<float>((size_t)KMAX * c->ffn);
  const int lm_tiles = (c->vocab + 127) / 128;
  unsigned long long* part = cv.take<unsigned long long>((size_t)KMAX * std::max(lm_grid, lm_tiles));
  float* logits = cv.take<float>((size_t)KMAX * c->vocab);
  const int group = c->n_heads / std::max(1, c->n_kv_heads);
  float* attn_ws = cv.take<float>((size_t)c->n_kv_heads * KMAX * attn_max_splits(c->max_seq) * group * (c->head_dim + 2));
  int* attn_cnt = cv.take<int>((size_t)c->n_kv_heads * KMAX);
  const bool tc = tc_shapes_ok(c);
  __nv_bfloat16 *xa_b = nullptr, *attn_b = nullptr, *act_b = nullptr;
  float *inv = nullptr, *ws = nullptr, *ssp_b = nullptr;
  int* cnt = nullptr;
  uint8_t* tiled = nullptr;
  if (tc) {
    xa_b = cv.take<__nv_bfloat16>((size_t)KMAX * c->d_model);
    attn_b = cv.take<__nv_bfloat16>((size_t)KMAX * c->n_heads * c->head_dim);
    act_b = cv.take<__nv_bfloat16>((size_t)KMAX * c->ffn);
    inv = cv.take<float>(KMAX);
    ssp_b = cv.take<float>((size_t)KMAX * (c->d_model / 128));
    ws = cv.take<float>((size_t)256 * 2 * 128 * KMAX);  // >= grid (SM count) x 2 partial tiles of 128 x 16
    cnt = cv.take<int>(std::max(lm_tiles, 4096));
    const int hh = c->n_heads * c->head_dim;
    const size_t per_layer = tc::tiled_bytes(ncols, c->d_model) + tc::tiled_bytes(c->d_model, hh) +
                             tc::tiled_bytes(2 * c->ffn, c->d_model) + tc::tiled_bytes(c->d_model, c->ffn);
    tiled = cv.take<uint8_t>(per_layer * c->n_layers + tc::tiled_bytes(c->vocab, c->d_model));
  }
  int* fsched = nullptr;
  unsigned long long* fbest = nullptr;
  float* fws = nullptr;
  int* fcnt = nullptr;
  __nv_bfloat16* fnorms = nullptr;
  __nv_bfloat16* fxb = nullptr;
  float* fsspb = nullptr;
  long long* ftflag = nullptr;
  int* fagrp = nullptr;
  float* fattn_ws = nullptr;
  int* fattn_cnt = nullptr;
  if (tc) {
    int mt;
    size_t wsf;
    int cints;
    fw_sizes(c, sh, &wsf, &cints, &mt);
    fsched = cv.take<int>(fw::sched_ints(c->n_layers));
    fbest = cv.take<unsigned long long>(KMAX);
    fws = cv.take<float>(std::max<size_t>(wsf, 1));
    fcnt = cv.take<int>((size_t)cints);
    fxb = cv.take<__nv_bfloat16>((size_t)KMAX * c->d_model);
    fsspb = cv.take<float>((size_t)KMAX * (c->d_model / 128));
    ftflag = cv.take<long long>((size_t)4 * mt * (fw::kCounterInts / 2));
    fagrp = cv.take<int>((size_t)c->n_layers * c->n_kv_heads * fw::kCounterInts);
    fnorms = cv.take<__nv_bfloat16>((size_t)(2 * c->n_layers + 1) * c->d_model);
    fattn_ws = cv.take<float>((size_t)c->n_kv_heads * KMAX * fw::attn_splits(c->max_seq) * group * (c->head_dim + 2));
    fattn_cnt = cv.take<int>((size_t)c->n_kv_heads * KMAX * fw::kCounterInts);
  }
  const bool clok = tc && cl::supported(c->d_model, c->n_heads, c->n_kv_heads, c->head_dim, c->ffn, c->vocab);
  float* clh = nullptr;
  unsigned long long* clacc = nullptr;
  int* clsync = nullptr;
  if (clok) {
    clh = cv.take<float>(cl::h_bytes(c->d_model) / 4);
    clacc = cv.take<unsigned long long>(cl::acc_bytes(c->d_model) / 8);
    clsync = cv.take<int>(cl::sync_ints());
  }
  const bool gvok = tc && gv::supported(c->d_model, c->n_heads, c->n_kv_heads, c->head_dim, c->ffn, c->vocab);
  int* gsync = nullptr;
  float *gss = nullptr, *gattn = nullptr;
  if (gvok) {
    gsync = cv.take<int>(gv::sync_ints(c->n_kv_heads));
    gss = cv.take<float>(gv::ss_floats());
    gattn = cv.take<float>(gv::attn_ws_floats(c->n_kv_heads, group, c->head_dim, c->max_seq));
  }
  if (m) {
    m->attn_ws = attn_ws; m->attn_cnt = attn_cnt;
    m->fw_sched = fsched; m->fw_best = fbest; m->fw_ws = fws; m->fw_tile_cnt = fcnt; m->fw_norms = fnorms;
    m->fw_attn_ws = fattn_ws; m->fw_attn_cnt = fattn_cnt;
    if (tc) {
      size_t wsf;
      int cints, mt;
      fw_sizes(c, sh, &wsf, &cints, &mt);
      m->fw_ws_floats = std::max<size_t>(wsf, 1);
      m->fw_cnt_ints = (size_t)cints;
      m->fw_attn_cnt_ints = (size_t)c->n_kv_heads * KMAX * fw::kCounterInts;
    }
    m->gv_ok = gvok; m->gv_sync = gsync; m->gv_ss = gss; m->gv_attn_ws = gattn;
    m->cl_ok = clok; m->cl_h = clh; m->cl_acc = clacc; m->cl_sync = clsync;
    m->fw_xb = fxb; m->fw_sspb = fsspb; m->fw_tflag = ftflag; m->fw_agrp = fagrp;
    m->tc = tc; m->xa_b = xa_b; m->attn_b = attn_b; m->act_b = act_b; m->inv = inv; m->ssp = ssp_b; m->tc_ws = ws; m->tc_cnt = cnt; m->tiled = tiled;
    m->seq = seq; m->tok = tok; m->api_ctl = ctl; m->kc = kc; m->vc = vc; m->h = h; m->qkv = qkv;
    m->attn = attn; m->act = act; m->part = part; m->logits = logits; m->lm_grid = lm_grid;
    m->kv_layer_elems = (size_t)c->n_kv_heads * c->max_seq * c->head_dim;
  }
  return align_up(cv.off, 256);
}

static size_t hash_carve(int max_seq, void* base, amusd_model* m, int script_len = 0) {
  Carver cv(base);
  SeqHdr* seq = cv.take<SeqHdr>(1);
  int* tok = cv.take<int>(max_seq + 1);
  StepCtl* ctl = cv.take<StepCtl>(1);
  unsigned long long* chain = cv.take<unsigned long long>(max_seq + 2);
  int* script = script_len ? cv.take<int>(script_len) : nullptr;
  if (m) { m->seq = seq; m->tok = tok; m->api_ctl = ctl; m->chain = chain; m->script = script; }
  return align_up(cv.off, 256);
}

// One kernel of a transformer forward: which = 0 QKV gemv, 1 attention, 2 O
// gemv, 3 gate/up gemv, 4 down gemv (per layer), 5 LM head, 6 argmax reduce,
// 7 embedding.
static int tf_kernel(amusd_model* m, StepCtl* ctl, int nr, int l, int which, cudaStream_t st, bool pdl,
                     bool want_logits) {
  const amusd_tf_config& c = m->cfg;
  const int dt = c.dtype;
  const size_t wsz = dt == AMUSD_BF16 ? 2 : 4;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads;
  const int ncols = (H + 2 * KV) * hd;
  GemvArgs g{};
  g.ctl = ctl; g.eps = c.norm_eps; g.eos = c.eos_token; g.exclude_eos = c.exclude_eos;
  switch (which) {
    case 7:
      CUDA_TRY(launch_embed(dt, ctl, m->w.embed, m->h, d, st, pdl));
      break;
    case 0:  // QKV (attention RMSNorm fused)
      g.x = m->h; g.ldx = d; g.gamma = m->w.attn_norm[l]; g.W = m->w.wqkv[l]; g.N = ncols; g.K = d;
      g.kc = gemv_kc(nr, d); g.out = m->qkv; g.ldo = ncols;
      CUDA_TRY(launch_gemv(nr, dt, kEpiStore, g, st, pdl));
      break;
    case 1: {  // attention (RoPE + KV append fused)
      AttnArgs at{};
      at.ctl = ctl; at.qkv = m->qkv;
      at.kc = (char*)m->kc + (size_t)l * m->kv_layer_elems * wsz;
      at.vc = (char*)m->vc + (size_t)l * m->kv_layer_elems * wsz;
      at.cos = m->w.rope_cos; at.sin = m->w.rope_sin; at.out = m->attn; at.ldo = H * hd;
      at.H = H; at.KV = KV; at.hd = hd; at.S = c.max_seq; at.scale = 1.0f / sqrtf((float)hd);
      at.ws = m->attn_ws; at.counters = m->attn_cnt; at.max_splits = attn_max_splits(c.max_seq);
      CUDA_TRY(launch_attention(dt, at, st, pdl));
      break;
    }
    case 2:  // O projection + residual
      g.x = m->attn; g.ldx = H * hd; g.W = m->w.wo[l]; g.N = d; g.K = H * hd;
      g.kc = gemv_kc(nr, H * hd); g.out = m->h; g.ldo = d;
      CUDA_TRY(launch_gemv(nr, dt, kEpiResid, g, st, pdl));
      break;
    case 3:  // gate/up (MLP RMSNorm + SiLU*mul fused)
      g.x = m->h; g.ldx = d; g.gamma = m->w.mlp_norm[l]; g.W = m->w.wgate[l]; g.W2 = m->w.wup[l];
      g.N = c.ffn; g.K = d; g.kc = gemv_kc(nr, d); g.out = m->act; g.ldo = c.ffn;
      CUDA_TRY(launch_gemv(nr, dt, kEpiGateUp, g, st, pdl));
      break;
    case 4:  // down projection + residual
      g.x = m->act; g.ldx = c.ffn; g.W = m->w.wdown[l]; g.N = d; g.K = c.ffn; g.kc = gemv_kc(nr, c.ffn);
      g.out = m->h; g.ldo = d;
      CUDA_TRY(launch_gemv(nr, dt, kEpiResid, g, st, pdl));
      break;
    case 5:  // final RMSNorm + LM head + per-CTA argmax
      g.x = m->h; g.ldx = d; g.gamma = m->w.final_norm; g.W = m->w.lm_head; g.N = c.vocab; g.K = d;
      g.kc = gemv_kc(nr, d); g.part = m->part; g.logits = want_logits ? m->logits : nullptr;
      CUDA_TRY(launch_gemv(nr, dt, kEpiArgmax, g, st, pdl));
      break;
    case 6:
      CUDA_TRY(launch_argmax_final(ctl, m->part, m->lm_grid, st, pdl));
      break;
    default:
      return fail(AMUSD_ERR_INVALID_INPUT, "unknown kernel id");
  }
  return AMUSD_OK;
}

// One kernel of the tensor-core forward (bf16, 16 rows): which = 0 QKV gemm,
// 1 attention, 2 O gemm (+residual, emits mlp-norm input), 3 gate/up gemm,
// 4 down gemm (+residual, emits next attn-norm input) per layer; 5 LM-head
// gemm, 6 argmax reduce, 7 embedding (emits layer-0 attn-norm input).
static int tc_kernel(amusd_model* m, StepCtl* ctl, int l, int which, cudaStream_t st, bool pdl,
                     bool want_logits = false) {
  const amusd_tf_config& c = m->cfg;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads;
  const int ncols = (H + 2 * KV) * hd;
  tc::TcArgs g{};
  g.ctl = ctl; g.eos = c.eos_token; g.exclude_eos = c.exclude_eos; g.ws = m->tc_ws; g.counters = m->tc_cnt;
  g.ssp_tiles = d / 128; g.norm_dim = (float)d; g.eps = c.norm_eps;
  switch (which) {
    case 7: CUDA_TRY(tc::launch_embed_tc(ctl, m->w.embed, m->h, m->w.attn_norm[0], m->xa_b, m->ssp, d, st, pdl)); break;
    case 0:
      g.epi = tc::kTcStoreScaled; g.ntiles = ncols / 128; g.kb = d / 64; g.N = ncols; g.ssp_in = m->ssp;
      g.out = m->qkv; g.ldo = ncols;
      g.wt = m->wt_qkv[l];
      CUDA_TRY(tc::launch_gemm_tc(m->map_xa, g, st, pdl));
      break;
    case 1: {
      AttnArgs at{};
      at.ctl = ctl; at.qkv = m->qkv;
      at.kc = (char*)m->kc + (size_t)l * m->kv_layer_elems * 2;
      at.vc = (char*)m->vc + (size_t)l * m->kv_layer_elems * 2;
      at.cos = m->w.rope_cos; at.sin = m->w.rope_sin; at.out = nullptr; at.out_b = m->attn_b; at.ldo = H * hd;
      at.H = H; at.KV = KV; at.hd = hd; at.S = c.max_seq; at.scale = 1.0f / sqrtf((float)hd);
      at.ws = m->attn_ws; at.counters = m->attn_cnt; at.max_splits = attn_max_splits(c.max_seq);
      at.blocked = 1;  // the tensor-core QKV tiles are group-blocked
      CUDA_TRY(launch_attention(c.dtype, at, st, pdl));
      break;
    }
    case 2:
      g.epi = tc::kTcResid; g.ntiles = d / 128; g.kb = H * hd / 64; g.N = d; g.out = m->h; g.ldo = d;
      g.xnext = m->xa_b; g.gnext = (const __nv_bfloat16*)m->w.mlp_norm[l]; g.ssp = m->ssp;
      g.wt = m->wt_o[l];
      CUDA_TRY(tc::launch_gemm_tc(m->map_attn, g, st, pdl));
      break;
    case 3:
      g.epi = tc::kTcGateUp; g.ntiles = c.ffn / 64; g.kb = d / 64; g.N = c.ffn; g.ssp_in = m->ssp;
      g.out_b = m->act_b; g.ldo = c.ffn;
      g.wt = m->wt_gu[l];
      CUDA_TRY(tc::launch_gemm_tc(m->map_xa, g, st, pdl));
      break;
    case 4:
      g.epi = tc::kTcResid; g.ntiles = d / 128; g.kb = c.ffn / 64; g.N = d; g.out = m->h; g.ldo = d;
      g.xnext = m->xa_b; g.ssp = m->ssp;
      g.gnext = (const __nv_bfloat16*)(l + 1 < c.n_layers ? m->w.attn_norm[l + 1] : m->w.final_norm);
      g.wt = m->wt_d[l];
      CUDA_TRY(tc::launch_gemm_tc(m->map_act, g, st, pdl));
      break;
    case 5:
      g.epi = tc::kTcArgmax; g.ntiles = c.vocab / 128; g.kb = d / 64; g.N = c.vocab; g.ssp_in = m->ssp;
      g.part = m->part; g.logits = want_logits ? m->logits : nullptr;
      g.wt = m->wt_lm;
      CUDA_TRY(tc::launch_gemm_tc(m->map_xa, g, st, pdl));
      break;
    case 6: CUDA_TRY(launch_argmax_final(ctl, m->part, c.vocab / 128, st, pdl)); break;
    default: return fail(AMUSD_ERR_INVALID_INPUT, "unknown kernel id");
  }
  return AMUSD_OK;
}

static bool use_fw(const amusd_model* m) {
  return m->kind == 0 && m->tc && m->fw_ready && fw_enabled() && m->path == AMUSD_PATH_PERSISTENT;
}
// Persistent SIMT decode forward (decode_gv.cu): the draft's path (AMUSD_PATH_DECODE).
static bool use_gv(const amusd_model* m) {
  return m->kind == 0 && m->gv_ok && m->gv_wt && m->path == AMUSD_PATH_DECODE;
}
// Cluster decode forward (decode_cl.cu): the draft's path (AMUSD_PATH_CLUSTER).
static bool use_cl(const amusd_model* m) {
  return m->kind == 0 && m->cl_ok && m->cl_wt && m->path == AMUSD_PATH_CLUSTER;
}
// A persistent forward (tcgen05 work queue, decode or cluster decode): one launch, grid from fw_grid.
static bool use_persistent(const amusd_model* m) { return use_fw(m) || use_gv(m) || use_cl(m); }
// Rows one forward of this model can carry (host-driven API forwards are chunked to it).
static int max_rows(const amusd_model* m) { return use_cl(m) ? cl::kMaxRows : KMAX; }
// Per-kernel tcgen05 path for 16-row forwards (2-row draft steps take the SIMT GEMVs).
static bool use_tc(const amusd_model* m, int nr) {
  return m->kind == 0 && m->tc && nr > 2 && m->path != AMUSD_PATH_SIMT;
}

// The whole forward as one persistent launch (forward_tc.cu).
static int fw_forward(amusd_model* m, StepCtl* ctl, cudaStream_t st, bool want_logits) {
  const amusd_tf_config& c = m->cfg;
  if (m->tp.tp_size > 1 && !m->tp_connected)
    return fail(AMUSD_ERR_INVALID_INPUT, "tensor-parallel shard used before amusd_tp_connect");
  fw::FwArgs a = m->fw_args;
  if (m->fw_part_ok && m->fw_grid < num_sms()) {  // co-located AMUSD draft: larger work items
    if (m->fw_part_grid != m->fw_grid) {
      fw::FwArgs t = m->fw_args;
      size_t wsf;
      int ci, mt;
      fw::build_kinds(m->fw_view, fw_units(), &t, &wsf, &ci, &mt, m->fw_grid);
      std::memcpy(m->fw_kinds_part, t.g, sizeof(t.g));
      m->fw_part_grid = m->fw_grid;
    }
    std::memcpy(a.g, m->fw_kinds_part, sizeof(a.g));
  }
  a.ctl = ctl; a.sched = m->fw_sched;
  a.embed = (const __nv_bfloat16*)m->w.embed; a.norms = m->fw_norms;
  a.h = m->h; a.xa = m->xa_b; a.ssp = m->ssp; a.qkv = m->qkv; a.attn_b = m->attn_b;
  a.xb = m->fw_xb; a.sspb = m->fw_sspb; a.tflag = m->fw_tflag; a.agrp = m->fw_agrp;
  a.kcache = (char*)m->kc; a.vcache = (char*)m->vc; a.kv_layer_bytes = (long long)m->kv_layer_elems * 2;
  a.ws = m->fw_ws; a.tile_cnt = m->fw_tile_cnt; a.attn_ws = m->fw_attn_ws; a.attn_cnt = m->fw_attn_cnt;
  a.cos = m->w.rope_cos; a.sin = m->w.rope_sin; a.best = m->fw_best; a.logits = want_logits ? m->logits : nullptr;
  a.d = c.d_model; a.H = c.n_heads; a.KV = c.n_kv_heads; a.hd = c.head_dim; a.S = c.max_seq;
  a.max_splits = fw::attn_splits(c.max_seq); a.vocab = c.vocab; a.eos = c.eos_token; a.exclude_eos = c.exclude_eos;
  a.scale = 1.0f / sqrtf((float)c.head_dim); a.eps = c.norm_eps;
  a.dbg = m->fw_dbg; a.dbg_items = m->fw_dbg_items;
  a.ab_req = m->fw_ab_req; a.ab_done = m->fw_ab_done;
  // L2 prefetch window (bytes of weights ahead of the grab pointer), AMUSD_FW_L2_MB
  a.prefetch_items = (int)((size_t)env_int("AMUSD_FW_L2_MB", 0) * (1 << 20) / ((size_t)fw_units() * 16384));
  a.inflight = env_int("AMUSD_FW_INFLIGHT", 0);
  a.prefetch_next = env_int("AMUSD_FW_PREFETCH_NEXT", 0);  // measured: L2 prefetch costs more than it hides
  a.debug = env_int("AMUSD_FW_DEBUG", 0);
  a.fine = env_int("AMUSD_FW_FINE", 0);  // per-tile deps measured slower: CTAs run their queues in order
  CUDA_TRY(fw::launch_forward(a, m->map_xa, m->map_attn, m->map_act, m->map_xb, m->fw_grid, m->fw_stages, st));
  if (a.ab_req)
    CUDA_TRY(fw::launch_cut_cleanup(m->fw_sched, ctl, m->fw_ws, m->fw_ws_floats, m->fw_tile_cnt, m->fw_cnt_ints,
                                    m->fw_attn_cnt, m->fw_attn_cnt_ints, m->fw_best, st));
  return AMUSD_OK;
}

// The whole forward as one persistent SIMT launch (decode_gv.cu).
static int gv_forward(amusd_model* m, StepCtl* ctl, cudaStream_t st, bool want_logits) {
  const amusd_tf_config& c = m->cfg;
  gv::GvArgs a;
  std::memset(&a, 0, sizeof(a));
  const gv::Layout t = gv::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers);
  a.wt = m->gv_wt; a.wt_layer_bytes = t.layer_bytes; a.wt_off_o = t.off_o; a.wt_off_gu = t.off_gu;
  a.wt_off_down = t.off_down; a.wt_lm = m->gv_wt + t.lm_off;
  a.embed = (const __nv_bfloat16*)m->w.embed;
  a.norms = m->fw_norms;
  a.cos = m->w.rope_cos; a.sin = m->w.rope_sin;
  a.ctl = ctl;
  a.kcache = (char*)m->kc; a.vcache = (char*)m->vc; a.kv_layer_bytes = (long long)m->kv_layer_elems * 2;
  a.h = m->h; a.xa = m->xa_b; a.xb = m->fw_xb; a.qkv = m->qkv; a.attn_b = m->attn_b; a.act_b = m->act_b;
  a.ss = m->gv_ss; a.attn_ws = m->gv_attn_ws; a.sync = m->gv_sync; a.best = m->fw_best;
  a.logits = want_logits ? m->logits : nullptr;
  a.ab_req = m->fw_ab_req; a.ab_done = m->fw_ab_done;
  a.cuts = m->fw_sched ? fw::cut_counter(m->fw_sched) : nullptr;
  a.d = c.d_model; a.H = c.n_heads; a.KV = c.n_kv_heads; a.hd = c.head_dim; a.ffn = c.ffn; a.vocab = c.vocab;
  a.L = c.n_layers; a.S = c.max_seq; a.eos = c.eos_token; a.exclude_eos = c.exclude_eos;
  a.eps = c.norm_eps; a.scale = 1.0f / sqrtf((float)c.head_dim);
  a.stages = std::max(2, std::min(gv::max_stages(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn),
                                  env_int("AMUSD_GV_STAGES", 99)));
  a.max_splits = gv::attn_splits(c.max_seq);
  const int grid = m->fw_grid > 0 ? m->fw_grid : model_sms(m);
  if (m->fw_dbg && (size_t)m->fw_dbg_items * 8 >= (size_t)grid * (gv::kDbgEvents + 9 * 24)) a.dbg = m->fw_dbg;
  a.debug = env_int("AMUSD_GV_DEBUG", 0);
  a.l2_ahead = env_int("AMUSD_GV_L2", 0);
  CUDA_TRY(gv::launch(a, grid, st));
  return AMUSD_OK;
}

// The whole forward as one cluster-decode launch (decode_cl.cu).
static int cl_forward(amusd_model* m, StepCtl* ctl, cudaStream_t st, bool want_logits) {
  const amusd_tf_config& c = m->cfg;
  cl::ClArgs a;
  std::memset(&a, 0, sizeof(a));
  const cl::Layout t = cl::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers);
  a.wt = m->cl_wt; a.layer_bytes = t.layer_bytes; a.off_o = t.off_o; a.off_gu = t.off_gu; a.off_dn = t.off_dn;
  a.wt_lm = m->cl_wt + t.lm_off;
  a.embed = (const __nv_bfloat16*)m->w.embed;
  a.norms = m->fw_norms;
  a.cos = m->w.rope_cos; a.sin = m->w.rope_sin;
  a.ctl = ctl;
  a.kcache = (char*)m->kc; a.vcache = (char*)m->vc; a.kv_layer_bytes = (long long)m->kv_layer_elems * 2;
  a.h = m->cl_h; a.acc = m->cl_acc; a.sync = m->cl_sync; a.best = m->fw_best;
  a.logits = want_logits ? m->logits : nullptr;
  a.ab_req = m->fw_ab_req; a.ab_done = m->fw_ab_done;
  a.cuts = m->fw_sched ? fw::cut_counter(m->fw_sched) : nullptr;
  a.d = c.d_model; a.H = c.n_heads; a.KV = c.n_kv_heads; a.hd = c.head_dim; a.ffn = c.ffn; a.vocab = c.vocab;
  a.L = c.n_layers; a.S = c.max_seq; a.eos = c.eos_token; a.exclude_eos = c.exclude_eos;
  a.eps = c.norm_eps; a.scale = 1.0f / sqrtf((float)c.head_dim);
  a.stages = std::max(2, std::min(cl::max_stages(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim),
                                  env_int("AMUSD_CL_STAGES", 99)));
  a.debug = env_int("AMUSD_GV_DEBUG", 0);
  a.l2_ahead = env_int("AMUSD_CL_L2", 0);
  const int grid = cl::grid_for(a, m->fw_grid > 0 ? m->fw_grid : model_sms(m));
  if (m->fw_dbg && (size_t)m->fw_dbg_items * 8 >= (size_t)grid * cl::kDbgPerLayer * c.n_layers) a.dbg = m->fw_dbg;
  if (grid <= 0) return fail(AMUSD_ERR_UNSUPPORTED, "cluster decode: too few SMs for one 8-CTA cluster per KV head");
  CUDA_TRY(cl::launch(a, grid, st));
  return AMUSD_OK;
}

// Enqueue one forward of `m` driven by control block `ctl` (rows <= nr).
static int model_forward(amusd_model* m, StepCtl* ctl, int nr, cudaStream_t st, bool pdl, bool want_logits) {
  if (m->kind == 1) {
    CUDA_TRY(launch_hash_forward(ctl, m->chain, m->vocab, m->eos, m->exclude_eos, m->agree, m->agree_always,
                                 m->agree_thr, m->script, m->script_len, m->eos_position, st));
    return AMUSD_OK;
  }
  // co-located AMUSD draft (fw_part_ok): the cluster kernel's grid barrier needs every cluster
  // resident, which the verify forward beside it does not guarantee -> the work-queue forward
  if (use_cl(m) && !m->fw_part_ok) return cl_forward(m, ctl, st, want_logits);
  if (use_gv(m) && !m->fw_part_ok) return gv_forward(m, ctl, st, want_logits);
  if ((use_cl(m) || use_gv(m)) && m->fw_ready) return fw_forward(m, ctl, st, want_logits);
  if (use_fw(m)) return fw_forward(m, ctl, st, want_logits);
  if (!m->row_major) return fail(AMUSD_ERR_UNSUPPORTED, "row-major weights released: persistent path only");
  if (use_tc(m, nr)) {
    if (int r = tc_kernel(m, ctl, 0, 7, st, pdl)) return r;
    for (int l = 0; l < m->cfg.n_layers; ++l)
      for (int k = 0; k < 5; ++k)
        if (int r = tc_kernel(m, ctl, l, k, st, pdl)) return r;
    for (int k = 5; k < 7; ++k)
      if (int r = tc_kernel(m, ctl, 0, k, st, pdl, want_logits)) return r;
    return AMUSD_OK;
  }
  if (int r = tf_kernel(m, ctl, nr, 0, 7, st, pdl, false)) return r;
  for (int l = 0; l < m->cfg.n_layers; ++l)
    for (int k = 0; k < 5; ++k)
      if (int r = tf_kernel(m, ctl, nr, l, k, st, pdl, false)) return r;
  if (int r = tf_kernel(m, ctl, nr, 0, 5, st, pdl, want_logits)) return r;
  return tf_kernel(m, ctl, nr, 0, 6, st, pdl, false);
}

static int model_kernels_per_forward(const amusd_model* m, int nr = KMAX) {
  if (m->kind == 1) return 1;
  if (use_persistent(m)) return 1;
  if (use_tc(m, nr)) return 1 + 5 * m->cfg.n_layers + 2;
  return 1 + 5 * m->cfg.n_layers + 2;
}

extern "C" {

int amusd_abi_version(void) { return AMUSD_ABI_VERSION; }
const char* amusd_last_error(void) { return g_err.c_str(); }

size_t amusd_tf_state_bytes(const amusd_tf_config* cfg) { return cfg ? tf_carve(cfg, nullptr, nullptr) : 0; }
size_t amusd_tf_shard_state_bytes(const amusd_tf_config* cfg, const amusd_tp_shard* sh) {
  return cfg ? tf_carve(cfg, nullptr, nullptr, sh) : 0;
}

}  // extern "C"

static int tf_create(amusd_model** out, const amusd_tf_config* cfg, const amusd_tp_shard* sh,
                     const amusd_tf_weights* w, void* state, size_t state_bytes) {
  if (!out || !cfg || !w || !state) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  const amusd_tf_config& c = *cfg;
  if (c.vocab < 2 || c.d_model <= 0 || c.n_layers <= 0 || c.n_layers > AMUSD_MAX_LAYERS || c.n_heads <= 0 ||
      c.n_kv_heads <= 0 || c.n_heads % c.n_kv_heads || c.head_dim % 8 || c.head_dim > 256 || c.ffn <= 0 ||
      c.max_seq < 2)
    return fail(AMUSD_ERR_INVALID_INPUT, "invalid transformer config");
  const int vocab_total = sh ? sh->vocab_total : c.vocab;
  if (!(0 <= c.eos_token && c.eos_token < vocab_total))
    return fail(AMUSD_ERR_INVALID_INPUT, "eos_token out of range");  // models.py:98-101
  if (sh) {
    if (sh->tp_size < 2 || sh->tp_size > fw::kMaxTp || sh->tp_rank < 0 || sh->tp_rank >= sh->tp_size)
      return fail(AMUSD_ERR_INVALID_INPUT, "tp_rank / tp_size out of range (2 <= tp_size <= 8)");
    if (sh->n_kv_heads_full <= 0 || sh->n_heads_full % sh->n_kv_heads_full ||
        sh->n_heads_full / sh->n_kv_heads_full != c.n_heads / c.n_kv_heads || c.n_kv_heads > sh->n_kv_heads_full ||
        c.ffn > sh->ffn_full || sh->vocab_offset < 0 || sh->vocab_offset + c.vocab > sh->vocab_total)
      return fail(AMUSD_ERR_INVALID_INPUT, "tensor-parallel shard inconsistent with the unsharded model");
    if (c.dtype != AMUSD_BF16 || !c.use_tensor_cores || !fw_enabled())
      return fail(AMUSD_ERR_UNSUPPORTED, "tensor-parallel shards run on the persistent bf16 tcgen05 forward only");
  }
  if (c.d_model % 256 || c.ffn % 256 || (c.n_heads * c.head_dim) % 256)
    return fail(AMUSD_ERR_UNSUPPORTED, "d_model, ffn and n_heads*head_dim must be multiples of 256");
  if (c.dtype != AMUSD_F32 && c.dtype != AMUSD_BF16) return fail(AMUSD_ERR_INVALID_INPUT, "bad dtype");
  if (state_bytes < tf_carve(cfg, nullptr, nullptr, sh)) return fail(AMUSD_ERR_INVALID_INPUT, "state buffer too small");
  {
    const int group = c.n_heads / c.n_kv_heads;
    if (!(c.head_dim == 64 || c.head_dim == 128) || !(group == 2 || group == 4 || group == 8))
      return fail(AMUSD_ERR_UNSUPPORTED, "attention kernels support head_dim 64/128 and GQA groups 2/4/8");
  }
  amusd_model* m = new amusd_model();
  m->kind = 0;
  m->cfg = c;
  m->w = *w;
  m->vocab = vocab_total;  // token ids (a shard's LM head covers cfg.vocab of them)
  m->eos = c.eos_token;
  m->exclude_eos = c.exclude_eos;
  m->max_seq = c.max_seq;
  if (sh) m->tp = *sh;
  tf_carve(cfg, state, m, sh);
  if (sh && !m->tc) {
    delete m;
    return fail(AMUSD_ERR_UNSUPPORTED, "tensor-parallel shard shape does not fit the tcgen05 tiles");
  }
  if (m->tc) {
    const int d = c.d_model, ncols = (c.n_heads + 2 * c.n_kv_heads) * c.head_dim, hh = c.n_heads * c.head_dim;
    bool ok = true;
    uint8_t* p = m->tiled;
    cudaError_t e = cudaSuccess;
    auto place = [&](const void* src, const void* src2, int N, int K, bool qkv = false) -> const uint8_t* {
      const uint8_t* at = p;
      if (e == cudaSuccess)
        e = qkv ? tc::launch_tile_weights(src, src2, p, N, K, 0, c.n_heads, c.n_kv_heads, c.head_dim)
                : tc::launch_tile_weights(src, src2, p, N, K, 0);
      p += tc::tiled_bytes(src2 ? 2 * N : N, K);
      return at;
    };
    for (int l = 0; l < c.n_layers; ++l) {
      m->wt_qkv.push_back(place(w->wqkv[l], nullptr, ncols, d, true));  // group-blocked q|k|v
      m->wt_o.push_back(place(w->wo[l], nullptr, d, hh));
      m->wt_gu.push_back(place(w->wgate[l], w->wup[l], c.ffn, d));
      m->wt_d.push_back(place(w->wdown[l], nullptr, d, c.ffn));
    }
    m->wt_lm = place(w->lm_head, nullptr, c.vocab, d);
    if (e == cudaSuccess) {  // persistent forward: packed norms + GEMM kinds (kernel parameters)
      const size_t dbytes = (size_t)d * 2;
      for (int l = 0; l < c.n_layers && e == cudaSuccess; ++l) {
        e = cudaMemcpy(m->fw_norms + (size_t)(2 * l) * d, w->attn_norm[l], dbytes, cudaMemcpyDeviceToDevice);
        if (e == cudaSuccess)
          e = cudaMemcpy(m->fw_norms + (size_t)(2 * l + 1) * d, w->mlp_norm[l], dbytes, cudaMemcpyDeviceToDevice);
      }
      if (e == cudaSuccess)
        e = cudaMemcpy(m->fw_norms + (size_t)(2 * c.n_layers) * d, w->final_norm, dbytes, cudaMemcpyDeviceToDevice);
      fw::ModelView v{};
      v.d = d; v.H = c.n_heads; v.KV = c.n_kv_heads; v.hd = c.head_dim; v.ffn = c.ffn; v.vocab = c.vocab;
      v.L = c.n_layers; v.S = c.max_seq;
      v.fuse = fw_fuse();
      v.wt_layer0 = m->wt_qkv[0];
      v.wt_layer_bytes = c.n_layers > 1 ? (long long)(m->wt_qkv[1] - m->wt_qkv[0]) : 0;
      v.wt_lm = m->wt_lm; v.norms = m->fw_norms;
      v.h = m->h; v.qkv = m->qkv; v.xa = m->xa_b; v.act_b = m->act_b;
      v.xb = m->fw_xb; v.ssp = m->ssp; v.sspb = m->fw_sspb;
      view_shard(&v, sh);
      size_t wsf;
      int mt, cints;
      if (!fw::build_kinds(v, fw_units(), &m->fw_args, &wsf, &cints, &mt)) {
        delete m;
        return fail(AMUSD_ERR_UNSUPPORTED, "tensor-parallel shard: a rank's O / down K slice is not a whole number of "
                                           "the unsharded model's split-K chunks (set AMUSD_FW_UNITS_O / _DOWN)");
      }
      if (sh) { m->fw_args.vocab_off = sh->vocab_offset; m->fw_args.tp = 1; }  // tp = n at amusd_tp_connect
      m->fw_view = v;
      m->fw_ready = e == cudaSuccess && c.max_seq <= fw::max_positions();  // else the per-kernel path
      m->fw_grid = model_sms(m);
      m->fw_stages = env_int("AMUSD_FW_STAGES", fw_max_stages(c, 1));
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    ok &= tc::make_map(&m->map_xa, m->xa_b, KMAX, d, KMAX);
    ok &= tc::make_map(&m->map_attn, m->attn_b, KMAX, hh, KMAX);
    ok &= tc::make_map(&m->map_act, m->act_b, KMAX, c.ffn, KMAX);
    ok &= tc::make_map(&m->map_xb, m->fw_xb, KMAX, d, KMAX);
    if (!ok || e != cudaSuccess) {
      delete m;
      return fail(AMUSD_ERR_CUDA, std::string("tcgen05 path setup failed: ") +
                                      (e != cudaSuccess ? cudaGetErrorString(e) : "cuTensorMapEncodeTiled"));
    }
  }
  if (sh && !m->fw_ready) {
    delete m;
    return fail(AMUSD_ERR_UNSUPPORTED, "tensor-parallel shard needs the persistent forward (max_seq too long?)");
  }
  *out = m;
  return AMUSD_OK;
}

extern "C" {

int amusd_tf_create(amusd_model** out, const amusd_tf_config* cfg, const amusd_tf_weights* w, void* state,
                    size_t state_bytes) {
  return tf_create(out, cfg, nullptr, w, state, state_bytes);
}
int amusd_tf_create_shard(amusd_model** out, const amusd_tf_config* cfg, const amusd_tp_shard* shard,
                          const amusd_tf_weights* w, void* state, size_t state_bytes) {
  if (!shard) return fail(AMUSD_ERR_INVALID_INPUT, "null shard");
  return tf_create(out, cfg, shard, w, state, state_bytes);
}

int amusd_peer_enable(int device, int peer) {
  if (device == peer) return AMUSD_OK;
  int ok = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&ok, device, peer));
  if (!ok) return fail(AMUSD_ERR_UNSUPPORTED, "no peer access between the two GPUs");
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); e = cudaSuccess; }
  cudaSetDevice(cur);
  CUDA_TRY(e);
  return AMUSD_OK;
}

int amusd_tp_export(amusd_model* m, amusd_tp_peer* out) {
  if (!m || !out) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (m->kind != 0 || m->tp.tp_size < 2) return fail(AMUSD_ERR_INVALID_INPUT, "not a tensor-parallel shard");
  *out = amusd_tp_peer{};
  out->ws = m->fw_ws; out->tile_cnt = m->fw_tile_cnt; out->best = m->fw_best; out->sched = m->fw_sched;
  out->lm_items = m->fw_args.g[fw::kGLm].nitems;
  return AMUSD_OK;
}

int amusd_tp_connect(amusd_model* m, const amusd_tp_peer* peers, int n) {
  if (!m || !peers) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (m->kind != 0 || m->tp.tp_size < 2) return fail(AMUSD_ERR_INVALID_INPUT, "not a tensor-parallel shard");
  if (n != m->tp.tp_size) return fail(AMUSD_ERR_INVALID_INPUT, "need one peer entry per rank (n == tp_size)");
  if (peers[m->tp.tp_rank].ws != (void*)m->fw_ws || peers[m->tp.tp_rank].sched != (void*)m->fw_sched)
    return fail(AMUSD_ERR_INVALID_INPUT, "peers[tp_rank] must be this shard's own words");
  int lm = 0;
  for (int i = 0; i < n; ++i) {
    if (!peers[i].ws || !peers[i].tile_cnt || !peers[i].best || !peers[i].sched || peers[i].lm_items < 1)
      return fail(AMUSD_ERR_INVALID_INPUT, "incomplete peer entry");
    m->fw_args.peer_ws[i] = (unsigned long long*)peers[i].ws;
    m->fw_args.peer_cnt[i] = (int*)peers[i].tile_cnt;
    m->fw_args.peer_best[i] = (unsigned long long*)peers[i].best;
    m->fw_args.peer_sched[i] = (int*)peers[i].sched;
    lm += peers[i].lm_items;
  }
  m->fw_args.tp = n;
  m->fw_args.lm_items_total = lm;
  m->tp_connected = true;
  return AMUSD_OK;
}

size_t amusd_hash_state_bytes(int max_seq) { return hash_carve(max_seq, nullptr, nullptr); }

int amusd_hash_create(amusd_model** out, uint64_t seed, int vocab, int eos, int exclude_eos, double rho,
                      int max_seq, void* state, size_t state_bytes) {
  if (!out || !state) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (vocab < 2) return fail(AMUSD_ERR_INVALID_INPUT, "vocab_size must be >= 2");  // models.py:96
  if (!(0 <= eos && eos < vocab)) return fail(AMUSD_ERR_INVALID_INPUT, "eos_token out of range");
  if (exclude_eos && vocab < 3) return fail(AMUSD_ERR_INVALID_INPUT, "exclude_eos requires vocab_size >= 3");
  if (max_seq < 2) return fail(AMUSD_ERR_INVALID_INPUT, "max_seq must be >= 2");
  if (rho > 1.0) return fail(AMUSD_ERR_INVALID_INPUT, "agreement_rho must be in [0, 1]");  // models.py:290
  if (rho >= 0.0 && rho < 1.0 && vocab - (exclude_eos ? 1 : 0) < 2)
    return fail(AMUSD_ERR_INVALID_INPUT, "vocabulary too small to hold a disagreeing token alternative");
  if (state_bytes < amusd_hash_state_bytes(max_seq)) return fail(AMUSD_ERR_INVALID_INPUT, "state buffer too small");
  amusd_model* m = new amusd_model();
  m->kind = 1;
  m->seed = seed;
  m->vocab = vocab;
  m->eos = eos;
  m->exclude_eos = exclude_eos;
  m->max_seq = max_seq;
  m->agree = rho >= 0.0;
  m->agree_always = rho >= 1.0;
  m->agree_thr = m->agree_always ? ~0ull : (rho >= 0.0 ? (unsigned long long)(rho * 18446744073709551616.0) : 0ull);
  hash_carve(max_seq, state, m);
  *out = m;
  return AMUSD_OK;
}

size_t amusd_scripted_state_bytes(int max_seq, int script_len) {
  return hash_carve(max_seq, nullptr, nullptr, std::max(script_len, 1));
}

int amusd_scripted_create(amusd_model** out, const int32_t* script, int script_len, int vocab, int eos,
                          int eos_position, int max_seq, void* state, size_t state_bytes, void* stream) {
  if (!out || !state || !script) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (vocab < 2) return fail(AMUSD_ERR_INVALID_INPUT, "vocab_size must be >= 2");  // models.py:96
  if (!(0 <= eos && eos < vocab)) return fail(AMUSD_ERR_INVALID_INPUT, "eos_token out of range");
  if (script_len < 1) return fail(AMUSD_ERR_INVALID_INPUT, "script must contain at least one token");  // models.py:333
  for (int i = 0; i < script_len; ++i)
    if (script[i] < 0 || script[i] >= vocab)
      return fail(AMUSD_ERR_INVALID_INPUT, "token " + std::to_string(script[i]) + " out of vocabulary range [0, " +
                                               std::to_string(vocab) + ")");
  if (eos_position < 0) return fail(AMUSD_ERR_INVALID_INPUT, "eos_position must be >= 1");  // models.py:336 (0 = none)
  if (max_seq < 2) return fail(AMUSD_ERR_INVALID_INPUT, "max_seq must be >= 2");
  if (state_bytes < amusd_scripted_state_bytes(max_seq, script_len))
    return fail(AMUSD_ERR_INVALID_INPUT, "state buffer too small");
  amusd_model* m = new amusd_model();
  m->kind = 1;
  m->vocab = vocab;
  m->eos = eos;
  m->max_seq = max_seq;
  m->script_len = script_len;
  m->eos_position = eos_position;
  hash_carve(max_seq, state, m, script_len);
  cudaError_t e = cudaMemcpyAsync(m->script, script, sizeof(int) * script_len, cudaMemcpyHostToDevice,
                                  (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    delete m;
    return fail(AMUSD_ERR_CUDA, std::string("script upload: ") + cudaGetErrorString(e));
  }
  *out = m;
  return AMUSD_OK;
}

int amusd_model_destroy(amusd_model* m) {
  delete m;
  return AMUSD_OK;
}

int amusd_model_set_timeline(amusd_model* m, void* buf, size_t bytes) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  m->fw_dbg = (long long*)buf;
  m->fw_dbg_items = buf ? (int)std::min<size_t>(bytes / 64, 1 << 20) : 0;
  return AMUSD_OK;
}

int amusd_model_set_path(amusd_model* m, int path) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (path < AMUSD_PATH_PERSISTENT || path > AMUSD_PATH_CLUSTER) return fail(AMUSD_ERR_INVALID_INPUT, "unknown path");
  if (path == AMUSD_PATH_CLUSTER && (m->kind != 0 || !m->cl_ok))
    return fail(AMUSD_ERR_UNSUPPORTED, "the cluster decode forward needs a bf16 model with d_model <= 2048 (64-multiple), "
                                       "16-row output blocks, head_dim 64/128 and <= 8 query heads per KV head");
  if (path == AMUSD_PATH_CLUSTER && !m->cl_wt)
    return fail(AMUSD_ERR_INVALID_INPUT, "attach the cluster decode weight layout first (amusd_model_set_cluster)");
  if (path == AMUSD_PATH_DECODE && (m->kind != 0 || !m->gv_ok))
    return fail(AMUSD_ERR_UNSUPPORTED, "the decode forward needs a bf16 model with 64-multiple GEMV widths, 16-row "
                                       "output blocks, head_dim 64/128 and <= 8 query heads per KV head");
  if (path == AMUSD_PATH_DECODE && !m->gv_wt)
    return fail(AMUSD_ERR_INVALID_INPUT, "attach the decode weight layout first (amusd_model_set_decode)");
  if (path != AMUSD_PATH_SIMT && m->kind == 0 && !m->tc)
    return fail(AMUSD_ERR_UNSUPPORTED, "tensor-core paths need a bf16 model with 128-aligned shapes");
  if (m->kind == 0 && path != AMUSD_PATH_PERSISTENT && !m->row_major)
    return fail(AMUSD_ERR_UNSUPPORTED, "the row-major weights were released: only the persistent path remains");
  m->path = path;
  return AMUSD_OK;
}

size_t amusd_cluster_bytes(amusd_model* m) {
  if (!m || m->kind != 0 || !m->cl_ok) return 0;
  const amusd_tf_config& c = m->cfg;
  return (size_t)cl::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers).total;
}

int amusd_model_set_cluster(amusd_model* m, void* buf, size_t bytes) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (!buf) {
    if (m->path == AMUSD_PATH_CLUSTER) return fail(AMUSD_ERR_INVALID_INPUT, "the cluster decode path is selected");
    m->cl_wt = nullptr;
    return AMUSD_OK;
  }
  if (m->kind != 0 || !m->cl_ok) return fail(AMUSD_ERR_UNSUPPORTED, "this model's shapes do not take the cluster decode");
  if (!m->row_major) return fail(AMUSD_ERR_UNSUPPORTED, "the row-major weights were released");
  if (bytes < amusd_cluster_bytes(m)) return fail(AMUSD_ERR_INVALID_INPUT, "cluster decode weight buffer too small");
  const amusd_tf_config& c = m->cfg;
  const cl::Layout t = cl::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers);
  uint8_t* dst = (uint8_t*)buf;
  for (int l = 0; l < c.n_layers; ++l)
    CUDA_TRY(cl::tile_layer(m->w.wqkv[l], m->w.wo[l], m->w.wgate[l], m->w.wup[l], m->w.wdown[l], c.d_model, c.n_heads,
                            c.n_kv_heads, c.head_dim, c.ffn, dst + (size_t)l * t.layer_bytes, 0));
  CUDA_TRY(cl::tile_lm(m->w.lm_head, c.vocab, c.d_model, dst + t.lm_off, 0));
  CUDA_TRY(cudaDeviceSynchronize());
  m->cl_wt = dst;
  return AMUSD_OK;
}

size_t amusd_decode_bytes(amusd_model* m) {
  if (!m || m->kind != 0 || !m->gv_ok) return 0;
  const amusd_tf_config& c = m->cfg;
  return (size_t)gv::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers).total;
}

int amusd_model_set_decode(amusd_model* m, void* buf, size_t bytes) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (!buf) {
    if (m->path == AMUSD_PATH_DECODE) return fail(AMUSD_ERR_INVALID_INPUT, "the decode path is selected");
    m->gv_wt = nullptr;
    return AMUSD_OK;
  }
  if (m->kind != 0 || !m->gv_ok)
    return fail(AMUSD_ERR_UNSUPPORTED, "this model's shapes do not take the decode forward");
  if (!m->row_major) return fail(AMUSD_ERR_UNSUPPORTED, "the row-major weights were released");
  if (bytes < amusd_decode_bytes(m)) return fail(AMUSD_ERR_INVALID_INPUT, "decode weight buffer too small");
  const amusd_tf_config& c = m->cfg;
  const gv::Layout t = gv::layout(c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn, c.vocab, c.n_layers);
  uint8_t* dst = (uint8_t*)buf;
  const int ncols = (c.n_heads + 2 * c.n_kv_heads) * c.head_dim, hh = c.n_heads * c.head_dim;
  for (int l = 0; l < c.n_layers; ++l) {
    uint8_t* lw = dst + (size_t)l * t.layer_bytes;
    CUDA_TRY(gv::tile_weights(m->w.wqkv[l], nullptr, ncols, c.d_model, lw, 0));
    CUDA_TRY(gv::tile_weights(m->w.wo[l], nullptr, c.d_model, hh, lw + t.off_o, 0));
    CUDA_TRY(gv::tile_weights(m->w.wgate[l], m->w.wup[l], 2 * c.ffn, c.d_model, lw + t.off_gu, 0));
    CUDA_TRY(gv::tile_weights(m->w.wdown[l], nullptr, c.d_model, c.ffn, lw + t.off_down, 0));
  }
  CUDA_TRY(gv::tile_weights(m->w.lm_head, nullptr, c.vocab, c.d_model, dst + t.lm_off, 0));
  CUDA_TRY(cudaDeviceSynchronize());
  m->gv_wt = dst;
  return AMUSD_OK;
}

int amusd_model_release_row_major(amusd_model* m) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (m->kind != 0 || !m->tc || !m->fw_ready)
    return fail(AMUSD_ERR_UNSUPPORTED, "only a tensor-core model on the persistent path can drop its row-major weights");
  if (m->path != AMUSD_PATH_PERSISTENT)
    return fail(AMUSD_ERR_UNSUPPORTED, "row-major weights are in use by the selected forward path");
  CUDA_TRY(cudaDeviceSynchronize());  // no launch in flight reads them
  for (int l = 0; l < m->cfg.n_layers; ++l)
    m->w.wqkv[l] = m->w.wo[l] = m->w.wgate[l] = m->w.wup[l] = m->w.wdown[l] = nullptr;
  if (m->w.lm_head != m->w.embed) m->w.lm_head = nullptr;
  m->row_major = false;
  return AMUSD_OK;
}

size_t amusd_prefill_bytes(amusd_model* m, int max_tokens) {
  if (!m || m->kind != 0 || max_tokens < 1) return 0;
  const amusd_tf_config& c = m->cfg;
  return pf::work_bytes(max_tokens, c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn);
}

int amusd_model_set_prefill(amusd_model* m, void* buf, size_t bytes, int max_tokens) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (!buf) { m->pf_ready = false; return AMUSD_OK; }
  if (m->kind != 0 || !m->tc || !m->fw_ready)
    return fail(AMUSD_ERR_UNSUPPORTED, "the prefill runs bf16 tcgen05 transformer models only");
  if (max_tokens < 1 || bytes < amusd_prefill_bytes(m, max_tokens))
    return fail(AMUSD_ERR_INVALID_INPUT, "prefill buffer too small");
  const amusd_tf_config& c = m->cfg;
  pf::carve(&m->pf, buf, max_tokens, c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn);
  if (!pf::make_maps(&m->pf, c.d_model, c.n_heads * c.head_dim, c.ffn))
    return fail(AMUSD_ERR_CUDA, "prefill tensor maps (cuTensorMapEncodeTiled) failed");
  m->pf_ready = true;
  return AMUSD_OK;
}

int amusd_model_set_max_grid(amusd_model* m, int sms) {
  if (!m || sms < 0) return fail(AMUSD_ERR_INVALID_INPUT, "bad argument");
  if (m->kind != 0) return AMUSD_OK;
  m->max_grid = sms;
  if (m->fw_ready) m->fw_grid = model_sms(m);
  return AMUSD_OK;
}

int amusd_model_set_grid(amusd_model* m, int sms) {
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (sms < 0 || sms > num_sms()) return fail(AMUSD_ERR_INVALID_INPUT, "sms out of range");
  m->grid_override = sms;
  return AMUSD_OK;
}

}  // extern "C"

// ------------------------------------------------- MockModel parity path
static int sync_from_device(amusd_model* m, cudaStream_t st) {
  if (!m->dirty) return AMUSD_OK;
  SeqHdr h;
  CUDA_TRY(cudaMemcpyAsync(&h, m->seq, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  m->htok.resize(h.len);
  if (h.len) CUDA_TRY(cudaMemcpyAsync(m->htok.data(), m->tok, sizeof(int) * h.len, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  m->len = h.len;
  m->kv_len = h.kv_len;
  m->pred_valid = false;
  m->dirty = false;
  return AMUSD_OK;
}

static int push_header(amusd_model* m, cudaStream_t st) {
  SeqHdr h{};
  h.len = m->len;
  h.kv_len = m->kv_len;
  h.prompt_len = m->prompt_len;
  h.cap = m->max_seq;
  h.pred_valid = 0;
  CUDA_TRY(cudaMemcpyAsync(m->seq, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  return AMUSD_OK;
}

// Forward explicit rows (positions pos0..) on the model's API control block;
// returns the predictions (host) after a stream sync.
static int api_forward(amusd_model* m, int pos0, const int* rows_tok, int rows, int* preds, cudaStream_t st) {
  StepCtl c{};
  c.active = 1;
  c.rows = rows;
  c.pos0 = pos0;
  c.npend = rows;
  for (int i = 0; i < rows; ++i) c.tok[i] = rows_tok[i];
  CUDA_TRY(cudaMemcpyAsync(m->api_ctl, &c, sizeof(c), cudaMemcpyHostToDevice, st));
  // tensor-core models always run the 16-row tcgen05 forward (identical
  // arithmetic to the engines' verify steps); SIMT models pick 2 or 16 rows,
  // which give identical per-row results (same per-lane k order).
  const int nr = (m->tc || rows > 2) ? KMAX : 2;
  int r = model_forward(m, m->api_ctl, nr, st, false, true);
  if (r) return r;
  m->last_rows = rows;
  if (preds) {
    CUDA_TRY(cudaMemcpyAsync(preds, m->api_ctl->preds, sizeof(int) * rows, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  return AMUSD_OK;
}

// Prompt positions [0, n) into the KV cache as dense GEMMs over all n tokens (prefill.cu):
// the decode forward would re-stream every weight once per 16 positions.
static int prefill_forward(amusd_model* m, int n, cudaStream_t st) {
  const amusd_tf_config& c = m->cfg;
  pf::Work& W = m->pf;
  const int d = c.d_model, H = c.n_heads, KV = c.n_kv_heads, hd = c.head_dim, L = c.n_layers;
  const int ncols = (H + 2 * KV) * hd, hh = H * hd;
  auto gemm = [&](const CUtensorMap& mx, const uint8_t* wt, int ntiles, int K, int epi, float* out,
                  __nv_bfloat16* out_b, int ldo) -> cudaError_t {
    pf::GemmArgs g{};
    g.wt = wt; g.ntiles = ntiles; g.kb = K / 64; g.M = n; g.epi = epi; g.out = out; g.out_b = out_b; g.ldo = ldo;
    g.inv = W.inv;
    return pf::launch_gemm(mx, g, st);
  };
  CUDA_TRY(pf::launch_embed(m->tok, (const __nv_bfloat16*)m->w.embed, W.h, n, d, st));
  for (int l = 0; l < L; ++l) {
    __nv_bfloat16* kc = (__nv_bfloat16*)m->kc + (size_t)l * m->kv_layer_elems;
    __nv_bfloat16* vc = (__nv_bfloat16*)m->vc + (size_t)l * m->kv_layer_elems;
    CUDA_TRY(pf::launch_norm(W.h, m->fw_norms + (size_t)(2 * l) * d, W.x, W.inv, n, d, c.norm_eps, st));
    CUDA_TRY(gemm(W.map_x_d, m->wt_qkv[l], ncols / 128, d, pf::kEpStoreScaled, W.qkv, nullptr, ncols));
    CUDA_TRY(pf::launch_rope_kv(W.qkv, m->w.rope_cos, m->w.rope_sin, kc, vc, n, H, KV, hd, c.max_seq, st));
    if (l == L - 1) break;  // the last layer's K / V is all the decode steps need
    CUDA_TRY(pf::launch_attention(W.qkv, kc, vc, W.x, n, H, KV, hd, c.max_seq, 1.0f / sqrtf((float)hd), st));
    CUDA_TRY(gemm(W.map_x_hh, m->wt_o[l], d / 128, hh, pf::kEpResid, W.h, nullptr, d));
    CUDA_TRY(pf::launch_norm(W.h, m->fw_norms + (size_t)(2 * l + 1) * d, W.x, W.inv, n, d, c.norm_eps, st));
    CUDA_TRY(gemm(W.map_x_d, m->wt_gu[l], c.ffn / 64, d, pf::kEpGateUp, nullptr, W.act, c.ffn));
    CUDA_TRY(gemm(W.map_act, m->wt_d[l], d / 128, c.ffn, pf::kEpResid, W.h, nullptr, d));
  }
  return AMUSD_OK;
}

static int prefill_min_tokens() {
  static int v = -1;
  if (v < 0) v = std::max(1, env_int("AMUSD_PREFILL_MIN", 64));
  return v;
}

// Bring the cache up to len-1 (at most `keep` pending tokens stay uncached).
static int catch_up(amusd_model* m, int keep, cudaStream_t st) {
  if (m->kv_len >= m->len) m->kv_len = m->len - 1;
  const int todo = m->len - keep - m->kv_len;
  if (m->pf_ready && m->kv_len == 0 && m->tp.tp_size < 2 && m->tc && m->fw_ready && todo >= prefill_min_tokens() &&
      todo <= m->pf.max_tokens) {
    if (int r = prefill_forward(m, todo, st)) return r;
    m->kv_len = todo;
  }
  while (m->len - m->kv_len > keep) {
    const int rows = std::min(max_rows(m), m->len - m->kv_len - keep);
    int r = api_forward(m, m->kv_len, m->htok.data() + m->kv_len, rows, nullptr, st);
    if (r) return r;
    m->kv_len += rows;
  }
  return AMUSD_OK;
}

static int validate_tokens(const amusd_model* m, const int32_t* t, int n) {
  for (int i = 0; i < n; ++i)
    if (t[i] < 0 || t[i] >= m->vocab)
      return fail(AMUSD_ERR_INVALID_INPUT, "token " + std::to_string(t[i]) + " out of vocabulary range [0, " +
                                               std::to_string(m->vocab) + ")");
  return AMUSD_OK;
}

extern "C" {

int amusd_init_state(amusd_model* m, const int32_t* prompt, int n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (n <= 0) return fail(AMUSD_ERR_INVALID_INPUT, "prompt must be non-empty");  // models.py:111
  if (int r = validate_tokens(m, prompt, n)) return r;
  if (n + 1 > m->max_seq) return fail(AMUSD_ERR_INVALID_INPUT, "prompt exceeds max_seq");
  m->htok.assign(prompt, prompt + n);
  m->prompt_len = n;
  m->len = n;
  m->kv_len = 0;
  m->pred_valid = false;
  m->dirty = false;
  CUDA_TRY(cudaMemcpyAsync(m->tok, prompt, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  if (m->kind == 1) CUDA_TRY(launch_hash_seed(m->chain, m->seed, st));
  if (int r = catch_up(m, 1, st)) return r;
  if (int r = push_header(m, st)) return r;
  CUDA_TRY(cudaStreamSynchronize(st));
  return AMUSD_OK;
}

int amusd_next_token(amusd_model* m, int32_t* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m || !out) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (int r = sync_from_device(m, st)) return r;
  if (m->pred_valid) { *out = m->pred; return AMUSD_OK; }
  if (int r = catch_up(m, max_rows(m), st)) return r;
  const int rows = m->len - m->kv_len;
  int preds[KMAX];
  if (int r = api_forward(m, m->kv_len, m->htok.data() + m->kv_len, rows, preds, st)) return r;
  m->kv_len = m->len;
  m->pred = preds[rows - 1];
  m->pred_valid = true;
  *out = m->pred;
  return push_header(m, st);
}

int amusd_advance(amusd_model* m, const int32_t* tokens, int n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (int r = sync_from_device(m, st)) return r;
  if (n <= 0) return fail(AMUSD_ERR_INVALID_INPUT, "advance requires at least one token");  // models.py:128
  if (int r = validate_tokens(m, tokens, n)) return r;
  if (m->len + n + 1 > m->max_seq) return fail(AMUSD_ERR_INVALID_INPUT, "sequence exceeds max_seq");
  CUDA_TRY(cudaMemcpyAsync(m->tok + m->len, tokens, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  m->htok.insert(m->htok.end(), tokens, tokens + n);
  m->len += n;
  m->pred_valid = false;
  if (int r = push_header(m, st)) return r;
  CUDA_TRY(cudaStreamSynchronize(st));
  return AMUSD_OK;
}

int amusd_rollback(amusd_model* m, int position, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m) return fail(AMUSD_ERR_INVALID_INPUT, "null model");
  if (int r = sync_from_device(m, st)) return r;
  if (position > m->len)  // models.py:140-147
    return fail(AMUSD_ERR_INVALID_ROLLBACK, "rollback position " + std::to_string(position) +
                                                " exceeds prefix length " + std::to_string(m->len));
  if (position < m->prompt_len)
    return fail(AMUSD_ERR_INVALID_ROLLBACK, "rollback position " + std::to_string(position) +
                                                " is below prompt length " + std::to_string(m->prompt_len));
  if (position == m->len) return AMUSD_OK;
  m->len = position;
  m->htok.resize(position);
  m->kv_len = std::min(m->kv_len, position);  // cache-length truncate, no copy
  m->pred_valid = false;
  if (int r = push_header(m, st)) return r;
  CUDA_TRY(cudaStreamSynchronize(st));
  return AMUSD_OK;
}

int amusd_verify_tokens(amusd_model* m, const int32_t* cands, int n, int32_t* preds, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m || !preds) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (int r = sync_from_device(m, st)) return r;
  if (n <= 0) return fail(AMUSD_ERR_INVALID_INPUT, "verify_tokens requires at least one candidate");
  if (int r = validate_tokens(m, cands, n)) return r;
  if (m->len + n + 1 > m->max_seq) return fail(AMUSD_ERR_INVALID_INPUT, "sequence exceeds max_seq");
  if (int r = catch_up(m, 1, st)) return r;
  // rows: [pending, c_0 .. c_{n-2}] in chunks of KMAX; chunk i continues at
  // the positions after chunk i-1 (teacher forcing; cache beyond len is scratch)
  std::vector<int> rows_tok;
  rows_tok.push_back(m->htok[m->len - 1]);
  for (int j = 0; j + 1 < n; ++j) rows_tok.push_back(cands[j]);
  int pos = m->kv_len, done = 0;
  int buf[KMAX];
  while (done < (int)rows_tok.size()) {
    const int rows = std::min(max_rows(m), (int)rows_tok.size() - done);
    if (int r = api_forward(m, pos, rows_tok.data() + done, rows, buf, st)) return r;
    for (int i = 0; i < rows; ++i) preds[done + i] = buf[i];
    done += rows;
    pos += rows;
  }
  m->kv_len = m->len;
  m->pred = preds[0];
  m->pred_valid = true;
  return push_header(m, st);
}

int amusd_prefix_length(amusd_model* m, int* out) {
  if (!m || !out) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (int r = sync_from_device(m, 0)) return r;
  *out = m->len;
  return AMUSD_OK;
}

int amusd_last_logits(amusd_model* m, float* out, int rows, void* stream) {
  if (!m || !out) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (m->kind != 0) return fail(AMUSD_ERR_UNSUPPORTED, "logits exist only for transformer models");
  rows = std::min(rows, m->last_rows);
  CUDA_TRY(cudaMemcpyAsync(out, m->logits, sizeof(float) * (size_t)rows * m->cfg.vocab, cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return AMUSD_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ session
struct amusd_session {
  amusd_model* draft = nullptr;
  amusd_model* verify = nullptr;
  amusd_session_desc d{};
  int cap = 0;
  MailboxHdr* mb_local = nullptr;
  MailboxHdr* mb_peer = nullptr;
  StepCtl* dctl = nullptr;
  StepCtl* vctl = nullptr;
  TraceDev dtrace{}, vtrace{};
  CoinDev coin{};
  int* prompt_dev = nullptr;
  int prompt_cap = 0;
  cudaStream_t capture = nullptr;
  cudaGraphExec_t exec[5][2] = {};
  bool use_pdl = true;
  // tensor-parallel verify group (amusd_session_set_tp): 1 leader, 2 follower
  int tp_role = 0;
  TpInbox* tp_inbox = nullptr;  // this session's inbox (carved; used when a follower)
  TpInbox* tp_out[kMaxTpOut] = {};
  int tp_nout = 0;
};

static int mailbox_cap(const amusd_session_desc* d) { return d->max_new_tokens + 4 * KMAX + 64; }

static size_t session_carve(const amusd_session_desc* d, int coin_cap, int prompt_cap, void* base,
                            amusd_session* s) {
  Carver cv(base);
  StepCtl* dctl = cv.take<StepCtl>(1);
  StepCtl* vctl = cv.take<StepCtl>(1);
  amusd_trace_event* dev = cv.take<amusd_trace_event>(d->trace_cap);
  amusd_trace_event* vev = cv.take<amusd_trace_event>(d->trace_cap);
  int* counts = cv.take<int>(2);
  unsigned long long* hash = cv.take<unsigned long long>(coin_cap + 2);
  unsigned char* onpath = cv.take<unsigned char>(coin_cap + 2);
  int* prompt = cv.take<int>(prompt_cap);
  TpInbox* inbox = cv.take<TpInbox>(1);
  if (s) {
    s->tp_inbox = inbox;
    s->dctl = dctl; s->vctl = vctl;
    s->dtrace = TraceDev{dev, counts, d->trace_cap};
    s->vtrace = TraceDev{vev, counts + 1, d->trace_cap};
    s->coin.hash = hash; s->coin.onpath = onpath;
    s->prompt_dev = prompt; s->prompt_cap = prompt_cap;
  }
  return align_up(cv.off, 256);
}

static int session_max_seq(const amusd_session_desc* d) { return d->prompt_len + mailbox_cap(d) + 8; }

static ProtoArgs make_args(amusd_session* s) {
  ProtoArgs a{};
  a.mb_local = s->mb_local;
  a.mb_peer = s->mb_peer;
  a.cap = s->cap;
  a.P = s->d.prompt_len;
  a.N = s->d.max_new_tokens;
  a.lead = s->d.max_draft_lead;
  a.max_window = s->d.max_window;
  a.k = s->d.draft_window_k;
  if (s->draft) { a.dseq = s->draft->seq; a.dtok = s->draft->tok; }
  if (s->verify) { a.vseq = s->verify->seq; a.vtok = s->verify->tok; a.vocab_v = s->verify->vocab; a.eos_v = s->verify->eos; }
  a.dctl = s->dctl;
  a.vctl = s->vctl;
  a.dtrace = s->dtrace;
  a.vtrace = s->vtrace;
  a.coin = s->coin;
  a.jitter_ns = s->d.jitter_ns;
  a.jitter_seed = s->d.jitter_seed;
  a.min_window = std::max(1, env_int("AMUSD_VERIFY_MIN_WINDOW", 1));
  a.wait_ns = 1000ll * env_int("AMUSD_VERIFY_WAIT_US", 0);
  if (s->tp_role == 1) {
    for (int i = 0; i < s->tp_nout; ++i) a.tp_out[i] = s->tp_out[i];
    a.tp_nout = s->tp_nout;
  } else if (s->tp_role == 2) {
    a.tp_in = s->tp_inbox;
  }
  return a;
}

extern "C" {

size_t amusd_mailbox_bytes(int capacity_tokens) { return mailbox_bytes(capacity_tokens); }
int amusd_mailbox_capacity(const amusd_session_desc* d) { return d ? mailbox_cap(d) : 0; }

size_t amusd_session_bytes(const amusd_session_desc* d) {
  if (!d) return 0;
  return session_carve(d, session_max_seq(d), std::max(d->prompt_len, 1), nullptr, nullptr);
}

int amusd_session_create(amusd_session** out, amusd_model* draft, amusd_model* verify, const amusd_session_desc* d,
                         void* mem, size_t mem_bytes, void* mb_local, void* mb_peer) {
  if (!out || !d || !mem || !mb_local) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (!draft && !verify) return fail(AMUSD_ERR_INVALID_INPUT, "session needs a draft or a verify model");
  // a device model holds ONE sequence (KV cache, schedule counters, split-K workspace):
  // the same handle as both draft and verify would run two forwards over the same state
  if (draft == verify)
    return fail(AMUSD_ERR_INVALID_INPUT, "draft and verify must be distinct device models (one sequence per model)");
  if (d->prompt_len < 1) return fail(AMUSD_ERR_INVALID_INPUT, "prompt_length must be >= 1");
  if (d->max_new_tokens < 1) return fail(AMUSD_ERR_INVALID_INPUT, "max_new_tokens must be >= 1");
  if (d->draft_window_k < 1 || d->draft_window_k > KMAX - 1)
    return fail(AMUSD_ERR_INVALID_INPUT, "draft_window_k must be in [1, 15]");
  if (d->max_draft_lead < 0) return fail(AMUSD_ERR_INVALID_INPUT, "max_draft_lead must be >= 1 when set");
  if (d->max_window < 1 || d->max_window > KMAX) return fail(AMUSD_ERR_INVALID_INPUT, "max_window must be in [1, 16]");
  if (d->rho < 0.0 || d->rho > 1.0) return fail(AMUSD_ERR_INVALID_INPUT, "rho must be in [0, 1]");
  if (d->trace_cap < 1) return fail(AMUSD_ERR_INVALID_INPUT, "trace_cap must be >= 1");
  if (mem_bytes < amusd_session_bytes(d)) return fail(AMUSD_ERR_INVALID_INPUT, "session buffer too small");
  const int need = d->prompt_len + d->max_new_tokens + KMAX + 2;
  if (verify && verify->max_seq < need) return fail(AMUSD_ERR_INVALID_INPUT, "verify max_seq too small for prompt + max_new_tokens");
  if (draft && draft->max_seq < need) return fail(AMUSD_ERR_INVALID_INPUT, "draft max_seq too small for prompt + max_new_tokens");
  amusd_session* s = new amusd_session();
  s->draft = draft;
  s->verify = verify;
  s->d = *d;
  s->cap = mailbox_cap(d);
  s->mb_local = (MailboxHdr*)mb_local;
  s->mb_peer = mb_peer ? (MailboxHdr*)mb_peer : (MailboxHdr*)mb_local;
  session_carve(d, session_max_seq(d), std::max(d->prompt_len, 1), mem, s);
  s->coin.mode = draft ? d->coin_mode : AMUSD_COIN_NONE;
  s->coin.always = d->rho >= 1.0;  // int(1.0 * 2**64) == 2**64 > every hash
  s->coin.thr = s->coin.always ? ~0ull : (unsigned long long)(d->rho * 18446744073709551616.0);
  if (draft) { s->coin.vocab = draft->vocab; s->coin.eos = draft->eos; s->coin.exclude_eos = draft->exclude_eos; }
  s->coin.canon = d->canon;
  s->coin.canon_len = d->canon ? d->canon_len : 0;
  if (s->coin.mode == AMUSD_COIN_NONE) { s->coin.hash = nullptr; s->coin.onpath = nullptr; }
  const char* nopdl = getenv("AMUSD_NO_PDL");
  s->use_pdl = !(nopdl && nopdl[0] == '1');
  if (cudaStreamCreateWithFlags(&s->capture, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    return fail(AMUSD_ERR_CUDA, "stream create failed");
  }
  *out = s;
  return AMUSD_OK;
}

int amusd_session_tp_inbox(amusd_session* s, void** out) {
  if (!s || !out) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  *out = s->tp_inbox;
  return AMUSD_OK;
}

int amusd_session_set_tp(amusd_session* s, int role, void* const* followers, int n) {
  if (!s) return fail(AMUSD_ERR_INVALID_INPUT, "null session");
  if (role < 0 || role > 2) return fail(AMUSD_ERR_INVALID_INPUT, "role must be 0 (none), 1 (leader) or 2 (follower)");
  if (role != 0 && !s->verify) return fail(AMUSD_ERR_INVALID_INPUT, "tensor-parallel roles need a verify model");
  if (role == 1 && (n < 1 || n > kMaxTpOut || !followers))
    return fail(AMUSD_ERR_INVALID_INPUT, "leader needs 1..7 follower inboxes");
  for (auto& e : s->exec)  // the loops capture the role: rebuild them
    for (auto& x : e)
      if (x) { cudaGraphExecDestroy(x); x = nullptr; }
  s->tp_role = role;
  s->tp_nout = role == 1 ? n : 0;
  for (int i = 0; i < s->tp_nout; ++i) s->tp_out[i] = (TpInbox*)followers[i];
  return AMUSD_OK;
}

int amusd_session_destroy(amusd_session* s) {
  if (!s) return AMUSD_OK;
  for (auto& e : s->exec)
    for (auto& x : e)
      if (x) cudaGraphExecDestroy(x);
  if (s->capture) cudaStreamDestroy(s->capture);
  delete s;
  return AMUSD_OK;
}

int amusd_session_reset(amusd_session* s, const int32_t* prompt, int n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!s || !prompt) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  if (n != s->d.prompt_len) return fail(AMUSD_ERR_INVALID_INPUT, "prompt length differs from the session's");
  for (amusd_model* m : {s->draft, s->verify}) {
    if (!m) continue;
    if (int r = sync_from_device(m, st)) return r;
    if (m->len != n || m->prompt_len != n)
      return fail(AMUSD_ERR_INVALID_INPUT, "models must hold init_state(prompt) before a run");
    if (m->kv_len > m->len - 1) m->kv_len = m->len - 1;
    if (int r = push_header(m, st)) return r;
  }
  CUDA_TRY(cudaMemcpyAsync(s->prompt_dev, prompt, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  ProtoArgs a = make_args(s);
  CUDA_TRY(launch_session_reset(a, s->prompt_dev, s->d.coin_seed, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return AMUSD_OK;
}

}  // extern "C"

// Capture the body of one actor's loop into `body`.
static int capture_body(amusd_session* s, int engine, int actor, cudaGraph_t body, cudaGraphConditionalHandle h) {
  ProtoArgs a = make_args(s);
  a.cond = h;
  a.has_cond = 1;
  cudaStream_t st = s->capture;
  CUDA_TRY(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  int r = AMUSD_OK;
  // Co-located AMUSD: early-launched (PDL) verify CTAs would hold the second
  // SM slot and starve the draft stream -- measured 146 vs 221 tok/s on B200.
  const bool pdl = s->use_pdl && engine != AMUSD_ENGINE_ASYNC;
  const bool colo = engine == AMUSD_ENGINE_ASYNC;
  // Co-located AMUSD: the draft and the verify forward run at the same time on DISJOINT SM
  // sets (each persistent CTA fills an SM; grids summing to <= #SMs can always co-run, and
  // the work-queue kernel needs no particular grid size).  Other engines own the GPU.
  const int draft_sms = std::max(1, std::min(num_sms() - 1, env_int("AMUSD_FW_DRAFT_GRID", 64)));
  for (amusd_model* m : {s->draft, s->verify}) {
    if (!m || !use_persistent(m)) continue;
    m->fw_stages = env_int("AMUSD_FW_STAGES", fw_max_stages(m->cfg, 1));
    m->fw_grid = model_sms(m);
    if (colo) m->fw_grid = m == s->draft ? draft_sms : num_sms() - draft_sms;
    // AMUSD_FW_COLO_SHARED=1 (experiment): both forwards on every SM, rings sized for two CTAs
    // per SM (the work-queue kernel needs no co-residency, so any overlap is safe)
    if (colo && env_int("AMUSD_FW_COLO_SHARED", 0)) {
      m->fw_grid = model_sms(m);
      m->fw_stages = env_int("AMUSD_FW_STAGES", fw_max_stages(m->cfg, 2));
    }
    m->fw_part_ok = colo && m == s->draft;
  }
  auto fwd = [&](amusd_model* m, StepCtl* c, int nr) { if (!r) r = model_forward(m, c, nr, st, pdl, false); };
  auto pk = [&](int which, int arg) { if (!r && proto_launch(which, a, st, arg) != cudaSuccess) r = fail(AMUSD_ERR_CUDA, "protocol launch failed"); };
  if (engine == AMUSD_ENGINE_AUTOREGRESSIVE) {
    pk(kArBegin, 0); fwd(s->verify, s->vctl, KMAX); pk(kArEnd, 0);
  } else if (engine == AMUSD_ENGINE_SYNC) {
    pk(kSyncRoundBegin, 0);
    for (int i = 0; i < s->d.draft_window_k; ++i) {
      pk(kSyncDraftBegin, i); fwd(s->draft, s->dctl, 2); pk(kSyncDraftEnd, 0);
    }
    pk(kSyncVerifyBegin, 0); fwd(s->verify, s->vctl, KMAX); pk(kSyncVerifyEnd, 0);
  } else if (actor == 0) {
    // a rollback request or completion raised during the draft forward discards its token
    // (k_draft_end): cut the forward short (AMUSD_FW_CUT=0 disables)
    if (env_int("AMUSD_FW_CUT", 1)) {
      s->draft->fw_ab_req = &s->mb_local->vb.rb_req;
      s->draft->fw_ab_done = &s->mb_local->vb.complete;
    }
    pk(kDraftBegin, 0); fwd(s->draft, s->dctl, 2); pk(kDraftEnd, 0);
    s->draft->fw_ab_req = s->draft->fw_ab_done = nullptr;
  } else {
    pk(kVerifyBegin, 0); fwd(s->verify, s->vctl, KMAX); pk(kVerifyEnd, 0);
  }
  cudaGraph_t g2 = body;
  cudaError_t e = cudaStreamEndCapture(st, &g2);
  for (amusd_model* m : {s->draft, s->verify}) {  // parity API launches own the GPU again
    if (!m || !use_persistent(m)) continue;
    m->fw_part_ok = false;
    m->fw_stages = env_int("AMUSD_FW_STAGES", fw_max_stages(m->cfg, 1));
    m->fw_grid = model_sms(m);
  }
  if (r) return r;
  CUDA_TRY(e);
  return AMUSD_OK;
}

static int build_loop(amusd_session* s, int engine, int actor, cudaGraphExec_t* out) {
  cudaGraph_t g;
  CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CUDA_TRY(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  if (int r = capture_body(s, engine, actor, p.conditional.phGraph_out[0], h)) {
    cudaGraphDestroy(g);
    return r;
  }
  cudaError_t e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(e);
  return AMUSD_OK;
}

extern "C" {

// Build (capture + instantiate) the engine's graphs without launching them.
int amusd_session_build(amusd_session* s, int engine) {
  if (!s) return fail(AMUSD_ERR_INVALID_INPUT, "null session");
  if (engine < 0 || engine > AMUSD_ENGINE_ASYNC_VERIFY) return fail(AMUSD_ERR_INVALID_INPUT, "unknown engine");
  const bool need_d = engine != AMUSD_ENGINE_AUTOREGRESSIVE && engine != AMUSD_ENGINE_ASYNC_VERIFY;
  const bool need_v = engine != AMUSD_ENGINE_ASYNC_DRAFT;
  if (need_d && !s->draft) return fail(AMUSD_ERR_INVALID_INPUT, "engine needs a draft model");
  if (need_v && !s->verify) return fail(AMUSD_ERR_INVALID_INPUT, "engine needs a verify model");
  const int actors[2] = {need_d && engine != AMUSD_ENGINE_AUTOREGRESSIVE && engine != AMUSD_ENGINE_SYNC,
                         need_v || engine == AMUSD_ENGINE_SYNC};
  for (int actor = 0; actor < 2; ++actor)
    if (actors[actor] && !s->exec[engine][actor])
      if (int r = build_loop(s, engine, actor, &s->exec[engine][actor])) return r;
  CUDA_TRY(cudaDeviceSynchronize());
  return AMUSD_OK;
}

int amusd_session_launch(amusd_session* s, int engine, void* verify_stream, void* draft_stream) {
  if (!s) return fail(AMUSD_ERR_INVALID_INPUT, "null session");
  if (engine < 0 || engine > AMUSD_ENGINE_ASYNC_VERIFY) return fail(AMUSD_ERR_INVALID_INPUT, "unknown engine");
  const bool need_d = engine != AMUSD_ENGINE_AUTOREGRESSIVE && engine != AMUSD_ENGINE_ASYNC_VERIFY;
  const bool need_v = engine != AMUSD_ENGINE_ASYNC_DRAFT;
  if (need_d && !s->draft) return fail(AMUSD_ERR_INVALID_INPUT, "engine needs a draft model");
  if (need_v && !s->verify) return fail(AMUSD_ERR_INVALID_INPUT, "engine needs a verify model");
  if (engine == AMUSD_ENGINE_SYNC && s->d.draft_window_k + 1 > KMAX)
    return fail(AMUSD_ERR_INVALID_INPUT, "draft_window_k too large");
  const int actors[2] = {need_d && engine != AMUSD_ENGINE_AUTOREGRESSIVE && engine != AMUSD_ENGINE_SYNC,
                         need_v || engine == AMUSD_ENGINE_SYNC};
  for (int actor = 0; actor < 2; ++actor) {
    if (!actors[actor]) continue;
    if (!s->exec[engine][actor])
      if (int r = build_loop(s, engine, actor, &s->exec[engine][actor])) return r;
  }
  if (s->draft) s->draft->dirty = true;
  if (s->verify) s->verify->dirty = true;
  if (actors[1]) CUDA_TRY(cudaGraphLaunch(s->exec[engine][1], (cudaStream_t)verify_stream));
  if (actors[0]) CUDA_TRY(cudaGraphLaunch(s->exec[engine][0], (cudaStream_t)(draft_stream ? draft_stream : verify_stream)));
  return AMUSD_OK;
}

int amusd_session_info(amusd_session* s, amusd_run_info* info, int32_t* V, int v_cap, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!s || !info) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  MailboxHdr h;
  int counts[2];
  CUDA_TRY(cudaMemcpyAsync(&h, s->mb_local, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(counts, s->dtrace.count, sizeof(counts), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  info->p_v = h.vb.p_v;
  info->p_d = h.db.p_d;
  info->complete = h.vb.complete;
  info->error = h.vb.error ? h.vb.error : h.db.error;
  info->verify_steps = h.vb.verify_steps;
  info->rollbacks = h.vb.rollbacks;
  info->drafted = h.db.drafted;
  info->acks = h.db.acks;
  info->n_draft_events = counts[0];
  info->n_verify_events = counts[1];
  info->draft_iters = h.db.iters;
  info->verify_iters = h.vb.iters;
  info->draft_cuts = 0;
  if (s->draft && s->draft->kind == 0 && s->draft->fw_sched) {
    CUDA_TRY(cudaMemcpyAsync(&info->draft_cuts, fw::cut_counter(s->draft->fw_sched), sizeof(int),
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (V && v_cap > 0) {
    const int nv = std::min(v_cap, std::max(0, h.vb.p_v - s->d.prompt_len));
    if (nv) CUDA_TRY(cudaMemcpyAsync(V, mb_V(s->mb_local, s->cap), sizeof(int) * nv, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return AMUSD_OK;
}

int amusd_session_trace(amusd_session* s, int actor, amusd_trace_event* out, int cap, int* n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!s || !out || !n) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  const TraceDev& t = actor == 0 ? s->dtrace : s->vtrace;
  int cnt = 0;
  CUDA_TRY(cudaMemcpyAsync(&cnt, t.count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *n = cnt;
  const int k = std::min(std::min(cnt, cap), t.cap);
  if (k) CUDA_TRY(cudaMemcpyAsync(out, t.ev, sizeof(amusd_trace_event) * k, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return AMUSD_OK;
}

int amusd_time_forward(amusd_model* m, int rows, int which, int layer, int iters, float* ms, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!m || !ms || iters < 1) return fail(AMUSD_ERR_INVALID_INPUT, "bad argument");
  if (rows < 1 || rows > KMAX) return fail(AMUSD_ERR_INVALID_INPUT, "rows must be in [1, 16]");
  if (m->kind == 0 && which >= 0 && (layer < 0 || layer >= m->cfg.n_layers))
    return fail(AMUSD_ERR_INVALID_INPUT, "layer out of range");
  if (int r = sync_from_device(m, st)) return r;
  const int pos0 = std::max(0, std::min(m->kv_len, m->max_seq - rows - 1));
  StepCtl c{};
  c.active = 1; c.rows = rows; c.pos0 = pos0; c.npend = rows;
  for (int i = 0; i < rows; ++i) c.tok[i] = (i * 7919 + 3) % m->vocab;
  CUDA_TRY(cudaMemcpyAsync(m->api_ctl, &c, sizeof(c), cudaMemcpyHostToDevice, st));
  const int nr = rows <= 2 ? 2 : KMAX;
  auto once = [&]() -> int {
    if (which < 0 || m->kind == 1) return model_forward(m, m->api_ctl, nr, st, false, false);
    if (use_tc(m, nr)) return tc_kernel(m, m->api_ctl, layer, which, st, false);
    return tf_kernel(m, m->api_ctl, nr, layer, which, st, false, false);
  };
  const int grid0 = m->fw_grid;
  if (m->grid_override > 0) m->fw_grid = m->grid_override;
  struct Restore { amusd_model* m; int g; ~Restore() { m->fw_grid = g; } } restore{m, grid0};
  if (int r = once()) return r;  // warm-up
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i)
    if (int r = once()) return r;
  CUDA_TRY(cudaEventRecord(e1, st));
  CUDA_TRY(cudaEventSynchronize(e1));
  float t = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = t / iters;
  return AMUSD_OK;
}

int amusd_session_kernels_per_step(amusd_session* s, int engine, int* draft_step, int* verify_step) {
  if (!s || !draft_step || !verify_step) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  *draft_step = s->draft ? model_kernels_per_forward(s->draft, 2) + 2 : 0;
  // the AMUSD draft's persistent forward is followed by the cut cleanup (a no-op launch when not cut)
  // (co-located AMUSD runs a decode-path draft on the work-queue forward too, see model_forward)
  const bool wq = s->draft && (use_fw(s->draft) || (engine == AMUSD_ENGINE_ASYNC && use_persistent(s->draft)));
  if ((engine == AMUSD_ENGINE_ASYNC || engine == AMUSD_ENGINE_ASYNC_DRAFT) && wq && env_int("AMUSD_FW_CUT", 1))
    *draft_step += 1;
  *verify_step = s->verify ? model_kernels_per_forward(s->verify, KMAX) + 2 : 0;
  if (engine == AMUSD_ENGINE_SYNC) *verify_step += 1;
  return AMUSD_OK;
}

}  // extern "C"

// -------------------------------------------------------- weight fill
__global__ void k_fill_uniform(void* dst, int dtype, size_t n, unsigned long long seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long z = mix64(seed + i);
    const float u = (float)(z >> 40) * (1.0f / 16777216.0f);  // [0, 1)
    const float v = scale * (2.0f * u - 1.0f);
    if (dtype == AMUSD_BF16) ((__nv_bfloat16*)dst)[i] = __float2bfloat16(v);
    else ((float*)dst)[i] = v;
  }
}

extern "C" int amusd_fill_uniform(void* dst, int dtype, size_t n, uint64_t seed, float scale, void* stream) {
  if (!dst) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  k_fill_uniform<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(dst, dtype, n, seed, scale);
  CUDA_TRY(cudaGetLastError());
  return AMUSD_OK;
}

// ------------------------------------------------------------ split pair
extern "C" {

int amusd_ipc_export(void* ptr, uint8_t handle[64], size_t* offset) {
  if (!ptr || !handle || !offset) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(AMUSD_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range = (PFN_cuMemGetAddressRange_v3020)p;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(AMUSD_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(handle, &h, 64);
  *offset = (size_t)((CUdeviceptr)ptr - base);
  return AMUSD_OK;
}

int amusd_ipc_import(const uint8_t handle[64], size_t offset, void** ptr, void** base) {
  if (!handle || !ptr || !base) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* b = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
  *base = b;
  *ptr = (char*)b + offset;
  return AMUSD_OK;
}

int amusd_ipc_close(void* base) {
  if (!base) return AMUSD_OK;
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return AMUSD_OK;
}

}  // extern "C"

__global__ void k_device_clock(long long* out) { *out = globaltimer(); }

extern "C" int amusd_device_clock(int64_t* ns, void* scratch, void* stream) {
  if (!ns || !scratch) return fail(AMUSD_ERR_INVALID_INPUT, "null argument");
  long long* d = (long long*)scratch;  // caller-owned 8-byte device buffer (the library never allocates)
  k_device_clock<<<1, 1, 0, (cudaStream_t)stream>>>(d);
  CUDA_TRY(cudaGetLastError());
  long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  *ns = v;
  return AMUSD_OK;
}
