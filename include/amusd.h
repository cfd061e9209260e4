/*
 * amusd.h -- C-ABI of the B200-native AMUSD draft/verify decode path.
 *
 * The reference (pkg/src/specdec) is pure Python with two duck-typed plug-in
 * points and no FFI.  This header is the boundary a
 * maintainer binds (ctypes stub in INTEGRATION.md); every entry point names the
 * reference interface it replaces.  Conventions:
 *   - plain pointers and sizes only; no torch types;
 *   - all DEVICE memory (weights, KV cache, activations, mailbox, trace rings,
 *     canonical table) is allocated by the caller and passed in; the library
 *     never allocates device memory.  Host-side handles (graphs, TMA
 *     descriptors) are owned by the opaque amusd_model / amusd_session;
 *   - every function returns an amusd_status; amusd_last_error() gives text;
 *   - streams are cudaStream_t passed as void*.
 */
#ifndef AMUSD_H
#define AMUSD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMUSD_ABI_VERSION 1
#define AMUSD_KMAX 16          /* rows in one forward: verify window + pending */
#define AMUSD_MAX_LAYERS 128

/* Status codes; the Python wrapper maps them onto the reference hierarchy
 * (errors.py:4-29). */
typedef enum {
  AMUSD_OK = 0,
  AMUSD_ERR_INVALID_INPUT = 1,    /* InvalidInputError       errors.py:8  */
  AMUSD_ERR_INVALID_ROLLBACK = 2, /* InvalidRollbackError    errors.py:12 */
  AMUSD_ERR_PROTOCOL = 3,         /* ProtocolViolationError  errors.py:16 */
  AMUSD_ERR_CUDA = 4,             /* SpecDecError (runtime)  errors.py:4  */
  AMUSD_ERR_UNSUPPORTED = 5       /* SpecDecError                          */
} amusd_status;

typedef enum { AMUSD_F32 = 0, AMUSD_BF16 = 1 } amusd_dtype;

/* Engines (engines.py:279-301, 534-561). */
typedef enum {
  AMUSD_ENGINE_AUTOREGRESSIVE = 0, /* decode_autoregressive    engines.py:279 */
  AMUSD_ENGINE_SYNC = 1,           /* decode_speculative_sync  engines.py:290 */
  AMUSD_ENGINE_ASYNC = 2,          /* decode_speculative_async engines.py:534 */
  AMUSD_ENGINE_ASYNC_DRAFT = 3,    /* draft loop only (draft GPU of a split pair) */
  AMUSD_ENGINE_ASYNC_VERIFY = 4    /* verify loop only (verify GPU of a split pair) */
} amusd_engine;

/* Draft agreement coin (models.py:271-314). */
typedef enum {
  AMUSD_COIN_NONE = 0,  /* draft emits its own greedy token                       */
  AMUSD_COIN_SELF = 1,  /* agreed = the draft's own greedy token (coin on its prefix) */
  AMUSD_COIN_CANON = 2  /* agreed = canonical verify token while on the canonical
                           path (transformer pairs)       */
} amusd_coin_mode;

typedef struct amusd_model amusd_model;
typedef struct amusd_session amusd_session;

/* ---------------------------------------------------------------- models */

/* Llama-style decoder shape (builder-defined). */
typedef struct {
  int vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, ffn;
  int max_seq;       /* KV capacity in tokens                         */
  int dtype;         /* amusd_dtype of weights and KV cache           */
  int eos_token;
  int exclude_eos;   /* mask eos from the argmax (models.py:256-261)  */
  float norm_eps;
  int use_tensor_cores; /* bf16 only: tcgen05 GEMMs for >2-row forwards */
} amusd_tf_config;

/* Device pointers, row-major [out][in]; dtype per config (norms are always
 * the model dtype; rope tables are fp32 [max_seq][head_dim/2]). */
typedef struct {
  const void* embed;       /* [vocab][d]                     */
  const void* lm_head;     /* [vocab][d]; == embed when tied  */
  const void* final_norm;  /* [d]                             */
  const float* rope_cos;
  const float* rope_sin;
  const void* attn_norm[AMUSD_MAX_LAYERS]; /* [d]                       */
  const void* wqkv[AMUSD_MAX_LAYERS];      /* [(H+2*KV)*hd][d]          */
  const void* wo[AMUSD_MAX_LAYERS];        /* [d][H*hd]                 */
  const void* mlp_norm[AMUSD_MAX_LAYERS];  /* [d]                       */
  const void* wgate[AMUSD_MAX_LAYERS];     /* [ffn][d]                  */
  const void* wup[AMUSD_MAX_LAYERS];       /* [ffn][d]                  */
  const void* wdown[AMUSD_MAX_LAYERS];     /* [d][ffn]                  */
} amusd_tf_weights;

/* Bytes of device state (KV cache + activations + sequence state). */
size_t amusd_tf_state_bytes(const amusd_tf_config* cfg);
int amusd_tf_create(amusd_model** out, const amusd_tf_config* cfg, const amusd_tf_weights* w,
                    void* state, size_t state_bytes);

/* splitmix64 hash-chain model (models.py:203-268): the device test double (K7).
 * agreement_rho < 0: HashChainModel; in [0,1]: AgreementDraftModel whose
 * forward applies the prefix-keyed agreement coin (models.py:271-314). */
size_t amusd_hash_state_bytes(int max_seq);
int amusd_hash_create(amusd_model** out, uint64_t seed, int vocab, int eos_token, int exclude_eos,
                      double agreement_rho, int max_seq, void* state, size_t state_bytes);

/* ScriptedModel (models.py:317-346): the prediction at 1-based absolute
 * position p is script[(p-1) % script_len], or eos_token at eos_position
 * (0 = none) -- pins eos-terminated run lengths (pkg/tests/test_engines.py:66-76).
 * The script (host buffer) is copied into the caller's state buffer. */
size_t amusd_scripted_state_bytes(int max_seq, int script_len);
int amusd_scripted_create(amusd_model** out, const int32_t* script, int script_len, int vocab, int eos_token,
                          int eos_position, int max_seq, void* state, size_t state_bytes, void* stream);

int amusd_model_destroy(amusd_model* m);

/* Tensor-parallel shard of a transformer (BASELINE config 4: the verify model
 * sharded over tp_size GPUs; not in the reference, which has no transformer).
 * The amusd_tf_config passed with it describes the SHARD: n_heads / n_kv_heads
 * / ffn / vocab are this rank's slice -- whole KV groups (QKV column-parallel,
 * O row-parallel), whole gate/up features (gate/up column-parallel, down
 * row-parallel), whole 128-row vocab tiles of the LM head.  The embedding and
 * the norms are replicated.  Only the persistent forward runs shards: the O and
 * down partials are red.added into EVERY rank's int64 split-K accumulators
 * over peer memory (the allreduce fused into the GEMM epilogue) and the LM-head
 * argmax keys into every rank's, so every rank computes the same predictions --
 * bit-identical to the unsharded forward (the shard takes the unsharded
 * model's split-K chunking).  Replaces nothing in the reference: its only
 * parallelism is the two actor threads (engines.py:448-459). */
typedef struct {
  int tp_rank, tp_size;        /* 2 <= tp_size <= 8 */
  int n_heads_full, n_kv_heads_full, ffn_full;  /* the unsharded model */
  int vocab_offset;            /* global vocab id of this shard's first LM-head row */
  int vocab_total;             /* embedding rows (valid token ids) */
} amusd_tp_shard;
/* One rank's cross-rank words (device pointers, valid in the exporting process;
 * translate through CUDA IPC for another process). */
typedef struct {
  void* ws;        /* int64 split-K accumulators */
  void* tile_cnt;  /* split-K tile counters */
  void* best;      /* argmax keys */
  void* sched;     /* schedule block (LM-head arrival counter) */
  int lm_items;    /* LM-head work items of this rank */
  int pad;
} amusd_tp_peer;
size_t amusd_tf_shard_state_bytes(const amusd_tf_config* cfg, const amusd_tp_shard* shard);
int amusd_tf_create_shard(amusd_model** out, const amusd_tf_config* cfg, const amusd_tp_shard* shard,
                          const amusd_tf_weights* w, void* state, size_t state_bytes);
int amusd_tp_export(amusd_model* m, amusd_tp_peer* out);
/* All ranks' words in rank order (n == tp_size, this rank's own included);
 * required before the shard's first forward. */
int amusd_tp_connect(amusd_model* m, const amusd_tp_peer* peers, int n);
/* One process driving several GPUs: let `device` load/store/atomically update `peer`'s HBM. */
int amusd_peer_enable(int device, int peer);

/* Forward implementation of a bf16 tensor-core-shaped transformer (perf A/B
 * and parity tests; not in the reference, whose models are Python mocks):
 * 0 = persistent tcgen05 forward (default, one launch per forward),
 * 1 = per-kernel tcgen05 path (1 + 5L + 2 launches), 2 = SIMT GEMV path,
 * 3 = persistent SIMT decode forward (decode_gv.cu: one launch, static
 *     per-CTA row partitions, fused RMSNorm + GEMV over the row-major weights;
 *     the draft model's path -- its forwards carry 1-2 rows),
 * 4 = cluster decode forward (decode_cl.cu: one 8-CTA cluster per KV head
 *     does QKV + attention + the O slice with DSMEM hand-offs, two grid-wide
 *     dependencies per layer; <= 8 rows per forward).
 * Applies to launches enqueued afterwards (sessions capture it per engine). */
enum { AMUSD_PATH_PERSISTENT = 0, AMUSD_PATH_KERNELS = 1, AMUSD_PATH_SIMT = 2, AMUSD_PATH_DECODE = 3,
       AMUSD_PATH_CLUSTER = 4 };
int amusd_model_set_path(amusd_model* m, int path);
/* The decode forward (AMUSD_PATH_DECODE) streams its own weight layout: 16-row x 512-K
 * units, 16-byte chunks swizzled for ldmatrix.  amusd_decode_bytes = its size (0: shapes not
 * supported); amusd_model_set_decode tiles the row-major weights into the caller's buffer
 * (the library never allocates), buf = NULL detaches it. */
size_t amusd_decode_bytes(amusd_model* m);
/* The cluster decode forward's weight layout (per layer: QKV / O by KV group, gate/up and
 * down^T by 16-feature block); same contract as amusd_decode_bytes / amusd_model_set_decode. */
size_t amusd_cluster_bytes(amusd_model* m);
int amusd_model_set_cluster(amusd_model* m, void* buf, size_t bytes);
int amusd_model_set_decode(amusd_model* m, void* buf, size_t bytes);
/* Drop the caller's row-major layer weights from the model (the persistent path
 * reads only its tile-contiguous copy): afterwards the caller may free them
 * (8B: 16 GB) and only AMUSD_PATH_PERSISTENT remains selectable. */
int amusd_model_release_row_major(amusd_model* m);
/* Perf analysis only: run amusd_time_forward's persistent launches on `sms`
 * SMs (0 = all), e.g. the share a co-located session gives the model. */
int amusd_model_set_grid(amusd_model* m, int sms);
/* Compute-bound prompt prefill (init_state models.py:109-118):
 * with a workspace set, init_state of a bf16 tcgen05 model caches prompts of
 * >= 64 positions (AMUSD_PREFILL_MIN) as dense M128 N256 tcgen05 GEMMs over all
 * prompt tokens plus a causal attention, instead of 16-row decode forwards.
 * buf = NULL detaches it.  The caller owns the memory (the library never allocates). */
size_t amusd_prefill_bytes(amusd_model* m, int max_tokens);
int amusd_model_set_prefill(amusd_model* m, void* buf, size_t bytes, int max_tokens);
/* Cap every persistent launch of the model (API forwards and non-co-located
 * engine loops) at `sms` CTAs (0 = all SMs).  Ranks of a tensor-parallel group
 * emulated on ONE GPU need this: their forwards wait on each other, so their
 * grids must be co-resident (sum <= SM count). */
int amusd_model_set_max_grid(amusd_model* m, int sms);
/* Perf analysis only: record a per-work-item timeline of the persistent
 * forward into a device buffer (64 bytes per item; NULL disables). */
int amusd_model_set_timeline(amusd_model* m, void* buf, size_t bytes);

/* MockModel interface (models.py:85-200): synchronous on `stream`, host token
 * buffers.  Used by the parity path; the decode loops below never call it. */
int amusd_init_state(amusd_model* m, const int32_t* prompt, int n, void* stream);       /* models.py:109 */
int amusd_next_token(amusd_model* m, int32_t* out, void* stream);                        /* models.py:120 */
int amusd_advance(amusd_model* m, const int32_t* tokens, int n, void* stream);            /* models.py:125 */
int amusd_rollback(amusd_model* m, int position, void* stream);                           /* models.py:133 */
int amusd_verify_tokens(amusd_model* m, const int32_t* cands, int n, int32_t* preds,
                        void* stream);                                                    /* models.py:151 */
int amusd_prefix_length(amusd_model* m, int* out);                                        /* models.py:72  */
/* Raw last-row logits of the most recent forward (debug/parity; fp32, vocab entries). */
int amusd_last_logits(amusd_model* m, float* out, int rows, void* stream);

/* ------------------------------------------------------------- sessions */

typedef struct {
  int prompt_len;
  int max_new_tokens;     /* DecodeConfig.max_new_tokens  engines.py:61 */
  int draft_window_k;     /* DecodeConfig.draft_window_k  engines.py:62 */
  int max_draft_lead;     /* DecodeConfig.max_draft_lead  engines.py:63 (0 = None) */
  int max_window;         /* verify rows cap, <= AMUSD_KMAX            */
  int coin_mode;          /* amusd_coin_mode                           */
  double rho;             /* agreement probability                      */
  uint64_t coin_seed;     /* hash-chain seed of the coin                */
  const int32_t* canon;   /* device [canon_len] absolute tokens (COIN_CANON) */
  int canon_len;
  int trace_cap;          /* events per actor ring                      */
  int jitter_ns;          /* device-side poll jitter (ThreadExecutor.poll_jitter_ms analog) */
  uint64_t jitter_seed;
} amusd_session_desc;

/* Mailbox = SharedDecodeState (coordination.py:114-275) in HBM. */
int amusd_mailbox_capacity(const amusd_session_desc* d); /* tokens per D/V buffer */
size_t amusd_mailbox_bytes(int capacity_tokens);
size_t amusd_session_bytes(const amusd_session_desc* d);

/* draft or verify may be NULL for one half of a split pair.  mb_peer is the
 * peer GPU's mailbox mapped over NVLink (NULL when co-located). */
int amusd_session_create(amusd_session** out, amusd_model* draft, amusd_model* verify,
                         const amusd_session_desc* d, void* mem, size_t mem_bytes,
                         void* mb_local, void* mb_peer);
int amusd_session_destroy(amusd_session* s);
/* Tensor-parallel verify group (BASELINE config 4): the leader rank's
 * k_verify_begin snapshots the draft window and pushes the step control into
 * every follower's inbox (peer memory); followers run the same loop on it.
 * role 0 = none, 1 = leader (followers = the followers' inboxes, n <= 7),
 * 2 = follower.  Sessions of one group must run the same engine. */
int amusd_session_tp_inbox(amusd_session* s, void** out);
int amusd_session_set_tp(amusd_session* s, int role, void* const* followers, int n);

/* Reset the mailbox, coin chain and trace rings for a fresh run; the models
 * must already hold init_state(prompt).  Prompt is a host buffer. */
int amusd_session_reset(amusd_session* s, const int32_t* prompt, int n, void* stream);

/* Launch one engine as device-driven CUDA graphs (conditional WHILE loops):
 * no host sync inside; returns after enqueueing. ASYNC uses both streams. */
int amusd_session_launch(amusd_session* s, int engine, void* verify_stream, void* draft_stream);
/* Capture + instantiate an engine's graphs without launching (launch does it on
 * first use).  A split pair builds both halves first: instantiation may wait
 * for the device, which must not happen while the peer's loop is spinning. */
int amusd_session_build(amusd_session* s, int engine);

/* Verified stream V and counters after a run (host buffers). */
typedef struct {
  int p_v, p_d, complete, error;
  int verify_steps, rollbacks, drafted, acks;
  int n_draft_events, n_verify_events;
  int draft_iters, verify_iters;  /* loop-body executions (launch accounting) */
  int draft_cuts;                 /* draft forwards cut short by a rollback/completion (cumulative) */
} amusd_run_info;
int amusd_session_info(amusd_session* s, amusd_run_info* info, int32_t* V, int v_cap, void* stream);

/* Trace events (metrics.py:60-72): kind 0 draft_token, 1 verify_accept,
 * 2 verify_correct, 3 rollback; times in ns from %globaltimer. */
typedef struct {
  int64_t t_ns;
  int64_t busy_ns;
  int32_t kind, pos_lo, pos_hi, draft_accepted;
} amusd_trace_event;
int amusd_session_trace(amusd_session* s, int actor /*0 draft, 1 verify*/, amusd_trace_event* out,
                        int cap, int* n, void* stream);

/* ---------------------------------------------------------------- misc */
int amusd_abi_version(void);
const char* amusd_last_error(void);
/* Benchmark helper: `iters` eager launches of one model forward over `rows`
 * rows at the current cache position (state is not advanced), timed with
 * CUDA events on `stream`; *ms = mean ms per launch.  which = -1 whole
 * forward, else one kernel of layer `layer`: 0 QKV gemv, 1 attention, 2 O
 * gemv, 3 gate/up gemv, 4 down gemv, 5 LM-head gemv, 6 argmax reduce. */
int amusd_time_forward(amusd_model* m, int rows, int which, int layer, int iters, float* ms, void* stream);
/* Number of kernels one step of `engine` launches (gpu_launches accounting). */
int amusd_session_kernels_per_step(amusd_session* s, int engine, int* draft_step, int* verify_step);
/* Device-side deterministic weight fill: w[i] = scale * u(splitmix64(seed + i)),
 * u uniform in [-1,1) -- used for synthetic bf16/fp32 weights. */
int amusd_fill_uniform(void* dst, int dtype, size_t n, uint64_t seed, float scale, void* stream);

/* ---------------------------------------------- split pair (2 GPUs) */
/* The draft GPU and the verify GPU each own a mailbox copy and store into the
 * peer's copy over NVLink (coordination.py:114-275 across a device boundary).
 * Export a device buffer as a CUDA IPC handle (64 bytes) plus its offset in
 * the underlying allocation; import maps the peer's buffer into this process
 * (peer access enabled lazily).  amusd_ipc_close unmaps an imported base. */
int amusd_ipc_export(void* ptr, uint8_t handle[64], size_t* offset);
int amusd_ipc_import(const uint8_t handle[64], size_t offset, void** ptr, void** base);
int amusd_ipc_close(void* base);
/* %globaltimer of this device (ns), for aligning the two GPUs' trace clocks;
 * `scratch` is a caller-owned device buffer of >= 8 bytes. */
int amusd_device_clock(int64_t* ns, void* scratch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AMUSD_H */
