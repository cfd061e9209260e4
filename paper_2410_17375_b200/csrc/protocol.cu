// protocol.cu -- the AMUSD draft/verify protocol as device kernels.
//
// The reference runs two Python threads around one shared object
// (engines.py:409-531, coordination.py:114-275).  Here each actor is a chain
// of kernels on its own stream (or GPU) inside a CUDA-graph WHILE loop:
//
//   draft  : k_draft_begin  -> model forward -> k_draft_end      (engines.py:332-352)
//   verify : k_verify_begin -> model forward -> k_verify_end     (engines.py:355-401)
//
// and they talk only through the HBM mailbox (internal.h) with
// release/acquire flags.  Every field keeps the reference's single writer;
// the reference's two-writer rollback flag (set at coordination.py:255,
// cleared at :209) becomes two monotone epochs rb_req (verify) / rb_ack
// (draft): "pending" == rb_req != rb_ack.
//
// Rollback is a cache-length truncate (kv_len := target-1) plus the
// correction becoming the pending token -- no copy and no host sync
// (coordination.py:188-211).
#include "common.cuh"
#include "internal.h"
#include "protocol.h"

namespace amusd {

constexpr long long kSpinTimeoutNs = 20ll * 1000 * 1000 * 1000;  // 20 s: fail loudly, never hang
enum { kErrTimeout = 1, kErrTarget = 2, kErrCapacity = 3 };

AMUSD_DEV void stop_loop(const ProtoArgs& a, StepCtl* c) {
  c->active = 0;
  if (a.has_cond) cudaGraphSetConditional(a.cond, 0);
}

AMUSD_DEV void trace_push(const TraceDev& t, long long now, long long busy, int kind, int lo, int hi, int acc) {
  if (!t.ev) return;
  const int i = *t.count;
  if (i < t.cap) {
    amusd_trace_event e;
    e.t_ns = now;
    e.busy_ns = busy;
    e.kind = kind;
    e.pos_lo = lo;
    e.pos_hi = hi;
    e.draft_accepted = acc;
    t.ev[i] = e;
  }
  *t.count = i + 1;
}

// Coin chain over the draft prefix: hash[n] after n tokens (models.py:218-227).
AMUSD_DEV void coin_push(const CoinDev& c, int n, int tok) {
  if (!c.hash) return;
  c.hash[n + 1] = mix64(c.hash[n] ^ (unsigned long long)(unsigned)tok);
  c.onpath[n + 1] = c.onpath[n] && n < c.canon_len && c.canon[n] == tok;
}
// Token the draft publishes for prefix length n given its own greedy `pred`.
AMUSD_DEV int coin_pick(const CoinDev& c, int n, int pred) {
  int agreed;
  if (c.mode == AMUSD_COIN_SELF) agreed = pred;  // AgreementDraftModel._token_from_hash (models.py:300-304)
  else if (c.mode == AMUSD_COIN_CANON && c.onpath[n] && n < c.canon_len) agreed = c.canon[n];
  else return pred;
  if (c.always) return agreed;  // rho == 1: int(2**64) exceeds every hash
  return coin_token(c.hash[n], agreed, c.thr, c.vocab, c.eos, c.exclude_eos);
}

// Device-side poll jitter (ThreadExecutor.poll_jitter_ms, engines.py:464-469).
AMUSD_DEV void jitter(const ProtoArgs& a, unsigned long long salt, int step) {
  if (a.jitter_ns <= 0) return;
  const unsigned long long r = mix64(a.jitter_seed ^ (salt << 32) ^ (unsigned long long)step);
  const long long until = globaltimer() + (long long)(r % (unsigned long long)a.jitter_ns);
  while (globaltimer() < until) __nanosleep(64);
}

AMUSD_DEV void mb_write_both(int* peer, int* local, int v) {
  st_release(peer, v);
  if (local != peer) st_release(local, v);
}

// ------------------------------------------------------------------ draft
// draft_loop_step priority: complete > rollback-ack > lead cap > generate
// (engines.py:337-352).  The ack and the next generation share one step.
__global__ void k_draft_begin(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.dctl;
  SeqHdr* s = a.dseq;
  MailboxHdr* L = a.mb_local;
  MailboxHdr* R = a.mb_peer;
  c->active = 0;
  R->db.iters += 1;
  if (L != R) L->db.iters = R->db.iters;
  jitter(a, 0x0D, *a.dtrace.count);
  const long long t_enter = globaltimer();
  const int seq_limit = min(s->cap, a.P + a.cap) - 1;
  for (;;) {
    if (ld_acquire(&L->vb.complete) || ld_volatile(&L->vb.error)) { stop_loop(a, c); return; }
    const int req = ld_acquire(&L->vb.rb_req);
    if (req != c->rb_ack_local) {  // acknowledge_rollback (coordination.py:188-211)
      const int target = ld_volatile(&L->vb.rb_target);
      const int corr = ld_volatile(&L->vb.rb_correction);
      const int pd = s->len;
      if (!(a.P < target && target <= pd)) {
        mb_write_both(&R->db.error, &L->db.error, kErrTarget);
        stop_loop(a, c);
        return;
      }
      a.dtok[target - 1] = corr;           // rollback(target-1) + advance([c])
      if (s->kv_len > target - 1) s->kv_len = target - 1;
      s->len = target;
      s->pred_valid = 0;
      coin_push(a.coin, target - 1, corr);
      mb_D(R)[target - 1 - a.P] = corr;    // D.truncate_to + append(c)
      // stamp before publishing: the peer may act on the ack at once, and the merged
      // trace orders events by these stamps
      const long long now = globaltimer();
      st_release(&R->db.p_d, target);      // p_d = target
      R->db.acks += 1;
      c->rb_ack_local = req;
      st_release(&R->db.rb_ack, req);      // clear the request (epoch)
      trace_push(a.dtrace, now, now - c->t0, 3, target, pd, 0);
      continue;
    }
    const bool capped = (a.lead > 0 && s->len - ld_acquire(&L->vb.p_v) >= a.lead) || s->len >= seq_limit;
    if (!capped) break;
    if (globaltimer() - t_enter > kSpinTimeoutNs) {
      mb_write_both(&R->db.error, &L->db.error, kErrTimeout);
      stop_loop(a, c);
      return;
    }
    __nanosleep(100);
  }
  const int npend = s->len - s->kv_len;
  c->npend = npend;
  c->rows = npend;
  c->pos0 = s->kv_len;
  for (int i = 0; i < npend; ++i) c->tok[i] = a.dtok[s->kv_len + i];
  c->t0 = globaltimer();
  c->active = 1;
}

// Publish the drafted token (publish_draft_token, coordination.py:183-186).
// A token whose forward overlapped a rollback request is discarded
// (simulator.py:292-297); the next begin acknowledges.
__global__ void k_draft_end(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.dctl;
  if (!c->active) return;
  SeqHdr* s = a.dseq;
  MailboxHdr* L = a.mb_local;
  MailboxHdr* R = a.mb_peer;
  const int n = s->len;
  const int tok = coin_pick(a.coin, n, c->preds[c->rows - 1]);
  s->kv_len = n;
  if (ld_acquire(&L->vb.complete) || ld_acquire(&L->vb.rb_req) != c->rb_ack_local) return;
  a.dtok[n] = tok;
  coin_push(a.coin, n, tok);
  s->len = n + 1;
  s->pred_valid = 0;
  mb_D(R)[n - a.P] = tok;
  const long long now = globaltimer();  // stamp before publishing (trace order)
  st_release(&R->db.p_d, n + 1);
  R->db.drafted += 1;
  trace_push(a.dtrace, now, now - c->t0, 0, n + 1, n + 1, 0);
}

// ----------------------------------------------------------------- verify
// Wait for a non-empty window outside a rollback handshake, then snapshot
// (p_v, p_d] once (read_draft_window, coordination.py:217-228).
// Tensor-parallel leader: push this step's control (or the stop) to every follower.
AMUSD_DEV void tp_push(const ProtoArgs& a, const StepCtl* c, int seq, int stop) {
  for (int i = 0; i < a.tp_nout; ++i) {
    TpInbox* o = a.tp_out[i];
    o->stop = stop;
    if (!stop) {
      o->ctl.npend = c->npend; o->ctl.m = c->m; o->ctl.rows = c->rows; o->ctl.pos0 = c->pos0;
      for (int j = 0; j < KMAX; ++j) { o->ctl.tok[j] = c->tok[j]; o->ctl.cand[j] = c->cand[j]; }
    }
    st_release(&o->seq, seq);
  }
}

// Tensor-parallel follower: the leader's snapshot of this step (same iteration count).
AMUSD_DEV void tp_follow(const ProtoArgs& a, StepCtl* c, MailboxHdr* L) {
  L->vb.iters += 1;
  const int want = L->vb.iters;
  const TpInbox* in = a.tp_in;
  const long long t_enter = globaltimer();
  while (ld_acquire(&in->seq) < want) {
    if (globaltimer() - t_enter > kSpinTimeoutNs) {
      L->vb.error = kErrTimeout;
      L->vb.complete = 1;
      stop_loop(a, c);
      return;
    }
    __nanosleep(64);
  }
  if (ld_volatile(&in->stop)) {
    L->vb.complete = 1;
    stop_loop(a, c);
    return;
  }
  c->npend = in->ctl.npend; c->m = in->ctl.m; c->rows = in->ctl.rows; c->pos0 = in->ctl.pos0;
  for (int j = 0; j < KMAX; ++j) { c->tok[j] = in->ctl.tok[j]; c->cand[j] = in->ctl.cand[j]; }
  c->t0 = globaltimer();
  c->active = 1;
}

__global__ void k_verify_begin(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  SeqHdr* s = a.vseq;
  MailboxHdr* L = a.mb_local;
  MailboxHdr* R = a.mb_peer;
  c->active = 0;
  if (a.tp_in) {
    tp_follow(a, c, L);
    return;
  }
  R->vb.iters += 1;
  if (L != R) L->vb.iters = R->vb.iters;
  jitter(a, 0x5E, *a.vtrace.count);
  const long long t_enter = globaltimer();
  long long t_first = 0;
  int pd;
  for (;;) {
    if (ld_volatile(&L->db.error)) {  // draft-side violation: end the run
      mb_write_both(&R->vb.error, &L->vb.error, ld_volatile(&L->db.error));
      mb_write_both(&R->vb.complete, &L->vb.complete, 1);
      tp_push(a, c, L->vb.iters, 1);
      stop_loop(a, c);
      return;
    }
    if (ld_acquire(&L->db.rb_ack) == c->rb_ack_local) {
      pd = ld_acquire(&L->db.p_d);
      if (pd > s->len) {
        if (pd - s->len >= a.min_window) break;
        const long long now = globaltimer();
        if (!t_first) t_first = now;
        else if (now - t_first >= a.wait_ns) break;
      }
    }
    if (globaltimer() - t_enter > kSpinTimeoutNs) {
      mb_write_both(&R->vb.error, &L->vb.error, kErrTimeout);
      mb_write_both(&R->vb.complete, &L->vb.complete, 1);
      tp_push(a, c, L->vb.iters, 1);
      stop_loop(a, c);
      return;
    }
    __nanosleep(64);
  }
  const int pv = s->len, npend = pv - s->kv_len;
  const int m = min(pd - pv, a.max_window - npend + 1);
  const int* D = mb_D(L);
  for (int j = 0; j < m; ++j) c->cand[j] = ld_volatile(&D[pv - a.P + j]);
  for (int i = 0; i < npend; ++i) c->tok[i] = a.vtok[s->kv_len + i];
  for (int j = 0; j + 1 < m; ++j) c->tok[npend + j] = c->cand[j];
  c->npend = npend;
  c->m = m;
  c->rows = npend + m - 1;
  c->pos0 = s->kv_len;
  c->t0 = globaltimer();
  c->active = 1;
  tp_push(a, c, L->vb.iters, 0);
}

// K1 epilogue: accept the matched prefix + correction, publish to V, raise
// the rollback request, signal completion (engines.py:376-393,
// coordination.py:230-260).  No bonus token (engines.py:366-367).
__global__ void k_verify_end(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  if (!c->active) return;
  SeqHdr* s = a.vseq;
  MailboxHdr* L = a.mb_local;
  MailboxHdr* R = a.mb_peer;
  const int m = c->m, npend = c->npend, pv0 = s->len;
  int miss = -1;
  for (int j = 0; j < m; ++j)
    if (c->cand[j] != c->preds[npend - 1 + j]) { miss = j; break; }
  const int na = miss < 0 ? m : miss + 1;
  bool eos_hit = false;
  int* Vl = mb_V(L, a.cap);
  int* Vr = mb_V(R, a.cap);
  for (int j = 0; j < na; ++j) {
    const int t = (j == miss) ? c->preds[npend - 1 + j] : c->cand[j];
    a.vtok[pv0 + j] = t;
    Vl[pv0 - a.P + j] = t;
    if (Vr != Vl) Vr[pv0 - a.P + j] = t;
    eos_hit |= (t == a.eos_v);
  }
  const int pv = pv0 + na;
  s->len = pv;
  s->kv_len = pv - 1;
  s->pred_valid = 0;
  const long long now = globaltimer();  // stamp before publishing (trace order)
  mb_write_both(&R->vb.p_v, &L->vb.p_v, pv);
  R->vb.verify_steps += 1;
  if (L != R) L->vb.verify_steps = R->vb.verify_steps;
  if (miss >= 0) {  // request_rollback(target = p_v, correction)
    R->vb.rb_target = pv;
    R->vb.rb_correction = a.vtok[pv - 1];
    if (L != R) { L->vb.rb_target = pv; L->vb.rb_correction = a.vtok[pv - 1]; }
    R->vb.rollbacks += 1;
    if (L != R) L->vb.rollbacks = R->vb.rollbacks;
    c->rb_ack_local += 1;
    mb_write_both(&R->vb.rb_req, &L->vb.rb_req, c->rb_ack_local);
  }
  trace_push(a.vtrace, now, now - c->t0, miss >= 0 ? 2 : 1, pv0 + 1, pv, miss >= 0 ? miss : m);
  if (eos_hit || pv - a.P >= a.N) {
    mb_write_both(&R->vb.complete, &L->vb.complete, 1);
    stop_loop(a, c);
  }
}

// ---------------------------------------------------------- autoregressive
// AutoregressiveStepper.next_unit (engines.py:150-157).
__global__ void k_ar_begin(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  a.mb_local->vb.iters += 1;
  SeqHdr* s = a.vseq;
  const int npend = s->len - s->kv_len;
  c->npend = npend;
  c->rows = npend;
  c->m = 1;
  c->pos0 = s->kv_len;
  for (int i = 0; i < npend; ++i) c->tok[i] = a.vtok[s->kv_len + i];
  c->t0 = globaltimer();
  c->active = 1;
}

__global__ void k_ar_end(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  if (!c->active) return;
  SeqHdr* s = a.vseq;
  MailboxHdr* L = a.mb_local;
  const int t = c->preds[c->rows - 1];
  const int n = s->len;
  a.vtok[n] = t;
  s->len = n + 1;
  s->kv_len = n;
  s->pred_valid = 0;
  mb_V(L, a.cap)[n - a.P] = t;
  L->vb.p_v = n + 1;
  L->vb.verify_steps += 1;
  const long long now = globaltimer();
  trace_push(a.vtrace, now, now - c->t0, 1, n + 1, n + 1, 0);
  if (t == a.eos_v || n + 1 - a.P >= a.N) {
    L->vb.complete = 1;
    stop_loop(a, c);
  }
}

// ------------------------------------------------------------ synchronous
// SyncSpeculativeStepper (engines.py:160-259) as one device loop body:
// round_begin, k x (draft_begin, draft forward, draft_end), verify_begin,
// verify forward (k+1 rows: the last one yields the bonus), verify_end.
__global__ void k_sync_round_begin(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  a.mb_local->vb.iters += 1;
  const int verified = a.vseq->len - a.P;
  c->kr = min(a.k, a.N - verified);  // engines.py:190-191
  c->ncand = 0;
  c->t0 = globaltimer();
}

__global__ void k_sync_draft_begin(ProtoArgs a, int i) {
  if (threadIdx.x != 0) return;
  StepCtl* d = a.dctl;
  SeqHdr* s = a.dseq;
  if (i >= a.vctl->kr) { d->active = 0; return; }
  const int npend = s->len - s->kv_len;
  d->npend = npend;
  d->rows = npend;
  d->pos0 = s->kv_len;
  for (int j = 0; j < npend; ++j) d->tok[j] = a.dtok[s->kv_len + j];
  d->t0 = globaltimer();
  d->active = 1;
}

__global__ void k_sync_draft_end(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* d = a.dctl;
  if (!d->active) return;
  SeqHdr* s = a.dseq;
  StepCtl* v = a.vctl;
  const int n = s->len;
  const int tok = coin_pick(a.coin, n, d->preds[d->rows - 1]);
  s->kv_len = n;
  a.dtok[n] = tok;
  coin_push(a.coin, n, tok);
  s->len = n + 1;
  v->cand[v->ncand++] = tok;
  a.mb_local->db.drafted += 1;
  const long long now = globaltimer();
  trace_push(a.dtrace, now, now - d->t0, 0, n + 1, n + 1, 0);
}

__global__ void k_sync_verify_begin(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  SeqHdr* s = a.vseq;
  const int npend = s->len - s->kv_len;
  c->npend = npend;
  c->m = c->kr;
  c->rows = npend + c->kr;
  c->pos0 = s->kv_len;
  for (int i = 0; i < npend; ++i) c->tok[i] = a.vtok[s->kv_len + i];
  for (int j = 0; j < c->kr; ++j) c->tok[npend + j] = c->cand[j];
  c->t0 = globaltimer();
  c->active = 1;
}

__global__ void k_sync_verify_end(ProtoArgs a) {
  if (threadIdx.x != 0) return;
  StepCtl* c = a.vctl;
  SeqHdr* vs = a.vseq;
  SeqHdr* ds = a.dseq;
  MailboxHdr* L = a.mb_local;
  const int kr = c->kr, npend = c->npend, frontier = vs->len;
  int miss = -1;
  for (int j = 0; j < kr; ++j)
    if (c->cand[j] != c->preds[npend - 1 + j]) { miss = j; break; }
  const int na = miss < 0 ? kr + 1 : miss + 1;
  bool eos_hit = false;
  int* V = mb_V(L, a.cap);
  for (int j = 0; j < na; ++j) {
    const int t = (j < kr && j != miss) ? c->cand[j] : c->preds[npend - 1 + j];
    a.vtok[frontier + j] = t;
    V[frontier - a.P + j] = t;
    eos_hit |= (t == a.eos_v);
  }
  vs->len = frontier + na;
  vs->kv_len = frontier + na - 1;
  vs->pred_valid = 0;
  if (miss < 0) {  // draft advances the bonus (engines.py:221)
    const int t = a.vtok[frontier + kr];
    a.dtok[ds->len] = t;
    coin_push(a.coin, ds->len, t);
    ds->len += 1;
  } else {         // draft rollback(frontier) + advance(accepted) (engines.py:227-228)
    for (int j = miss; j < na; ++j) {
      a.dtok[frontier + j] = a.vtok[frontier + j];
      coin_push(a.coin, frontier + j, a.vtok[frontier + j]);
    }
    ds->len = frontier + na;
    if (ds->kv_len > ds->len - 1) ds->kv_len = ds->len - 1;
  }
  ds->pred_valid = 0;
  L->vb.p_v = frontier + na;
  L->db.p_d = ds->len;
  L->vb.verify_steps += 1;
  const bool done = eos_hit || frontier + na - a.P >= a.N;
  const long long now = globaltimer();
  trace_push(a.vtrace, now, now - c->t0, miss >= 0 ? 2 : 1, frontier + 1, frontier + na, miss >= 0 ? miss : kr);
  if (miss >= 0) {
    L->vb.rollbacks += 1;
    if (!done) trace_push(a.dtrace, now, 0, 3, frontier + miss + 1, frontier + kr, 0);
  }
  if (done) {
    L->vb.complete = 1;
    stop_loop(a, c);
  }
}

// ------------------------------------------------------------------ reset
// Fresh SharedDecodeState (coordination.py:117-140) + coin chain over the
// prompt.  The models already hold init_state(prompt).
__global__ void k_session_reset(ProtoArgs a, const int* prompt, unsigned long long coin_seed) {
  if (threadIdx.x != 0) return;
  {  // each GPU of a split pair resets its own copy (host barrier follows)
    MailboxHdr* m = a.mb_local;
    m->vb.p_v = a.P; m->vb.rb_req = 0; m->vb.rb_target = 0; m->vb.rb_correction = 0;
    m->vb.complete = 0; m->vb.error = 0; m->vb.verify_steps = 0; m->vb.rollbacks = 0; m->vb.iters = 0;
    m->db.p_d = a.P; m->db.rb_ack = 0; m->db.error = 0; m->db.drafted = 0; m->db.acks = 0; m->db.iters = 0;
  }
  if (a.dctl) { a.dctl->rb_ack_local = 0; a.dctl->active = 0; a.dctl->t0 = globaltimer(); }
  if (a.vctl) { a.vctl->rb_ack_local = 0; a.vctl->active = 0; a.vctl->t0 = globaltimer(); }
  if (a.dtrace.count) *a.dtrace.count = 0;
  if (a.vtrace.count) *a.vtrace.count = 0;
  if (a.tp_in) { a.tp_in->seq = 0; a.tp_in->stop = 0; }
  if (a.coin.hash) {
    a.coin.hash[0] = mix64(coin_seed);
    a.coin.onpath[0] = 1;
    for (int n = 0; n < a.P; ++n) coin_push(a.coin, n, prompt[n]);
  }
}

// ----------------------------------------------- hash-chain model (K7)
// One "forward" of the chain: row j incorporates token tok[j] at absolute
// index pos0+j (h[pos0+j+1] = splitmix64(h[pos0+j] ^ tok)) and predicts the
// next token from it (models.py:221-235, 256-268).
__global__ void k_hash_forward(StepCtl* c, unsigned long long* h, int vocab, int eos, int exclude_eos, int agree,
                               int always, unsigned long long thr, const int* script, int script_len, int eos_pos) {
  pdl_wait();
  if (threadIdx.x != 0 || !c->active) return;
  for (int j = 0; j < c->rows; ++j) {
    const int p = c->pos0 + j;
    if (script) {
      // ScriptedModel._predict (models.py:340-344): the token at 1-based absolute position
      // prefix_length + 1, where prefix_length = p + 1 after consuming row j
      const int pos1 = p + 2;
      c->preds[j] = pos1 == eos_pos ? eos : script[(pos1 - 1) % script_len];
      continue;
    }
    const unsigned long long hp = mix64(h[p] ^ (unsigned long long)(unsigned)c->tok[j]);
    h[p + 1] = hp;
    const int base = chain_draw(hp, vocab, eos, exclude_eos);
    // AgreementDraftModel._token_from_hash (models.py:300-304)
    c->preds[j] = (!agree || always) ? base : coin_token(hp, base, thr, vocab, eos, exclude_eos);
  }
  pdl_launch();
}

__global__ void k_hash_seed(unsigned long long* h, unsigned long long seed) { h[0] = mix64(seed); }

// ---------------------------------------------------------- launchers
cudaError_t proto_launch(int which, const ProtoArgs& a, cudaStream_t st, int arg) {
  switch (which) {
    case kDraftBegin: k_draft_begin<<<1, 32, 0, st>>>(a); break;
    case kDraftEnd: k_draft_end<<<1, 32, 0, st>>>(a); break;
    case kVerifyBegin: k_verify_begin<<<1, 32, 0, st>>>(a); break;
    case kVerifyEnd: k_verify_end<<<1, 32, 0, st>>>(a); break;
    case kArBegin: k_ar_begin<<<1, 32, 0, st>>>(a); break;
    case kArEnd: k_ar_end<<<1, 32, 0, st>>>(a); break;
    case kSyncRoundBegin: k_sync_round_begin<<<1, 32, 0, st>>>(a); break;
    case kSyncDraftBegin: k_sync_draft_begin<<<1, 32, 0, st>>>(a, arg); break;
    case kSyncDraftEnd: k_sync_draft_end<<<1, 32, 0, st>>>(a); break;
    case kSyncVerifyBegin: k_sync_verify_begin<<<1, 32, 0, st>>>(a); break;
    case kSyncVerifyEnd: k_sync_verify_end<<<1, 32, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_session_reset(const ProtoArgs& a, const int* prompt_dev, unsigned long long coin_seed,
                                 cudaStream_t st) {
  k_session_reset<<<1, 32, 0, st>>>(a, prompt_dev, coin_seed);
  return cudaGetLastError();
}

cudaError_t launch_hash_forward(StepCtl* c, unsigned long long* h, int vocab, int eos, int excl, int agree, int always,
                                unsigned long long thr, const int* script, int script_len, int eos_pos,
                                cudaStream_t st) {
  k_hash_forward<<<1, 32, 0, st>>>(c, h, vocab, eos, excl, agree, always, thr, script, script_len, eos_pos);
  return cudaGetLastError();
}
cudaError_t launch_hash_seed(unsigned long long* h, unsigned long long seed, cudaStream_t st) {
  k_hash_seed<<<1, 1, 0, st>>>(h, seed);
  return cudaGetLastError();
}
}  // namespace amusd
