// internal.h -- device-side records shared by the protocol and model kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/amusd.h"

namespace amusd {

constexpr int KMAX = AMUSD_KMAX;

// Mailbox = SharedDecodeState (coordination.py:114-275) laid out in HBM.
// Two 128-byte blocks, one per writer (single-writer discipline,
// coordination.py:6-12), then the D and V token buffers.  In a split pair
// each GPU holds a copy; a writer stores into the PEER copy (NVLink P2P) and,
// for host read-back, its own; readers poll only their local copy.
struct alignas(128) MbVerifyBlock {  // written by verify, polled by draft
  int p_v;            // verified frontier (absolute)       coordination.py:137
  int rb_req;         // rollback request epoch             coordination.py:240
  int rb_target;      // RollbackRequest.target             coordination.py:110
  int rb_correction;  // RollbackRequest.correction_token   coordination.py:111
  int complete;       // completion flag                    coordination.py:257
  int error;          // protocol-violation word (0 = ok)
  int verify_steps, rollbacks;
  int iters;          // verify loop iterations (kernel-launch accounting)
  int pad[23];
};
struct alignas(128) MbDraftBlock {  // written by draft, polled by verify
  int p_d;            // draft frontier (absolute)          coordination.py:136
  int rb_ack;         // rollback acknowledgment epoch      coordination.py:188
  int error;
  int drafted, acks;
  int iters;          // draft loop iterations (kernel-launch accounting)
  int pad[26];
};
struct MailboxHdr {
  MbVerifyBlock vb;
  MbDraftBlock db;
  // followed by: int D[cap]; int V[cap];
};
inline size_t mailbox_bytes(int cap) { return sizeof(MailboxHdr) + 2 * sizeof(int) * (size_t)cap; }
__host__ __device__ inline int* mb_D(MailboxHdr* m) { return (int*)(m + 1); }
__host__ __device__ inline int* mb_V(MailboxHdr* m, int cap) { return (int*)(m + 1) + cap; }

// Per-model sequence state (ModelState, models.py:58-82) with the
// pending-token scheme: tokens[0..len) is the prefix, positions [0, kv_len)
// are in the model cache (KV / hash chain), kv_len <= len - 1 in steady state.
struct SeqHdr {
  int len;
  int kv_len;
  int prompt_len;
  int cap;
  int pred_valid;  // cached next_token for the current prefix (parity API)
  int pred;
  int pad[2];
};

// Per-actor step control: written by the actor's begin kernel, read by the
// model forward, written back (preds) by the forward's last kernel.
struct StepCtl {
  int active;          // 0 => every kernel of this step returns at once
  int rows;            // rows forwarded this step (<= KMAX)
  int pos0;            // absolute 0-based position of row 0 (= kv_len)
  int npend;           // pending prefix tokens forwarded first
  int m;               // candidates in the window (verify) / drafted (sync)
  int rb_ack_local;    // draft: last acknowledged epoch; verify: last request epoch
  int kr;              // sync: drafts this round
  int ncand;           // sync: drafted so far this round
  long long t0;        // %globaltimer at step start
  int tok[KMAX];       // row input tokens
  int cand[KMAX];      // candidates under verification
  int preds[KMAX];     // model predictions per row
};

// Tensor-parallel verify group (BASELINE config 4): the leader rank's
// k_verify_begin snapshots the draft window once and pushes the step control
// into every follower rank's inbox (peer HBM, payload then st.release.sys of
// seq); followers run the same sharded forward and k_verify_end on identical
// inputs, so every rank reaches the same predictions and the same sequence
// state without further messages.
struct alignas(128) TpInbox {
  int seq;    // the leader's verify iteration this payload belongs to
  int stop;   // 1: the leader ended its loop in k_verify_begin (error / timeout)
  int pad[30];
  StepCtl ctl;
};
constexpr int kMaxTpOut = 7;

struct TraceDev {
  amusd_trace_event* ev;
  int* count;
  int cap;
};

struct CoinDev {
  int mode;                 // amusd_coin_mode
  unsigned long long thr;   // int(rho * 2**64), models.py:298
  int always;               // rho == 1.0
  int vocab, eos, exclude_eos;
  unsigned long long* hash; // [cap+1] chain after n tokens of the DRAFT prefix
  unsigned char* onpath;    // [cap+1] prefix == canonical prefix
  const int* canon;         // absolute canonical tokens (prompt included)
  int canon_len;
};

// Everything a protocol kernel needs for one side (draft or verify).
struct ProtoArgs {
  MailboxHdr* mb_local;
  MailboxHdr* mb_peer;      // == mb_local when co-located
  int cap;                  // mailbox D/V capacity
  int P, N, lead, max_window, k;
  SeqHdr* dseq; int* dtok;  // draft sequence state (may be null on verify-only side)
  SeqHdr* vseq; int* vtok;  // verify sequence state
  StepCtl* dctl;
  StepCtl* vctl;
  TraceDev dtrace, vtrace;
  CoinDev coin;
  int vocab_v, eos_v;       // verify model vocab / eos (completion check)
  int jitter_ns;
  unsigned long long jitter_seed;
  // AMUSD verify pacing (timing only: any interleaving of the two loops is a valid AMUSD run):
  // a step waits until the draft window holds >= min_window tokens or wait_ns have passed
  // since the first one appeared (1 / 0 = verify whatever is there, the reference's pacing)
  int min_window;
  long long wait_ns;
  cudaGraphConditionalHandle cond;
  int has_cond;
  TpInbox* tp_out[kMaxTpOut];  // leader: the followers' inboxes
  int tp_nout;
  TpInbox* tp_in;              // follower: this rank's inbox (null otherwise)
};

}  // namespace amusd
