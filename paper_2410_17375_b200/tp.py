"""Tensor-parallel verify model (BASELINE config 4: 1B draft + a TP-sharded verify).

The reference has no transformer and no parallelism beyond its two actor
threads (engines.py:448-459); north_star asks for the verify model sharded
over GPUs with an allreduce over NVLink.  Layout (Megatron-style, per rank):

* QKV column-parallel by whole KV groups (each rank owns G query heads per
  group plus that group's K/V head, its KV cache and its attention items);
* O row-parallel over the same heads;
* gate/up column-parallel over whole feature blocks, down row-parallel;
* LM head vocab-parallel over whole 128-row tiles;
* embedding and RMSNorm weights replicated, residual stream replicated.

The two allreduces per layer are not separate collectives: the persistent
forward's split-K epilogue red.adds each O / down chunk's exact int64 partial
into EVERY rank's accumulator over peer memory (NVLink P2P atomics) and bumps
every rank's tile count; each rank merges the all-rank sum itself
(csrc/forward_tc.cu).  The LM head's (value, first-index) argmax keys go to
every rank the same way.  Integer adds commute, so every rank computes the same
residual stream -- bit-identical to the unsharded forward, whose chunking the
shards take (amusd_tf_create_shard).

Engines:

* ``TPGroup.decode_autoregressive`` / ``decode_speculative_sync``: every rank
  runs the reference stepper's device loop on its shard (sync-SD with a draft
  replica per rank); their inputs are identical by construction, so no step
  control is exchanged.
* ``TPGroup.decode_speculative_async``: the draft on its own GPU (config 4:
  GPU0) publishes into the LEADER rank's mailbox copy; the leader's
  k_verify_begin snapshots the window and pushes the step control into every
  follower's inbox (csrc/protocol.cu tp_push / tp_follow).

One process holds all ranks here (one Python thread per rank, one stream per
rank); on one GPU the ranks' grids are capped so that their forwards are
co-resident (``amusd_model_set_max_grid``).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, replace
from typing import Sequence

import torch

from . import _lib as L
from .engines import DecodeConfig, DecodeResult, DeviceSession, _model_of, finalize_tokens
from .errors import InvalidInputError, SpecDecError
from .metrics import summarize, trace_from_device
from .models import (CudaModel, TransformerConfig, rope_tables, settle, synthetic_weight, weight_names)

__all__ = ["ShardSpec", "shard_spec", "TransformerShard", "TPGroup"]


@dataclass(frozen=True)
class ShardSpec:
    """Rank `rank` of `size`: global KV groups [kv0, kv1), ffn features [f0, f1), vocab rows [v0, v1)."""
    rank: int
    size: int
    kv0: int
    kv1: int
    f0: int
    f1: int
    v0: int
    v1: int


def _even(n: int, size: int, rank: int) -> tuple:
    base, extra = divmod(n, size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_spec(cfg: TransformerConfig, rank: int, size: int) -> ShardSpec:
    """Balanced contiguous shards: KV groups, ffn in 2048-feature blocks (256 when too few) so that
    the unsharded model's down-projection chunks never straddle two ranks, vocab in 128-row tiles."""
    if not 2 <= size <= 8 or not 0 <= rank < size:
        raise InvalidInputError("tensor parallelism needs 2 <= size <= 8 and 0 <= rank < size")
    if cfg.n_kv_heads < size:
        raise InvalidInputError(f"{cfg.n_kv_heads} KV heads cannot be sharded over {size} ranks")
    if cfg.vocab_size % 128 or cfg.ffn % 256:
        raise InvalidInputError("vocab must be a multiple of 128 and ffn of 256 for tensor parallelism")
    kv0, kv1 = _even(cfg.n_kv_heads, size, rank)
    blk = 2048 if cfg.ffn % 2048 == 0 and cfg.ffn // 2048 >= size else 256
    b0, b1 = _even(cfg.ffn // blk, size, rank)
    t0, t1 = _even(cfg.vocab_size // 128, size, rank)
    return ShardSpec(rank, size, kv0, kv1, b0 * blk, b1 * blk, t0 * 128, t1 * 128)


def _slice_weight(cfg: TransformerConfig, sp: ShardSpec, leaf: str, t: torch.Tensor) -> torch.Tensor:
    G, hd, H, KV = cfg.n_heads // cfg.n_kv_heads, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    if leaf == "wqkv":  # [q (H) | k (KV) | v (KV)] heads -> this rank's groups, same order
        q = t[sp.kv0 * G * hd: sp.kv1 * G * hd]
        k = t[H * hd + sp.kv0 * hd: H * hd + sp.kv1 * hd]
        v = t[(H + KV) * hd + sp.kv0 * hd: (H + KV) * hd + sp.kv1 * hd]
        return torch.cat([q, k, v]).contiguous()
    if leaf == "wo":
        return t[:, sp.kv0 * G * hd: sp.kv1 * G * hd].contiguous()
    if leaf in ("wgate", "wup"):
        return t[sp.f0: sp.f1].contiguous()
    if leaf == "wdown":
        return t[:, sp.f0: sp.f1].contiguous()
    if leaf == "lm_head":
        return t[sp.v0: sp.v1].contiguous()
    return t  # embed, norms: replicated


class TransformerShard(CudaModel):
    """One rank's shard of a Llama-style verify model (persistent tcgen05 forward only).

    Weights are the seeded synthetic model's (``TransformerModel(config, seed=...)`` holds the
    identical unsharded tensors) or slices of caller-provided full `weights`.  Tokens and
    predictions are global vocabulary ids; ``last_logits`` returns this rank's vocab slice."""

    def __init__(self, config: TransformerConfig, rank: int, size: int, seed: int = 0, device=None,
                 init_std: float = 0.02, weights: dict | None = None):
        super().__init__(config.vocab_size, config.eos_token, device)
        if config.dtype != "bf16" or not config.use_tensor_cores:
            raise InvalidInputError("tensor-parallel shards are bf16 tcgen05 models")
        self.config = config
        self.spec = sp = shard_spec(config, rank, size)
        G = config.n_heads // config.n_kv_heads
        self.local = replace(config, n_heads=(sp.kv1 - sp.kv0) * G, n_kv_heads=sp.kv1 - sp.kv0, ffn=sp.f1 - sp.f0,
                             vocab_size=sp.v1 - sp.v0, tied=False)
        keep = {}
        for i, n in enumerate(weight_names(config)):
            full = (weights[n].to(device=self.device, dtype=torch.bfloat16) if weights is not None
                    else synthetic_weight(config, i, n, torch.bfloat16, seed, init_std, self.device))
            leaf = n.split(".")[-1]
            keep[n] = _slice_weight(config, sp, leaf, full)
            if config.tied and n == "embed":
                keep["lm_head"] = _slice_weight(config, sp, "lm_head", full)
            del full
        self.weights = keep
        cos, sin = rope_tables(config)
        self.rope_cos, self.rope_sin = cos.to(self.device), sin.to(self.device)
        lc = self.local
        cfg = L.TfConfig(vocab=lc.vocab_size, d_model=lc.d_model, n_layers=lc.n_layers, n_heads=lc.n_heads,
                         n_kv_heads=lc.n_kv_heads, head_dim=lc.head_dim, ffn=lc.ffn, max_seq=lc.max_seq, dtype=L.BF16,
                         eos_token=lc.eos_token, exclude_eos=int(lc.exclude_eos), norm_eps=lc.norm_eps,
                         use_tensor_cores=1)
        shard = L.TpShard(tp_rank=rank, tp_size=size, n_heads_full=config.n_heads, n_kv_heads_full=config.n_kv_heads,
                          ffn_full=config.ffn, vocab_offset=sp.v0, vocab_total=config.vocab_size)
        w = L.TfWeights()
        p = lambda t: C.c_void_p(t.data_ptr())
        w.embed, w.lm_head, w.final_norm = p(keep["embed"]), p(keep["lm_head"]), p(keep["final_norm"])
        w.rope_cos, w.rope_sin = p(self.rope_cos), p(self.rope_sin)
        for l in range(config.n_layers):
            for leaf in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate", "wup", "wdown"):
                getattr(w, leaf)[l] = keep[f"layers.{l}.{leaf}"].data_ptr()
        self._cfg_c, self._shard_c, self._w_c = cfg, shard, w
        nbytes = self._lib.amusd_tf_shard_state_bytes(C.byref(cfg), C.byref(shard))
        self._state = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        settle(self.device)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_tf_create_shard(C.byref(self._h), C.byref(cfg), C.byref(shard), C.byref(w),
                                                    C.c_void_p(self._state.data_ptr()), nbytes))
            # the persistent forward streams only its tile-contiguous copy: drop the row-major slices
            L.check(self._lib.amusd_model_release_row_major(self._h))
        for n in [n for n in keep if not (n == "embed" or n.endswith("norm"))]:
            del keep[n]
        torch.cuda.empty_cache()

    def export(self) -> L.TpPeer:
        out = L.TpPeer()
        L.check(self._lib.amusd_tp_export(self._h, C.byref(out)))
        return out

    def connect(self, peers: Sequence[L.TpPeer]) -> None:
        arr = (L.TpPeer * len(peers))(*peers)
        L.check(self._lib.amusd_tp_connect(self._h, arr, len(peers)))

    def kernels_per_forward(self) -> int:
        return 1

    def last_logits(self, rows: int = 1):
        """fp32 logits of this rank's vocab rows [v0, v1) for the last `rows` forwarded rows."""
        out = torch.empty((rows, self.local.vocab_size), dtype=torch.float32)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_last_logits(self._h, C.cast(out.data_ptr(), C.POINTER(C.c_float)), rows,
                                                torch.cuda.current_stream(self.device).cuda_stream))
        return out


class TPGroup:
    """The `size` shards of one verify model, driven from this process (one thread per rank).

    ``devices``: one per rank (default: all on the current GPU -- a one-GPU emulation whose ranks
    share the SMs).  Ranks on one device get ``sms // ranks_on_device`` SMs each; ``reserve_sms``
    leaves SMs for a draft on the same device."""

    def __init__(self, config: TransformerConfig, size: int, seed: int = 0, devices=None, init_std: float = 0.02,
                 weights: dict | None = None, reserve_sms: int = 0):
        if devices is None:
            devices = [torch.device("cuda", torch.cuda.current_device())] * size
        devices = [torch.device(d) for d in devices]
        if len(devices) != size:
            raise InvalidInputError("one device per rank")
        self.config, self.size, self.devices = config, size, devices
        lib = L.load()
        for a in {d.index for d in devices}:
            for b in {d.index for d in devices}:
                L.check(lib.amusd_peer_enable(a, b))
        self.shards = [TransformerShard(config, r, size, seed, devices[r], init_std, weights) for r in range(size)]
        per_dev = {}
        for d in devices:
            per_dev[d.index] = per_dev.get(d.index, 0) + 1
        for s in self.shards:
            n = per_dev[s.device.index]
            if n > 1 or reserve_sms:
                sms = torch.cuda.get_device_properties(s.device).multi_processor_count
                s.set_max_grid((sms - reserve_sms) // n)
        peers = [s.export() for s in self.shards]
        for s in self.shards:
            s.connect(peers)
        self.streams = []
        for d in devices:
            with torch.cuda.device(d):
                self.streams.append((torch.cuda.Stream(), torch.cuda.Stream()))
        self.vocab_size, self.eos_token = config.vocab_size, config.eos_token

    # -------------------------------------------------------------- plumbing
    def run(self, fn) -> list:
        """fn(rank, shard, (verify_stream, draft_stream)) on every rank concurrently (one thread each)."""
        out, errs = [None] * self.size, []

        def body(r):
            try:
                with torch.cuda.device(self.devices[r]), torch.cuda.stream(self.streams[r][0]):
                    out[r] = fn(r, self.shards[r], self.streams[r])
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errs.append(e)
        th = [threading.Thread(target=body, args=(r,)) for r in range(self.size)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out

    def first_logits(self, prompt: Sequence[int]):
        """Full-vocabulary logits of the prediction after `prompt` (the ranks' slices concatenated)
        and every rank's greedy token (all equal: the all-rank argmax)."""
        def f(r, s, st):
            state = s.init_state(prompt)
            tok = s.next_token(state)
            return s.last_logits(1)[0], tok
        res = self.run(f)
        return torch.cat([x[0] for x in res]), [x[1] for x in res]

    # ---------------------------------------------------------------- engines
    def _sessions(self, drafts, prompt_len, config, engine_kw=None):
        return [DeviceSession(drafts[r] if drafts else None, self.shards[r], prompt_len, config,
                              stream_pair=self.streams[r], **(engine_kw or {})) for r in range(self.size)]

    def _run_sessions(self, sessions, engine, prompt):
        def prep(r, s, st):
            sessions[r].prepare(prompt)
            st[0].synchronize()
        self.run(prep)
        for s in sessions:   # graphs first: instantiation may wait for the device
            with torch.cuda.device(s.device):
                L.check(s.lib.amusd_session_build(s._h, engine))
        ev = []
        for s in sessions:
            ev.append(s.launch(engine))
        return [s.collect(*e) for s, e in zip(sessions, ev)]

    def _agree(self, outs):
        ref = outs[0].verified
        for r, o in enumerate(outs[1:], 1):
            if o.verified != ref:
                raise SpecDecError(f"tensor-parallel rank {r} diverged from rank 0")
        return outs[0]

    def decode_autoregressive(self, prompt: Sequence[int], config: DecodeConfig, return_outputs=False):
        """AutoregressiveStepper (engines.py:139-157) on the sharded verify model."""
        sess = self._sessions(None, len(prompt), config)
        outs = self._run_sessions(sess, L.ENGINE_AR, list(prompt))
        o = self._agree(outs)
        res = self._result(o.verified, o.draft_rows, o.verify_rows, len(prompt), config)
        return (res, outs) if return_outputs else res

    def decode_speculative_sync(self, drafts: Sequence, prompt: Sequence[int], config: DecodeConfig, canon=None,
                                return_outputs=False):
        """SyncSpeculativeStepper (engines.py:160-259): rank r drafts with its own replica drafts[r]
        (identical weights -> identical drafts), so the ranks' windows agree without messages."""
        if len(drafts) != self.size:
            raise InvalidInputError("one draft replica per rank")
        canon_r = [canon.to(_model_of(d).device) if canon is not None else None for d in drafts]
        sess = [DeviceSession(drafts[r], self.shards[r], len(prompt), config, canon=canon_r[r],
                              stream_pair=self.streams[r]) for r in range(self.size)]
        outs = self._run_sessions(sess, L.ENGINE_SYNC, list(prompt))
        o = self._agree(outs)
        res = self._result(o.verified, o.draft_rows, o.verify_rows, len(prompt), config)
        return (res, outs) if return_outputs else res

    def decode_speculative_async(self, draft, prompt: Sequence[int], config: DecodeConfig, canon=None,
                                 max_window: int = L.KMAX, return_outputs=False):
        """AMUSD (engines.py:534-561 semantics) with the draft on its own device and the verify
        model sharded: the draft <-> leader mailbox pair of the split layout, plus the leader's
        window broadcast to the followers."""
        prompt = list(prompt)
        dm = _model_of(draft)
        if canon is None and getattr(draft, "coin_mode", L.COIN_NONE) == L.COIN_CANON:
            ar = self.decode_autoregressive(prompt, DecodeConfig(max_new_tokens=config.max_new_tokens + L.KMAX))
            canon = torch.tensor(prompt + ar.tokens, dtype=torch.int32)
        mbytes = DeviceSession.mailbox_bytes(len(prompt), config)
        mb_d = torch.zeros(mbytes, dtype=torch.uint8, device=dm.device)
        mbs = [torch.zeros(mbytes, dtype=torch.uint8, device=d) for d in self.devices]
        with torch.cuda.device(dm.device):
            dstreams = (torch.cuda.Stream(), torch.cuda.Stream())
        sd = DeviceSession(draft, None, len(prompt), config, max_window=max_window,
                           canon=canon.to(dm.device) if canon is not None else None, mb_local=mb_d,
                           mb_peer=mbs[0].data_ptr(), stream_pair=dstreams)
        sv = [DeviceSession(None, self.shards[r], len(prompt), config, max_window=max_window, mb_local=mbs[r],
                            mb_peer=mb_d.data_ptr() if r == 0 else None, stream_pair=self.streams[r])
              for r in range(self.size)]
        lib = L.load()
        inboxes = []
        for s in sv[1:]:
            p = C.c_void_p()
            L.check(lib.amusd_session_tp_inbox(s._h, C.byref(p)))
            L.check(lib.amusd_session_set_tp(s._h, 2, None, 0))
            inboxes.append(p)
        arr = (C.c_void_p * len(inboxes))(*[p.value for p in inboxes])
        L.check(lib.amusd_session_set_tp(sv[0]._h, 1, arr, len(inboxes)))
        # prefill: the draft alone, the verify ranks together (their forwards meet in peer memory)
        with torch.cuda.device(dm.device), torch.cuda.stream(dstreams[0]):
            sd.prepare(prompt)
            dstreams[0].synchronize()

        def prep(r, s, st):
            sv[r].prepare(prompt)
            st[0].synchronize()
        self.run(prep)
        with torch.cuda.device(dm.device):
            L.check(lib.amusd_session_build(sd._h, L.ENGINE_ASYNC_DRAFT))
        for s in sv:
            with torch.cuda.device(s.device):
                L.check(lib.amusd_session_build(s._h, L.ENGINE_ASYNC_VERIFY))
        for d in {dm.device.index, *(d.index for d in self.devices)}:
            torch.cuda.synchronize(d)
        # launch every loop (no cross-stream waits: the loops spin on each other's words)
        ev = []
        for s, eng in [(x, L.ENGINE_ASYNC_VERIFY) for x in sv] + [(sd, L.ENGINE_ASYNC_DRAFT)]:
            vs, _ = s.streams()
            with torch.cuda.device(s.device):
                start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                start.record(vs)
                L.check(lib.amusd_session_launch(s._h, eng, vs.cuda_stream, vs.cuda_stream))
                end.record(vs)
                ev.append((start, end))
            for m in (s.draft, s.verify):
                if m is not None:
                    _model_of(m)._fresh = None
        outs = [s.collect(*e) for s, e in zip(sv + [sd], ev)]
        vouts, dout = outs[:-1], outs[-1]
        if not vouts[0].info.complete:
            raise SpecDecError("tensor-parallel AMUSD ended without completion")
        self._agree(vouts)
        res = self._result(vouts[0].verified, dout.draft_rows, vouts[0].verify_rows, len(prompt), config)
        return (res, outs) if return_outputs else res

    def _result(self, verified, draft_rows, verify_rows, prompt_len, config) -> DecodeResult:
        tokens, finished_by = finalize_tokens(verified, self.eos_token, config.max_new_tokens)
        trace = trace_from_device(draft_rows, verify_rows, prompt_len, prompt_len + len(tokens))
        return DecodeResult(tokens, finished_by, summarize(trace), trace)
