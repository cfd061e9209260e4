"""AMUSD with the draft and the verify model on separate GPUs (BASELINE config 2).

The paper's deployment: draft on GPU0, verify on GPU1,
coordinated through shared state.  Here each GPU owns one copy of the HBM
mailbox (SharedDecodeState, coordination.py:114-275); every field keeps its
single writer, which stores into the PEER's copy over NVLink P2P
(`st.release.sys`) while readers poll their local copy (`ld.acquire.sys`):
D / p_d / rb_ack are written by the draft into the verify GPU's copy, V /
p_v / the rollback request / completion by the verify into the draft GPU's
copy (and its own, for read-back).  The device loops are the same protocol
kernels as the co-located engine (engines AMUSD_ENGINE_ASYNC_DRAFT /
_ASYNC_VERIFY of libamusd).

Two ways to run it:

* ``decode_speculative_async_split(model, prompt, config, link=SplitLink())``
  -- one process per GPU under ``torch.distributed`` (torchrun, 2 ranks):
  the draft rank passes its draft model, the verify rank its verify model.
  The mailbox copies are exchanged as CUDA IPC handles, the canonical path
  (AgreementDraft's coin input) is sent from the verify rank to the draft
  rank, the two device clocks are aligned for the trace, and both ranks get
  the same ``DecodeResult``.
* ``decode_speculative_async_split(draft, prompt, config, verify=verify)`` --
  one process holding both models (possibly on one GPU): two sessions, two
  mailbox copies, the same split protocol.  This is how the split protocol is
  tested when only one GPU is available.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib as L
from .engines import DecodeConfig, DecodeResult, DeviceSession, _model_of, canonical_path, finalize_tokens
from .errors import InvalidInputError, SpecDecError
from .metrics import summarize, trace_from_device
from .models import settle


class SplitLink:
    """Host-side link between the draft rank and the verify rank.

    Only object collectives over ``torch.distributed`` (any backend, gloo
    included): handle / metadata exchange, the canonical path, clock samples
    and the trace rows.  Nothing on the decode path goes through it.
    """

    def __init__(self, group=None, draft_rank: int = 0, verify_rank: int = 1):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise InvalidInputError("SplitLink needs an initialised torch.distributed process group")
        self.dist, self.group = dist, group
        if dist.get_world_size(group) != 2:
            raise InvalidInputError("a split pair is exactly two ranks (draft, verify)")
        self.draft_rank, self.verify_rank = draft_rank, verify_rank
        me = dist.get_rank(group)
        if me not in (draft_rank, verify_rank):
            raise InvalidInputError("this rank is neither the draft nor the verify rank")
        self.role = "draft" if me == draft_rank else "verify"

    def exchange(self, obj):
        """Send `obj` to the peer, return the peer's object (all_gather of two)."""
        out = [None, None]
        self.dist.all_gather_object(out, obj, group=self.group)
        me = 0 if self.dist.get_rank(self.group) == min(self.draft_rank, self.verify_rank) else 1
        return out[1 - me]

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)


@dataclass
class _Half:
    session: DeviceSession
    mailbox: torch.Tensor
    stream: torch.cuda.Stream
    engine: int
    peer_base: int = 0          # imported IPC base (distributed mode) to close after the run


def _export(lib, t: torch.Tensor) -> tuple:
    h = (C.c_uint8 * 64)()
    off = C.c_size_t()
    L.check(lib.amusd_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
    return bytes(h), off.value


def _import(lib, handle: bytes, offset: int) -> tuple:
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    ptr, base = C.c_void_p(), C.c_void_p()
    L.check(lib.amusd_ipc_import(h, offset, C.byref(ptr), C.byref(base)))
    return ptr.value, base.value


# The last distributed run of this process: its actor's loop iterations and kernels per step
# (bench.py's gpu_launches).
last_run: dict = {}


def _clock(lib, dev, stream) -> int:
    v = C.c_int64()
    with torch.cuda.device(dev):
        scratch = torch.empty(1, dtype=torch.int64, device=dev)
        torch.cuda.current_stream(dev).synchronize()
        L.check(lib.amusd_device_clock(C.byref(v), C.c_void_p(scratch.data_ptr()), stream.cuda_stream))
    return v.value


def _coin_meta(draft) -> dict:
    return {"coin_mode": int(getattr(draft, "coin_mode", L.COIN_NONE)),
            "rho": getattr(draft, "agreement_rho", None), "coin_seed": getattr(draft, "coin_seed", 0)}


def _result(verified, draft_rows, verify_rows, prompt_len, eos, config) -> DecodeResult:
    tokens, finished_by = finalize_tokens(verified, eos, config.max_new_tokens)
    trace = trace_from_device(draft_rows, verify_rows, prompt_len, prompt_len + len(tokens))
    return DecodeResult(tokens, finished_by, summarize(trace), trace)


def _mark_stale(session: DeviceSession) -> None:
    """The loop advances the models' device state: the next run must init_state again."""
    for m in (session.draft, session.verify):
        if m is not None:
            _model_of(m)._fresh = None


def _run_halves(halves, prompt) -> list:
    """Reset both mailbox copies, then launch both loops with no cross-stream waits
    (the verify loop spins on the draft's tokens: a stream dependency would deadlock)."""
    lib = L.load()
    for h in halves:  # graphs first: instantiation may wait for the device (see amusd_session_build)
        with torch.cuda.device(h.session.device):
            L.check(lib.amusd_session_build(h.session._h, h.engine))
    for h in halves:
        h.session.prepare(prompt)
    for h in halves:
        torch.cuda.synchronize(h.session.device)
    events = []
    for h in halves:
        dev = h.session.device
        with torch.cuda.device(dev):
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(h.stream)
            L.check(lib.amusd_session_launch(h.session._h, h.engine, h.stream.cuda_stream, h.stream.cuda_stream))
            end.record(h.stream)
            events.append((start, end))
        _mark_stale(h.session)
    outs = []
    for h, (start, end) in zip(halves, events):
        with torch.cuda.device(h.session.device):
            h.stream.synchronize()
        outs.append((h, start.elapsed_time(end)))
    return outs


def _collect(half: _Half):
    s = half.session
    lib = L.load()
    info = L.RunInfo()
    with torch.cuda.device(s.device):
        st = half.stream.cuda_stream
        L.check(lib.amusd_session_info(s._h, C.byref(info), s._v_buf, s.mb_cap, st))
        rows = []
        for actor in (0, 1):
            cnt = C.c_int()
            L.check(lib.amusd_session_trace(s._h, actor, s._trace_buf, len(s._trace_buf), C.byref(cnt), st))
            if cnt.value > len(s._trace_buf):
                raise SpecDecError(f"trace ring overflow ({cnt.value} events)")
            rows.append([(e.t_ns, e.busy_ns, e.kind, e.pos_lo, e.pos_hi, e.draft_accepted)
                         for e in s._trace_buf[:cnt.value]])
    if info.error:
        raise SpecDecError(f"device mailbox reported protocol error code {info.error}")
    return info, rows, list(s._v_buf[:max(0, info.p_v - s.prompt_len)])


def decode_speculative_async_split(model, prompt: Sequence[int], config: DecodeConfig, *, verify=None,
                                   link: SplitLink | None = None, max_window: int = L.KMAX):
    """AMUSD (engines.py:534-561 semantics) with draft and verify on separate devices.

    Distributed: pass `link` and this rank's model (draft on the draft rank, verify on
    the verify rank).  Single process: pass the draft as `model` and `verify=`.
    Returns ``(DecodeResult, (draft_ms, verify_ms))`` -- the result on both ranks in
    distributed mode, and each side's device-timed decode milliseconds.
    """
    if len(prompt) == 0:
        raise InvalidInputError("prompt must be non-empty")
    lib = L.load()
    prompt = list(prompt)
    N = config.max_new_tokens
    if link is None:  # ---------------------------------------------- one process
        if verify is None:
            raise InvalidInputError("single-process split needs verify=")
        draft = model
        dm, vm = _model_of(draft), _model_of(verify)
        canon = None
        if getattr(draft, "coin_mode", L.COIN_NONE) == L.COIN_CANON:
            canon = canonical_path(verify, prompt, N + L.KMAX).to(dm.device)
        mbytes = DeviceSession.mailbox_bytes(len(prompt), config)
        mb_d = torch.zeros(mbytes, dtype=torch.uint8, device=dm.device)
        mb_v = torch.zeros(mbytes, dtype=torch.uint8, device=vm.device)
        sd = DeviceSession(draft, None, len(prompt), config, max_window=max_window, canon=canon,
                           mb_local=mb_d, mb_peer=mb_v.data_ptr())
        sv = DeviceSession(None, verify, len(prompt), config, max_window=max_window,
                           mb_local=mb_v, mb_peer=mb_d.data_ptr())
        with torch.cuda.device(dm.device):
            st_d = torch.cuda.Stream()
        with torch.cuda.device(vm.device):
            st_v = torch.cuda.Stream()
        halves = [_Half(sv, mb_v, st_v, L.ENGINE_ASYNC_VERIFY), _Half(sd, mb_d, st_d, L.ENGINE_ASYNC_DRAFT)]
        timed = _run_halves(halves, prompt)
        vinfo, vrows, verified = _collect(halves[0])
        _, drows, _ = _collect(halves[1])
        if not vinfo.complete:
            raise SpecDecError("split pair ended without completion")
        res = _result(verified, drows[0], vrows[1], len(prompt), vm.eos_token, config)
        return res, (timed[1][1], timed[0][1])
    # ------------------------------------------------------------- distributed
    role = link.role
    m = _model_of(model)
    dev = m.device
    meta = {"role": role, "eos": m.eos_token, "vocab": m.vocab_size}
    if role == "draft":
        meta.update(_coin_meta(model))
    peer = link.exchange(meta)
    if peer["role"] == role:
        raise InvalidInputError("both ranks claim the same role")
    coin = meta if role == "draft" else peer
    canon_list = None
    if role == "verify" and coin["coin_mode"] == L.COIN_CANON:
        canon_list = canonical_path(model, prompt, N + L.KMAX).tolist()
    received = link.exchange(canon_list)    # verify -> draft (the draft sends None)
    canon = None
    if role == "draft" and received:
        canon = torch.tensor(received, dtype=torch.int32, device=dev)
    mbytes = DeviceSession.mailbox_bytes(len(prompt), config)
    mb = torch.zeros(mbytes, dtype=torch.uint8, device=dev)
    settle(dev)
    handle, off = _export(lib, mb)
    peer_handle, peer_off = link.exchange((handle, off))
    peer_ptr, peer_base = _import(lib, peer_handle, peer_off)
    try:
        if role == "draft":
            s = DeviceSession(model, None, len(prompt), config, max_window=max_window, canon=canon, mb_local=mb,
                              mb_peer=peer_ptr)
        else:
            s = DeviceSession(None, model, len(prompt), config, max_window=max_window, mb_local=mb,
                              mb_peer=peer_ptr)
        with torch.cuda.device(dev):
            st = torch.cuda.Stream()
        half = _Half(s, mb, st, L.ENGINE_ASYNC_DRAFT if role == "draft" else L.ENGINE_ASYNC_VERIFY, peer_base)
        with torch.cuda.device(dev):
            L.check(lib.amusd_session_build(s._h, half.engine))  # before either loop can spin
        s.prepare(prompt)
        torch.cuda.synchronize(dev)
        link.barrier()                      # both copies reset before any peer store
        clk = _clock(lib, dev, st)
        peer_clk = link.exchange(clk)       # sampled right after a barrier: offset within the barrier skew
        with torch.cuda.device(dev):
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(st)
            L.check(lib.amusd_session_launch(s._h, half.engine, st.cuda_stream, st.cuda_stream))
            _mark_stale(s)
            end.record(st)
            st.synchronize()
        ms = start.elapsed_time(end)
        info, rows, verified = _collect(half)
        last_run.clear()
        last_run.update({"role": role, "iters": info.draft_iters if role == "draft" else info.verify_iters,
                         "kernels_per_step": half.session.kernels_per_step(half.engine)[0 if role == "draft" else 1]})
        mine = rows[0] if role == "draft" else rows[1]
        if role == "draft":  # express the draft events on the verify GPU's clock
            shift = peer_clk - clk
            mine = [(r[0] + shift,) + tuple(r[1:]) for r in mine]
        theirs = link.exchange({"rows": mine, "ms": ms, "verified": verified if role == "verify" else None,
                                "complete": bool(info.complete)})
        link.barrier()                      # the peer is done storing into our copy
    finally:
        lib.amusd_ipc_close(C.c_void_p(peer_base))
    drows, vrows = (mine, theirs["rows"]) if role == "draft" else (theirs["rows"], mine)
    v_tokens = verified if role == "verify" else theirs["verified"]
    eos = m.eos_token if role == "verify" else peer["eos"]
    res = _result(v_tokens, drows, vrows, len(prompt), eos, config)
    return res, ((ms, theirs["ms"]) if role == "draft" else (theirs["ms"], ms))
