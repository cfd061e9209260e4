"""The three decoding strategies, executed as device-driven CUDA-graph loops.

Same entry points, arguments and results as the reference
(pkg/src/specdec/engines.py:52-88, 279-301, 534-561):

* ``decode_autoregressive(verify, prompt, config)``  -- one verify forward per token
* ``decode_speculative_sync(draft, verify, prompt, config)`` -- k drafts, batch verify, bonus/correction
* ``decode_speculative_async(draft, verify, prompt, config, executor=None)`` -- AMUSD

The per-token work never returns to the host: each engine is one (sync/AR)
or two (AMUSD: draft stream + verify stream) CUDA graphs whose bodies are
WHILE loops over the protocol kernels and the model forwards; completion is
decided on the device.  ``CudaAsyncExecutor`` is the executor plug-in
(engines.py:424-432 contract): it fills ``shared.V`` and returns a trace that
passes ``DecodeTrace.validate``.
"""
from __future__ import annotations

import ctypes as C
import weakref
from collections import OrderedDict
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib as L
from .coordination import SharedDecodeState
from .errors import InvalidInputError, ProtocolViolationError, SpecDecError
from .metrics import DecodeStats, DecodeTrace, summarize, trace_from_device
from .models import AgreementDraft, CudaModel, ModelState, settle

FINISHED_BY_EOS = "eos"
FINISHED_BY_LENGTH = "length_limit"


@dataclass(frozen=True)
class DecodeConfig:
    """Run limits shared by all strategies (engines.py:52-78)."""
    max_new_tokens: int
    draft_window_k: int = 4
    max_draft_lead: int | None = None
    seed: int = 0

    def __post_init__(self) -> None:
        if self.max_new_tokens < 1:
            raise InvalidInputError(f"max_new_tokens must be >= 1, got {self.max_new_tokens}")
        if self.draft_window_k < 1:
            raise InvalidInputError(f"draft_window_k must be >= 1, got {self.draft_window_k}")
        if self.max_draft_lead is not None and self.max_draft_lead < 1:
            raise InvalidInputError(f"max_draft_lead must be >= 1 when set, got {self.max_draft_lead}")


@dataclass(frozen=True)
class DecodeResult:
    """Generated tokens (prompt excluded), termination cause, stats, trace (engines.py:81-88)."""
    tokens: list
    finished_by: str
    stats: DecodeStats
    trace: DecodeTrace


def find_mismatch(candidates: Sequence[int], predictions: Sequence[int]):
    """Smallest 1-based index where the sequences differ, else None (engines.py:91-100).

    The device implementation is the scan at the top of k_verify_end."""
    if len(candidates) != len(predictions):
        raise InvalidInputError(
            f"length mismatch: {len(candidates)} candidates vs {len(predictions)} predictions")
    for i, (c, p) in enumerate(zip(candidates, predictions)):
        if c != p:
            return i + 1
    return None


def finalize_tokens(verified: Sequence[int], eos_token: int, max_new_tokens: int):
    """Cap at max_new_tokens, then end at the first eos (engines.py:103-113)."""
    capped = list(verified[:max_new_tokens])
    if eos_token in capped:
        return capped[: capped.index(eos_token) + 1], FINISHED_BY_EOS
    return capped, FINISHED_BY_LENGTH


# --------------------------------------------------------------------------- #
# Device sessions
# --------------------------------------------------------------------------- #

def _model_of(m):
    inner = m.model if isinstance(m, AgreementDraft) else m
    if not isinstance(inner, CudaModel):
        raise InvalidInputError(
            f"{type(m).__name__} is not a device model: the CUDA engines drive CudaModel instances "
            "(HashChainModel, AgreementDraftModel, TransformerModel, AgreementDraft)")
    return inner


_STREAMS: dict = {}


def streams(device) -> tuple:
    """(verify_stream, draft_stream) for a device.

    AMUSD_STREAM_PRIO = equal (default) | verify_high | draft_high.  Purely a
    scheduling knob for the co-located pair (never changes tokens)."""
    key = torch.device(device).index or 0
    if key not in _STREAMS:
        import os
        mode = os.environ.get("AMUSD_STREAM_PRIO", "equal")
        pv, pd = {"verify_high": (-1, 0), "draft_high": (0, -1)}.get(mode, (0, 0))
        with torch.cuda.device(key):
            _STREAMS[key] = (torch.cuda.Stream(priority=pv), torch.cuda.Stream(priority=pd))
    return _STREAMS[key]


@dataclass
class RunOutput:
    verified: list
    info: L.RunInfo
    draft_rows: list
    verify_rows: list
    device_ms: float


class DeviceSession:
    """libamusd session: mailbox + control blocks + trace rings + cached graphs.

    One per (draft, verify, prompt length, limits, coin); reusable across runs.
    """

    def __init__(self, draft, verify, prompt_len: int, config: DecodeConfig, *, max_window: int = L.KMAX,
                 canon: torch.Tensor | None = None, trace_cap: int | None = None, jitter_ns: int = 0,
                 jitter_seed: int = 0, mb_peer: int | None = None, mb_local: torch.Tensor | None = None,
                 stream_pair: tuple | None = None):
        self.lib = L.load()
        # (verify, draft) streams; default the device's shared pair.  Ranks of a tensor-parallel
        # group emulated on one GPU need their own: their forwards wait on each other.
        self._stream_pair = stream_pair
        # weak: a cached session must not keep its models (GBs of HBM) alive (see _session)
        self._draft = weakref.ref(draft) if draft is not None else None
        self._verify = weakref.ref(verify) if verify is not None else None
        dm = _model_of(draft) if draft is not None else None
        vm = _model_of(verify) if verify is not None else None
        if dm is not None and dm is vm:
            raise InvalidInputError("draft and verify must be distinct device models: a CudaModel holds one "
                                    "live sequence (KV cache and forward workspace)")
        self.device = (vm or dm).device
        self.config = config
        self.prompt_len = prompt_len
        coin_mode = getattr(draft, "coin_mode", L.COIN_NONE) if draft is not None else L.COIN_NONE
        if coin_mode == L.COIN_CANON and canon is None:
            raise InvalidInputError("AgreementDraft needs the canonical verify path (canon)")
        self.canon = canon
        n = config.max_new_tokens
        cap = trace_cap or ((config.draft_window_k + 2) * (n + 2 * L.KMAX) + 16 * (n + 64) + 1024)
        self.desc = L.SessionDesc(
            prompt_len=prompt_len, max_new_tokens=n, draft_window_k=config.draft_window_k,
            max_draft_lead=config.max_draft_lead or 0, max_window=max_window, coin_mode=coin_mode,
            rho=float(getattr(draft, "agreement_rho", None) or 0.0) if coin_mode != L.COIN_NONE else 0.0,
            coin_seed=getattr(draft, "coin_seed", 0), canon=C.c_void_p(canon.data_ptr()) if canon is not None else None,
            canon_len=int(canon.numel()) if canon is not None else 0, trace_cap=cap, jitter_ns=jitter_ns,
            jitter_seed=jitter_seed)
        self.mb_cap = self.lib.amusd_mailbox_capacity(C.byref(self.desc))
        mbytes = self.lib.amusd_mailbox_bytes(self.mb_cap)
        sbytes = self.lib.amusd_session_bytes(C.byref(self.desc))
        self.mailbox = mb_local if mb_local is not None else torch.zeros(mbytes, dtype=torch.uint8, device=self.device)
        self.mem = torch.zeros(sbytes, dtype=torch.uint8, device=self.device)
        self._h = C.c_void_p()
        L.check(self.lib.amusd_session_create(
            C.byref(self._h), dm.handle if dm else None, vm.handle if vm else None, C.byref(self.desc),
            C.c_void_p(self.mem.data_ptr()), sbytes, C.c_void_p(self.mailbox.data_ptr()),
            C.c_void_p(mb_peer) if mb_peer else None))
        settle(self.device)
        self._trace_buf = (L.TraceEvent * cap)()
        self._v_buf = (C.c_int32 * (self.mb_cap + 1))()

    @property
    def draft(self):
        return self._draft() if self._draft is not None else None

    @property
    def verify(self):
        return self._verify() if self._verify is not None else None

    @staticmethod
    def mailbox_bytes(prompt_len: int, config: DecodeConfig) -> int:
        lib = L.load()
        d = L.SessionDesc(prompt_len=prompt_len, max_new_tokens=config.max_new_tokens)
        return lib.amusd_mailbox_bytes(lib.amusd_mailbox_capacity(C.byref(d)))

    def kernels_per_step(self, engine: int) -> tuple:
        d, v = C.c_int(), C.c_int()
        L.check(self.lib.amusd_session_kernels_per_step(self._h, engine, C.byref(d), C.byref(v)))
        return d.value, v.value

    def streams(self) -> tuple:
        return self._stream_pair or streams(self.device)

    def prepare(self, prompt: Sequence[int]) -> None:
        """init_state(prompt) on the models (GPU prefill) and reset the mailbox."""
        vs, ds = self.streams()
        with torch.cuda.device(self.device), torch.cuda.stream(vs):
            for m in (self.draft, self.verify):
                if m is not None and _model_of(m)._fresh != tuple(prompt):
                    m.init_state(prompt)
            L.check(self.lib.amusd_session_reset(self._h, L.int_array(prompt), len(prompt), vs.cuda_stream))

    def launch(self, engine: int) -> tuple:
        """Enqueue the engine's graph(s); returns (start_event, end_event) on the verify stream."""
        vs, ds = self.streams()
        with torch.cuda.device(self.device):
            start, end, dend = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            start.record(vs)
            ds.wait_event(start)
            L.check(self.lib.amusd_session_launch(self._h, engine, vs.cuda_stream, ds.cuda_stream))
            for m in (self.draft, self.verify):
                if m is not None:
                    _model_of(m)._fresh = None
            dend.record(ds)
            vs.wait_event(dend)
            end.record(vs)
        return start, end

    def collect(self, start=None, end=None) -> RunOutput:
        vs, _ = self.streams()
        with torch.cuda.device(self.device):
            vs.synchronize()
            ms = start.elapsed_time(end) if start is not None else 0.0
            info = L.RunInfo()
            L.check(self.lib.amusd_session_info(self._h, C.byref(info), self._v_buf, self.mb_cap, vs.cuda_stream))
            rows = []
            for actor in (0, 1):
                cnt = C.c_int()
                L.check(self.lib.amusd_session_trace(self._h, actor, self._trace_buf, len(self._trace_buf),
                                                     C.byref(cnt), vs.cuda_stream))
                if cnt.value > len(self._trace_buf):
                    raise SpecDecError(f"trace ring overflow ({cnt.value} events > {len(self._trace_buf)})")
                k = cnt.value
                rows.append([(e.t_ns, e.busy_ns, e.kind, e.pos_lo, e.pos_hi, e.draft_accepted)
                             for e in self._trace_buf[:k]])
        if info.error:
            raise ProtocolViolationError(f"device mailbox reported protocol error code {info.error} "
                                         "(1 = spin timeout, 2 = bad rollback target)")
        nv = max(0, info.p_v - self.prompt_len)
        return RunOutput(list(self._v_buf[:nv]), info, rows[0], rows[1], ms)

    def run(self, engine: int, prompt: Sequence[int]) -> RunOutput:
        self.prepare(prompt)
        start, end = self.launch(engine)
        out = self.collect(start, end)
        if not out.info.complete:
            raise SpecDecError("device loop ended without completion")
        return out

    def __del__(self):
        try:
            if self._h:
                L.load().amusd_session_destroy(self._h)
        except Exception:
            pass


# Cached sessions / canonical paths, keyed by model identity.  Entries hold their models
# only weakly and are evicted when a model (or AgreementDraft wrapper) is collected; the
# session cache is also LRU-bounded, so a caller looping over models never accumulates HBM.
_SESSIONS: "OrderedDict" = OrderedDict()
_CANON: dict = {}
_TRACKED: set = set()
MAX_SESSIONS = 16


def clear_sessions() -> None:
    """Drop cached device sessions and canonical paths."""
    _SESSIONS.clear()
    _CANON.clear()


def _evict(key: int) -> None:
    _TRACKED.discard(key)
    for k in [k for k in _SESSIONS if key in (k[0], k[1])]:
        del _SESSIONS[k]
    for k in [k for k in _CANON if k[0] == key]:
        del _CANON[k]


def _track(obj) -> None:
    if obj is not None and id(obj) not in _TRACKED:
        _TRACKED.add(id(obj))
        weakref.finalize(obj, _evict, id(obj))


def _session(draft, verify, prompt_len, config, **kw) -> DeviceSession:
    canon = kw.get("canon")
    key = (id(draft), id(verify), prompt_len, config.max_new_tokens, config.draft_window_k, config.max_draft_lead,
           kw.get("max_window", L.KMAX), kw.get("jitter_ns", 0), kw.get("jitter_seed", 0),
           None if canon is None else canon.data_ptr(), getattr(draft, "agreement_rho", None))
    s = _SESSIONS.get(key)
    if s is None:
        _track(draft)
        _track(verify)
        s = DeviceSession(draft, verify, prompt_len, config, **kw)
        _SESSIONS[key] = s
        while len(_SESSIONS) > MAX_SESSIONS:
            _SESSIONS.popitem(last=False)
    else:
        _SESSIONS.move_to_end(key)
    return s


def canonical_path(verify, prompt: Sequence[int], n: int) -> torch.Tensor:
    """prompt + the verify model's greedy continuation (AR on the GPU), as a device int32 tensor.

    Used by AgreementDraft's coin.  Cached per (model, prompt, n).
    """
    vm = _model_of(verify)
    key = (id(vm), tuple(prompt), n)
    if key not in _CANON:
        _track(vm)
        cfg = DecodeConfig(max_new_tokens=n)
        out = _session(None, verify, len(prompt), cfg).run(L.ENGINE_AR, prompt)
        toks = list(prompt) + out.verified
        _CANON[key] = torch.tensor(toks, dtype=torch.int32, device=vm.device)
        settle(vm.device)
    return _CANON[key]


def _canon_for(draft, verify, prompt, config):
    if getattr(draft, "coin_mode", L.COIN_NONE) != L.COIN_CANON:
        return None
    return canonical_path(verify, prompt, config.max_new_tokens + L.KMAX)


def _result(out: RunOutput, prompt_len: int, eos: int, config: DecodeConfig) -> DecodeResult:
    tokens, finished_by = finalize_tokens(out.verified, eos, config.max_new_tokens)
    trace = trace_from_device(out.draft_rows, out.verify_rows, prompt_len, prompt_len + len(tokens))
    return DecodeResult(tokens, finished_by, summarize(trace), trace)


def _check_prompt(model, prompt):
    if len(prompt) == 0:
        raise InvalidInputError("prompt must be non-empty")
    _model_of(model)._validate_tokens(prompt)


def decode_autoregressive(verify_model, prompt: Sequence[int], config: DecodeConfig) -> DecodeResult:
    """Greedy one-token-at-a-time decoding on the verify model (engines.py:279-287)."""
    _check_prompt(verify_model, prompt)
    s = _session(None, verify_model, len(prompt), config)
    return _result(s.run(L.ENGINE_AR, prompt), len(prompt), verify_model.eos_token, config)


def decode_speculative_sync(draft_model, verify_model, prompt: Sequence[int], config: DecodeConfig) -> DecodeResult:
    """Synchronous speculative decoding (engines.py:290-301); output equals AR."""
    _check_prompt(verify_model, prompt)
    if config.draft_window_k > L.KMAX - 1:
        raise InvalidInputError(f"draft_window_k must be <= {L.KMAX - 1} on the device engine")
    canon = _canon_for(draft_model, verify_model, prompt, config)
    s = _session(draft_model, verify_model, len(prompt), config, canon=canon)
    return _result(s.run(L.ENGINE_SYNC, prompt), len(prompt), verify_model.eos_token, config)


class CudaAsyncExecutor:
    """Executor plug-in running AMUSD's two loops on the GPU (engines.py:409-531 contract).

    ``max_window`` caps the verify rows per step (<= 16); ``poll_jitter_ns`` /
    ``jitter_seed`` inject seeded device-side delays at the poll points
    (ThreadExecutor.poll_jitter_ms analog) -- neither may change tokens.
    """

    def __init__(self, max_window: int = L.KMAX, poll_jitter_ns: int = 0, jitter_seed: int = 0):
        if not 1 <= max_window <= L.KMAX:
            raise InvalidInputError(f"max_window must be in [1, {L.KMAX}]")
        self.max_window = max_window
        self.poll_jitter_ns = poll_jitter_ns
        self.jitter_seed = jitter_seed
        self.last_run: RunOutput | None = None

    def run(self, shared, draft_model, draft_state: ModelState, verify_model, verify_state: ModelState,
            config: DecodeConfig) -> DecodeTrace:
        prompt = getattr(verify_state, "prompt", None)
        if prompt is None:
            raise InvalidInputError("verify_state must come from a device model's init_state")
        canon = _canon_for(draft_model, verify_model, prompt, config)
        s = _session(draft_model, verify_model, len(prompt), config, canon=canon, max_window=self.max_window,
                     jitter_ns=self.poll_jitter_ns, jitter_seed=self.jitter_seed)
        out = s.run(L.ENGINE_ASYNC, prompt)
        self.last_run = out
        shared.publish_verified(out.verified)
        if hasattr(shared, "mirror_device"):
            shared.mirror_device([], out.info.p_d)
        tokens, _ = finalize_tokens(out.verified, verify_model.eos_token, config.max_new_tokens)
        return trace_from_device(out.draft_rows, out.verify_rows, len(prompt), len(prompt) + len(tokens))


def decode_speculative_async(draft_model, verify_model, prompt: Sequence[int], config: DecodeConfig,
                             executor=None) -> DecodeResult:
    """AMUSD: concurrent draft and verify loops with rollback recovery (engines.py:534-561)."""
    _check_prompt(verify_model, prompt)
    if executor is None:
        executor = CudaAsyncExecutor()
    shared = SharedDecodeState(prompt_length=len(prompt), max_new_tokens=config.max_new_tokens,
                               max_draft_lead=config.max_draft_lead)
    draft_state = draft_model.init_state(prompt)
    verify_state = verify_model.init_state(prompt)
    trace = executor.run(shared, draft_model, draft_state, verify_model, verify_state, config)
    tokens, finished_by = finalize_tokens(shared.verified_tokens(), verify_model.eos_token, config.max_new_tokens)
    return DecodeResult(tokens, finished_by, summarize(trace), trace)
