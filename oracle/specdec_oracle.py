"""CPU restatement of the reference AMUSD protocol -- TEST INFRASTRUCTURE ONLY.

Pinned bit-exactly against tests/golden/*.json (generated from the unmodified
reference by oracle/make_golden.py); see tests/test_oracle_golden.py.

Every function cites the reference ``pkg/src/specdec`` file:line it restates.
The structure is deliberately different from the reference (plain functions
over small state records, one event loop per engine) -- it is a second,
independent statement of the same algorithm, used to check the CUDA path.
"""
from __future__ import annotations

import heapq
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
AGREE_SALT = 0xD1B54A32D192ED03      # models.py:46
DISAGREE_SALT = 0x8CB92BA72F3D8DD7   # models.py:47

EOS = "eos"                # engines.py:48
LENGTH = "length_limit"    # engines.py:49


# --------------------------------------------------------------------------
# splitmix64 hash chain (models.py:15-30, 50-55, 203-314)
# --------------------------------------------------------------------------

def mix64(x: int) -> int:
    """splitmix64 finalizer with the golden-gamma increment (models.py:50-55)."""
    z = (x + GOLDEN_GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rho_threshold(rho: float) -> int:
    """int(rho * 2**64) exactly as models.py:298 computes it (float product)."""
    return int(rho * 2.0 ** 64)


def draw_excluding(h: int, vocab: int, eos: int, exclude_eos: bool) -> int:
    """Base chain draw, eos-skipping if configured (models.py:256-261)."""
    if not exclude_eos:
        return h % vocab
    r = h % (vocab - 1)
    return r + (r >= eos)


def different_token(h: int, agreed: int, vocab: int, eos: int, exclude_eos: bool) -> int:
    """Uniform draw over the vocabulary minus {agreed (, eos)} (models.py:306-314)."""
    skip = sorted({agreed, eos} if exclude_eos else {agreed})
    d = mix64(h ^ DISAGREE_SALT) % (vocab - len(skip))
    for s in skip:
        d += d >= s
    return d


def coin_token(h: int, agreed: int, thr: int, vocab: int, eos: int, exclude_eos: bool) -> int:
    """Agreement coin keyed on the prefix hash (models.py:300-304)."""
    if mix64(h ^ AGREE_SALT) < thr:
        return agreed
    return different_token(h, agreed, vocab, eos, exclude_eos)


@dataclass
class SeqState:
    """Incremental per-sequence state: tokens + per-position cache (models.py:58-82)."""
    prompt_len: int
    tokens: list
    cache: list = field(default_factory=list)


class ChainOracle:
    """HashChainModel (rho=None) or AgreementDraftModel (rho given).

    cache[i] = h_i, len(cache) == len(tokens) + 1 (models.py:203-231).
    """

    def __init__(self, seed: int, vocab: int, eos: int, exclude_eos: bool = False, rho: float | None = None):
        self.seed, self.vocab, self.eos, self.exclude_eos = seed & M64, vocab, eos, exclude_eos
        self.rho = rho
        self.thr = None if rho is None else rho_threshold(rho)
        self.eos_token = eos

    def token_from_hash(self, h: int) -> int:
        base = draw_excluding(h, self.vocab, self.eos, self.exclude_eos)
        if self.thr is None:
            return base
        return coin_token(h, base, self.thr, self.vocab, self.eos, self.exclude_eos)

    def start(self, prompt: Sequence[int]) -> SeqState:
        st = SeqState(len(prompt), [], [mix64(self.seed)])
        self.extend(st, prompt)
        return st

    def predict(self, st: SeqState) -> int:
        return self.token_from_hash(st.cache[-1])

    def extend(self, st: SeqState, toks: Sequence[int]) -> None:
        h = st.cache[-1]
        for t in toks:
            h = mix64(h ^ t)
            st.cache.append(h)
        st.tokens.extend(toks)

    def crop(self, st: SeqState, n: int) -> None:
        if not st.prompt_len <= n <= len(st.tokens):
            raise ValueError(f"rollback position {n} outside [{st.prompt_len}, {len(st.tokens)}]")
        del st.tokens[n:]
        del st.cache[n + 1:]

    def verify(self, st: SeqState, cands: Sequence[int]) -> list:
        """Teacher-forced predictions, non-mutating (models.py:237-250)."""
        h, out = st.cache[-1], []
        for t in cands:
            out.append(self.token_from_hash(h))
            h = mix64(h ^ t)
        return out


class ScriptOracle:
    """Position-indexed table model with forced eos (models.py:317-346)."""

    def __init__(self, script: Sequence[int], vocab: int, eos: int, eos_position: int | None = None):
        self.script, self.vocab, self.eos_token, self.eos_position = list(script), vocab, eos, eos_position

    def _at(self, pos1: int) -> int:
        if self.eos_position is not None and pos1 == self.eos_position:
            return self.eos_token
        return self.script[(pos1 - 1) % len(self.script)]

    def start(self, prompt):
        return SeqState(len(prompt), list(prompt))

    def predict(self, st):
        return self._at(len(st.tokens) + 1)

    def extend(self, st, toks):
        st.tokens.extend(toks)

    def crop(self, st, n):
        del st.tokens[n:]

    def verify(self, st, cands):
        base = len(st.tokens)
        return [self._at(base + 1 + j) for j in range(len(cands))]


# --------------------------------------------------------------------------
# Small engine helpers (engines.py:91-113)
# --------------------------------------------------------------------------

def first_mismatch(cands: Sequence[int], preds: Sequence[int]):
    """1-based index of the first disagreement, else None (engines.py:91-100)."""
    if len(cands) != len(preds):
        raise ValueError("length mismatch")
    return next((i + 1 for i, (c, p) in enumerate(zip(cands, preds)) if c != p), None)


def finalize(verified: Sequence[int], eos: int, n: int):
    """Cap at n then cut after the first eos (engines.py:103-113)."""
    head = list(verified[:n])
    if eos in head:
        return head[: head.index(eos) + 1], EOS
    return head, LENGTH


def accept_window(window: Sequence[int], preds: Sequence[int]):
    """(accepted, matched, corrected) for one async verify step (engines.py:376-383)."""
    i = first_mismatch(window, preds)
    if i is None:
        return list(window), len(window), False
    return list(window[: i - 1]) + [preds[i - 1]], i - 1, True


# --------------------------------------------------------------------------
# Latency model (simulator.py:70-103) and the trace schema (metrics.py:60-231)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Latency:
    draft_base_ms: float = 0.0
    draft_per_token_ms: float = 10.0
    verify_base_ms: float = 25.0
    verify_per_token_ms: float = 0.0
    rollback_overhead_ms: float = 0.0

    def draft(self, b: int) -> float:
        return self.draft_base_ms + self.draft_per_token_ms * b

    def verify(self, b: int) -> float:
        return self.verify_base_ms + self.verify_per_token_ms * b


# trace row = [t_ms, actor, kind, pos_lo, pos_hi, busy_ms, draft_accepted]
DRAFT, VERIFY = "draft", "verify"
K_DRAFT, K_ACCEPT, K_CORRECT, K_ROLLBACK, K_COMPLETE = (
    "draft_token", "verify_accept", "verify_correct", "rollback", "complete")


def merge_logs(draft_log: list, verify_log: list) -> list:
    """Protocol-ordered merge of per-actor logs (metrics.py:146-186).

    Each log entry is (t_ms, seq, row). A rollback is held back until a
    correction is outstanding; otherwise (t, seq) order decides. Timestamps
    are clamped non-decreasing afterwards.
    """
    out, owed, last = [], False, 0.0
    i = j = 0
    while i < len(draft_log) or j < len(verify_log):
        if i == len(draft_log):
            use_d = False
        elif j == len(verify_log):
            use_d = True
        elif draft_log[i][2][2] == K_ROLLBACK:
            use_d = owed
        else:
            use_d = draft_log[i][:2] < verify_log[j][:2]
        row = list(draft_log[i][2] if use_d else verify_log[j][2])
        i, j = (i + 1, j) if use_d else (i, j + 1)
        owed = True if row[2] == K_CORRECT else (False if row[2] == K_ROLLBACK else owed)
        if row[0] < last:
            row[0] = last
        last = row[0]
        out.append(row)
    return out


def validate_trace(rows: list) -> None:
    """metrics.py:83-107."""
    if not rows:
        raise ValueError("trace has no events")
    if sum(r[2] == K_COMPLETE for r in rows) != 1 or rows[-1][2] != K_COMPLETE:
        raise ValueError("trace must end with exactly one complete event")
    last, owed = 0.0, False
    for r in rows:
        if r[0] < last - 1e-9:
            raise ValueError("trace timestamps must be non-decreasing")
        last = max(last, r[0])
        if r[2] in (K_ACCEPT, K_CORRECT) and owed:
            raise ValueError("verify event before the pending correction was rolled back")
        if r[2] == K_CORRECT:
            owed = True
        elif r[2] == K_ROLLBACK:
            if not owed:
                raise ValueError("rollback without a preceding correction")
            owed = False


def trace_stats(rows: list, prompt_len: int) -> dict:
    """metrics.py:207-231."""
    validate_trace(rows)
    done = rows[-1]
    gen = done[4] - prompt_len
    if gen < 1:
        raise ValueError("complete trace reports no generated tokens")
    ver = [r for r in rows if r[2] in (K_ACCEPT, K_CORRECT)]
    published = sum(r[4] - r[3] + 1 for r in ver)
    return {
        "generated_tokens": gen,
        "total_ms": done[0],
        "mean_ms_per_token": done[0] / gen,
        "verify_steps": len(ver),
        "accepted_per_verify_step": published / len(ver) if ver else 0.0,
        "rollbacks": sum(r[2] == K_CORRECT for r in ver),
        "drafted_tokens": sum(r[2] == K_DRAFT for r in rows),
        "wasted_draft_tokens": sum(r[4] - r[3] + 1 for r in rows if r[2] == K_ROLLBACK),
    }


# --------------------------------------------------------------------------
# Serial engines as unit generators (engines.py:139-259)
# unit = (actor, kind, pos_lo, pos_hi, batch, draft_accepted, completed)
# --------------------------------------------------------------------------

def ar_units(verify, prompt, n):
    """Autoregressive oracle (engines.py:139-157). Yields units; returns verified list."""
    st = verify.start(prompt)
    out = []
    while True:
        t = verify.predict(st)
        verify.extend(st, [t])
        out.append(t)
        pos = len(prompt) + len(out)
        done = t == verify.eos_token or len(out) >= n
        yield (VERIFY, K_ACCEPT, pos, pos, 1, 0, done), out
        if done:
            return


def sync_units(draft, verify, prompt, n, k):
    """Synchronous speculative rounds with bonus/correction (engines.py:160-259)."""
    ds, vs = draft.start(prompt), verify.start(prompt)
    P = len(prompt)
    out = []
    while True:
        want = min(k, n - len(out))
        cands = []
        for _ in range(want):
            t = draft.predict(ds)
            draft.extend(ds, [t])
            cands.append(t)
            pos = P + len(out) + len(cands)
            yield (DRAFT, K_DRAFT, pos, pos, 1, 0, False), out
        frontier = P + len(out)
        preds = verify.verify(vs, cands)
        miss = first_mismatch(cands, preds)
        if miss is None:
            verify.extend(vs, cands)
            bonus = verify.predict(vs)
            verify.extend(vs, [bonus])
            acc = cands + [bonus]
            draft.extend(ds, [bonus])
            kind, matched = K_ACCEPT, len(cands)
        else:
            acc = cands[: miss - 1] + [preds[miss - 1]]
            verify.extend(vs, acc)
            draft.crop(ds, frontier)
            draft.extend(ds, acc)
            kind, matched = K_CORRECT, miss - 1
        out.extend(acc)
        done = verify.eos_token in acc or len(out) >= n
        yield (VERIFY, kind, frontier + 1, frontier + len(acc), len(cands), matched, done), out
        if done:
            return
        if miss is not None:
            yield (DRAFT, K_ROLLBACK, frontier + miss, frontier + len(cands), 0, 0, False), out


def run_serial(units_iter, prompt_len, eos, n):
    """Drain a unit generator; returns (tokens, finished_by, verified, units)."""
    units, verified = [], []
    for unit, verified in units_iter:
        units.append(unit)
    toks, by = finalize(verified, eos, n)
    return toks, by, list(verified), units


def sim_serial(units, prompt_len, tokens, latency: Latency) -> list:
    """Virtual-clock timing of a serial engine (simulator.py:156-196)."""
    dlog, vlog, seq, now = [], [], 0, 0.0
    for actor, kind, lo, hi, batch, acc, _done in units:
        cost = (latency.draft(batch) if kind == K_DRAFT else
                latency.rollback_overhead_ms if kind == K_ROLLBACK else latency.verify(batch))
        now = now + cost
        (dlog if actor == DRAFT else vlog).append((now, seq, [now, actor, kind, lo, hi, cost, acc]))
        seq += 1
    fin = prompt_len + len(tokens)
    vlog.append((now, seq, [now, VERIFY, K_COMPLETE, fin, fin, 0.0, 0]))
    return merge_logs(dlog, vlog)


def decode_ar(verify, prompt, n):
    toks, by, _, units = run_serial(ar_units(verify, prompt, n), len(prompt), verify.eos_token, n)
    return toks, by, units


def decode_sync(draft, verify, prompt, n, k):
    toks, by, _, units = run_serial(sync_units(draft, verify, prompt, n, k), len(prompt), verify.eos_token, n)
    return toks, by, units


# --------------------------------------------------------------------------
# Asynchronous AMUSD protocol (coordination.py:114-275, engines.py:332-401)
# --------------------------------------------------------------------------

class Mailbox:
    """Single-writer coordination record (coordination.py:114-275).

    D/p_d written by the draft side only; V/p_v/rollback/complete by verify.
    """

    def __init__(self, prompt_len: int, n: int, lead: int | None):
        self.P, self.n, self.lead = prompt_len, n, lead
        self.D, self.V = [], []
        self.p_d = self.p_v = prompt_len
        self.rb = None           # (target, correction)
        self.complete = False
        self.acks = 0

    def capped(self) -> bool:
        return self.lead is not None and self.p_d - self.p_v >= self.lead

    def window(self) -> list:
        assert self.rb is None, "window read during pending rollback"
        hi = self.p_d
        return self.D[self.p_v - self.P: hi - self.P]

    def publish_draft(self, t: int) -> None:
        self.D.append(t)
        self.p_d += 1

    def ack(self, draft, ds) -> None:
        """acknowledge_rollback (coordination.py:188-211)."""
        target, c = self.rb
        assert self.P < target <= self.p_d
        draft.crop(ds, target - 1)
        draft.extend(ds, [c])
        del self.D[target - 1 - self.P:]
        self.D.append(c)
        self.p_d = target
        self.rb = None
        self.acks += 1
        assert self.p_d == self.p_v and self.D[: self.p_d - self.P] == self.V

    def publish_verified(self, toks: list) -> None:
        assert self.rb is None and toks
        self.V.extend(toks)
        self.p_v += len(toks)


def draft_step(mb: Mailbox, draft, ds) -> str:
    """complete > rollback-ack > lead cap > generate (engines.py:332-352)."""
    if mb.complete:
        return "stopped"
    if mb.rb is not None:
        mb.ack(draft, ds)
        return "rolled_back"
    if mb.capped():
        return "idle"
    t = draft.predict(ds)
    draft.extend(ds, [t])
    mb.publish_draft(t)
    return "generated"


def verify_step(mb: Mailbox, verify, vs, window=None):
    """One verify iteration (engines.py:355-401). Returns (kind, matched, corrected) or None when idle."""
    if window is None:
        window = mb.window()
    if not window:
        return None
    preds = verify.verify(vs, window)
    acc, matched, corrected = accept_window(window, preds)
    verify.extend(vs, acc)
    mb.publish_verified(acc)
    if corrected:
        assert mb.rb is None
        mb.rb = (mb.p_v, acc[-1])
    done = verify.eos_token in acc or mb.p_v - mb.P >= mb.n
    if done:
        assert not mb.complete
        mb.complete = True
    return ("done" if done else ("corrected" if corrected else "accepted")), matched, corrected


def sim_async(draft, verify, prompt, n, lead, latency: Latency):
    """Virtual-clock AMUSD (simulator.py:214-396): deterministic tokens + trace.

    Returns (tokens, finished_by, trace_rows, mailbox).
    """
    P = len(prompt)
    mb = Mailbox(P, n, lead)
    ds, vs = draft.start(prompt), verify.start(prompt)
    heap, seq = [], [0]
    dlog, vlog, lseq = [], [], [0]
    st = {"draft": "running", "verify": "idle", "d_since": 0.0, "v_since": 0.0}

    def push(t, actor, what, payload=None):
        heapq.heappush(heap, (t, 0 if actor == VERIFY else 1, seq[0], what, payload))
        seq[0] += 1

    def log(actor, row):
        (dlog if actor == DRAFT else vlog).append((row[0], lseq[0], row))
        lseq[0] += 1

    def draft_go(now):
        st["draft"], st["d_since"] = "running", now
        push(now + latency.draft(1), DRAFT, "fwd")

    def verify_go(now):
        w = mb.window()
        if not w:
            st["verify"] = "idle"
            return
        st["verify"], st["v_since"] = "busy", now
        push(now + latency.verify(len(w)), VERIFY, "fwd", w)

    draft_go(0.0)
    while True:
        now, _, _, what, payload = heapq.heappop(heap)
        if what == "end":
            break
        if what == "fwd" and payload is None:          # draft forward finished
            if mb.complete:
                st["draft"] = "stopped"
                continue
            if mb.rb is not None:                      # in-flight token discarded
                st["draft"] = "recovering"
                push(now + latency.rollback_overhead_ms, DRAFT, "ack")
                continue
            assert draft_step(mb, draft, ds) == "generated"
            log(DRAFT, [now, DRAFT, K_DRAFT, mb.p_d, mb.p_d, now - st["d_since"], 0])
            if st["verify"] == "idle":
                verify_go(now)
            if mb.capped():
                st["draft"] = "capped"
            else:
                draft_go(now)
        elif what == "ack":
            before = mb.p_d
            if draft_step(mb, draft, ds) == "stopped":
                st["draft"] = "stopped"
                continue
            log(DRAFT, [now, DRAFT, K_ROLLBACK, mb.p_d, before, now - st["d_since"], 0])
            st["verify"] = "idle"
            draft_go(now)
        else:                                          # verify forward finished
            v_before = mb.p_v
            kind, matched, corrected = verify_step(mb, verify, vs, window=payload)
            log(VERIFY, [now, VERIFY, K_CORRECT if corrected else K_ACCEPT, v_before + 1, mb.p_v,
                         now - st["v_since"], matched])
            if kind == "done":
                toks, _ = finalize(mb.V, verify.eos_token, n)
                log(VERIFY, [now, VERIFY, K_COMPLETE, P + len(toks), P + len(toks), 0.0, 0])
                st["verify"] = "done"
                push(now, VERIFY, "end")
                continue
            if corrected:
                st["verify"] = "awaiting_ack"
                if st["draft"] == "capped":
                    st["d_since"], st["draft"] = now, "recovering"
                    push(now + latency.rollback_overhead_ms, DRAFT, "ack")
                continue
            if st["draft"] == "capped" and not mb.capped():
                draft_go(now)
            verify_go(now)
    toks, by = finalize(mb.V, verify.eos_token, n)
    return toks, by, merge_logs(dlog, vlog), mb


def thread_async(draft, verify, prompt, n, lead=None, on_event: Callable | None = None):
    """Two-thread AMUSD executor (engines.py:409-531) for CPU timing.

    Returns (tokens, finished_by, counters, wall_s). Post-completion draft
    work is discarded (the reference can log it after ``complete``;
    SURVEY.md section 0.6).
    """
    P = len(prompt)
    mb = Mailbox(P, n, lead)
    ds, vs = draft.start(prompt), verify.start(prompt)
    cnt = {"drafted": 0, "verify_steps": 0, "rollbacks": 0, "acks": 0}
    errs = []

    def dloop():
        try:
            while not errs:
                time.sleep(0)
                r = draft_step(mb, draft, ds)
                if r == "stopped":
                    return
                if r == "generated":
                    cnt["drafted"] += 1
                elif r == "rolled_back":
                    cnt["acks"] += 1
        except BaseException as e:  # pragma: no cover - propagated below
            errs.append(e)

    def vloop():
        try:
            while not errs:
                time.sleep(0)
                if mb.rb is not None:
                    continue
                r = verify_step(mb, verify, vs)
                if r is None:
                    continue
                cnt["verify_steps"] += 1
                cnt["rollbacks"] += r[2]
                if r[0] == "done":
                    return
        except BaseException as e:  # pragma: no cover
            errs.append(e)

    t0 = time.perf_counter()
    th = [threading.Thread(target=dloop), threading.Thread(target=vloop)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    if errs:
        raise errs[0]
    toks, by = finalize(mb.V, verify.eos_token, n)
    return toks, by, cnt, wall


def canonical_disagreements(draft, verify, prompt, count):
    """Rollback-count theorem oracle (pkg/tests/test_engines.py:293-321):
    positions (1-based, generated index) where draft != verify along the
    canonical greedy path, plus the canonical path itself."""
    ds, vs = draft.start(prompt), verify.start(prompt)
    path, dis = [], []
    for i in range(count):
        v = verify.predict(vs)
        d = draft.predict(ds)
        if d != v:
            dis.append(i + 1)
        path.append(v)
        verify.extend(vs, [v])
        draft.extend(ds, [v])
    return path, dis
