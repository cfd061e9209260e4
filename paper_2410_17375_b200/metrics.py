"""Trace and statistics schema of a decode run.

Same event vocabulary, field names and statistics as the reference
(pkg/src/specdec/metrics.py:42-231), so a trace produced by the GPU loops
passes the reference's own ``summarize`` unchanged (duck-typed: ``events``,
``validate()``, ``clock``, ``prompt_length``).

On the GPU the events are written by the protocol kernels into per-actor
device rings stamped with %globaltimer; ``trace_from_device`` turns them
into a merged, protocol-ordered ``DecodeTrace``.
"""
from __future__ import annotations

import csv
import io
from dataclasses import asdict, dataclass, field, replace

from .errors import InvalidInputError

ACTOR_DRAFT = "draft"
ACTOR_VERIFY = "verify"

DRAFT_TOKEN = "draft_token"
VERIFY_ACCEPT = "verify_accept"
VERIFY_CORRECT = "verify_correct"
ROLLBACK = "rollback"
COMPLETE = "complete"
VERIFY_KINDS = (VERIFY_ACCEPT, VERIFY_CORRECT)

CLOCK_WALL = "wall"
CLOCK_VIRTUAL = "virtual"
CLOCK_DEVICE = "wall"  # %globaltimer is a wall clock (ns); reported as "wall"

TRACE_CSV_COLUMNS = ["t_ms", "actor", "kind", "pos_lo", "pos_hi", "busy_ms", "draft_accepted"]
TIMELINE_CSV_COLUMNS = ["t_ms", "verified_tokens"]  # metrics.py:57

# device event kind codes (include/amusd.h amusd_trace_event)
_DEVICE_KINDS = {0: DRAFT_TOKEN, 1: VERIFY_ACCEPT, 2: VERIFY_CORRECT, 3: ROLLBACK}


@dataclass(frozen=True)
class TraceEvent:
    """One protocol event (metrics.py:60-72)."""
    t_ms: float
    actor: str
    kind: str
    pos_lo: int
    pos_hi: int
    busy_ms: float = 0.0
    draft_accepted: int = 0

    @property
    def token_count(self) -> int:
        return self.pos_hi - self.pos_lo + 1


@dataclass
class DecodeTrace:
    """Time-ordered events of one run (metrics.py:75-107)."""
    clock: str
    prompt_length: int
    events: list = field(default_factory=list)

    def validate(self) -> None:
        ev = self.events
        if not ev:
            raise InvalidInputError("trace has no events")
        if sum(e.kind == COMPLETE for e in ev) != 1 or ev[-1].kind != COMPLETE:
            raise InvalidInputError("trace must end with exactly one complete event")
        newest, owed = 0.0, False
        for e in ev:
            if e.t_ms < newest - 1e-9:
                raise InvalidInputError("trace timestamps must be non-decreasing")
            newest = max(newest, e.t_ms)
            if e.kind in VERIFY_KINDS and owed:
                raise InvalidInputError("verify event before the pending correction was rolled back")
            if e.kind == VERIFY_CORRECT:
                owed = True
            elif e.kind == ROLLBACK:
                if not owed:
                    raise InvalidInputError("rollback without a preceding correction")
                owed = False


def merge_actor_logs(draft: list, verify: list) -> list:
    """Merge per-actor (t_ms, seq, TraceEvent) logs in protocol order.

    Same rule as TraceRecorder.build (metrics.py:146-186): a rollback is placed
    only once a correction is outstanding, otherwise (t, seq) decides; then
    timestamps are clamped non-decreasing.
    """
    out, owed, last = [], False, 0.0
    i = j = 0
    while i < len(draft) or j < len(verify):
        if i >= len(draft):
            pick_draft = False
        elif j >= len(verify):
            pick_draft = True
        elif draft[i][2].kind == ROLLBACK:
            pick_draft = owed
        else:
            pick_draft = draft[i][:2] < verify[j][:2]
        ev = draft[i][2] if pick_draft else verify[j][2]
        if pick_draft:
            i += 1
        else:
            j += 1
        if ev.kind == VERIFY_CORRECT:
            owed = True
        elif ev.kind == ROLLBACK:
            owed = False
        if ev.t_ms < last:
            ev = replace(ev, t_ms=last)
        last = ev.t_ms
        out.append(ev)
    return out


def trace_from_device(draft_rows, verify_rows, prompt_length: int, final_pos: int) -> DecodeTrace:
    """Build a DecodeTrace from device ring records (t_ns, busy_ns, kind, lo, hi, acc).

    Draft work that lands after the verify side signalled completion is
    dropped (it can never be observed by the protocol; the reference
    ThreadExecutor races on it -- SURVEY.md section 0.6).
    """
    all_rows = list(draft_rows) + list(verify_rows)
    if not verify_rows:
        raise InvalidInputError("device trace has no verify events")
    t0 = min(r[0] - r[1] for r in all_rows)
    t_done = max(r[0] for r in verify_rows)
    seq = 0
    logs = {ACTOR_DRAFT: [], ACTOR_VERIFY: []}
    for actor, rows in ((ACTOR_VERIFY, verify_rows), (ACTOR_DRAFT, draft_rows)):
        for t_ns, busy_ns, kind, lo, hi, acc in rows:
            if actor == ACTOR_DRAFT and t_ns > t_done:
                continue
            ev = TraceEvent((t_ns - t0) / 1e6, actor, _DEVICE_KINDS[kind], int(lo), int(hi), busy_ns / 1e6, int(acc))
            logs[actor].append((ev.t_ms, seq, ev))
            seq += 1
    # Each ring is already in true program order (single writer, sequential
    # kernels); %globaltimer can differ by a few hundred ns between SMs, so
    # rings are never re-sorted -- only merged, then clamped.
    events = merge_actor_logs(logs[ACTOR_DRAFT], logs[ACTOR_VERIFY])
    t_end = max((t_done - t0) / 1e6, events[-1].t_ms if events else 0.0)
    events.append(TraceEvent(t_end, ACTOR_VERIFY, COMPLETE, final_pos, final_pos))
    return DecodeTrace(clock=CLOCK_DEVICE, prompt_length=prompt_length, events=events)


@dataclass(frozen=True)
class DecodeStats:
    """Run statistics (metrics.py:189-204)."""
    clock: str
    generated_tokens: int
    total_ms: float
    mean_ms_per_token: float
    verify_steps: int
    accepted_per_verify_step: float
    rollbacks: int
    drafted_tokens: int
    wasted_draft_tokens: int

    def to_dict(self) -> dict:
        return asdict(self)


def summarize(trace: DecodeTrace) -> DecodeStats:
    """Statistics of a complete trace (metrics.py:207-231)."""
    trace.validate()
    last = trace.events[-1]
    generated = last.pos_hi - trace.prompt_length
    if generated < 1:
        raise InvalidInputError("complete trace reports no generated tokens")
    steps = [e for e in trace.events if e.kind in VERIFY_KINDS]
    published = sum(e.token_count for e in steps)
    return DecodeStats(
        clock=trace.clock,
        generated_tokens=generated,
        total_ms=last.t_ms,
        mean_ms_per_token=last.t_ms / generated,
        verify_steps=len(steps),
        accepted_per_verify_step=published / len(steps) if steps else 0.0,
        rollbacks=sum(e.kind == VERIFY_CORRECT for e in steps),
        drafted_tokens=sum(e.kind == DRAFT_TOKEN for e in trace.events),
        wasted_draft_tokens=sum(e.token_count for e in trace.events if e.kind == ROLLBACK),
    )


def trace_to_csv(trace: DecodeTrace) -> str:
    """Event CSV with the reference's stable columns (metrics.py:338-346)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(TRACE_CSV_COLUMNS)
    for e in trace.events:
        w.writerow([repr(e.t_ms), e.actor, e.kind, e.pos_lo, e.pos_hi, repr(e.busy_ms), e.draft_accepted])
    return buf.getvalue()


def busy_intervals(trace: DecodeTrace, actor: str) -> list:
    """Merged busy intervals of one actor (metrics.py:301-314)."""
    spans = sorted((e.t_ms - e.busy_ms, e.t_ms) for e in trace.events if e.actor == actor and e.busy_ms > 0.0)
    merged = []
    for lo, hi in spans:
        if merged and lo <= merged[-1][1] + 1e-9:
            merged[-1] = (merged[-1][0], max(merged[-1][1], hi))
        else:
            merged.append((lo, hi))
    return merged


def overlap_ms(a: list, b: list) -> float:
    """Length of the intersection of two merged interval lists (metrics.py:317-330)."""
    total, i, j = 0.0, 0, 0
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if hi > lo:
            total += hi - lo
        if a[i][1] <= b[j][1]:
            i += 1
        else:
            j += 1
    return total


def read_trace_csv(path, clock: str, prompt_length: int) -> DecodeTrace:
    """Rebuild a trace from an event CSV written by ``trace_to_csv`` (metrics.py:358-374)."""
    events = []
    with open(path, newline="", encoding="utf-8") as fh:
        rows = csv.reader(fh)
        if next(rows, None) != TRACE_CSV_COLUMNS:
            raise InvalidInputError(f"unexpected trace CSV header in {path}")
        for t_ms, actor, kind, lo, hi, busy, acc in rows:
            events.append(TraceEvent(float(t_ms), actor, kind, int(lo), int(hi), float(busy), int(acc)))
    return DecodeTrace(clock=clock, prompt_length=prompt_length, events=events)


def export_timeline(trace: DecodeTrace) -> list:
    """Cumulative verified tokens over time, capped at the generated count (metrics.py:282-298)."""
    trace.validate()
    cap = trace.events[-1].pos_hi - trace.prompt_length
    series, done = [(0.0, 0)], 0
    for e in trace.events:
        if e.kind in VERIFY_KINDS:
            done = min(done + e.token_count, cap)
            series.append((e.t_ms, done))
    return series


def timeline_to_csv(series) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(TIMELINE_CSV_COLUMNS)
    for t_ms, n in series:
        w.writerow([repr(t_ms), n])
    return buf.getvalue()


def compare_table(entries) -> dict:
    """Speedup of each (label, mean_ms_per_token) over the first (metrics.py:264-276)."""
    if len(entries) < 2:
        raise InvalidInputError("a comparison needs at least two entries")
    base = entries[0][1]
    return {"baseline": entries[0][0],
            "rows": [{"label": k, "mean_ms_per_token": v, "speedup": base / v} for k, v in entries]}


def compare_text(table: dict) -> str:
    width = max(len("strategy"), *(len(r["label"]) for r in table["rows"]))
    out = [f"{'strategy':<{width}}  {'mean ms/token':>14}  {'speedup':>8}"]
    out += [f"{r['label']:<{width}}  {r['mean_ms_per_token']:>14.3f}  {r['speedup']:>7.2f}x" for r in table["rows"]]
    return "\n".join(out)
