"""Simulator calibration.

Measured forward latencies of the CUDA models are fed into the reference's OWN
virtual-clock simulator -- ``specdec.simulator.LatencyModel`` /
``specdec.simulate`` (pkg/src/specdec/simulator.py:70-103, 399-435), imported
unmodified from the offline install in ``baseline/_ref`` -- which replays the
reference's step functions (engines.py:332-401) under those latencies.  The
result is the protocol-level prediction of AR / sync-SD / AMUSD tokens/s for a
pair whose actors do not share a GPU (the paper's split pair, BASELINE
config 2), the best sync-SD k and the effect of ``max_draft_lead``.  ``bench.py``
prints it next to the measured engines.

The acceptance process is the reference's own ``make_agreement_pair``
(models.py:349-365): the draft agrees with the verify model's greedy token with
probability rho per position -- the same coin the CUDA ``AgreementDraft``
applies to the transformer pair.
"""
from __future__ import annotations

import importlib
import statistics
import sys
from dataclasses import asdict, dataclass
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def load_specdec():
    """The unmodified reference package (``baseline/_ref``); ImportError when absent."""
    if "specdec" in sys.modules:
        return sys.modules["specdec"]
    ref = ROOT / "baseline" / "_ref"
    if (ref / "specdec" / "__init__.py").exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    return importlib.import_module("specdec")


@dataclass(frozen=True)
class Latencies:
    """Fitted forward costs (ms), the LatencyModel fields (simulator.py:70-103)."""
    draft_base_ms: float
    draft_per_token_ms: float
    verify_base_ms: float
    verify_per_token_ms: float
    ctx: int

    def latency_model(self, S):
        return S.LatencyModel(draft_base_ms=self.draft_base_ms, draft_per_token_ms=self.draft_per_token_ms,
                              verify_base_ms=self.verify_base_ms, verify_per_token_ms=self.verify_per_token_ms)


def fit_linear(points: dict) -> tuple:
    """Least-squares (base, per_row) of {rows: ms}; per_row clamped at >= 0."""
    xs, ys = list(points), [points[k] for k in points]
    if len(xs) == 1:
        return 0.0, ys[0] / xs[0]
    mx, my = statistics.fmean(xs), statistics.fmean(ys)
    sxx = sum((x - mx) ** 2 for x in xs)
    slope = max(0.0, sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx)
    return max(0.0, my - slope * mx), slope


def forward_ms(model, rows: int, iters: int = 10) -> float:
    """One persistent forward of `rows` token rows at the model's current context (CUDA events)."""
    import ctypes as C

    import torch

    from . import _lib as L
    lib = L.load()
    ms = C.c_float()
    L.check(lib.amusd_time_forward(model.handle, rows, -1, 0, iters, C.byref(ms),
                                   torch.cuda.current_stream().cuda_stream))
    return ms.value


def measure(draft, verify, ctx: int, verify_rows=(1, 2, 4, 8, 16)) -> Latencies:
    """Latencies of `draft` (1-row decode step) and `verify` (window of m rows) at context `ctx`.

    The draft's cost is charged per token (draft_per_token_ms, base 0) as the reference models
    it; the verify cost is fitted as base + per_row over `verify_rows`.  Both models are left
    holding a synthetic prefix of length ctx (call init_state again before decoding)."""
    prompt = [(7919 * i + 3) % 30000 + 3 for i in range(ctx)]
    verify.init_state(prompt)
    vb, vp = fit_linear({m: forward_ms(verify, m) for m in verify_rows})
    draft.init_state(prompt)
    d1 = forward_ms(draft, 1, iters=20)
    return Latencies(0.0, d1, vb, vp, ctx)


def predict(lat: Latencies, rho: float, n_tokens: int = 512, ks=(2, 3, 4, 5, 6, 8), lead=None,
            seeds=range(5), vocab: int = 32000, prompt=(1, 2, 3, 4)) -> dict:
    """tokens/s predicted by the reference simulator (mean over seeds), per engine."""
    S = load_specdec()
    lm = lat.latency_model(S)

    def run(kind, k, seed):
        d, v = S.make_agreement_pair(seed, rho, vocab, eos_token=2, exclude_eos=True)
        cfg = S.DecodeConfig(max_new_tokens=n_tokens, draft_window_k=k, max_draft_lead=lead)
        res, trace = S.simulate(kind, d if kind != "autoregressive" else None, v, list(prompt), cfg, lm)
        return len(res.tokens) / (res.stats.total_ms / 1000.0)

    out = {"ar": statistics.fmean(run("autoregressive", 4, s) for s in seeds)}
    sync = {k: statistics.fmean(run("sync_speculative", k, s) for s in seeds) for k in ks}
    out["sync_k4"] = sync.get(4)
    best = max(sync, key=sync.get)
    out["sync_best"] = {"k": best, "tokens_per_s": round(sync[best], 3)}
    out["amusd"] = statistics.fmean(run("async_speculative", 4, s) for s in seeds)
    out["amusd_vs_sync_k4"] = out["amusd"] / out["sync_k4"] if out["sync_k4"] else None
    out["amusd_vs_ar"] = out["amusd"] / out["ar"]
    return {k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}


def calibrate(draft, verify, ctx: int, rhos=(0.8, 0.9), n_tokens: int = 512, lead=None) -> dict:
    """measure() + predict() for each rho: the calibration record bench.py prints."""
    lat = measure(draft, verify, ctx)
    return {"latency_ms": {k: round(v, 5) if isinstance(v, float) else v for k, v in asdict(lat).items()},
            "simulator": "specdec.simulate (unmodified reference, simulator.py:399-435)",
            "assumes": "draft and verify on separate GPUs (no HBM/SM sharing): the split pair",
            "predicted_tokens_per_s": {f"rho{r}": predict(lat, r, n_tokens=n_tokens, lead=lead) for r in rhos}}
