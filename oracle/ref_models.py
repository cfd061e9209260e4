"""The UNMODIFIED reference engines driving the numpy decoder -- TEST/BASELINE
INFRASTRUCTURE ONLY.

The reference (``specdec``, pkg/src/specdec) is pure Python with duck-typed
model and executor plug-ins.  This module plugs the
fp32 numpy Llama restatement (``ref_decoder.RefDecoder``) into the
reference's OWN ``MockModel`` hooks (models.py:171-185) so that the
reference's own ``decode_autoregressive`` / ``decode_speculative_sync`` /
``decode_speculative_async(ThreadExecutor)`` (engines.py:279-301, 409-561)
run unchanged over transformer arithmetic.  Used by

* ``bench.py --impl reference`` and the GPU arm's ``cpu_baseline`` (the
  reference's CPU path timed on the host cores), and
* tests that check the CUDA engines against the reference engines.

``specdec`` is imported from ``baseline/_ref`` (the offline pip install that
travels to the GPU box) or, in the build container, from
``/root/reference/pkg/src``.  Nothing in ``paper_2410_17375_b200`` imports
this module.
"""
from __future__ import annotations

import importlib
import os
import sys
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .ref_decoder import DecState, RefDecoder, TfShape, bf16_round
from .specdec_oracle import coin_token, mix64, rho_threshold

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def load_reference():
    """The unmodified reference package ``specdec`` (None when not installed)."""
    if "specdec" in sys.modules:
        return sys.modules["specdec"]
    for p in _CANDIDATES:
        if (p / "specdec" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return importlib.import_module("specdec")
    return None


def reference_origin() -> str:
    S = load_reference()
    return str(Path(S.__file__).resolve().parent) if S else "unavailable"


# ------------------------------------------------------------------ weights
def _uniform_chunk(sub: int, lo: int, hi: int, scale: np.float32) -> np.ndarray:
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    x = (np.arange(lo, hi, dtype=np.uint64) + np.uint64(sub)) & M
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return scale * (np.float32(2.0) * u - np.float32(1.0))


def synthetic_weights(names_shapes: list, seed: int, bf16: bool, std: float = 0.02, threads: int | None = None,
                      chunk: int = 1 << 24) -> dict:
    """Host twin of TransformerModel._synthetic / amusd_fill_uniform (api.cu k_fill_uniform):
    the same splitmix64 counter stream per weight, norms = 1, optionally rounded to bf16 --
    so a CPU model holds bit-identical weights without touching a GPU.  ``names_shapes`` is
    weight_names() order with shapes (the per-weight seed depends on the index)."""
    threads = threads or os.cpu_count() or 1
    scale = np.float32(std * np.sqrt(3.0))
    out = {}
    with ThreadPoolExecutor(threads) as ex:
        for i, (name, shp) in enumerate(names_shapes):
            if name.endswith("norm"):
                out[name] = np.ones(shp, dtype=np.float32)
                continue
            n = int(np.prod(shp))
            sub = (seed * 0x9E3779B97F4A7C15 + (i + 1) * 0xD1B54A32D192ED03) & ((1 << 64) - 1)
            buf = np.empty(n, dtype=np.float32)

            def work(lo, buf=buf, sub=sub):
                hi = min(n, lo + chunk)
                v = _uniform_chunk(sub, lo, hi, scale)
                buf[lo:hi] = bf16_round(v) if bf16 else v
            list(ex.map(work, range(0, n, chunk)))
            out[name] = buf.reshape(shp)
    return out


# ------------------------------------------------------------- model plug-ins
@dataclass
class _DecCache:
    """ModelState.cache of the transformer plug-in: the KV cache plus the greedy
    prediction after every prefix length (the hash chain's per-position cache analog,
    models.py:203-209), so a crop is a truncate and needs no forward."""
    st: DecState
    preds: list = field(default_factory=list)
    spec: tuple | None = None   # (candidates, K, V, preds) of the last verify_tokens (pure scratch)
    hashes: list = field(default_factory=list)   # coin draft only: prefix hashes


def make_models(S=None):
    """Classes over the given reference package: (DecoderModel, CoinDraftModel, ShimExecutor)."""
    S = S or load_reference()
    if S is None:
        raise ImportError("reference package specdec not found (baseline/_ref or /root/reference)")
    from specdec.models import MockModel

    class DecoderModel(MockModel):
        """RefDecoder behind the reference's MockModel hooks (models.py:171-185)."""

        def __init__(self, dec: RefDecoder):
            super().__init__(dec.s.vocab, dec.s.eos)
            self.dec = dec

        def _initial_cache(self):
            return _DecCache(DecState(0, []))

        def _extend(self, state, tokens):
            state.tokens.extend(tokens)
            c = state.cache
            tokens = list(tokens)
            if c.spec is not None:
                # advance(accepted) after verify_tokens: the accepted prefix that equals the
                # candidates already has its K/V and predictions from the verify forward
                cands, K, V, pr = c.spec
                c.spec = None
                n0 = c.st.k[0].shape[1]
                j = 0
                while j < len(tokens) and j < len(cands) - 1 and tokens[j] == cands[j]:
                    j += 1
                if j:
                    c.st.k = [k[:, : n0 + j] for k in K]
                    c.st.v = [v[:, : n0 + j] for v in V]
                    c.st.tokens.extend(tokens[:j])
                    c.preds.extend(pr[1:j + 1])
                    tokens = tokens[j:]
                if not tokens:
                    return
            logits = self.dec.forward(c.st, tokens)
            c.preds.extend(self.dec.argmax(r) for r in logits)

        def _crop_cache(self, state, position):
            c = state.cache
            c.spec = None
            c.st.k = [k[:, :position] for k in c.st.k]
            c.st.v = [v[:, :position] for v in c.st.v]
            del c.st.tokens[position:]
            del c.preds[position:]

        def _predict(self, state):
            return state.cache.preds[len(state.tokens) - 1]

        def verify_tokens(self, state, candidates):
            """Teacher-forced predictions in ONE batched forward on a scratch view (the
            base class clones the cache: unusable for tensors)."""
            self._check_owner(state)
            if len(candidates) == 0:
                raise S.InvalidInputError("verify_tokens requires at least one candidate")
            self._validate_tokens(candidates)
            c = state.cache
            preds = [self._predict(state)]
            if len(candidates) > 1:
                lg = self.dec.forward(c.st, list(candidates[:-1]), commit=False)
                preds += [self.dec.argmax(r) for r in lg]
                c.spec = (list(candidates), self.dec.scratch[0], self.dec.scratch[1], list(preds))
            return preds

    class CoinDraftModel(DecoderModel):
        """AgreementDraft restated over the reference hooks: while the prefix equals the
        verify model's canonical greedy path it emits the canonical token with probability
        rho (AgreementDraftModel's prefix-keyed coin, models.py:271-314), otherwise its own
        greedy token (mirrors csrc/protocol.cu coin_pick)."""

        def __init__(self, dec: RefDecoder, canon: list, rho: float, coin_seed: int = 1234):
            super().__init__(dec)
            self.canon, self.rho, self.seed = list(canon), rho, coin_seed
            self.thr = rho_threshold(rho)

        def _initial_cache(self):
            c = super()._initial_cache()
            c.hashes = [mix64(self.seed)]
            return c

        def _extend(self, state, tokens):
            super()._extend(state, tokens)
            for t in tokens:
                state.cache.hashes.append(mix64(state.cache.hashes[-1] ^ t))

        def _crop_cache(self, state, position):
            super()._crop_cache(state, position)
            del state.cache.hashes[position + 1:]

        def _coin(self, toks, hashes, own):
            n = len(toks)
            if n < len(self.canon) and toks == self.canon[:n]:
                a = self.canon[n]
                if self.rho >= 1.0:
                    return a
                return coin_token(hashes[n], a, self.thr, self.dec.s.vocab, self.dec.s.eos, self.dec.s.exclude_eos)
            return own

        def _predict(self, state):
            return self._coin(state.tokens, state.cache.hashes, super()._predict(state))

        def verify_tokens(self, state, candidates):
            base = super().verify_tokens(state, candidates)
            toks, hs, out = list(state.tokens), list(state.cache.hashes), []
            for j, c in enumerate(candidates):
                out.append(self._coin(toks, hs, base[j]))
                toks.append(c)
                hs.append(mix64(hs[-1] ^ c))
            return out

    class ShimExecutor(S.ThreadExecutor):
        """The reference ThreadExecutor, unchanged, plus the SURVEY.md section 0.6 shim:
        with millisecond forwards the draft thread can log a draft event after the verify
        thread's ``complete`` (engines.py:342-352 vs 482-488), which DecodeTrace.validate
        rejects.  Tokens are unaffected; the shim drops events after ``complete`` and
        records the executor's wall time (``last_wall_s``: decode only, prefill excluded)."""

        def run(self, shared, draft_model, draft_state, verify_model, verify_state, config):
            import time
            t0 = time.perf_counter()
            trace = super().run(shared, draft_model, draft_state, verify_model, verify_state, config)
            self.last_wall_s = time.perf_counter() - t0
            ev = trace.events
            idx = next((i for i, e in enumerate(ev) if e.kind == "complete"), None)
            if idx is not None and idx != len(ev) - 1:
                self.dropped = len(ev) - 1 - idx
                trace = S.DecodeTrace(clock=trace.clock, prompt_length=trace.prompt_length, events=ev[:idx + 1])
            return trace

    return DecoderModel, CoinDraftModel, ShimExecutor


def shape_of(cfg, kv_bf16: bool, act_bf16: bool = False, acc64: bool = False) -> TfShape:
    """TfShape of a paper_2410_17375_b200.TransformerConfig (duck-typed)."""
    return TfShape(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn,
                   eos=cfg.eos_token, exclude_eos=cfg.exclude_eos, eps=cfg.norm_eps, theta=cfg.rope_theta,
                   kv_bf16=kv_bf16, act_bf16=act_bf16, acc64=acc64)
