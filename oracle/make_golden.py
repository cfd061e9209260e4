"""Generate golden fixtures under tests/golden/ by running the REAL reference.

Test infrastructure only (see oracle/__init__.py). This script imports the
unmodified reference package ``specdec`` from ``/root/reference/pkg/src``
(read-only) and records its outputs, so that the oracle restatement in
``oracle/specdec_oracle.py`` -- and, through it, the CUDA path -- can be pinned
against the reference on a machine where ``/root/reference`` does not exist.

Run:  python oracle/make_golden.py  [--ref /root/reference/pkg/src]

Cases follow the reference's own tests:
  * hash chain / splitmix64 known answers  -- pkg/tests/test_models.py:22-69, 190-194
  * agreement-pair draws                    -- pkg/tests/test_models.py:252-313
  * verify_tokens teacher forcing           -- pkg/tests/test_models.py:196-227
  * AR / sync / async-sim engine outputs    -- pkg/tests/test_engines.py:78-371
  * the >=1000-config equivalence campaign  -- pkg/tests/test_acceptance.py:37-66
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "tests" / "golden"


def _import_reference(path: str):
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)
    import specdec  # noqa: F401  (the unmodified reference)
    return specdec


def _trace_rows(trace):
    return [[e.t_ms, e.actor, e.kind, e.pos_lo, e.pos_hi, e.busy_ms, e.draft_accepted] for e in trace.events]


def _stats(stats):
    d = stats.to_dict()
    return d


def gen_hashchain(sd):
    rng = random.Random(0x5EED)
    out = {"splitmix64": [], "chain_next": [], "agreement": [], "verify_tokens": []}
    xs = [0, 1, 2, (1 << 64) - 1, 0x9E3779B97F4A7C15, 42, 7, 1234]
    xs += [rng.getrandbits(64) for _ in range(40)]
    out["splitmix64"] = [[str(x), str(sd.splitmix64(x))] for x in xs]
    # plain chain next-token (incl. the reference's frozen vectors)
    cases = [(42, [1, 2, 3], 101, 100, False), (7, [5, 6], 101, 100, False)]
    for _ in range(300):
        vocab = rng.randint(3, 140000)
        seed = rng.getrandbits(64)
        prefix = [rng.randrange(vocab) for _ in range(rng.randint(1, 24))]
        eos = rng.randrange(vocab)
        cases.append((seed, prefix, vocab, eos, rng.random() < 0.5))
    for seed, prefix, vocab, eos, excl in cases:
        m = sd.HashChainModel(seed=seed, vocab_size=vocab, eos_token=eos, exclude_eos=excl)
        st = m.init_state(prefix)
        out["chain_next"].append({"seed": str(seed), "prefix": prefix, "vocab": vocab, "eos": eos,
                                  "exclude_eos": excl, "next": m.next_token(st)})
    for _ in range(400):
        vocab = rng.choice([3, 4, 11, 101, 997, 32000, 128256])
        seed = rng.getrandbits(64)
        rho = rng.choice([0.0, 0.25, 0.5, 0.8, 0.9, 1.0])
        eos = rng.randrange(vocab)
        excl = rng.random() < 0.5
        prefix = [rng.randrange(vocab) for _ in range(rng.randint(1, 16))]
        d, v = sd.make_agreement_pair(seed, rho, vocab, eos, exclude_eos=excl)
        out["agreement"].append({"seed": str(seed), "rho": rho, "vocab": vocab, "eos": eos, "exclude_eos": excl,
                                 "prefix": prefix, "draft_next": d.next_token(d.init_state(prefix)),
                                 "verify_next": v.next_token(v.init_state(prefix))})
    cases = [(9, [4, 5], [10, 11, 12, 13], 101)]
    for _ in range(100):
        vocab = rng.randint(3, 5000)
        cases.append((rng.getrandbits(32), [rng.randrange(vocab) for _ in range(rng.randint(1, 5))],
                      [rng.randrange(vocab) for _ in range(rng.randint(1, 16))], vocab))
    for seed, prompt, cands, vocab in cases:
        m = sd.HashChainModel(seed=seed, vocab_size=vocab, eos_token=0)
        out["verify_tokens"].append({"seed": str(seed), "prompt": prompt, "cands": cands, "vocab": vocab,
                                     "preds": m.verify_tokens(m.init_state(prompt), cands)})
    return out


def _run_three(sd, draft, verify, prompt, config, latency):
    ar = sd.decode_autoregressive(verify, prompt, config)
    sy = sd.decode_speculative_sync(draft, verify, prompt, config)
    sim = sd.decode_speculative_async(draft, verify, prompt, config,
                                      executor=sd.SimulatedExecutor(latency))
    return ar, sy, sim


def gen_engines(sd):
    """Engine outputs with full virtual-clock traces (deterministic)."""
    rng = random.Random(0xE9)
    cases = []
    specs = []
    for rho in (0.0, 0.3, 0.6, 0.8, 0.9, 1.0):
        for _ in range(6):
            specs.append(dict(seed=rng.getrandbits(48), rho=rho, vocab=rng.choice([101, 503, 5000, 32000]),
                              eos=0, exclude_eos=rng.random() < 0.6,
                              prompt=[rng.randrange(3, 100) for _ in range(rng.randint(1, 8))],
                              n=rng.choice([1, 2, 7, 40, 128]), k=rng.choice([1, 2, 4, 8]),
                              lead=rng.choice([None, None, 1, 3, 16]),
                              draft_ms=rng.choice([0.377, 5.0, 10.0]), verify_ms=rng.choice([2.29, 12.0, 25.0]),
                              rb_ms=rng.choice([0.0, 0.0, 1.5])))
    for s in specs:
        draft, verify = sd.make_agreement_pair(s["seed"], s["rho"], s["vocab"], s["eos"], exclude_eos=s["exclude_eos"])
        config = sd.DecodeConfig(max_new_tokens=s["n"], draft_window_k=s["k"], max_draft_lead=s["lead"])
        latency = sd.LatencyModel(draft_per_token_ms=s["draft_ms"], verify_base_ms=s["verify_ms"],
                                  rollback_overhead_ms=s["rb_ms"])
        ar, sy, sim = _run_three(sd, draft, verify, s["prompt"], config, latency)
        _, sync_sim_trace = sd.simulate("sync_speculative", draft, verify, s["prompt"], config, latency)
        _, ar_sim_trace = sd.simulate("autoregressive", None, verify, s["prompt"], config, latency)
        case = dict(s, seed=str(s["seed"]))
        case.update(
            ar_tokens=ar.tokens, ar_finished_by=ar.finished_by,
            sync_tokens=sy.tokens, sync_finished_by=sy.finished_by,
            sync_stats={k: v for k, v in _stats(sy.stats).items() if k not in ("total_ms", "mean_ms_per_token", "clock")},
            sync_sim_trace=_trace_rows(sync_sim_trace),
            ar_sim_trace=_trace_rows(ar_sim_trace),
            async_tokens=sim.tokens, async_finished_by=sim.finished_by,
            async_stats=_stats(sim.stats), async_trace=_trace_rows(sim.trace),
        )
        cases.append(case)
    # scripted eos cases (pkg/tests/test_engines.py:66-76, 302-312)
    scripted = []
    for eos_at in (1, 2, 7, 13):
        for k in (1, 4):
            prompt = [1, 2, 3]
            verify = sd.ScriptedModel([5, 6, 7], vocab_size=100, eos_token=99, eos_position=len(prompt) + eos_at)
            draft = sd.ScriptedModel([5, 6, 8], vocab_size=100, eos_token=99)
            config = sd.DecodeConfig(max_new_tokens=50, draft_window_k=k)
            ar, sy, sim = _run_three(sd, draft, verify, prompt, config, sd.LatencyModel())
            scripted.append(dict(script_verify=[5, 6, 7], script_draft=[5, 6, 8], eos_position=len(prompt) + eos_at,
                                 prompt=prompt, k=k, n=50, ar_tokens=ar.tokens, ar_finished_by=ar.finished_by,
                                 sync_tokens=sy.tokens, async_tokens=sim.tokens, async_finished_by=sim.finished_by,
                                 async_trace=_trace_rows(sim.trace)))
    # finalize_tokens / find_mismatch known answers (pkg/tests/test_engines.py:33-61)
    fin = []
    for verified, eos, n in [([5, 9, 6, 7], 9, 10), ([1, 2, 3, 4], 9, 3), ([1, 2, 3, 9], 9, 3), ([9], 9, 1), ([4, 4, 9, 9], 9, 4)]:
        toks, by = sd.finalize_tokens(verified, eos, n)
        fin.append(dict(verified=verified, eos=eos, n=n, tokens=toks, finished_by=by))
    return {"cases": cases, "scripted": scripted, "finalize": fin}


def gen_campaign(sd):
    """The reference's acceptance campaign inputs + reference outputs.

    Mirrors pkg/tests/test_acceptance.py:37-66 exactly (same RNG stream), and
    records the oracle tokens, finished_by and the canonical disagreement
    count along the verified path (the rollback-count theorem,
    pkg/tests/test_engines.py:293-321) for every configuration.
    """
    rng = random.Random(0xACCE97)
    rows = []
    for rho, n, k in itertools.product((0.0, 0.25, 0.5, 0.8, 0.95, 1.0), (1, 2, 17, 128), (1, 4, 8)):
        for trial in range(14):
            seed = rng.getrandbits(48)
            exclude = trial % 3 != 0
            vocab = rng.choice([101, 503, 5000])
            lead = rng.choice([None, None, 1, 4])
            dms = rng.choice([5.0, 10.0, 15.0])
            vms = rng.choice([12.0, 25.0, 40.0])
            prompt = [rng.randrange(vocab) for _ in range(rng.randint(1, 6))]
            draft, verify = sd.make_agreement_pair(seed, rho, vocab, eos_token=0, exclude_eos=exclude)
            config = sd.DecodeConfig(max_new_tokens=n, draft_window_k=k, max_draft_lead=lead, seed=seed)
            latency = sd.LatencyModel(draft_per_token_ms=dms, verify_base_ms=vms)
            ar, sy, sim = _run_three(sd, draft, verify, prompt, config, latency)
            assert ar.tokens == sy.tokens == sim.tokens
            rows.append([rho, n, k, str(seed), int(exclude), vocab, lead, dms, vms, prompt,
                         ar.tokens, ar.finished_by, sy.stats.verify_steps, sy.stats.rollbacks,
                         sim.stats.verify_steps, sim.stats.rollbacks, sim.stats.wasted_draft_tokens])
    cols = ["rho", "n", "k", "seed", "exclude_eos", "vocab", "lead", "draft_ms", "verify_ms", "prompt",
            "tokens", "finished_by", "sync_verify_steps", "sync_rollbacks", "async_verify_steps",
            "async_rollbacks", "async_wasted"]
    return {"columns": cols, "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("SPECDEC_REF", "/root/reference/pkg/src"))
    args = ap.parse_args()
    sd = _import_reference(args.ref)
    OUT.mkdir(parents=True, exist_ok=True)
    for name, fn in (("hashchain", gen_hashchain), ("engines", gen_engines), ("campaign", gen_campaign)):
        data = fn(sd)
        data["_generated_by"] = "oracle/make_golden.py from the unmodified reference specdec " + sd.__version__
        (OUT / f"{name}.json").write_text(json.dumps(data, separators=(",", ":")))
        print(name, (OUT / f"{name}.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
