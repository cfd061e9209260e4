"""GPU protocol parity: device hash-chain models + the CUDA engines vs the
reference's golden vectors and the CPU oracle (bit-exact integer work).

Mirrors the reference tests: pkg/tests/test_models.py (chain/agreement/
verify_tokens/rollback), test_engines.py (engines, rollback-count theorem,
jitter), test_acceptance.py (the >= 1000-config equivalence campaign).
"""
import random

import pytest

from oracle import specdec_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2410_17375_b200")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    P.engines.clear_sessions()


def _pair(seed, rho, vocab, eos, excl, max_seq=1024):
    return P.make_agreement_pair(seed, rho, vocab, eos, exclude_eos=excl, max_seq=max_seq)


def test_chain_next_token_golden(golden):
    for c in golden("hashchain")["chain_next"][:120]:
        m = P.HashChainModel(int(c["seed"]), c["vocab"], c["eos"], c["exclude_eos"], max_seq=64)
        assert m.next_token(m.init_state(c["prefix"])) == c["next"]


def test_agreement_draws_golden(golden):
    for c in golden("hashchain")["agreement"][:150]:
        d, v = _pair(int(c["seed"]), c["rho"], c["vocab"], c["eos"], c["exclude_eos"], max_seq=64)
        assert d.next_token(d.init_state(c["prefix"])) == c["draft_next"]
        assert v.next_token(v.init_state(c["prefix"])) == c["verify_next"]


def test_verify_tokens_golden(golden):
    cases = golden("hashchain")["verify_tokens"]
    for c in cases[:60]:
        m = P.HashChainModel(int(c["seed"]), c["vocab"], 0, max_seq=64)
        st = m.init_state(c["prompt"])
        assert m.verify_tokens(st, c["cands"]) == c["preds"]
        assert st.prefix_length == len(c["prompt"])  # not mutated (models.py:151-169)


def test_rollback_semantics():
    m = P.HashChainModel(5, 100, 0, max_seq=64)
    st = m.init_state([7])
    m.advance(st, [10, 11, 12])
    m.rollback(st, 2)
    m.advance(st, [20, 21])
    ref = O.ChainOracle(5, 100, 0)
    assert m.next_token(st) == ref.predict(ref.start([7, 10, 20, 21]))
    with pytest.raises(P.InvalidRollbackError):
        m.rollback(st, 0)
    with pytest.raises(P.InvalidRollbackError):
        m.rollback(st, 99)
    with pytest.raises(P.InvalidInputError):
        m.advance(st, [])
    with pytest.raises(P.InvalidInputError):
        m.advance(st, [100])
    other = P.HashChainModel(5, 100, 0, max_seq=64)
    with pytest.raises(P.InvalidInputError):
        other.next_token(st)


def test_rollback_soundness_random_interleavings():
    rng = random.Random(77)
    m = P.HashChainModel(31, 500, 0, max_seq=256)
    ref = O.ChainOracle(31, 500, 0)
    for _ in range(20):
        prompt = [rng.randrange(500) for _ in range(rng.randint(1, 4))]
        st = m.init_state(prompt)
        toks = list(prompt)
        for _ in range(rng.randint(1, 20)):
            if rng.random() < 0.6 or len(toks) == len(prompt):
                add = [rng.randrange(500) for _ in range(rng.randint(1, 3))]
                m.advance(st, add)
                toks += add
            else:
                n = rng.randint(len(prompt), len(toks))
                m.rollback(st, n)
                del toks[n:]
            if rng.random() < 0.3:
                assert m.next_token(st) == ref.predict(ref.start(toks))
        assert m.next_token(st) == ref.predict(ref.start(toks))


def _check_run(d, v, prompt, n, k, lead, executor=None):
    cfg = P.DecodeConfig(max_new_tokens=n, draft_window_k=k, max_draft_lead=lead)
    ar = P.decode_autoregressive(v, prompt, cfg)
    sy = P.decode_speculative_sync(d, v, prompt, cfg)
    asy = P.decode_speculative_async(d, v, prompt, cfg, executor=executor)
    return ar, sy, asy


def test_engine_cases_golden(golden):
    for c in golden("engines")["cases"]:
        seed = int(c["seed"])
        d, v = _pair(seed, c["rho"], c["vocab"], c["eos"], c["exclude_eos"], max_seq=len(c["prompt"]) + c["n"] + 64)
        ar, sy, asy = _check_run(d, v, c["prompt"], c["n"], c["k"], c["lead"])
        assert (ar.tokens, ar.finished_by) == (c["ar_tokens"], c["ar_finished_by"])
        assert (sy.tokens, sy.finished_by) == (c["sync_tokens"], c["sync_finished_by"])
        # sync-SD schedule is deterministic: its stats match the reference exactly
        for key, val in c["sync_stats"].items():
            assert getattr(sy.stats, key) == pytest.approx(val), key
        assert (asy.tokens, asy.finished_by) == (c["async_tokens"], c["async_finished_by"])
        # rollback-count theorem (pkg/tests/test_engines.py:293-321)
        dd = O.ChainOracle(seed, c["vocab"], c["eos"], c["exclude_eos"], rho=c["rho"])
        vv = O.ChainOracle(seed, c["vocab"], c["eos"], c["exclude_eos"])
        verified = max(e.pos_hi for e in asy.trace.events if e.kind.startswith("verify_")) - len(c["prompt"])
        _, dis = O.canonical_disagreements(dd, vv, c["prompt"], verified)
        assert asy.stats.rollbacks == len(dis)
        # gap-free monotone p_v (test_acceptance.py criterion 5)
        frontier = len(c["prompt"])
        for e in asy.trace.events:
            if e.kind in ("verify_accept", "verify_correct"):
                assert e.pos_lo == frontier + 1
                frontier = e.pos_hi


def test_acceptance_campaign_on_gpu(golden):
    """All 1,008 reference campaign configs (pkg/tests/test_acceptance.py:37-66)."""
    g = golden("campaign")
    col = {k: i for i, k in enumerate(g["columns"])}
    count = 0
    for idx, r in enumerate(g["rows"]):
        seed, rho, vocab, excl = int(r[col["seed"]]), r[col["rho"]], r[col["vocab"]], bool(r[col["exclude_eos"]])
        prompt, n, k, lead = r[col["prompt"]], r[col["n"]], r[col["k"]], r[col["lead"]]
        d, v = _pair(seed, rho, vocab, 0, excl, max_seq=len(prompt) + n + 64)
        ar, sy, asy = _check_run(d, v, prompt, n, k, lead)
        assert ar.tokens == r[col["tokens"]] and ar.finished_by == r[col["finished_by"]], idx
        assert sy.tokens == ar.tokens and sy.finished_by == ar.finished_by, idx
        assert sy.stats.verify_steps == r[col["sync_verify_steps"]] and sy.stats.rollbacks == r[col["sync_rollbacks"]]
        assert asy.tokens == ar.tokens and asy.finished_by == ar.finished_by, idx
        verified = max(e.pos_hi for e in asy.trace.events if e.kind.startswith("verify_")) - len(prompt)
        dd = O.ChainOracle(seed, vocab, 0, excl, rho=rho)
        vv = O.ChainOracle(seed, vocab, 0, excl)
        _, dis = O.canonical_disagreements(dd, vv, prompt, verified)
        assert asy.stats.rollbacks == len(dis), idx
        count += 1
        if idx % 64 == 63:
            P.engines.clear_sessions()
    assert count >= 1000


def test_jittered_device_schedules_keep_tokens():
    """>= 100 runs with seeded device-side poll jitter (criterion 5 analog)."""
    rng = random.Random(5)
    acks = 0
    for i in range(100):
        rho = rng.choice([0.0, 0.5, 0.7, 0.9])
        seed = rng.getrandbits(32)
        d, v = _pair(seed, rho, 997, 0, True, max_seq=128)
        ex = P.CudaAsyncExecutor(poll_jitter_ns=rng.choice([0, 2000, 20000]), jitter_seed=i,
                                 max_window=rng.choice([1, 4, 16]))
        cfg = P.DecodeConfig(max_new_tokens=40, max_draft_lead=rng.choice([None, 1, 3]))
        res = P.decode_speculative_async(d, v, [1, 2, 3, 4], cfg, executor=ex)
        vv = O.ChainOracle(seed, 997, 0, True)
        assert res.tokens == O.decode_ar(vv, [1, 2, 3, 4], 40)[0], i
        acks += sum(e.kind == "rollback" for e in res.trace.events)
        res.trace.validate()
    assert acks > 0


def test_livelock_freedom_rho_zero():
    d, v = _pair(23, 0.0, 5000, 0, True, max_seq=256)
    res = P.decode_speculative_async(d, v, [1, 2, 3, 4], P.DecodeConfig(max_new_tokens=100))
    assert res.tokens == O.decode_ar(O.ChainOracle(23, 5000, 0, True), [1, 2, 3, 4], 100)[0]
    assert res.stats.verify_steps == 100 and res.stats.rollbacks == 100


def test_full_agreement_no_rollbacks():
    d, v = _pair(9, 1.0, 997, 0, True, max_seq=256)
    res = P.decode_speculative_async(d, v, [1, 2, 3], P.DecodeConfig(max_new_tokens=40))
    assert res.stats.rollbacks == 0 and res.stats.wasted_draft_tokens == 0
    sy = P.decode_speculative_sync(d, v, [1, 2, 3], P.DecodeConfig(max_new_tokens=10, draft_window_k=4))
    assert sy.stats.verify_steps == 2 and sy.stats.accepted_per_verify_step == 5.0


@pytest.mark.parametrize("minw,wait_us", [(3, 200), (8, 50), (4, 20000)])
def test_verify_pacing_keeps_tokens(monkeypatch, minw, wait_us):
    """AMUSD_VERIFY_MIN_WINDOW / _WAIT_US change only when the verify loop starts a step: tokens
    stay the AR tokens, traces validate, and a step never waits forever (a window the draft cannot fill -- lead cap 2 < min window -- ends by the
    time bound)."""
    monkeypatch.setenv("AMUSD_VERIFY_MIN_WINDOW", str(minw))
    monkeypatch.setenv("AMUSD_VERIFY_WAIT_US", str(wait_us))
    P.engines.clear_sessions()  # the pacing is read when a session's graphs are built
    try:
        for seed, rho, lead in ((31, 0.7, None), (32, 0.9, 2), (33, 0.0, None)):
            d, v = _pair(seed, rho, 997, 0, True, max_seq=256)
            cfg = P.DecodeConfig(max_new_tokens=60, max_draft_lead=lead)
            res = P.decode_speculative_async(d, v, [1, 2, 3, 4], cfg)
            assert res.tokens == O.decode_ar(O.ChainOracle(seed, 997, 0, True), [1, 2, 3, 4], 60)[0], seed
            res.trace.validate()
    finally:
        P.engines.clear_sessions()
