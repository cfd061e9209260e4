"""Pin the CPU oracle restatement against golden vectors produced by the
unmodified reference (oracle/make_golden.py). CPU-only."""
import pytest

from oracle import specdec_oracle as O


def _pair(c):
    seed = int(c["seed"])
    d = O.ChainOracle(seed, c["vocab"], c["eos"], c["exclude_eos"], rho=c["rho"])
    v = O.ChainOracle(seed, c["vocab"], c["eos"], c["exclude_eos"])
    return d, v


def test_splitmix64(golden):
    for x, y in golden("hashchain")["splitmix64"]:
        assert O.mix64(int(x)) == int(y)


def test_chain_next(golden):
    cases = golden("hashchain")["chain_next"]
    # reference frozen answers (pkg/tests/test_models.py:57-69)
    assert cases[0]["next"] == 93 and cases[1]["next"] == 97
    for c in cases:
        m = O.ChainOracle(int(c["seed"]), c["vocab"], c["eos"], c["exclude_eos"])
        assert m.predict(m.start(c["prefix"])) == c["next"]


def test_agreement_draws(golden):
    for c in golden("hashchain")["agreement"]:
        d, v = _pair(c)
        assert d.predict(d.start(c["prefix"])) == c["draft_next"]
        assert v.predict(v.start(c["prefix"])) == c["verify_next"]


def test_verify_tokens(golden):
    cases = golden("hashchain")["verify_tokens"]
    assert cases[0]["preds"] == [2, 86, 40, 80]  # pkg/tests/test_models.py:190-194
    for c in cases:
        m = O.ChainOracle(int(c["seed"]), c["vocab"], 0)
        assert m.verify(m.start(c["prompt"]), c["cands"]) == c["preds"]


def test_finalize(golden):
    for c in golden("engines")["finalize"]:
        assert O.finalize(c["verified"], c["eos"], c["n"]) == (c["tokens"], c["finished_by"])


def _close_rows(a, b):
    assert len(a) == len(b)
    for ra, rb in zip(a, b):
        assert ra[1:5] == rb[1:5] and ra[6] == rb[6], (ra, rb)
        assert ra[0] == pytest.approx(rb[0], abs=1e-9) and ra[5] == pytest.approx(rb[5], abs=1e-9)


def test_engine_cases(golden):
    for c in golden("engines")["cases"]:
        d, v = _pair(c)
        lat = O.Latency(draft_per_token_ms=c["draft_ms"], verify_base_ms=c["verify_ms"],
                        rollback_overhead_ms=c["rb_ms"])
        toks, by, units = O.decode_ar(v, c["prompt"], c["n"])
        assert (toks, by) == (c["ar_tokens"], c["ar_finished_by"])
        _close_rows(O.sim_serial(units, len(c["prompt"]), toks, lat), c["ar_sim_trace"])
        stoks, sby, sunits = O.decode_sync(d, v, c["prompt"], c["n"], c["k"])
        assert (stoks, sby) == (c["sync_tokens"], c["sync_finished_by"])
        rows = O.sim_serial(sunits, len(c["prompt"]), stoks, lat)
        _close_rows(rows, c["sync_sim_trace"])
        st = O.trace_stats(rows, len(c["prompt"]))
        for key, val in c["sync_stats"].items():
            assert st[key] == pytest.approx(val), key
        atoks, aby, arows, _ = O.sim_async(d, v, c["prompt"], c["n"], c["lead"], lat)
        assert (atoks, aby) == (c["async_tokens"], c["async_finished_by"])
        _close_rows(arows, c["async_trace"])
        ast = O.trace_stats(arows, len(c["prompt"]))
        for key, val in c["async_stats"].items():
            if key != "clock":
                assert ast[key] == pytest.approx(val), key


def test_scripted_eos(golden):
    for c in golden("engines")["scripted"]:
        v = O.ScriptOracle(c["script_verify"], 100, 99, c["eos_position"])
        d = O.ScriptOracle(c["script_draft"], 100, 99)
        toks, by, _ = O.decode_ar(v, c["prompt"], c["n"])
        assert (toks, by) == (c["ar_tokens"], c["ar_finished_by"])
        assert O.decode_sync(d, v, c["prompt"], c["n"], c["k"])[0] == c["sync_tokens"]
        atoks, aby, arows, _ = O.sim_async(d, v, c["prompt"], c["n"], None, O.Latency())
        assert (atoks, aby) == (c["async_tokens"], c["async_finished_by"])
        _close_rows(arows, c["async_trace"])


def test_acceptance_campaign(golden):
    """All 1,008 reference campaign configs (pkg/tests/test_acceptance.py:37-66)."""
    g = golden("campaign")
    col = {k: i for i, k in enumerate(g["columns"])}
    assert len(g["rows"]) >= 1000
    for r in g["rows"]:
        seed, rho, vocab, excl = int(r[col["seed"]]), r[col["rho"]], r[col["vocab"]], bool(r[col["exclude_eos"]])
        d = O.ChainOracle(seed, vocab, 0, excl, rho=rho)
        v = O.ChainOracle(seed, vocab, 0, excl)
        prompt, n, k, lead = r[col["prompt"]], r[col["n"]], r[col["k"]], r[col["lead"]]
        toks, by, _ = O.decode_ar(v, prompt, n)
        assert (toks, by) == (r[col["tokens"]], r[col["finished_by"]])
        stoks, _, sunits = O.decode_sync(d, v, prompt, n, k)
        assert stoks == toks
        lat = O.Latency(draft_per_token_ms=r[col["draft_ms"]], verify_base_ms=r[col["verify_ms"]])
        atoks, _, arows, _ = O.sim_async(d, v, prompt, n, lead, lat)
        assert atoks == toks
        st = O.trace_stats(arows, len(prompt))
        assert st["verify_steps"] == r[col["async_verify_steps"]]
        assert st["rollbacks"] == r[col["async_rollbacks"]]
        assert st["wasted_draft_tokens"] == r[col["async_wasted"]]
        # rollback-count theorem along the verified path
        verified = max(x[4] for x in arows if x[2] in (O.K_ACCEPT, O.K_CORRECT)) - len(prompt)
        _, dis = O.canonical_disagreements(d, v, prompt, verified)
        assert st["rollbacks"] == len(dis)


def test_threaded_async_matches_ar():
    for seed in range(12):
        d = O.ChainOracle(seed, 503, 0, False, rho=0.7)
        v = O.ChainOracle(seed, 503, 0, False)
        toks, by, cnt, _ = O.thread_async(d, v, [1, 2, 3], 48)
        assert (toks, by) == O.decode_ar(v, [1, 2, 3], 48)[:2]
