"""GPU transformer parity: CUDA forwards vs the numpy fp32 oracle (oracle/ref_decoder.py).

fp32 path: token ids and the accept/rollback trace are bit-exact against the
CPU reference (logits within 2e-4 of the logit std -- summation order only).
bf16 path: logits within 3e-2 of the logit std of a CPU fp32 forward on the
same bf16 weights; AMUSD/sync tokens bit-exact vs GPU AR (batch invariance).
"""
import numpy as np
import pytest

from oracle import specdec_oracle as O
from oracle.ref_decoder import CanonCoinDraft, RefDecoder, TfShape

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2410_17375_b200")

FP32_LOGIT_TOL = 2e-4   # max |gpu - cpu| / std(cpu logits), fp32 weights
BF16_LOGIT_TOL = 3e-2   # same, bf16 weights + bf16 KV vs fp32 CPU on the bf16 weights
PROMPT = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    P.engines.clear_sessions()


def _shape(cfg, kv_bf16):
    return TfShape(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn,
                   eos=cfg.eos_token, exclude_eos=cfg.exclude_eos, eps=cfg.norm_eps, theta=cfg.rope_theta,
                   kv_bf16=kv_bf16)


def _pair(dtype, seed_v=1, seed_d=2):
    TC = P.TransformerConfig
    v = P.TransformerModel(TC.tiny_verify(dtype=dtype, max_seq=320), seed=seed_v)
    d = P.TransformerModel(TC.tiny_draft(dtype=dtype, max_seq=320), seed=seed_d)
    return d, v


def _oracle(model, kv_bf16=False):
    return RefDecoder(_shape(model.config, kv_bf16), model.host_weights(), tied=model.config.tied)


@pytest.fixture(scope="module")
def fp32_pair():
    return _pair("fp32")


@pytest.fixture(scope="module")
def bf16_pair():
    return _pair("bf16")


def _rel_err(gpu, cpu):
    return float(np.abs(gpu - cpu).max() / cpu.std())


def test_fp32_logits_and_next_token(fp32_pair):
    d, v = fp32_pair
    for m in (v, d):
        ref = _oracle(m)
        st = m.init_state(PROMPT)
        tok = m.next_token(st)
        rs = ref.start(PROMPT)
        assert _rel_err(m.last_logits(1).numpy()[0], rs.last_logits) < FP32_LOGIT_TOL
        assert tok == ref.predict(rs)


def test_fp32_verify_tokens_and_rollback(fp32_pair):
    _, v = fp32_pair
    ref = _oracle(v)
    st = v.init_state(PROMPT)
    rs = ref.start(PROMPT)
    cands = [5, 77, 901, 31000, 12, 12, 40, 3, 3, 9, 11, 2000, 17, 18, 19, 20, 21, 22]  # > KMAX: chunked
    assert v.verify_tokens(st, cands) == ref.verify(rs, cands)
    assert st.prefix_length == len(PROMPT)
    v.advance(st, cands[:5])
    ref.extend(rs, cands[:5])
    v.rollback(st, len(PROMPT) + 2)
    ref.crop(rs, len(PROMPT) + 2)
    v.advance(st, [600])
    ref.extend(rs, [600])
    assert v.next_token(st) == ref.predict(rs)


def test_fp32_engines_bit_exact_vs_cpu(fp32_pair):
    """AR / sync / AMUSD tokens and rollback counts == CPU fp32 oracle (natural + coin drafts)."""
    d, v = fp32_pair
    n = 48
    rv, rd = _oracle(v), _oracle(d)
    canon_toks, _, _ = O.decode_ar(rv, PROMPT, n + 16)
    cfg = P.DecodeConfig(max_new_tokens=n, draft_window_k=4)
    ar = P.decode_autoregressive(v, PROMPT, cfg)
    assert ar.tokens == canon_toks[:n]
    for rho in (None, 0.0, 0.8, 1.0):
        draft = d if rho is None else P.AgreementDraft(d, rho, coin_seed=1234)
        rdraft = rd if rho is None else CanonCoinDraft(rd, list(PROMPT) + canon_toks, rho, 1234)
        sy = P.decode_speculative_sync(draft, v, PROMPT, cfg)
        asy = P.decode_speculative_async(draft, v, PROMPT, cfg)
        assert sy.tokens == ar.tokens and asy.tokens == ar.tokens, rho
        # the CPU oracle's sync engine on the same models gives the same schedule
        otoks, _, ounits = O.decode_sync(rdraft, rv, PROMPT, n, 4)
        assert otoks == ar.tokens
        assert sy.stats.verify_steps == sum(u[1] in (O.K_ACCEPT, O.K_CORRECT) for u in ounits)
        assert sy.stats.rollbacks == sum(u[1] == O.K_CORRECT for u in ounits)
        verified = max(e.pos_hi for e in asy.trace.events if e.kind.startswith("verify_")) - len(PROMPT)
        _, dis = O.canonical_disagreements(rdraft, rv, PROMPT, verified)
        assert asy.stats.rollbacks == len(dis), rho


def test_bf16_logits_within_tolerance(bf16_pair):
    d, v = bf16_pair
    for m in (v, d):
        ref = _oracle(m, kv_bf16=True)
        st = m.init_state(PROMPT)
        m.next_token(st)
        rs = ref.start(PROMPT)
        err = _rel_err(m.last_logits(1).numpy()[0], rs.last_logits)
        assert err < BF16_LOGIT_TOL, err


def test_bf16_token_agreement_with_cpu(bf16_pair):
    _, v = bf16_pair
    ref = _oracle(v, kv_bf16=True)
    ar = P.decode_autoregressive(v, PROMPT, P.DecodeConfig(max_new_tokens=32))
    otoks, _, _ = O.decode_ar(ref, PROMPT, 32)
    match = sum(a == b for a, b in zip(ar.tokens, otoks)) / 32
    assert match >= 0.9, (ar.tokens, otoks)


def test_bf16_batch_invariance(bf16_pair):
    """The verify forward is row-independent: AMUSD/sync == AR bit-exactly in bf16."""
    d, v = bf16_pair
    cfg = P.DecodeConfig(max_new_tokens=96, draft_window_k=6)
    ar = P.decode_autoregressive(v, PROMPT, cfg)
    for draft in (d, P.AgreementDraft(d, 0.8), P.AgreementDraft(d, 0.95)):
        assert P.decode_speculative_sync(draft, v, PROMPT, cfg).tokens == ar.tokens
        for lead in (None, 2, 8):
            c2 = P.DecodeConfig(max_new_tokens=96, max_draft_lead=lead)
            res = P.decode_speculative_async(draft, v, PROMPT, c2)
            assert res.tokens == ar.tokens
            res.trace.validate()


def test_amusd_draft_cut_on_and_off(bf16_pair, monkeypatch):
    """AMUSD with the draft cut (a rollback raised mid-forward ends the draft forward at the
    grabbed prefix; the split state is re-armed) and without it: tokens == AR, valid traces,
    and the draft cut leaves no stale split-K state behind (a later AR run still matches)."""
    d, v = bf16_pair
    cfg = P.DecodeConfig(max_new_tokens=96)
    ar = P.decode_autoregressive(v, PROMPT, cfg)
    d_ar = P.decode_autoregressive(d, PROMPT, cfg).tokens  # before any cut forward
    for cut in ("0", "1"):
        monkeypatch.setenv("AMUSD_FW_CUT", cut)
        P.engines.clear_sessions()  # the knob is read when the session's graphs are captured
        cuts = []
        for rho in (0.5, 0.8):
            ex = P.CudaAsyncExecutor()
            res = P.decode_speculative_async(P.AgreementDraft(d, rho), v, PROMPT, cfg, executor=ex)
            assert res.tokens == ar.tokens, (cut, rho)
            res.trace.validate()
            cuts.append(ex.last_run.info.draft_cuts)   # cumulative per draft model
        if cut == "1":
            assert cuts[-1] > cuts0, "the cut arm never cut a draft forward"
        else:
            cuts0 = cuts[-1]
            assert cuts[0] == cuts[-1], "draft forwards were cut with AMUSD_FW_CUT=0"
        # the draft model's own greedy decode after cut forwards: unchanged (no stale
        # split-K accumulators / counters / argmax keys)
        assert P.decode_autoregressive(d, PROMPT, cfg).tokens == d_ar, cut
    P.engines.clear_sessions()


def test_llama_shapes_run():
    """1B/8B-shaped bf16 pair (reduced N): kernels handle the real shapes; AMUSD == AR."""
    TC = P.TransformerConfig
    v = P.TransformerModel(TC.llama_8b(max_seq=160), seed=11)
    d = P.TransformerModel(TC.llama_1b(max_seq=160), seed=12)
    cfg = P.DecodeConfig(max_new_tokens=24)
    ar = P.decode_autoregressive(v, PROMPT, cfg)
    res = P.decode_speculative_async(P.AgreementDraft(d, 0.8), v, PROMPT, cfg)
    assert res.tokens == ar.tokens
    sy = P.decode_speculative_sync(P.AgreementDraft(d, 0.8), v, PROMPT, cfg)
    assert sy.tokens == ar.tokens
    del v, d
    P.engines.clear_sessions()


def test_tcgen05_forward_matches_simt_and_cpu():
    """The tcgen05/TMA 16-row forward agrees with the SIMT forward and the CPU oracle (bf16 tolerance)."""
    import torch
    TC = P.TransformerConfig
    for maker in (TC.tiny_verify, TC.tiny_draft):
        tc = P.TransformerModel(maker(dtype="bf16", max_seq=256), seed=5)
        assert tc.config.use_tensor_cores
        simt = P.TransformerModel(maker(dtype="bf16", max_seq=256, use_tensor_cores=False),
                                  weights={k: v.clone() for k, v in tc.weights.items()})
        ref = _oracle(tc, kv_bf16=True)
        rs = ref.start(PROMPT)
        cands = [11, 22, 33, 44, 55, 66, 77]
        a = tc.verify_tokens(tc.init_state(PROMPT), cands)
        la = tc.last_logits(len(cands)).numpy()
        b = simt.verify_tokens(simt.init_state(PROMPT), cands)
        lb = simt.last_logits(len(cands)).numpy()
        lcpu = ref.forward(rs, cands[:-1], commit=False)
        assert _rel_err(la[1:], lcpu) < BF16_LOGIT_TOL
        assert _rel_err(la, lb) < BF16_LOGIT_TOL
        assert np.mean(np.array(a) == np.array(b)) >= 0.8
        torch.cuda.synchronize()


def test_tcgen05_llama8b_gemm_shapes():
    """8B-shaped verify: tcgen05 forward (stream-K over 148 SMs) vs SIMT forward on the same weights."""
    TC = P.TransformerConfig
    cfg = TC.llama_8b(max_seq=96, n_layers=2)
    tc = P.TransformerModel(cfg, seed=21)
    simt = P.TransformerModel(TC.llama_8b(max_seq=96, n_layers=2, use_tensor_cores=False), weights=tc.weights)
    prompt = PROMPT[:20]
    cands = [101, 202, 303, 404, 505]
    a = tc.verify_tokens(tc.init_state(prompt), cands)
    la = tc.last_logits(len(cands)).numpy()
    b = simt.verify_tokens(simt.init_state(prompt), cands)
    lb = simt.last_logits(len(cands)).numpy()
    assert _rel_err(la, lb) < 2 * BF16_LOGIT_TOL, _rel_err(la, lb)  # bf16 vs fp32 activations on both sides
    assert np.mean(np.array(a) == np.array(b)) >= 0.6


def test_persistent_forward_matches_kernel_path():
    """The one-launch persistent forward (forward_tc.cu) agrees with the per-kernel tcgen05
    path (same arithmetic up to split-K order) and is run-to-run deterministic."""
    TC = P.TransformerConfig
    cands = [11, 22, 33, 44, 55, 66, 77, 88, 99, 111, 122, 133, 144, 155, 166]
    for cfg, prompt in ((TC.tiny_verify(dtype="bf16", max_seq=320), PROMPT),
                        (TC.tiny_draft(dtype="bf16", max_seq=320), PROMPT * 9),  # 288 positions: 2 attention splits
                        (TC.llama_8b(max_seq=96, n_layers=2), PROMPT[:20])):
        m = P.TransformerModel(cfg, seed=31)
        runs = []
        for path in ("persistent", "persistent", "kernels"):
            m.set_path(path)
            preds = m.verify_tokens(m.init_state(prompt), cands)
            runs.append((preds, m.last_logits(len(cands)).numpy()))
        (p0, l0), (p1, l1), (p2, l2) = runs
        assert p0 == p1 and np.array_equal(l0, l1), "persistent forward is not deterministic"
        assert _rel_err(l0, l2) < BF16_LOGIT_TOL, _rel_err(l0, l2)  # bf16 intermediates, different split-K order
        assert np.mean(np.array(p0) == np.array(p2)) >= 0.9
        del m
    P.engines.clear_sessions()


@pytest.mark.parametrize("plen", [24, 126, 200, 300])
def test_persistent_forward_rows_invariant(plen):
    """A row's logits do not depend on how many rows share the persistent forward
    (prefixes crossing the 128-position attention split boundaries included)."""
    TC = P.TransformerConfig
    m = P.TransformerModel(TC.llama_1b(max_seq=352, n_layers=3), seed=32)
    prompt = (PROMPT * 10)[:plen]
    cands = [101, 202, 303, 404, 505, 606, 707]
    m.verify_tokens(m.init_state(prompt), cands)
    full = m.last_logits(len(cands)).numpy()
    for k in (1, 3, 5):
        m.verify_tokens(m.init_state(prompt), cands[:k])
        part = m.last_logits(k).numpy()
        assert np.array_equal(part, full[:k]), (plen, k, float(np.abs(part - full[:k]).max()))
    # incremental: advancing row by row (AR-style) gives the same last-row logits
    st = m.init_state(prompt)
    for j, c in enumerate(cands[:4]):
        m.next_token(st)
        m.advance(st, [c])
    m.next_token(st)
    inc = m.last_logits(1).numpy()[0]
    assert np.array_equal(inc, full[4]), (plen, float(np.abs(inc - full[4]).max()))
    del m
    P.engines.clear_sessions()
