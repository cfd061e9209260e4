"""GPU tests of the fused gate/up -> down persistent forward (AMUSD_FW_FUSE=1, csrc/forward_tc.cu:
every gate/up tile's epilogue feeds its 64 features' down-projection partial into the int64 down
accumulators; the down phase is one weight-less merge item per output tile).

* logits vs the bf16-faithful CPU oracle (tiny and Llama-3.2-1B shapes, 1 row and a 6-row
  window) and vs the unfused forward on the same weights;
* batch invariance: a row's logits do not depend on the rows sharing the forward nor on window
  vs incremental forwards (bit-exact);
* the full-depth 1B draft within 2x the fp32 noise floor of the oracle;
* the engines with fused models: AMUSD / sync-SD tokens == AR, the draft cut fires, and the
  co-located (partial-grid) draft takes the fused kinds too.
"""
import numpy as np
import pytest

from oracle.ref_decoder import RefDecoder
from oracle.ref_models import shape_of

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2410_17375_b200")

PROMPT = [(37 * i + 11) % 31000 + 3 for i in range(24)]
TOL = 3e-2  # max |gpu - cpu| / std(cpu logits), shallow models vs the bf16-faithful oracle


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    P.engines.clear_sessions()


def _rel(x, ref):
    return float(np.abs(x - ref).max() / ref.std())


def _model(monkeypatch, cfg, seed, fuse=True):
    monkeypatch.setenv("AMUSD_FW_FUSE", "1" if fuse else "0")  # read when the model is created
    m = P.TransformerModel(cfg, seed=seed)
    monkeypatch.delenv("AMUSD_FW_FUSE")
    return m


@pytest.mark.parametrize("shape,layers", [("tiny_draft", None), ("tiny_verify", None), ("llama_1b", 2)])
def test_fused_logits_vs_oracle(monkeypatch, shape, layers):
    TC = P.TransformerConfig
    kw = dict(dtype="bf16", max_seq=320) if shape.startswith("tiny") else dict(max_seq=320, n_layers=layers)
    cfg = getattr(TC, shape)(**kw)
    m = _model(monkeypatch, cfg, 5)
    rf = RefDecoder(shape_of(cfg, kv_bf16=True, act_bf16=True), m.host_weights(), tied=cfg.tied)
    prompt = (PROMPT * 12)[:150]
    st = m.init_state(prompt)
    m.next_token(st)
    gl = m.last_logits(1).numpy()[0]
    rs = rf.start(prompt)
    err = _rel(gl, rs.last_logits)
    print(f"{shape}: fused max|gpu-cpu|/std {err:.3e}")
    assert err < TOL, err
    cands = [101, 202, 303, 404, 505, 606]
    m.verify_tokens(st, cands)
    gw = m.last_logits(len(cands)).numpy()
    cw = np.concatenate([rs.last_logits[None], rf.forward(rs, cands[:-1], commit=False)])
    assert _rel(gw, cw) < TOL, _rel(gw, cw)
    del m
    u = _model(monkeypatch, cfg, 5, fuse=False)  # the unfused forward on the same weights
    st2 = u.init_state(prompt)
    u.next_token(st2)
    assert _rel(u.last_logits(1).numpy()[0], gl) < TOL
    del u
    P.engines.clear_sessions()


@pytest.mark.parametrize("plen", [40, 126, 250])
def test_fused_rows_invariant(monkeypatch, plen):
    TC = P.TransformerConfig
    m = _model(monkeypatch, TC.llama_1b(max_seq=352, n_layers=3), 32)
    prompt = (PROMPT * 12)[:plen]
    cands = [101, 202, 303, 404, 505, 606, 707]
    m.verify_tokens(m.init_state(prompt), cands)
    full = m.last_logits(len(cands)).numpy()
    for k in (1, 2, 3, 4, 5):
        m.verify_tokens(m.init_state(prompt), cands[:k])
        part = m.last_logits(k).numpy()
        assert np.array_equal(part, full[:k]), (plen, k, float(np.abs(part - full[:k]).max()))
    st = m.init_state(prompt)
    for c in cands[:4]:
        m.next_token(st)
        m.advance(st, [c])
    m.next_token(st)
    inc = m.last_logits(1).numpy()[0]
    assert np.array_equal(inc, full[4]), (plen, float(np.abs(inc - full[4]).max()))
    del m
    P.engines.clear_sessions()


def test_fused_full_depth_1b_vs_oracle(monkeypatch):
    import torch
    try:
        import psutil
        if psutil.virtual_memory().available < 12 * 2**30:
            pytest.skip("needs ~12 GB host RAM for the fp32 oracle")
    except ImportError:
        pass
    TC = P.TransformerConfig
    cfg = TC.llama_1b(max_seq=96)
    m = _model(monkeypatch, cfg, 1)
    w = m.host_weights()
    prompt = PROMPT + PROMPT[:8]
    st = m.init_state(prompt)
    m.next_token(st)
    gl = m.last_logits(1).numpy()[0]
    rf = RefDecoder(shape_of(cfg, kv_bf16=True, act_bf16=True), w, tied=cfg.tied)
    ref = rf.start(prompt).last_logits
    r64 = RefDecoder(shape_of(cfg, kv_bf16=True, act_bf16=True, acc64=True), w, tied=cfg.tied)
    floor = _rel(r64.start(prompt).last_logits, ref)
    err = _rel(gl, ref)
    print(f"llama_1b fused: max|gpu-cpu|/std {err:.3e} (fp32 noise floor {floor:.3e}); "
          f"argmax gpu {int(np.argmax(gl))} cpu {int(np.argmax(ref))}")
    assert err <= max(2.0 * floor, 1e-2), (err, floor)
    del m, w, rf, r64
    P.engines.clear_sessions()
    torch.cuda.empty_cache()


def test_fused_engines(monkeypatch):
    """AMUSD (co-located: the draft on a partial grid, draft cut on) and sync-SD with fused
    models: tokens == AR, valid traces, the cut fires, the draft's greedy decode unchanged."""
    TC = P.TransformerConfig
    v = _model(monkeypatch, TC.tiny_verify(dtype="bf16", max_seq=320), 3)
    d = _model(monkeypatch, TC.tiny_draft(dtype="bf16", max_seq=320), 4)
    cfg = P.DecodeConfig(max_new_tokens=96)
    ar = P.decode_autoregressive(v, PROMPT, cfg)
    d_ar = P.decode_autoregressive(d, PROMPT, cfg).tokens
    P.engines.clear_sessions()
    cuts = []
    for rho in (0.5, 0.8):
        ex = P.CudaAsyncExecutor()
        res = P.decode_speculative_async(P.AgreementDraft(d, rho), v, PROMPT, cfg, executor=ex)
        assert res.tokens == ar.tokens, rho
        res.trace.validate()
        cuts.append(ex.last_run.info.draft_cuts)
        syn = P.decode_speculative_sync(P.AgreementDraft(d, rho), v, PROMPT, cfg)
        assert syn.tokens == ar.tokens, rho
    print("draft cuts", cuts)
    assert sum(cuts) > 0
    assert P.decode_autoregressive(d, PROMPT, cfg).tokens == d_ar
    P.engines.clear_sessions()
