"""Pin the transformer oracle and exercise the reference's OWN engines over it (CPU).

1. ``oracle/ref_decoder.RefDecoder`` (numpy fp32 Llama restatement) against a
   third-party implementation, HF ``transformers.LlamaForCausalLM`` (the public
   Llama-3 architecture the build follows; SURVEY.md section 8(c) -- the reference
   itself has no transformer arithmetic): logits within 3e-5 of the logit std and
   the argmax equal at every prompt position, on the tiny config and a 2-layer
   Llama-3.2-1B-shaped config.
2. The unmodified reference engines (``specdec`` from baseline/_ref or
   /root/reference) driving RefDecoder through the MockModel hooks
   (oracle/ref_models.py): AR == sync == async(ThreadExecutor) tokens, rollbacks
   == canonical disagreements, traces validate.
3. The host weight generator is bit-identical to the device fill's host twin.
"""
import numpy as np
import pytest

from oracle.ref_decoder import RefDecoder, uniform_weights_like
from oracle.ref_models import load_reference, make_models, shape_of, synthetic_weights

HF_TOL = 3e-5  # fp32 rounding only: summation order of 2048..8192-long dots, fp32 (HF) vs fp64 (oracle) RoPE angles; measured 5e-6 (tiny), 1.05e-5 (1B-shaped)


def _cfg(kind):
    from paper_2410_17375_b200.models import TransformerConfig as TC
    if kind == "tiny":
        return TC.tiny_verify(dtype="fp32", max_seq=64)
    return TC.llama_1b(dtype="fp32", n_layers=2, max_seq=64)


def _weights(cfg, seed):
    from paper_2410_17375_b200.models import weight_names, weight_shape
    return synthetic_weights([(n, weight_shape(cfg, n)) for n in weight_names(cfg)], seed, bf16=False)


def _hf_logits(cfg, w, prompt):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    hc = tr.LlamaConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.d_model, intermediate_size=cfg.ffn,
                        num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                        num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.norm_eps,
                        rope_theta=cfg.rope_theta, tie_word_embeddings=cfg.tied, max_position_embeddings=256,
                        attention_bias=False, mlp_bias=False, torch_dtype="float32")
    hc._attn_implementation = "eager"
    model = tr.LlamaForCausalLM(hc).float().eval()
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    sd = {"model.embed_tokens.weight": t(w["embed"]), "model.norm.weight": t(w["final_norm"])}
    sd["lm_head.weight"] = t(w["embed"] if cfg.tied else w["lm_head"])
    for l in range(cfg.n_layers):
        p, q = f"layers.{l}.", f"model.layers.{l}."
        qkv = w[p + "wqkv"]
        sd[q + "self_attn.q_proj.weight"] = t(qkv[: H * hd])
        sd[q + "self_attn.k_proj.weight"] = t(qkv[H * hd:(H + KV) * hd])
        sd[q + "self_attn.v_proj.weight"] = t(qkv[(H + KV) * hd:])
        sd[q + "self_attn.o_proj.weight"] = t(w[p + "wo"])
        sd[q + "mlp.gate_proj.weight"] = t(w[p + "wgate"])
        sd[q + "mlp.up_proj.weight"] = t(w[p + "wup"])
        sd[q + "mlp.down_proj.weight"] = t(w[p + "wdown"])
        sd[q + "input_layernorm.weight"] = t(w[p + "attn_norm"])
        sd[q + "post_attention_layernorm.weight"] = t(w[p + "mlp_norm"])
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    with torch.no_grad():
        out = model(torch.tensor([prompt]), use_cache=False)
    return out.logits[0].float().numpy()


@pytest.mark.parametrize("kind", ["tiny", "1b_2layer"])
def test_ref_decoder_matches_hf_llama(kind):
    cfg = _cfg(kind)
    w = _weights(cfg, seed=5)
    prompt = [(977 * (i + 3)) % (cfg.vocab_size - 3) + 3 for i in range(32)]
    hf = _hf_logits(cfg, w, prompt)
    ref = RefDecoder(shape_of(cfg, kv_bf16=False), w, tied=cfg.tied)
    st = ref.start([prompt[0]])
    mine = np.concatenate([st.last_logits[None, :], ref.forward(st, prompt[1:])], axis=0)
    rel = float(np.abs(mine - hf).max() / hf.std())
    assert rel < HF_TOL, rel
    assert (mine.argmax(axis=1) == hf.argmax(axis=1)).all()


def test_synthetic_weights_match_host_twin():
    from paper_2410_17375_b200.models import TransformerConfig as TC, weight_names, weight_shape
    cfg = TC.tiny_draft(vocab_size=512, max_seq=64)
    shapes = {n: weight_shape(cfg, n) for n in weight_names(cfg)}
    a = uniform_weights_like(shapes, seed=7)
    b = synthetic_weights(list(shapes.items()), seed=7, bf16=False, chunk=1000)
    assert all(np.array_equal(a[k], b[k]) for k in a)
    c = synthetic_weights(list(shapes.items()), seed=7, bf16=True)
    assert all(np.array_equal(c[k].view(np.uint32) & 0xFFFF, np.zeros_like(c[k].view(np.uint32))) for k in c)


@pytest.fixture(scope="module")
def ref_pair():
    S = load_reference()
    if S is None:
        pytest.skip("reference package not installed")
    from paper_2410_17375_b200.models import TransformerConfig as TC
    vcfg = TC.tiny_verify(dtype="fp32", max_seq=256, vocab_size=4096)
    dcfg = TC.tiny_draft(dtype="fp32", max_seq=256, vocab_size=4096)
    rv = RefDecoder(shape_of(vcfg, False), _weights(vcfg, 1), tied=True)
    rd = RefDecoder(shape_of(dcfg, False), _weights(dcfg, 2), tied=True)
    return S, rv, rd


def test_reference_engines_over_decoder(ref_pair):
    """The reference's own AR / sync / async(ThreadExecutor) engines, unmodified, on the numpy decoder."""
    S, rv, rd = ref_pair
    Dec, Coin, Shim = make_models(S)
    prompt = [(31 * i + 7) % 4000 + 3 for i in range(16)]
    n = 24
    # bounded lead: the coin draft follows the canonical path only as far as `canon` reaches,
    # so the draft (<= verified + lead) must never outrun it (rho = 1 -> zero rollbacks)
    cfg = S.DecodeConfig(max_new_tokens=n, draft_window_k=4, max_draft_lead=32)
    verify = Dec(rv)
    ar = S.decode_autoregressive(verify, prompt, cfg)
    assert len(ar.tokens) == n and ar.finished_by == "length_limit"
    canon = list(prompt) + S.decode_autoregressive(verify, prompt, S.DecodeConfig(max_new_tokens=n + 72)).tokens
    assert canon[len(prompt):len(prompt) + n] == ar.tokens
    for rho in (0.0, 0.8, 1.0):
        draft = Coin(rd, canon, rho, 1234)
        sy = S.decode_speculative_sync(draft, verify, prompt, cfg)
        # the reference ThreadExecutor runs real threads: retry a run that raises, keeping the
        # traceback for the final failure
        errs = []
        for _ in range(3):
            ex = Shim()
            try:
                asy = S.decode_speculative_async(draft, verify, prompt, cfg, executor=ex)
                break
            except IndexError:
                import traceback
                errs.append(traceback.format_exc())
        else:
            raise AssertionError("reference async engine failed 3 times:\n" + errs[-1])
        assert sy.tokens == ar.tokens and asy.tokens == ar.tokens, rho
        asy.trace.validate()
        # rollback-count theorem (pkg/tests/test_engines.py:293-321) along the canonical path
        verified = max(e.pos_hi for e in asy.trace.events if e.kind.startswith("verify_")) - len(prompt)
        assert verified <= len(canon) - len(prompt), verified
        dis = [i for i in range(verified)
               if draft.next_token(_advanced(draft, prompt, canon, i)) != canon[len(prompt) + i]]
        assert asy.stats.rollbacks == len(dis), rho
        if rho == 1.0:
            assert asy.stats.rollbacks == 0 and sy.stats.rollbacks == 0


def _advanced(model, prompt, canon, i):
    st = model.init_state(prompt)
    if i:
        model.advance(st, canon[len(prompt):len(prompt) + i])
    return st


def test_decoder_plugin_rollback_and_verify(ref_pair):
    S, rv, _ = ref_pair
    Dec, _, _ = make_models(S)
    m = Dec(rv)
    st = m.init_state([5, 6, 7])
    cands = [9, 10, 11, 12]
    preds = m.verify_tokens(st, cands)
    seq = m.init_state([5, 6, 7])
    walk = []
    for c in cands:
        walk.append(m.next_token(seq))
        m.advance(seq, [c])
    assert preds == walk and st.prefix_length == 3
    m.advance(st, [1, 2, 3])
    m.rollback(st, 4)
    m.advance(st, [8])
    assert m.next_token(st) == m.next_token(m.init_state([5, 6, 7, 1, 8]))
    with pytest.raises(S.InvalidRollbackError):
        m.rollback(st, 2)
