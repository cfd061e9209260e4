"""Tensor-parallel verify model (BASELINE config 4) on one GPU: the ranks are emulated as
separate shards with their own streams and SM shares, talking through the same peer-memory
words (int64 split-K accumulators, tile counts, argmax keys, step-control inboxes) a
multi-GPU group uses over NVLink.

* The sharded forward is BIT-IDENTICAL to the unsharded persistent forward: the shards take
  the unsharded chunking, each O / down chunk's int64 partial lands in every rank's
  accumulator, integer sums commute (paper_2410_17375_b200/tp.py).
* AR / sync-SD / AMUSD on the sharded verify produce the unsharded model's AR tokens.
"""
import pytest

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2410_17375_b200")

PROMPT = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    P.engines.clear_sessions()


def _unsharded_logits(cfg, seed):
    m = P.TransformerModel(cfg, seed=seed)
    st = m.init_state(PROMPT)
    tok = m.next_token(st)
    return m, m.last_logits(1)[0], tok


@pytest.mark.parametrize("shape,layers,size", [("llama_8b", 2, 2), ("llama_8b", 2, 4), ("llama_70b", 1, 7)])
def test_tp_forward_bit_identical(shape, layers, size):
    import torch
    from paper_2410_17375_b200.tp import TPGroup
    cfg = getattr(P.TransformerConfig, shape)(n_layers=layers, max_seq=128)
    m, ref, tok = _unsharded_logits(cfg, seed=0)
    del m
    torch.cuda.empty_cache()
    g = TPGroup(cfg, size, seed=0)
    logits, toks = g.first_logits(PROMPT)
    assert toks == [tok] * size
    assert logits.shape == ref.shape
    diff = (logits - ref).abs().max().item()
    print(f"{shape} x{layers} TP-{size}: max|tp - unsharded| = {diff}")
    assert torch.equal(logits, ref), diff


@pytest.fixture(scope="module")
def tp_pair():
    import torch
    from paper_2410_17375_b200.tp import TPGroup
    TC = P.TransformerConfig
    vcfg = TC.llama_8b(n_layers=2, max_seq=256)
    dcfg = TC.llama_1b(n_layers=2, max_seq=256)
    ref = P.TransformerModel(vcfg, seed=0)
    n = 48
    ar = P.decode_autoregressive(ref, PROMPT, P.DecodeConfig(max_new_tokens=n + 16)).tokens
    del ref
    torch.cuda.empty_cache()
    g = TPGroup(vcfg, 2, seed=0, reserve_sms=48)
    return g, dcfg, ar, n


def test_tp_autoregressive(tp_pair):
    g, _, ar, n = tp_pair
    res = g.decode_autoregressive(PROMPT, P.DecodeConfig(max_new_tokens=n))
    assert res.tokens == ar[:n]
    res.trace.validate()


def test_tp_sync_and_amusd(tp_pair):
    import torch
    g, dcfg, ar, n = tp_pair
    canon = torch.tensor(PROMPT + ar, dtype=torch.int32)
    cfg = P.DecodeConfig(max_new_tokens=n)
    drafts = []
    for r in range(g.size):
        d = P.TransformerModel(dcfg, seed=1)
        d.set_max_grid(50)
        drafts.append(P.AgreementDraft(d, 0.8, coin_seed=1234))
    sy = g.decode_speculative_sync(drafts, PROMPT, cfg, canon=canon)
    assert sy.tokens == ar[:n]
    sy.trace.validate()
    dm = P.TransformerModel(dcfg, seed=1)
    dm.set_max_grid(48)
    res = g.decode_speculative_async(P.AgreementDraft(dm, 0.8, coin_seed=1234), PROMPT, cfg, canon=canon)
    assert res.tokens == ar[:n]
    res.trace.validate()
    print(f"TP-2 sync verify steps {sy.stats.verify_steps}, AMUSD verify steps {res.stats.verify_steps}, "
          f"rollbacks {res.stats.rollbacks}")
