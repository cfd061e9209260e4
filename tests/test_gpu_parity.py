"""GPU parity at the headline shapes and against the reference's OWN engines.

* Full-depth Llama-3.2-1B / Llama-3.1-8B-shaped bf16 models through the
  persistent tcgen05 forward (the bench path) vs the CPU fp32 oracle on the
  same bf16 weights (oracle/ref_decoder.py, pinned to HF Llama by
  tests/test_oracle_pinned.py): first-step logits within BF16_LOGIT_TOL of the
  logit std, and the first AR tokens, with the top-2 gap reported at any
  mismatch (near-ties only may differ: bf16 activations vs fp32).
* BASELINE config 1 exactly: tiny fp32 pair, 32-token prompt, 128 new tokens,
  AR / sync-SD / AMUSD on the GPU vs the unmodified reference engines
  (specdec from baseline/_ref) on the CPU decoders: tokens bit-exact, the
  sync-SD trace (every event's kind and positions) bit-exact, the AMUSD
  correction positions == the canonical disagreement positions.
* The drop-in claim: the reference's own
  decode_autoregressive / decode_speculative_sync / decode_speculative_async
  (executor=CudaAsyncExecutor()) driving the CUDA models.
* The reference's scripted-eos edge cases (ScriptedModel, models.py:317-346;
  pkg/tests/test_engines.py:66-76) on the device engines vs the goldens.
"""
import numpy as np
import pytest

from oracle import specdec_oracle as O
from oracle.ref_decoder import RefDecoder
from oracle.ref_models import load_reference, make_models, shape_of

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2410_17375_b200")

BF16_LOGIT_TOL = 3e-2   # max |gpu - cpu| / std(cpu logits): bf16 weights/activations/KV vs fp32 CPU (shallow)
# Full depth: the bf16-faithful oracle rounds exactly where the kernels round, so the GPU and the
# CPU differ in fp32 summation order only -- but a summation-order difference flips bf16 roundings
# of the activations, and 16 / 32 random-init layers amplify the flips.  The tolerance is therefore
# MEASURED, not guessed: the same oracle with float64 accumulation (a second summation order,
# acc64) sets the noise floor, and the GPU must sit within FLOOR_FACTOR x that floor (1B: floor
# 0.045 of the logit std, GPU 0.048).
FLOOR_FACTOR = 2.0
FLOOR_MIN = 1e-2
DEEP_BF16_TOL = 2e-1    # vs the pure-fp32 oracle (no activation rounding at all) at full depth
PROMPT32 = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    P.engines.clear_sessions()


def _ref():
    S = load_reference()
    if S is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    return S


def _host_ram_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except ImportError:
        return 0.0


@pytest.mark.parametrize("shape", ["llama_1b", "llama_8b"])
def test_bench_shapes_vs_cpu_oracle(shape):
    """Full-depth bench-shape forward (persistent tcgen05 path) vs the CPU oracle on the same
    bf16 weights: the bf16-faithful oracle (activations rounded where the kernels round them;
    only fp32 summation order differs) within FLOOR_FACTOR x the measured fp32 noise floor, the
    pure-fp32 oracle within
    DEEP_BF16_TOL (bf16 activation quantisation accumulated over 16 / 32 layers)."""
    import torch
    TC = P.TransformerConfig
    need = {"llama_1b": 12, "llama_8b": 70}[shape]
    if _host_ram_gb() < need:
        pytest.skip(f"needs ~{need} GB host RAM for the fp32 oracle")
    cfg = getattr(TC, shape)(max_seq=96)
    m = P.TransformerModel(cfg, seed={"llama_1b": 1, "llama_8b": 0}[shape])
    w = m.host_weights()
    rf = RefDecoder(shape_of(cfg, kv_bf16=True, act_bf16=True), w, tied=cfg.tied)
    n = 8
    ar = P.decode_autoregressive(m, PROMPT32, P.DecodeConfig(max_new_tokens=n)).tokens
    st = m.init_state(PROMPT32)
    m.next_token(st)
    gl = m.last_logits(1).numpy()[0]
    rs = rf.start(PROMPT32)
    ref = rs.last_logits
    rel = lambda x: float(np.abs(x - ref).max() / ref.std())
    r64 = RefDecoder(shape_of(cfg, kv_bf16=True, act_bf16=True, acc64=True), w, tied=cfg.tied)
    floor = rel(r64.start(PROMPT32).last_logits)
    del r64
    r32 = RefDecoder(shape_of(cfg, kv_bf16=True), w, tied=cfg.tied)
    l32 = r32.start(PROMPT32).last_logits
    del r32
    err = rel(gl)
    err32 = float(np.abs(gl - l32).max() / l32.std())
    tol = max(FLOOR_FACTOR * floor, FLOOR_MIN)
    print(f"{shape}: max|gpu-cpu|/std: bf16-faithful oracle {err:.3e} (fp32 noise floor {floor:.3e}, tol {tol:.3e}), "
          f"fp32 oracle {err32:.3e}; argmax gpu {int(np.argmax(gl))} cpu {int(np.argmax(ref))}")
    assert err <= tol, (err, floor)
    assert err32 < DEEP_BF16_TOL, err32
    cpu, gaps = [], []
    for i in range(n):
        z = np.array(rs.last_logits, dtype=np.float32)
        z[cfg.eos_token] = -np.inf
        top2 = np.sort(z)[-2:]
        cpu.append(rf.predict(rs))
        gaps.append(float((top2[1] - top2[0]) / rs.last_logits.std()))
        rf.extend(rs, [ar[i]])        # teacher-forced on the GPU's path: per-position comparison
    mism = [(i, ar[i], cpu[i], gaps[i]) for i in range(n) if ar[i] != cpu[i]]
    print(f"{shape}: AR tokens {n - len(mism)}/{n} equal to the faithful oracle; mismatches {mism}")
    # a mismatch is legitimate only at a near-tie (top-2 gap within the logit tolerance)
    assert all(g < 2 * tol for (_, _, _, g) in mism), mism
    del m, w, rf
    P.engines.clear_sessions()
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def cfg1_pair():
    TC = P.TransformerConfig
    v = P.TransformerModel(TC.tiny_verify(dtype="fp32", max_seq=256), seed=0)
    d = P.TransformerModel(TC.tiny_draft(dtype="fp32", max_seq=256), seed=1)
    rv = RefDecoder(shape_of(v.config, kv_bf16=False), v.host_weights(), tied=True)
    rd = RefDecoder(shape_of(d.config, kv_bf16=False), d.host_weights(), tied=True)
    return d, v, rd, rv


def test_config1_exact_vs_reference_engines(cfg1_pair):
    """BASELINE config 1: tiny fp32 pair, 32-token prompt, N=128 -- bit-exact vs the reference's engines."""
    S = _ref()
    Dec, Coin, Shim = make_models(S)
    d, v, rd, rv = cfg1_pair
    prompt = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]
    n, k = 128, 4
    verify = Dec(rv)
    ref_ar = S.decode_autoregressive(verify, prompt, S.DecodeConfig(max_new_tokens=n + 16, draft_window_k=k))
    canon = list(prompt) + ref_ar.tokens
    cfg = P.DecodeConfig(max_new_tokens=n, draft_window_k=k)
    ar = P.decode_autoregressive(v, prompt, cfg)
    assert ar.tokens == ref_ar.tokens[:n]
    for rho in (0.8, 0.9):
        rdraft = Coin(rd, canon, rho, 1234)
        gdraft = P.AgreementDraft(d, rho, coin_seed=1234)
        rsy = S.decode_speculative_sync(rdraft, verify, prompt, S.DecodeConfig(max_new_tokens=n, draft_window_k=k))
        gsy = P.decode_speculative_sync(gdraft, v, prompt, cfg)
        assert gsy.tokens == rsy.tokens == ar.tokens
        # sync-SD is deterministic in positions: the whole event sequence matches the reference's
        key = lambda t: [(e.actor, e.kind, e.pos_lo, e.pos_hi, e.draft_accepted) for e in t.events]
        assert key(gsy.trace) == key(rsy.trace), rho
        gas = P.decode_speculative_async(gdraft, v, prompt, cfg)
        assert gas.tokens == ar.tokens and gas.finished_by == ar.finished_by
        gas.trace.validate()
        # AMUSD correction positions == canonical disagreement positions (within the verified span)
        corr = sorted(e.pos_hi for e in gas.trace.events if e.kind == "verify_correct")
        verified = max(e.pos_hi for e in gas.trace.events if e.kind.startswith("verify_"))
        _, dis = O.canonical_disagreements(_Cpu(rdraft), _Cpu(verify), prompt, verified - len(prompt))
        assert corr == [len(prompt) + i for i in dis], rho


class _Cpu:
    """MockModel -> the oracle's start/predict/extend names (canonical_disagreements)."""

    def __init__(self, m):
        self.m = m

    def start(self, prompt):
        return self.m.init_state(prompt)

    def predict(self, st):
        return self.m.next_token(st)

    def extend(self, st, toks):
        self.m.advance(st, toks)


def test_reference_engines_drive_cuda_models(cfg1_pair):
    """the unmodified reference engines with the CUDA plug-ins."""
    S = _ref()
    d, v, _, _ = cfg1_pair
    prompt = PROMPT32[:20]
    n = 40
    ours = P.decode_autoregressive(v, prompt, P.DecodeConfig(max_new_tokens=n)).tokens
    cfg = S.DecodeConfig(max_new_tokens=n, draft_window_k=4)
    # MockModel path: the reference engines call next_token/advance/rollback/verify_tokens
    assert S.decode_autoregressive(v, prompt, cfg).tokens == ours
    assert S.decode_speculative_sync(d, v, prompt, cfg).tokens == ours
    # executor plug-in: the reference's decode_speculative_async with the device executor
    res = S.decode_speculative_async(P.AgreementDraft(d, 0.8), v, prompt, cfg, executor=P.CudaAsyncExecutor())
    assert res.tokens == ours
    res.trace.validate()
    assert res.stats.generated_tokens == n


def test_scripted_eos_goldens_on_device(golden):
    """eos at the first generated position / inside a verify window (the reference's goldens)."""
    for c in golden("engines")["scripted"]:
        v = P.ScriptedModel(c["script_verify"], 100, 99, eos_position=c["eos_position"], max_seq=128)
        d = P.ScriptedModel(c["script_draft"], 100, 99, max_seq=128)
        cfg = P.DecodeConfig(max_new_tokens=c["n"], draft_window_k=c["k"])
        ar = P.decode_autoregressive(v, c["prompt"], cfg)
        assert ar.tokens == c["ar_tokens"] and ar.finished_by == c["ar_finished_by"], c
        assert P.decode_speculative_sync(d, v, c["prompt"], cfg).tokens == c["sync_tokens"]
        for lead in (None, 1, 4):
            res = P.decode_speculative_async(d, v, c["prompt"], P.DecodeConfig(c["n"], c["k"], lead))
            assert res.tokens == c["async_tokens"] and res.finished_by == c["async_finished_by"], (c, lead)
            res.trace.validate()


def test_scripted_model_matches_reference_predictions():
    S = _ref()
    ref = S.ScriptedModel([4, 9, 1, 7], vocab_size=50, eos_token=3, eos_position=9)
    dev = P.ScriptedModel([4, 9, 1, 7], 50, 3, eos_position=9, max_seq=64)
    for prefix in ([1], [1, 2], [5, 5, 5, 5, 5, 5, 5], [1, 2, 3, 4, 5, 6, 7, 8], [2] * 12):
        assert dev.next_token(dev.init_state(prefix)) == ref.next_token(ref.init_state(prefix)), prefix
    st, rs = dev.init_state([1, 2]), ref.init_state([1, 2])
    cands = [6, 6, 6, 6, 6, 6, 6, 6, 6]
    assert dev.verify_tokens(st, cands) == ref.verify_tokens(rs, cands)


def test_release_row_major_keeps_results():
    """keep_row_major=False frees the row-major copy: same tokens, regenerated host weights, persistent only."""
    TC = P.TransformerConfig
    cfg = TC.llama_1b(max_seq=96, n_layers=2)
    a = P.TransformerModel(cfg, seed=9)
    b = P.TransformerModel(cfg, seed=9, keep_row_major=False)
    assert "layers.0.wqkv" not in b.weights
    conf = P.DecodeConfig(max_new_tokens=12)
    assert P.decode_autoregressive(a, PROMPT32, conf).tokens == P.decode_autoregressive(b, PROMPT32, conf).tokens
    wa, wb = a.host_weights(), b.host_weights()
    assert all(np.array_equal(wa[k], wb[k]) for k in wa)
    with pytest.raises(P.SpecDecError):
        b.set_path("simt")
    del a, b
    P.engines.clear_sessions()


def test_draft_equal_verify_rejected(cfg1_pair):
    _, v, _, _ = cfg1_pair
    with pytest.raises(P.InvalidInputError):
        P.decode_speculative_sync(v, v, PROMPT32[:8], P.DecodeConfig(max_new_tokens=4))
