"""CPU-only checks: the C-ABI library loads and exports every declared entry
point; host-side schema logic; the numpy decoder oracle is self-consistent."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    from paper_2410_17375_b200 import _lib as L
    lib = L.load()
    header = (ROOT / "include" / "amusd.h").read_text()
    names = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(amusd_\w+)\s*\(", header, re.M))
    assert len(names) >= 25
    bound = {n for n, _, _ in L.SIGNATURES}
    assert names == bound, names ^ bound
    for n in names:
        assert hasattr(lib, n), n
    assert lib.amusd_abi_version() == 1


def test_status_codes_map_to_reference_errors():
    from paper_2410_17375_b200 import _lib as L
    from paper_2410_17375_b200.errors import (InvalidInputError, InvalidRollbackError,
                                              ProtocolViolationError, SpecDecError)
    assert L._STATUS[1] is InvalidInputError and L._STATUS[2] is InvalidRollbackError
    assert L._STATUS[3] is ProtocolViolationError and issubclass(L._STATUS[4], SpecDecError)
    assert issubclass(InvalidInputError, ValueError) and issubclass(ProtocolViolationError, RuntimeError)


def test_session_and_model_sizes():
    import ctypes as C
    from paper_2410_17375_b200 import _lib as L
    from paper_2410_17375_b200.models import TransformerConfig
    lib = L.load()
    d = L.SessionDesc(prompt_len=32, max_new_tokens=512, draft_window_k=4, max_window=16, trace_cap=64)
    assert lib.amusd_mailbox_capacity(C.byref(d)) >= 512 + 16
    assert lib.amusd_session_bytes(C.byref(d)) > 0
    c8 = TransformerConfig.llama_8b()
    assert abs(c8.step_weight_bytes() / 1e9 - 15.010) < 0.01
    c1 = TransformerConfig.llama_1b()
    assert abs(c1.step_weight_bytes() / 1e9 - 2.472) < 0.01
    assert c8.kv_bytes_per_token() == 128 * 1024 and c1.kv_bytes_per_token() == 32 * 1024


def test_device_trace_conversion_and_validation():
    from paper_2410_17375_b200.metrics import summarize, trace_from_device
    # draft: tokens at 5,6,7 ; verify corrects at window [5..6] -> publishes 5,6 ; draft acks
    draft = [(100, 10, 0, 5, 5, 0), (200, 10, 0, 6, 6, 0), (300, 10, 0, 7, 7, 0), (450, 5, 3, 6, 7, 0),
             (560, 10, 0, 7, 7, 0), (9000, 10, 0, 8, 8, 0)]
    verify = [(400, 150, 2, 5, 6, 1), (600, 50, 1, 7, 7, 1)]
    tr = trace_from_device(draft, verify, 4, 7)
    tr.validate()
    st = summarize(tr)
    assert st.generated_tokens == 3 and st.rollbacks == 1 and st.verify_steps == 2
    assert st.wasted_draft_tokens == 2
    assert tr.events[-1].kind == "complete"
    assert all(e.t_ms <= tr.events[-1].t_ms for e in tr.events)
    assert st.drafted_tokens == 4  # the post-completion draft event was dropped


def test_oracle_decoder_self_consistency():
    from oracle.ref_decoder import RefDecoder, TfShape, uniform_weights_like
    from paper_2410_17375_b200.models import TransformerConfig, weight_names, weight_shape
    cfg = TransformerConfig.tiny_draft(vocab_size=512, max_seq=64)
    shapes = {n: weight_shape(cfg, n) for n in weight_names(cfg)}
    w = uniform_weights_like(shapes, seed=3)
    m = RefDecoder(TfShape(512, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn),
                   w, tied=True)
    st = m.start([5, 6, 7])
    cands = [9, 10, 11, 12]
    got = m.verify(st, cands)
    seq = m.start([5, 6, 7])
    exp = []
    for c in cands:
        exp.append(m.predict(seq))
        m.extend(seq, [c])
    assert got == exp and st.tokens == [5, 6, 7]
    m.extend(st, [1, 2, 3])
    m.crop(st, 4)
    m.extend(st, [8])
    fresh = m.start([5, 6, 7, 1, 8])
    assert m.predict(st) == m.predict(fresh)
    assert np.allclose(st.last_logits, fresh.last_logits, atol=1e-5)
