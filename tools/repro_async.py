"""Repro harness: tiny bf16 pair through AMUSD (async) at several leads (debugging aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_17375_b200 as P  # noqa: E402

PROMPT = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]
TC = P.TransformerConfig
v = P.TransformerModel(TC.tiny_verify(dtype="bf16", max_seq=320), seed=1)
d = P.TransformerModel(TC.tiny_draft(dtype="bf16", max_seq=320), seed=2)
cfg = P.DecodeConfig(max_new_tokens=96)
ar = P.decode_autoregressive(v, PROMPT, cfg)
for rho in [None, 0.8, 0.95]:
    draft = d if rho is None else P.AgreementDraft(d, rho)
    for lead in (None, 2, 8):
        res = P.decode_speculative_async(draft, v, PROMPT, P.DecodeConfig(max_new_tokens=96, max_draft_lead=lead))
        print(rho, lead, res.tokens == ar.tokens, flush=True)
