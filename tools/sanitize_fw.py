"""Tiny bf16 pair through the persistent forward, for compute-sanitizer
(memcheck / racecheck / synccheck): verify_tokens over 7 rows crossing a
128-position attention split, plus a short AMUSD decode."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_17375_b200 as P  # noqa: E402

TC = P.TransformerConfig
v = P.TransformerModel(TC.tiny_verify(dtype="bf16", max_seq=192), seed=5)
d = P.TransformerModel(TC.tiny_draft(dtype="bf16", max_seq=192), seed=6)
prompt = [(37 * i + 11) % 31000 + 3 for i in range(124)]
print(v.verify_tokens(v.init_state(prompt), [11, 22, 33, 44, 55, 66, 77]))
mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode == "all":
    res = P.decode_speculative_async(P.AgreementDraft(d, 0.8), v, prompt[:20], P.DecodeConfig(max_new_tokens=12))
    print(res.tokens)
