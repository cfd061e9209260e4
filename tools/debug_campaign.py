"""Run a slice of the golden campaign on the GPU and report every mismatch (debug aid)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_17375_b200 as P  # noqa: E402
from oracle import specdec_oracle as O  # noqa: E402

g = json.loads((Path(__file__).resolve().parents[1] / "tests/golden/campaign.json").read_text())
col = {k: i for i, k in enumerate(g["columns"])}
lo, hi = int(sys.argv[1]), int(sys.argv[2])
isolate = "--isolate" in sys.argv
bad = 0
for idx in range(lo, hi):
    r = g["rows"][idx]
    seed, rho, vocab, excl = int(r[col["seed"]]), r[col["rho"]], r[col["vocab"]], bool(r[col["exclude_eos"]])
    prompt, n, k, lead = r[col["prompt"]], r[col["n"]], r[col["k"]], r[col["lead"]]
    d, v = P.make_agreement_pair(seed, rho, vocab, 0, exclude_eos=excl, max_seq=len(prompt) + n + 64)
    cfg = P.DecodeConfig(max_new_tokens=n, draft_window_k=k, max_draft_lead=lead)
    ar = P.decode_autoregressive(v, prompt, cfg)
    res = {"ar": ar.tokens}
    if "--all" in sys.argv:
        res["sync"] = P.decode_speculative_sync(d, v, prompt, cfg).tokens
        res["async"] = P.decode_speculative_async(d, v, prompt, cfg).tokens
    for name, toks in res.items():
        if toks != r[col["tokens"]]:
            bad += 1
            print(f"idx {idx} {name} MISMATCH P={len(prompt)} n={n} k={k} lead={lead} excl={excl} vocab={vocab} "
                  f"rho={rho} dev={toks[:6]} ref={r[col['tokens']][:6]} len={len(toks)}/{len(r[col['tokens']])}", flush=True)
    if isolate or (idx % 64 == 63 and "--clear64" in sys.argv):
        P.engines.clear_sessions()
print("bad", bad, "of", hi - lo)
