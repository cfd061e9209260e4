"""Golden CLI artifacts from the UNMODIFIED reference command line -- TEST INFRASTRUCTURE.

Runs the reference ``specdec run`` (pkg/src/specdec/cli.py:328-359, backend
"concurrent": the real engines with ThreadExecutor) on model configs the CUDA
CLI also supports, and records what a drop-in must reproduce:

* ``tokens.json`` verbatim (tokens, finished_by, prompt_length);
* the ``stats.json`` key set, and the timing-independent stats: for AR and
  sync-SD every count; for AMUSD generated_tokens and rollbacks (== the
  canonical disagreements);
* the ``trace.csv`` header and the per-kind event counts of the deterministic
  engines.

Run here (the reference is importable in this container):
    python oracle/make_cli_golden.py [--ref /root/reference/pkg/src]
-> tests/golden/cli.json, checked by tests/test_cli.py on the GPU.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "tests" / "golden" / "cli.json"

SCRIPT = [7, 9, 11, 13, 5, 17, 19, 23, 29, 31, 37]
CASES = {
    "agreement_pair": {"prompt": [5, 6, 7, 8, 9], "model": {"kind": "agreement_pair", "seed": 3, "rho": 0.8,
                                                            "exclude_eos": True},
                       "decode": {"max_new_tokens": 40}},
    "agreement_pair_rho09_k6": {"prompt": [1, 2, 3, 4], "model": {"kind": "agreement_pair", "seed": 11, "rho": 0.9,
                                                                  "exclude_eos": True},
                                "decode": {"max_new_tokens": 64, "draft_window_k": 6}},
    "hash_chain": {"prompt": [2, 4, 6], "model": {"kind": "hash_chain", "seed": 42, "vocab_size": 101},
                   "decode": {"max_new_tokens": 30}},
    "scripted_eos": {"prompt": [1, 2, 3], "model": {"kind": "scripted", "vocab_size": 64, "eos_token": 2,
                                                    "eos_position": 12, "script_path": "@SCRIPT"},
                     "decode": {"max_new_tokens": 40}},
}
DETERMINISTIC = ("generated_tokens", "verify_steps", "accepted_per_verify_step", "rollbacks", "drafted_tokens",
                 "wasted_draft_tokens")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    a = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, a.ref)
    from specdec import cli as ref_cli  # the unmodified reference CLI
    out = {"script": SCRIPT, "cases": {}}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        (tmp / "script.json").write_text(json.dumps(SCRIPT))
        for name, cfg in CASES.items():
            cfg = json.loads(json.dumps(cfg).replace('"@SCRIPT"', json.dumps(str(tmp / "script.json"))))
            cfg["execution"] = {"backend": "concurrent", "out_dir": str(tmp / name)}
            p = tmp / f"{name}.json"
            p.write_text(json.dumps(cfg))
            assert ref_cli.main(["run", str(p)]) == 0, name
            case = {"config": CASES[name], "runs": {}}
            for strat in ("autoregressive", "sync_speculative", "async_speculative"):
                d = tmp / name / f"{strat}-t0"
                stats = json.loads((d / "stats.json").read_text())
                rows = list(csv.reader(io.StringIO((d / "trace.csv").read_text())))
                keep = DETERMINISTIC if strat != "async_speculative" else ("generated_tokens", "rollbacks")
                kinds = {}
                for r in rows[1:]:
                    kinds[r[2]] = kinds.get(r[2], 0) + 1
                case["runs"][strat] = {
                    "tokens_json": json.loads((d / "tokens.json").read_text()),
                    "stats_keys": sorted(stats),
                    "stats": {k: stats[k] for k in keep},
                    "trace_header": rows[0],
                    "trace_kinds": kinds if strat != "async_speculative" else None,
                }
            out["cases"][name] = case
    OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
