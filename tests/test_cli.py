"""CLI mirror of the reference `specdec` command (cli.py:72-472) on the CUDA engines."""
import json

import pytest

from paper_2410_17375_b200 import cli
from paper_2410_17375_b200.errors import ConfigError


@pytest.mark.parametrize("data,needle", [
    ({"bogus": 1}, "unknown top-level key 'bogus'"),
    ({"model": {"kind": "nope"}}, "model.kind"),
    ({"model": {"colour": 1}}, "unknown key 'model.colour'"),
    ({"model": {"vocab_size": 1}}, "model.vocab_size"),
    ({"model": {"eos_token": 40000}}, "model.eos_token"),
    ({"model": {"rho": 1.5}}, "model.rho"),
    ({"model": {"kind": "transformer", "shapes": "70b"}}, "model.shapes"),
    ({"decode": {"max_new_tokens": 0}}, "decode.max_new_tokens"),
    ({"decode": {"max_draft_lead": 0}}, "decode.max_draft_lead"),
    ({"execution": {"backend": "simulate"}}, "simulate"),
    ({"execution": {"strategies": ["fastest"]}}, "execution.strategies"),
    ({"execution": {"trials": 0}}, "execution.trials"),
    ({"prompt": []}, "prompt"),
    ({"latency": {"draft_ms": 1}}, "latency"),
])
def test_config_errors_name_the_field(data, needle):
    with pytest.raises(ConfigError) as e:
        cli.parse_config(data)
    assert needle in str(e.value)


def test_defaults_and_overrides(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"model": {"kind": "transformer"}, "execution": {"backend": "concurrent"}}))
    cfg = cli.load_config(p)
    assert cfg.model.kind == "transformer" and cfg.execution.strategies == cli.ENGINE_KINDS
    args = cli._parser().parse_args(["run", str(p), "--seed", "7", "--out-dir", str(tmp_path / "o")])
    cfg = cli._overrides(cfg, args)
    assert cfg.model.seed == 7 and cfg.execution.out_dir.endswith("o")
    assert cli.main(["run", str(tmp_path / "missing.json")]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["agreement_pair", "transformer"])
def test_compare_run_trace_on_gpu(tmp_path, capsys, kind):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = {"prompt": [5, 6, 7, 8, 9], "model": {"kind": kind, "seed": 3, "exclude_eos": True, "rho": 0.8},
           "decode": {"max_new_tokens": 40}, "execution": {"out_dir": str(tmp_path), "trials": 2}}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(cfg))
    assert cli.main(["compare", str(p)]) == 0      # output-equality gate (cli.py:377-385) passes
    table = json.loads((tmp_path / "compare.json").read_text())
    assert table["baseline"] == "autoregressive" and len(table["rows"]) == 3
    assert cli.main(["run", str(p)]) == 0
    toks = {s: json.loads((tmp_path / f"{s}-t0" / "tokens.json").read_text())["tokens"] for s in cli.ENGINE_KINDS}
    assert toks["sync_speculative"] == toks["autoregressive"] == toks["async_speculative"]
    stats = json.loads((tmp_path / "async_speculative-t0" / "stats.json").read_text())
    assert stats["generated_tokens"] == 40
    capsys.readouterr()
    assert cli.main(["trace", str(p), "async_speculative-t0"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "t_ms,verified_tokens" and lines[-1].endswith(",40")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["agreement_pair", "agreement_pair_rho09_k6", "hash_chain", "scripted_eos"])
def test_artifacts_match_reference_cli(tmp_path, case):
    """The CUDA CLI's artifacts against the UNMODIFIED reference CLI's on the same config
    (tests/golden/cli.json, oracle/make_cli_golden.py): tokens.json verbatim, the stats.json
    schema, every timing-independent statistic, the trace.csv header and (AR / sync-SD) the
    per-kind event counts."""
    import csv
    import io
    from pathlib import Path
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    gold = json.loads((Path(__file__).parent / "golden" / "cli.json").read_text())
    g = gold["cases"][case]
    cfg = json.loads(json.dumps(g["config"]))
    if cfg["model"].get("script_path") == "@SCRIPT":
        (tmp_path / "script.json").write_text(json.dumps(gold["script"]))
        cfg["model"]["script_path"] = str(tmp_path / "script.json")
    cfg["execution"] = {"backend": "cuda", "out_dir": str(tmp_path / "out")}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(cfg))
    assert cli.main(["run", str(p)]) == 0
    for strat, ref in g["runs"].items():
        d = tmp_path / "out" / f"{strat}-t0"
        assert json.loads((d / "tokens.json").read_text()) == ref["tokens_json"], strat
        stats = json.loads((d / "stats.json").read_text())
        assert sorted(stats) == ref["stats_keys"]
        assert {k: stats[k] for k in ref["stats"]} == ref["stats"], strat
        rows = list(csv.reader(io.StringIO((d / "trace.csv").read_text())))
        assert rows[0] == ref["trace_header"]
        if ref["trace_kinds"] is not None:
            kinds = {}
            for r in rows[1:]:
                kinds[r[2]] = kinds.get(r[2], 0) + 1
            assert kinds == ref["trace_kinds"], strat
