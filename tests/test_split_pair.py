"""Split pair (draft and verify on separate devices, BASELINE config 2).

* gloo, world_size 2, CPU: the host link (role assignment, object exchange,
  barrier) that carries the mailbox IPC handles, the canonical path, the clock
  samples and the trace rows between the two ranks.
* GPU: the split protocol itself -- two sessions, two mailbox copies, every
  field stored into the peer's copy -- emulated with both halves in one
  process on one GPU (only one GPU is available here); tokens == AR.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import specdec_oracle as O
import paper_2410_17375_b200 as P
from paper_2410_17375_b200.split import SplitLink, decode_speculative_async_split


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _link_worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        link = SplitLink()
        meta = {"role": link.role, "handle": bytes([rank]) * 64, "offset": 4096 * rank}
        peer = link.exchange(meta)
        link.barrier()
        canon = link.exchange([1, 2, 3, 4, 99] if link.role == "verify" else None)
        rows = link.exchange([(1000 + rank, 5, 0, 7, 7, 0)])
        q.put((rank, link.role, peer["role"], peer["handle"][:2], peer["offset"], canon, rows))
    finally:
        dist.destroy_process_group()


def test_split_link_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_link_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, role0, peer0, h0, off0, canon0, rows0), (r1, role1, peer1, h1, off1, canon1, rows1) = out
    assert (role0, peer0, role1, peer1) == ("draft", "verify", "verify", "draft")
    assert h0 == bytes([1, 1]) and off0 == 4096 and h1 == bytes([0, 0]) and off1 == 0
    assert canon0 == [1, 2, 3, 4, 99] and canon1 is None   # verify -> draft
    assert rows0 == [(1001, 5, 0, 7, 7, 0)] and rows1 == [(1000, 5, 0, 7, 7, 0)]


def test_split_link_requires_process_group():
    with pytest.raises(P.InvalidInputError):
        SplitLink()


@pytest.mark.gpu
def test_split_pair_emulated_hash_chain():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    for seed, rho in ((7, 0.8), (11, 0.5), (3, 1.0)):
        d, v = P.make_agreement_pair(seed, rho, 5000, 0, exclude_eos=True, max_seq=512)
        cfg = P.DecodeConfig(max_new_tokens=96)
        res, (dms, vms) = decode_speculative_async_split(d, [1, 2, 3, 4], cfg, verify=v)
        ref = O.decode_ar(O.ChainOracle(seed, 5000, 0, True), [1, 2, 3, 4], 96)[0]
        assert res.tokens == ref
        res.trace.validate()
        assert res.stats.generated_tokens == 96 and vms > 0
        # rollbacks == canonical disagreements (test_engines.py:293-321)
        od = O.ChainOracle(seed, 5000, 0, True, rho=rho) if rho < 1.0 else None
        if od is not None:
            verified = max(e.pos_hi for e in res.trace.events if e.kind.startswith("verify_")) - 4
            _, dis = O.canonical_disagreements(od, O.ChainOracle(seed, 5000, 0, True), [1, 2, 3, 4], verified)
            assert res.stats.rollbacks == len(dis)
    P.engines.clear_sessions()


@pytest.mark.gpu
def test_split_pair_emulated_transformer():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    TC = P.TransformerConfig
    v = P.TransformerModel(TC.tiny_verify(dtype="bf16", max_seq=192), seed=5)
    d = P.AgreementDraft(P.TransformerModel(TC.tiny_draft(dtype="bf16", max_seq=192), seed=6), 0.8)
    prompt = [(37 * i + 11) % 31000 + 3 for i in range(20)]
    cfg = P.DecodeConfig(max_new_tokens=64)
    ar = P.decode_autoregressive(v, prompt, cfg)
    res, _ = decode_speculative_async_split(d, prompt, cfg, verify=v)
    assert res.tokens == ar.tokens
    res.trace.validate()
    P.engines.clear_sessions()


@pytest.mark.gpu
def test_split_pair_two_processes_ipc():
    """The distributed path proper: two processes, mailbox copies exchanged as CUDA IPC
    handles (both on one GPU here; on two GPUs the peer stores go over NVLink)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "tools" / "split_check.py"), "48"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    out = {d["role"]: d for d in (json.loads(l) for l in r.stdout.splitlines() if l.startswith("{"))}
    assert out["draft"]["tokens"] == out["verify"]["tokens"] == out["verify"]["ar"] == out["draft"]["ar"]
    assert out["draft"]["rollbacks"] == out["verify"]["rollbacks"]
