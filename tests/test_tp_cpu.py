"""The tensor-parallel shard layout (paper_2410_17375_b200/tp.py shard_spec) as explicit
collectives over torch.distributed gloo, world sizes 2 and 7 (the 70B verify of BASELINE
config 4 uses 7 ranks): the sharded numpy decoder (oracle/ref_tp.py) reproduces the unsharded
decoder's logits up to fp32 summation order, and every rank sees the same argmax."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_17375_b200.models import TransformerConfig
from paper_2410_17375_b200.tp import shard_spec

# 8 KV heads (70B-like GQA), 7 ranks get 2+1+...+1 groups; ffn / vocab in whole 256 / 128 blocks
CFG = TransformerConfig(vocab_size=128 * 21, d_model=256, n_layers=2, n_heads=16, n_kv_heads=8, head_dim=32,
                        ffn=256 * 14, tied=False)


def _weights():
    from oracle.ref_decoder import bf16_round
    from paper_2410_17375_b200.models import weight_names, weight_shape
    rng = np.random.default_rng(7)
    w = {}
    for n in weight_names(CFG):
        shp = weight_shape(CFG, n)
        w[n] = np.ones(shp, np.float32) if n.endswith("norm") else bf16_round(rng.normal(0, 0.05, shp).astype(np.float32))
    return w


def _decoder():
    from oracle.ref_decoder import RefDecoder
    from oracle.ref_models import shape_of
    return RefDecoder(shape_of(CFG, kv_bf16=False), _weights(), tied=False)   # pure fp32: summation order only


def _worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from oracle.ref_tp import tp_logits
        dec = _decoder()
        toks = [(37 * i + 5) % CFG.vocab_size for i in range(12)]

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        def allgather(x):   # uneven vocab slices: object gather
            out = [None] * size
            dist.all_gather_object(out, np.ascontiguousarray(x))
            return out
        lg = tp_logits(dec, shard_spec(CFG, rank, size), toks, allreduce, allgather)
        from oracle.ref_decoder import DecState
        ref = dec.forward(DecState(len(toks), []), toks)
        err = float(np.abs(lg - ref).max() / ref.std())
        am = [int(x) for x in lg.argmax(axis=1)]
        q.put((rank, err, am, [int(x) for x in ref.argmax(axis=1)]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("size", [2, 7])
def test_tp_shards_equal_unsharded(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, am, ref_am in res:
        assert err < 1e-4, (rank, err)      # fp32 summation order only
        assert am == ref_am, rank
    assert len({tuple(r[2]) for r in res}) == 1   # every rank the same predictions


def test_shard_spec_covers_the_model():
    from paper_2410_17375_b200.models import TransformerConfig as TC
    for cfg, size in ((TC.llama_70b(), 7), (TC.llama_8b(), 2), (TC.llama_8b(), 4), (CFG, 7)):
        specs = [shard_spec(cfg, r, size) for r in range(size)]
        assert specs[0].kv0 == 0 and specs[-1].kv1 == cfg.n_kv_heads
        assert specs[0].f0 == 0 and specs[-1].f1 == cfg.ffn
        assert specs[0].v0 == 0 and specs[-1].v1 == cfg.vocab_size
        for a, b in zip(specs, specs[1:]):
            assert (a.kv1, a.f1, a.v1) == (b.kv0, b.f0, b.v0)
        assert all(s.kv1 > s.kv0 and s.f1 > s.f0 and s.v1 > s.v0 and s.v0 % 128 == 0 for s in specs)
