"""Tensor-parallel restatement of the numpy decoder -- TEST INFRASTRUCTURE ONLY.

The Megatron-style sharding of paper_2410_17375_b200/tp.py (QKV column-parallel
over whole KV groups, O row-parallel, gate/up column-parallel, down
row-parallel, LM head vocab-parallel, replicated residual) written over
``RefDecoder``'s arithmetic with EXPLICIT collectives: ``allreduce`` after O
and after down (2 per layer), ``allgather`` of the LM-head slices.  Run under
torch.distributed (gloo) by tests/test_tp_cpu.py, it checks that the shard
layout is a faithful factorisation of the unsharded forward (logits equal up to
fp32 summation order) -- the GPU's fused peer-memory reduction is then checked
bit-exactly against the unsharded GPU forward (tests/test_gpu_tp.py).
"""
from __future__ import annotations

import numpy as np

from .ref_decoder import RefDecoder


def tp_logits(dec: RefDecoder, spec, toks, allreduce, allgather) -> np.ndarray:
    """Full-vocabulary logits [m, vocab] of `toks` (positions 0..m-1, empty cache) computed by
    rank spec.rank's shard; `allreduce(x) -> sum over ranks`, `allgather(x) -> list by rank`."""
    s, w = dec.s, dec.w
    m = len(toks)
    pos = np.arange(m)
    H, KV, hd = s.heads, s.kv_heads, s.head_dim
    G = H // KV
    hl, kl = (spec.kv1 - spec.kv0) * G, spec.kv1 - spec.kv0
    h = w["embed"][np.asarray(toks)].astype(np.float32)
    for l in range(s.layers):
        p = f"layers.{l}."
        W = w[p + "wqkv"]
        wq = W[spec.kv0 * G * hd: spec.kv1 * G * hd]
        wk = W[H * hd + spec.kv0 * hd: H * hd + spec.kv1 * hd]
        wv = W[(H + KV) * hd + spec.kv0 * hd: (H + KV) * hd + spec.kv1 * hd]
        qkv = dec._normed_matmul(h, w[p + "attn_norm"], np.concatenate([wq, wk, wv]))
        q = dec._rope(qkv[:, : hl * hd].reshape(m, hl, hd), pos)
        k = dec._cast_kv(dec._rope(qkv[:, hl * hd:(hl + kl) * hd].reshape(m, kl, hd), pos))
        v = dec._cast_kv(qkv[:, (hl + kl) * hd:].reshape(m, kl, hd))
        scale = np.float32(1.0 / np.sqrt(np.float32(hd)))
        out = np.empty((m, hl, hd), dtype=np.float32)
        mask = np.arange(m)[None, :] > pos[:, None]
        for hh in range(hl):
            g = hh // G
            sc = (q[:, hh, :] @ k[:, g, :].T) * scale
            sc = np.where(mask, -np.inf, sc)
            sc = np.exp(sc - sc.max(axis=1, keepdims=True))
            sc = sc / sc.sum(axis=1, keepdims=True)
            out[:, hh, :] = sc @ v[:, g, :]
        wo = w[p + "wo"][:, spec.kv0 * G * hd: spec.kv1 * G * hd]
        h = h + allreduce(dec._mm(dec._act(out.reshape(m, hl * hd)), wo))            # allreduce 1
        x = dec._act(h * w[p + "mlp_norm"][None, :])
        inv = (1.0 / np.sqrt((h * h).mean(axis=1, keepdims=True) + np.float32(s.eps))).astype(np.float32)
        gg = dec._mm(x, w[p + "wgate"][spec.f0: spec.f1]) * inv
        uu = dec._mm(x, w[p + "wup"][spec.f0: spec.f1]) * inv
        a = dec._act((gg / (1.0 + np.exp(-gg))) * uu)
        h = h + allreduce(dec._mm(a, w[p + "wdown"][:, spec.f0: spec.f1]))           # allreduce 2
    local = dec._normed_matmul(h, w["final_norm"], dec.lm[spec.v0: spec.v1])
    return np.concatenate(allgather(local), axis=1)
