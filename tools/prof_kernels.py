"""Per-kernel eager timings (CUDA events) of the draft and verify forwards, plus
graph-loop vs eager step time.  Debug/perf aid; prints a table."""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402

lib = L.load()
TC = P.TransformerConfig
ms = 32 + 512 + 64
v = P.TransformerModel(TC.llama_8b(max_seq=ms), seed=0)
d = P.TransformerModel(TC.llama_1b(max_seq=ms), seed=1)
prompt = list(range(100, 132))
v.init_state(prompt)
d.init_state(prompt)


def t(m, rows, which, layer=0, iters=20):
    out = C.c_float()
    L.check(lib.amusd_time_forward(m.handle, rows, which, layer, iters, C.byref(out), torch.cuda.current_stream().cuda_stream))
    return out.value * 1000.0  # us


def table(m, rows, names, nbytes):
    c = m.config
    tot = 0.0
    print(f"--- {c.n_layers}L d={c.d_model} rows={rows}")
    for k, name in enumerate(names):
        us = t(m, rows, k, layer=c.n_layers // 2)
        b = nbytes(k)
        mult = c.n_layers if k < 5 else 1
        tot += us * mult
        print(f"  {name:12s} {us:8.2f} us  x{mult:3d}  {b/us/1e3 if b else 0:8.1f} GB/s  bytes={b}")
    full = t(m, rows, -1, iters=5)
    print(f"  sum-of-kernels {tot/1000:.3f} ms   whole forward {full/1000:.3f} ms   weights {c.step_weight_bytes()/1e9:.3f} GB -> {c.step_weight_bytes()/full/1e3:.0f} GB/s")


for m in (v, d):
    c = m.config
    e = c.elem_bytes
    qkv = c.qkv_rows * c.d_model * e
    o = c.d_model * c.n_heads * c.head_dim * e
    gu = 2 * c.ffn * c.d_model * e
    dn = c.ffn * c.d_model * e
    lm = c.vocab_size * c.d_model * e
    simt = ["qkv", "attention", "o", "gate_up", "down", "lm_head", "argmax"]
    table(m, 1, simt, lambda k: [qkv, 0, o, gu, dn, lm, 0][k])
    tcn = ["qkv", "attention", "o", "gate_up", "down", "lm_head", "argmax"]
    table(m, 4, tcn, lambda k: [qkv, 0, o, gu, dn, lm, 0][k])

# graph loop vs eager: AR decode of 64 tokens
cfg = P.DecodeConfig(max_new_tokens=64)
for name, m in (("verify", v), ("draft", d)):
    r = P.decode_autoregressive(m, prompt, cfg)
    r = P.decode_autoregressive(m, prompt, cfg)
    s = P.engines._session(None, m, len(prompt), cfg)
    s.prepare(prompt)
    st, en = s.launch(L.ENGINE_AR)
    out = s.collect(st, en)
    print(f"AR graph loop {name}: {out.device_ms/64:.3f} ms/token  (PDL={'off' if os.environ.get('AMUSD_NO_PDL') else 'on'})")
