import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2410_17375_b200 as P
TC = P.TransformerConfig
PROMPT = [(37 * i + 11) % 31000 + 3 for i in range(24)]
def run(fuse, shape, layers, plen, grid=0, **kw):
    os.environ["AMUSD_FW_FUSE"] = str(fuse)
    cfg = getattr(TC, shape)(max_seq=320, n_layers=layers, **kw)
    m = P.TransformerModel(cfg, seed=5)
    if grid:
        m.set_max_grid(grid)
    st = m.init_state((PROMPT * 12)[:plen])
    m.next_token(st)
    a = m.last_logits(1).numpy()[0]
    m.next_token(st)
    b = m.last_logits(1).numpy()[0]
    del m
    P.engines.clear_sessions()
    return a, b
for shape, kw in (("tiny_draft", dict(dtype="bf16")), ("llama_1b", {})):
    for layers in (2, 3):
        for grid in (1, 2, 16, 0):
            plen = 5
            a0, b0 = run(0, shape, layers, plen, grid, **kw)
            a1, b1 = run(1, shape, layers, plen, grid, **kw)
            print(shape, layers, plen, "grid", grid, "diff", float(np.abs(a1 - a0).max() / a0.std()), "std", float(a0.std()), float(a1.std()), flush=True)
