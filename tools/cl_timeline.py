"""Per-layer timeline of the cluster decode forward (decode_cl.cu): CTA 0 (a group cluster)
and the median over all CTAs of each mark, relative to the layer's phase-A start.

    python tools/cl_timeline.py [--ctx 32] [--rows 1] [--grid 0]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
MARKS = ["A.start", "x ready", "QKV done", "handoff1", "attention", "merge", "A.end(O)", "B.start", "x ready",
         "GU+act", "down", "-"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32)
    ap.add_argument("--rows", type=int, default=1)
    ap.add_argument("--grid", type=int, default=0)
    args = ap.parse_args()
    import torch
    import paper_2410_17375_b200 as P
    from paper_2410_17375_b200 import _lib as L
    lib = L.load()
    cfg = P.TransformerConfig.llama_1b(max_seq=max(1024, args.ctx + 64))
    m = P.TransformerModel(cfg, seed=1)
    m.set_path("cluster")
    m.init_state([(7 * i + 3) % 31000 + 3 for i in range(args.ctx)])
    nl = cfg.n_layers
    buf = torch.zeros(256 * 12 * nl, dtype=torch.int64, device="cuda")
    L.check(lib.amusd_model_set_timeline(m.handle, C.c_void_p(buf.data_ptr()), buf.numel() * 8))
    L.check(lib.amusd_model_set_grid(m.handle, args.grid))
    ms = C.c_float()
    L.check(lib.amusd_time_forward(m.handle, args.rows, -1, 0, 3, C.byref(ms), torch.cuda.current_stream().cuda_stream))
    L.check(lib.amusd_model_set_timeline(m.handle, None, 0))
    t = buf.view(256, nl, 12).cpu().numpy()
    G = int((t[:, 0, 0] != 0).sum())
    t = t[:G]
    print(f"forward {ms.value * 1000:.1f} us, grid {G}, rows {args.rows}")
    for l in (1, nl // 2):
        base = t[:, l, 0].min()
        cta0 = [(t[0, l, k] - base) / 1e3 if t[0, l, k] else float("nan") for k in range(11)]
        med = [np.median((t[:, l, k] - base)[t[:, l, k] > 0]) / 1e3 if (t[:, l, k] > 0).any() else float("nan")
               for k in range(11)]
        print(f"layer {l}:")
        for k in range(11):
            print(f"   {MARKS[k]:10s} cta0 {cta0[k]:7.2f} us   median {med[k]:7.2f} us")
    lay = [(t[:, l + 1, 0].min() - t[:, l, 0].min()) / 1e3 for l in range(nl - 1)]
    print(f"per layer {np.median(lay):.2f} us")


if __name__ == "__main__":
    main()
