"""One model, a few eager persistent forwards (ncu target).

  python tools/fw_one.py [--model 8b|1b] [--layers N] [--rows R] [--iters K] [--path persistent] [--grid SMS]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402
from paper_2410_17375_b200.models import device_stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="8b")
ap.add_argument("--layers", type=int, default=0)
ap.add_argument("--rows", type=int, default=1)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--pos", type=int, default=300)
ap.add_argument("--path", default="persistent")
ap.add_argument("--grid", type=int, default=0, help="SMs of the persistent launch (0 = all)")
a = ap.parse_args()
TC = P.TransformerConfig
kw = {"max_seq": max(640, a.pos + 64)}
if a.layers:
    kw["n_layers"] = a.layers
cfg = TC.llama_8b(**kw) if a.model == "8b" else TC.llama_1b(**kw)
m = P.TransformerModel(cfg, seed=3)
m.set_path(a.path)
m.init_state([(1234 * (i + 7)) % 31990 + 3 for i in range(a.pos)])
ms = C.c_float()
L.check(L.load().amusd_model_set_grid(m.handle, a.grid))
L.check(L.load().amusd_time_forward(m.handle, a.rows, -1, 0, a.iters, C.byref(ms), device_stream(m.device)))
gb = cfg.step_weight_bytes() / 1e9
print(f"{a.model} L={cfg.n_layers} rows={a.rows} {ms.value:.4f} ms  {gb / ms.value * 1e3:.1f} GB/s")
