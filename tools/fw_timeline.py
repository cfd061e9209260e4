"""Record the per-item timeline of one persistent forward (perf analysis).

  python tools/fw_timeline.py [--model 8b] [--layers 8] [--rows 1] --out gpurun_out/tl.npy
Columns: item, cta, phase, t_grab, t_issued, t_dep, t_mma, t_done, t_waited, t_epi_done (ns, globaltimer).
Attention items: t_issued = scores done, t_waited = inputs gathered, t_epi_done = P.V done,
t_dep = QKV dependency seen, t_mma = item returned.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402
from paper_2410_17375_b200.models import device_stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="8b")
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--rows", type=int, default=1)
ap.add_argument("--pos", type=int, default=300)
ap.add_argument("--out", default="gpurun_out/tl.npy")
ap.add_argument("--grid", type=int, default=0, help="SMs of the persistent launch (0 = all)")
a = ap.parse_args()
TC = P.TransformerConfig
kw = {"max_seq": 640}
if a.layers:
    kw["n_layers"] = a.layers
cfg = TC.llama_8b(**kw) if a.model == "8b" else TC.llama_1b(**kw)
m = P.TransformerModel(cfg, seed=3)
m.init_state([(1234 * (i + 7)) % 31990 + 3 for i in range(a.pos)])
lib = L.load()
buf = torch.zeros(1 << 17, 8, dtype=torch.int64, device="cuda")
L.check(lib.amusd_model_set_timeline(m.handle, C.c_void_p(buf.data_ptr()), buf.numel() * 8))
ms = C.c_float()
L.check(lib.amusd_model_set_grid(m.handle, a.grid))
L.check(lib.amusd_time_forward(m.handle, a.rows, -1, 0, 3, C.byref(ms), device_stream(m.device)))
torch.cuda.synchronize()
t = buf.cpu().numpy()
n = int((t[:, 1] != 0).sum())
t = t[:n]
out = np.zeros((n, 10), dtype=np.int64)
out[:, 0] = t[:, 0] & 0xFFFFF
out[:, 1] = (t[:, 0] >> 20) & 0xFFF
out[:, 2] = t[:, 0] >> 32
out[:, 3:8] = t[:, 1:6]
out[:, 8:10] = t[:, 6:8]  # merger: count-wait done, final epilogue done (before publish)
np.save(a.out, out)
print(f"{n} items, forward {ms.value:.4f} ms (timed with the timeline on)")
