"""Co-location probe: the 8B verify and 1B draft persistent forwards, each alone
on its SM share and both at once on disjoint SM sets (two streams, two host threads).

  python tools/colo_probe.py [--draft-sms 56] [--rows 3] [--iters 20]
"""
import argparse
import ctypes as C
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--draft-sms", type=int, default=56)
ap.add_argument("--rows", type=int, default=3)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--pos", type=int, default=300)
a = ap.parse_args()
lib = L.load()
TC = P.TransformerConfig
prompt = [(1234 * (i + 7)) % 31990 + 3 for i in range(a.pos)]
ver = P.TransformerModel(TC.llama_8b(max_seq=640), seed=3)
dra = P.TransformerModel(TC.llama_1b(max_seq=640), seed=4)
ver.init_state(prompt)
dra.init_state(prompt)
sms = torch.cuda.get_device_properties(0).multi_processor_count
sv, sd = torch.cuda.Stream(), torch.cuda.Stream()


def timed(m, rows, iters, st, out, key):
    ms = C.c_float()
    L.check(lib.amusd_time_forward(m.handle, rows, -1, 0, iters, C.byref(ms), C.c_void_p(st.cuda_stream)))
    out[key] = ms.value


for grid_v, grid_d in ((0, 0), (sms - a.draft_sms, a.draft_sms)):
    L.check(lib.amusd_model_set_grid(ver.handle, grid_v))
    L.check(lib.amusd_model_set_grid(dra.handle, grid_d))
    r = {}
    timed(ver, a.rows, a.iters, sv, r, "v")
    timed(dra, 1, a.iters * 3, sd, r, "d")
    print(f"alone   verify({grid_v or sms} SMs, {a.rows} rows) {r['v']:.3f} ms   draft({grid_d or sms} SMs) {r['d']:.3f} ms")
L.check(lib.amusd_model_set_grid(ver.handle, sms - a.draft_sms))
L.check(lib.amusd_model_set_grid(dra.handle, a.draft_sms))
r = {}
th = [threading.Thread(target=timed, args=(ver, a.rows, a.iters, sv, r, "v")),
      threading.Thread(target=timed, args=(dra, 1, a.iters * 4, sd, r, "d"))]
for t in th:
    t.start()
for t in th:
    t.join()
vb, db = ver.config.step_weight_bytes(), dra.config.step_weight_bytes()
print(f"concurrent verify {r['v']:.3f} ms  draft {r['d']:.3f} ms  "
      f"(HBM {vb / r['v'] / 1e6 + db / r['d'] / 1e6:.0f} GB/s combined while both run)")
