"""Eager forwards of the benchmark models for ncu (kernels inside CUDA graphs
with conditional nodes cannot be profiled): one AMUSD-like verify forward (4
rows) and one draft forward (1 row) through the persistent tcgen05 kernel,
each preceded by a warm-up launch.  `--steps N` instead replays N decode steps
eagerly (prefill + per step: verify forward, draft forward) so the launch list
shows the forward's share next to the prefill launches."""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--verify-rows", type=int, default=4)
ap.add_argument("--layers", type=int, default=0)
a = ap.parse_args()
TC = P.TransformerConfig
kw = {"max_seq": 608}
if a.layers:
    kw["n_layers"] = a.layers
v = P.TransformerModel(TC.llama_8b(**kw), seed=0)
d = P.TransformerModel(TC.llama_1b(**kw), seed=1)
prompt = [(1234 * (i + 7)) % 31990 + 3 for i in range(32)]
v.init_state(prompt)
d.init_state(prompt)
lib = L.load()
ms = C.c_float()
st = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
L.check(lib.amusd_time_forward(v.handle, a.verify_rows, -1, 0, 1, C.byref(ms), st))  # warm-up + 1 timed verify
L.check(lib.amusd_time_forward(d.handle, 1, -1, 0, 1, C.byref(ms), st))              # warm-up + 1 timed draft
torch.cuda.synchronize()
print("ok")
