"""Eager launches of individual verify/draft kernels for ncu (graph kernels with
conditional nodes cannot be profiled).  Usage: python tools/ncu_target.py [rows] [which...]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
which = [int(x) for x in sys.argv[2:]] or [0, 2, 3, 4, 5]
model = P.TransformerModel(P.TransformerConfig.llama_8b(max_seq=640, n_layers=int(__import__("os").environ.get("NCU_LAYERS", "2"))), seed=0)
lib = L.load()
ms = C.c_float()
for w in which:
    L.check(lib.amusd_time_forward(model.handle, rows, w, 0, 1, C.byref(ms), torch.cuda.current_stream().cuda_stream))
    print(w, ms.value)
torch.cuda.synchronize()
