"""One eager verify forward (16-row tcgen05 path) and one eager draft forward
(2-row SIMT path) of the benchmark models, for ncu launch lists / captures
(kernels inside CUDA graphs with conditional nodes cannot be profiled)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402

TC = P.TransformerConfig
v = P.TransformerModel(TC.llama_8b(max_seq=608), seed=0)
d = P.TransformerModel(TC.llama_1b(max_seq=608), seed=1)
lib = L.load()
ms = C.c_float()
st = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("forwards")
L.check(lib.amusd_time_forward(v.handle, 4, -1, 0, 1, C.byref(ms), st))  # warm-up + 1 timed verify forward
L.check(lib.amusd_time_forward(d.handle, 1, -1, 0, 1, C.byref(ms), st))  # warm-up + 1 timed draft forward
torch.cuda.synchronize()
print("ok")
