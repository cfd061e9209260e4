"""Time whole forwards of the 1B/8B-shaped models per path (persistent vs per-kernel).

  python tools/fw_bench.py [--paths persistent,kernels] [--rows 1,4,16] [--iters 20]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2410_17375_b200 as P  # noqa: E402
from paper_2410_17375_b200 import _lib as L  # noqa: E402
from paper_2410_17375_b200.models import device_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--paths", default="persistent,kernels")
    ap.add_argument("--rows", default="1,4,16")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--models", default="8b,1b")
    ap.add_argument("--pos", type=int, default=300)
    args = ap.parse_args()
    TC = P.TransformerConfig
    lib = L.load()
    out = {}
    prompt = [(1234 * (i + 7)) % 31990 + 3 for i in range(args.pos)]
    for name in args.models.split(","):
        cfg = TC.llama_8b(max_seq=640) if name == "8b" else TC.llama_1b(max_seq=640)
        m = P.TransformerModel(cfg, seed=3)
        m.init_state(prompt)
        gb = cfg.step_weight_bytes() / 1e9
        for path in args.paths.split(","):
            m.set_path(path)
            for rows in map(int, args.rows.split(",")):
                ms = C.c_float()
                L.check(lib.amusd_time_forward(m.handle, rows, -1, 0, args.iters, C.byref(ms), device_stream(m.device)))
                key = f"{name}/{path}/rows{rows}"
                out[key] = {"ms": round(ms.value, 4), "GB/s": round(gb / ms.value * 1e3, 1)}
                print(key, out[key], flush=True)
        del m
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
