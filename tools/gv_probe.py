"""Time the persistent forwards of the bench models in isolation (CUDA events): the SIMT decode
forward (decode_gv.cu) vs the tcgen05 work-queue forward (forward_tc.cu), per grid and rows.

    python tools/gv_probe.py [--models 1b,8b] [--grids 148,64] [--rows 1,2,4]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="1b")
    ap.add_argument("--grids", default="0,64")
    ap.add_argument("--rows", default="1,2")
    ap.add_argument("--paths", default="decode,persistent")
    ap.add_argument("--ctx", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2410_17375_b200 as P
    from paper_2410_17375_b200 import _lib as L
    lib = L.load()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    TC = P.TransformerConfig
    for name in args.models.split(","):
        cfg = {"1b": TC.llama_1b, "8b": TC.llama_8b}[name](max_seq=max(1024, args.ctx + 64))
        m = P.TransformerModel(cfg, seed=1)
        prompt = [(7 * i + 3) % 31000 + 3 for i in range(args.ctx)]
        for path in args.paths.split(","):
            m.set_path(path)
            st = m.init_state(prompt)
            m.next_token(st)
            for g in [int(x) for x in args.grids.split(",")]:
                L.check(lib.amusd_model_set_grid(m.handle, g))
                for rows in [int(x) for x in args.rows.split(",")]:
                    ms = C.c_float()
                    L.check(lib.amusd_time_forward(m.handle, rows, -1, 0, args.iters, C.byref(ms),
                                                   torch.cuda.current_stream().cuda_stream))
                    b = cfg.step_weight_bytes() + cfg.kv_bytes_per_token() * (args.ctx + rows)
                    gbs = b / ms.value / 1e6
                    print(json.dumps({"model": name, "path": path, "grid": g or "all", "rows": rows,
                                      "ms": round(ms.value, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)}),
                          flush=True)
            L.check(lib.amusd_model_set_grid(m.handle, 0))
        del m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
