"""Per-phase timeline of the persistent SIMT decode forward (decode_gv.cu): every CTA stamps
%globaltimer when it passes each grid barrier (phase start) and when it arrives at the next
(phase end).  Prints, per phase kind, the median over layers of: work (median / max over CTAs of
end - start) and the barrier gap (latest arrival of the previous phase -> median start).

    python tools/gv_timeline.py [--ctx 32] [--rows 1] [--grid 0]
"""
import argparse
import ctypes as C
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KINDS = ["qkv", "attn", "o", "gu", "down"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32)
    ap.add_argument("--rows", type=int, default=1)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--model", default="1b")
    args = ap.parse_args()
    import torch
    import paper_2410_17375_b200 as P
    from paper_2410_17375_b200 import _lib as L
    lib = L.load()
    TC = P.TransformerConfig
    cfg = {"1b": TC.llama_1b, "8b": TC.llama_8b}[args.model](max_seq=max(1024, args.ctx + 64))
    m = P.TransformerModel(cfg, seed=1)
    m.set_path("decode")
    prompt = [(7 * i + 3) % 31000 + 3 for i in range(args.ctx)]
    st = m.init_state(prompt)
    m.next_token(st)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    G = args.grid or sms
    nev = 2 * (5 * 128 + 1) + 2
    buf = torch.zeros(G * nev + G * 9 * 24, dtype=torch.int64, device="cuda")
    L.check(lib.amusd_model_set_timeline(m.handle, C.c_void_p(buf.data_ptr()), buf.numel() * 8))
    L.check(lib.amusd_model_set_grid(m.handle, args.grid))
    ms = C.c_float()
    L.check(lib.amusd_time_forward(m.handle, args.rows, -1, 0, 3, C.byref(ms), torch.cuda.current_stream().cuda_stream))
    L.check(lib.amusd_model_set_timeline(m.handle, None, 0))
    allb = buf.cpu().numpy().astype("int64")
    t = allb[:G * nev].reshape(G, nev)
    w = allb[G * nev:].reshape(G, 9, 6, 4)
    names = {0: "qkv", 1: "o", 2: "gu", 3: "down", 4: "lm"}
    for k in range(5):
        nb = w[:, :8, k, 0].sum()
        if nb:
            print(f"blocks {names[k]:5s}: {nb / G:7.1f} per CTA ({w[:, :8, k, 3].sum() / nb:.0f} units each); cycles per "
                  f"block: mma+waits {w[:, :8, k, 1].sum() / nb:8.0f}  epilogue {w[:, :8, k, 2].sum() / nb:8.0f}")
    for k in range(5):
        ph = w[:, 8, k, :]
        n = ph[:, 3].sum()
        if n:
            print(f"phase {names[k]:5s}: cycles per pass: start->x ready {ph[:, 0].sum() / n:7.0f}   blocks+epilogues {ph[:, 1].sum() / n:7.0f}")
    at = w[:, 0, 5, :]  # CTA warp-0 slot 5: attention marks (cycles from item start, summed)
    sel = at[at[:, 3] > 0]
    if len(sel):
        n = 16 * 4
        print("attention item (cycles from item start, mean over item CTAs / layers / launches): "
              f"inputs ready {sel[:, 0].mean() / n:.0f}, scores {sel[:, 1].mean() / n:.0f}, "
              f"softmax {sel[:, 2].mean() / n:.0f}, P.V+write {sel[:, 3].mean() / n:.0f}")
    nl = cfg.n_layers
    # events: [0] kernel start; then per phase p (5 per layer + LM): start (after the wait) and end
    # (arrive); layer-0 QKV has no wait: its start is event 0 (shared slot layout below)
    # event index: phase p -> start 2p (p>0: after grid_wait), end 2p+1; layer 0 QKV start = 0
    t0 = t[:, 0].min()
    nph = 5 * nl
    rows = []
    for p in range(nph):
        s = t[:, 2 * p] if p > 0 else t[:, 0]
        e = t[:, 2 * p + 1]
        work = e - s
        prev_end = t[:, 2 * p - 1].max() if p > 0 else t0
        rows.append((KINDS[p % 5], statistics.median(work.tolist()), work.max(), statistics.median(s.tolist()) - prev_end,
                     e.max() - t0))
    lm_s = t[:, 2 * nph]
    print(f"forward {ms.value * 1000:.1f} us (time_forward, 3 iters); timeline of the last launch, grid {G}, rows {args.rows}")
    for k in KINDS:
        rk = [r for r in rows if r[0] == k][1:]  # skip layer 0
        print(f"{k:5s} work median {statistics.median(r[1] for r in rk) / 1e3:7.2f} us  max {statistics.median(r[2] for r in rk) / 1e3:7.2f} us"
              f"   barrier gap {statistics.median(r[3] for r in rk) / 1e3:6.2f} us")
    per_layer = (rows[5 * (nl - 1) + 4][4] - rows[4][4]) / (nl - 1)
    print(f"per layer {per_layer / 1e3:.2f} us; LM phase start {statistics.median(lm_s.tolist()) - t0:.0f} ns after kernel start; "
          f"last layer end {rows[-1][4] / 1e3:.1f} us")


if __name__ == "__main__":
    main()
