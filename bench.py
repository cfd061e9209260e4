#!/usr/bin/env python
"""AMUSD decode benchmark (BASELINE.json metric): generated tokens/s, greedy,
bs=1, AMUSD vs sync-SD vs AR, with the HBM roofline of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl amusd|reference]

N=1 workload = BASELINE configs[2] (configs[1]'s pair co-located on one
B200): Llama-3.2-1B-shaped draft + Llama-3.1-8B-shaped verify, random-init
bf16, synthetic 32-token prompt, 512 new tokens, agreement coin rho=0.8.
A "step" is one full decode of 512 tokens.  N>1 (torchrun, one process per
GPU): every rank runs an independent co-located pair ("replicas"; weak
scaling, no data-path collective), value = all tokens / max-over-ranks time.

--impl reference times the CPU restatement of the reference path (oracle/,
numpy fp32, two-thread AMUSD executor) on the host cores, bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "generated tokens/sec (greedy, bs=1) AMUSD vs sync-SD vs AR; % HBM roofline"
WORKLOAD = ("cfg3: Llama-3.2-1B-shaped draft + Llama-3.1-8B-shaped verify co-located on 1xB200 "
            "(draft/verify on separate CUDA streams), random-init bf16, 32-token prompt, 512 new tokens")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amusd", choices=["amusd", "reference"])
    ap.add_argument("--new-tokens", type=int, default=512)
    ap.add_argument("--prompt-len", type=int, default=32)
    ap.add_argument("--rho", type=float, default=0.8)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--lead", type=int, default=0, help="max_draft_lead (0 = None)")
    ap.add_argument("--window", type=int, default=16)
    ap.add_argument("--shapes", default="1b8b", choices=["1b8b", "tiny"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=4)
    ap.add_argument("--profile-only", action="store_true", help="one AMUSD decode, no extras (for ncu)")
    ap.add_argument("--engines", default="ar,sync,amusd", help="subset of ar,sync,amusd to time")
    ap.add_argument("--no-extras", action="store_true", help="skip roofline/e2e/cpu legs (quick sweeps)")
    ap.add_argument("--draft-path-sync", default="persistent", choices=["persistent", "decode"],
                    help="draft forward for sync-SD (the draft owns the GPU): persistent SIMT decode kernel or the "
                         "tcgen05 work-queue forward")
    ap.add_argument("--draft-path-amusd", default="persistent", choices=["persistent", "decode"],
                    help="draft forward for co-located AMUSD (the draft gets its SM share)")
    ap.add_argument("--layout", default="auto", choices=["auto", "replicas", "split", "pairs"],
                    help="N>1: auto = the paper's split pair at N=2 (draft on rank 0's GPU, verify on rank 1's: "
                         "BASELINE config 2) and independent co-located pairs per GPU otherwise (replicas); "
                         "pairs = N/2 independent split pairs (BASELINE config 5 with --prompt-len 4096)")
    return ap.parse_args()


def synthetic_prompt(n: int, vocab: int) -> list:
    rng = random.Random(1234)
    return [rng.randrange(3, vocab) for _ in range(n)]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.path = gpu, None, None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows]
        loaded = [float(r[0]) for r in rows if float(r[2]) > 250.0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(float(r[1]) for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------- split pairs (configs 2 and 5)
def split_arm(args, rank: int, world: int, local_rank: int):
    """BASELINE config 2 (the paper's deployment, N=2) and config 5 (N/2 independent pairs,
    --layout pairs, long prompts via --prompt-len): in every pair the draft sits on one GPU
    (even rank) and the verify on the next (odd rank); the mailbox copies live in each GPU's HBM
    and are written by their single writers over NVLink P2P.  Pairs never communicate.

    value = all pairs' generated tokens / the device-timed decode (max over every GPU); e2e = the
    public API call (decode_speculative_async_split: host prompt in, prefill, IPC mailbox
    exchange, host tokens and trace out), wall clock, max over ranks; prefill (TTFT's GPU part) is
    timed separately; roofline = each GPU's persistent forward timed alone (CUDA events); the
    reference simulator's prediction for these latencies is printed beside the measurement
    (section 8(f)3)."""
    import torch
    import torch.distributed as dist
    import paper_2410_17375_b200 as P
    from paper_2410_17375_b200 import _lib as L
    from paper_2410_17375_b200 import calibrate as CB
    from paper_2410_17375_b200 import split as SP
    from paper_2410_17375_b200.split import SplitLink, decode_speculative_async_split
    if world % 2:
        raise SystemExit("split pairs need an even number of ranks")
    npairs = world // 2
    local_rank %= torch.cuda.device_count()   # fewer GPUs than ranks: functional check of the same path
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    groups = [dist.new_group([2 * p, 2 * p + 1]) for p in range(npairs)]
    link = SplitLink(group=groups[rank // 2])
    TC = P.TransformerConfig
    N, Plen = args.new_tokens, args.prompt_len
    max_seq = Plen + N + 64
    if link.role == "draft":
        base = P.TransformerModel(TC.llama_1b(max_seq=max_seq), seed=1, device=dev, keep_row_major=False)
        model = P.AgreementDraft(base, args.rho, coin_seed=1234)
    else:
        base = model = P.TransformerModel(TC.llama_8b(max_seq=max_seq), seed=0, device=dev, keep_row_major=False)
    if torch.cuda.device_count() < world:   # ranks share a GPU: keep their loops co-resident
        share = max(1, world // torch.cuda.device_count())
        base.set_max_grid(torch.cuda.get_device_properties(dev).multi_processor_count // share)
    cfg_m = base.config
    prompt = synthetic_prompt(Plen, 128256)
    cfg = P.DecodeConfig(max_new_tokens=N, draft_window_k=args.k, max_draft_lead=args.lead or None)
    for _ in range(args.warmup):
        decode_speculative_async_split(model, prompt, cfg, link=link, max_window=args.window)
    total, toks, launches, ref_tokens, prefill = 0.0, 0, 0, None, []
    dist.barrier()
    torch.cuda.synchronize()
    cm = ClockSampler(local_rank).__enter__()
    for _ in range(args.steps):
        # prefill timed apart (CUDA events); the decode below then starts from the fresh state
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        base.init_state(prompt)
        e1.record()
        e1.synchronize()
        prefill.append(e0.elapsed_time(e1))
        res, (dms, vms) = decode_speculative_async_split(model, prompt, cfg, link=link, max_window=args.window)
        total += max(dms, vms)      # device-timed, max over the pair's two GPUs
        toks += len(res.tokens)
        launches += SP.last_run["iters"] * SP.last_run["kernels_per_step"]   # this rank's GPU
        ref_tokens = ref_tokens or res.tokens
        if res.tokens != ref_tokens:
            raise SystemExit("split-pair output changed between runs -- parity broken")
    torch.cuda.synchronize()
    cm.__exit__(None, None, None)
    # parity: the pair's tokens equal the verify model's own greedy (AR) path
    ar_ok = None
    if link.role == "verify":
        from paper_2410_17375_b200.engines import canonical_path
        ar_ok = canonical_path(model, prompt, N + L.KMAX).tolist()[Plen:Plen + len(ref_tokens)] == ref_tokens
    ar_ok = next(x for x in (ar_ok, link.exchange(ar_ok)) if x is not None)
    if not ar_ok:
        raise SystemExit("split-pair AMUSD output differs from the verify model's AR path -- parity broken")
    # e2e through the public API (wall clock around the whole call), max over every rank
    e2e_ms, e2e_toks = [], 0
    for _ in range(max(1, args.steps)):
        dist.barrier()
        t0 = time.perf_counter()
        r2, _ = decode_speculative_async_split(model, prompt, cfg, link=link, max_window=args.window)
        e2e_ms.append((time.perf_counter() - t0) * 1000.0)
        e2e_toks += len(r2.tokens)
    # the baselines on the SAME GPUs: AR and sync-SD (k) on the verify GPU with a draft replica
    # there (sync-SD is sequential: a second GPU gives it nothing but a cross-GPU handoff)
    base_lines = None
    if link.role == "verify" and not args.no_extras:
        from paper_2410_17375_b200.engines import DeviceSession, canonical_path, finalize_tokens
        rep = P.TransformerModel(TC.llama_1b(max_seq=max_seq), seed=1, device=dev, keep_row_major=False)
        if torch.cuda.device_count() < world:
            rep.set_max_grid(torch.cuda.get_device_properties(dev).multi_processor_count // max(1, world // torch.cuda.device_count()))
        canon = canonical_path(base, prompt, N + L.KMAX)
        base_lines = {}
        for name, sess, eng in (("ar", DeviceSession(None, base, Plen, cfg), L.ENGINE_AR),
                                ("sync_sd", DeviceSession(P.AgreementDraft(rep, args.rho, coin_seed=1234), base, Plen, cfg,
                                                          canon=canon), L.ENGINE_SYNC)):
            for _ in range(max(1, args.warmup)):
                base.init_state(prompt)
                rep.init_state(prompt)
                sess.run(eng, prompt)
            ms, nt = 0.0, 0
            for _ in range(args.steps):
                base.init_state(prompt)
                rep.init_state(prompt)
                sess.prepare(prompt)
                st_, en_ = sess.launch(eng)
                out = sess.collect(st_, en_)
                toks_b, _ = finalize_tokens(out.verified, base.eos_token, N)
                if toks_b != ref_tokens[:len(toks_b)]:
                    raise SystemExit(f"split arm {name} output differs from AMUSD's -- parity broken")
                ms += out.device_ms
                nt += len(toks_b)
            base_lines[name] = {"tokens_per_s": round(nt / (ms / 1000.0), 3), "ms_per_token": round(ms / nt, 4),
                                "gpus": "the verify GPU (draft replica co-resident)" if name == "sync_sd" else "the verify GPU"}
        del rep
        P.engines.clear_sessions()
        torch.cuda.empty_cache()
    # per-GPU roofline: each GPU's persistent forward alone (1 row) at the prompt's context
    base.init_state(prompt)
    fms = CB.forward_ms(base, 1, iters=20)
    fbytes = cfg_m.step_weight_bytes() + cfg_m.kv_bytes_per_token() * (Plen + 1)
    vrows = {m: CB.forward_ms(base, m) for m in (1, 2, 4, 8, 16)} if link.role == "verify" else None
    mine = {"rank": rank, "role": link.role, "ms": fms, "bytes": fbytes, "vrows": vrows, "toks": toks,
            "base_lines": base_lines,
            "total": total, "prefill": max(prefill), "e2e_ms": sum(e2e_ms), "e2e_toks": e2e_toks,
            "launches": launches, "clocks": cm.summary(), "verify_steps": res.stats.verify_steps,
            "rollbacks": res.stats.rollbacks, "drafted": res.stats.drafted_tokens}
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    if rank != 0:
        return
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    verify_ranks = [r for r in allr if r["role"] == "verify"]
    draft_ranks = [r for r in allr if r["role"] == "draft"]
    tok_all = sum(r["toks"] for r in verify_ranks)
    t_max = max(r["total"] for r in allr)
    v = tok_all / (t_max / 1000.0)
    gbs = {r["role"] + str(r["rank"] // 2): r["bytes"] / r["ms"] / 1e6 for r in allr}
    vr0 = verify_ranks[0]
    calib = None
    try:
        vb, vp = CB.fit_linear(vr0["vrows"])
        lat = CB.Latencies(0.0, draft_ranks[0]["ms"], vb, vp, Plen)
        calib = {"latency_ms": {"draft_per_token_ms": round(lat.draft_per_token_ms, 5),
                                "verify_base_ms": round(vb, 5), "verify_per_token_ms": round(vp, 5)},
                 "predicted_tokens_per_s_per_pair": {f"rho{r}": CB.predict(lat, r, n_tokens=N) for r in (args.rho, 0.9)}}
    except Exception as exc:
        calib = {"unavailable": f"{type(exc).__name__}: {exc}"}
    e2e_t = max(r["e2e_ms"] for r in allr)
    workload = ("cfg2: Llama-3.2-1B-shaped draft on GPU0 + Llama-3.1-8B-shaped verify on GPU1, P2P mailbox over "
                "NVLink" if npairs == 1 else
                f"cfg5: {npairs} independent split pairs (1B-shaped draft GPU | 8B-shaped verify GPU) on {world} GPUs")
    print(json.dumps({
        "metric": METRIC, "value": round(v, 2), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if npairs == 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, seeded prompt)",
        "config": {"workload": workload, "rho": args.rho, "new_tokens": N, "prompt_len": Plen,
                   "parallelism": f"{npairs} split pair(s) (draft | verify)", "gpus_visible": torch.cuda.device_count(),
                   "l2": "weights (17.5 GB) >> 126 MB L2: no flush needed"},
        "amusd": {"tokens_per_s": round(v, 3), "tokens_per_s_per_pair": round(v / npairs, 3),
                  "verify_steps": vr0["verify_steps"], "rollbacks": vr0["rollbacks"], "drafted": vr0["drafted"],
                  "tokens_equal_ar": bool(ar_ok)},
        "sync_sd": (vr0["base_lines"] or {}).get("sync_sd"), "ar": (vr0["base_lines"] or {}).get("ar"),
        "speedup_vs_sync": round(v / npairs / vr0["base_lines"]["sync_sd"]["tokens_per_s"], 3) if vr0["base_lines"] else None,
        "speedup_vs_ar": round(v / npairs / vr0["base_lines"]["ar"]["tokens_per_s"], 3) if vr0["base_lines"] else None,
        "prefill_ms": {"max_over_gpus": round(max(r["prefill"] for r in allr), 3),
                       "draft": round(max(r["prefill"] for r in draft_ranks), 3),
                       "verify": round(max(r["prefill"] for r in verify_ranks), 3),
                       "note": f"init_state of the {Plen}-token prompt (not in value)"},
        "roofline": {"bound": "hbm", "kernel": "k_forward (persistent tcgen05 forward), 1 row, each GPU alone",
                     "achieved": round(vr0["bytes"] / vr0["ms"] / 1e6, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(vr0["bytes"] / vr0["ms"] / 1e6 / hbm_peak, 4), "traffic": None,
                     "per_gpu": {k: {"GB/s": round(x, 1), "frac": round(x / hbm_peak, 4)} for k, x in gbs.items()}},
        "calibration": calib,
        "cpu_baseline": None,
        "e2e": {"value": round(sum(r["e2e_toks"] for r in verify_ranks) / (e2e_t / 1000.0), 2), "unit": "tokens/s",
                "h2d_bytes_per_step": 4 * Plen * 2 * npairs, "d2h_bytes_per_step": 4 * (N + L.KMAX) * npairs,
                "includes": "prefill on both GPUs + IPC mailbox exchange + both loops + token/trace read-back"},
        "gpu_launches": int(sum(r["launches"] for r in allr)),
        "clocks": {f"rank{r['rank']}": r["clocks"] for r in allr}}))


# --------------------------------------------------------------- GPU arm
def gpu_arm(args, rank: int, world: int, local_rank: int):
    import torch
    import paper_2410_17375_b200 as P
    from paper_2410_17375_b200 import _lib as L
    from paper_2410_17375_b200.engines import DeviceSession, canonical_path, finalize_tokens

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    TC = P.TransformerConfig
    N, Plen = args.new_tokens, args.prompt_len
    max_seq = Plen + N + 2 * L.KMAX + 32
    if args.shapes == "tiny":
        vcfg, dcfg = TC.tiny_verify(max_seq=max_seq), TC.tiny_draft(max_seq=max_seq)
    else:
        vcfg, dcfg = TC.llama_8b(max_seq=max_seq), TC.llama_1b(max_seq=max_seq)
    # the verify keeps only its tcgen05 copy (the row-major one would be 16 GB more for the 8B);
    # the draft keeps both (the roofline block also tiles it for the decode forward)
    vm = P.TransformerModel(vcfg, seed=0, device=dev, keep_row_major=args.shapes == "tiny")
    dm = P.TransformerModel(dcfg, seed=1, device=dev)
    prompt = synthetic_prompt(Plen, vcfg.vocab_size)
    draft = P.AgreementDraft(dm, args.rho, coin_seed=1234)
    cfg = P.DecodeConfig(max_new_tokens=N, draft_window_k=args.k, max_draft_lead=args.lead or None)
    if args.profile_only:  # natural draft, no canonical AR pass: keeps the ncu launch list short
        s = DeviceSession(dm, vm, Plen, cfg, max_window=args.window)
        out = s.run(L.ENGINE_ASYNC, prompt)
        torch.cuda.synchronize()
        print(json.dumps({"profile_only": True, "verified": len(out.verified), "verify_steps": out.info.verify_steps,
                          "draft_iters": out.info.draft_iters}))
        return None
    canon = canonical_path(vm, prompt, N + L.KMAX)  # setup: the verify model's greedy path (coin input)
    sess = {
        "ar": (DeviceSession(None, vm, Plen, cfg), L.ENGINE_AR),
        "sync": (DeviceSession(draft, vm, Plen, cfg, canon=canon), L.ENGINE_SYNC),
        "amusd": (DeviceSession(draft, vm, Plen, cfg, canon=canon, max_window=args.window), L.ENGINE_ASYNC),
    }
    kd, kv = sess["amusd"][0].kernels_per_step(L.ENGINE_ASYNC)
    kd_sync, kv_sync = sess["sync"][0].kernels_per_step(L.ENGINE_SYNC)
    results, ref_tokens = {}, None
    sampler = None
    for name in ("ar", "sync", "amusd"):
        if name not in args.engines.split(","):
            continue
        s, eng = sess[name]
        if name in ("sync", "amusd") and args.shapes == "1b8b":
            dm.set_path(args.draft_path_sync if name == "sync" else args.draft_path_amusd)  # captured at graph build
        for _ in range(args.warmup):
            s.run(eng, prompt)
        per, toks, launches, stats = [], 0, 0, []
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        cm = ClockSampler(local_rank) if name == "amusd" else None
        if cm:
            cm.__enter__()
        pre_ms = []
        for _ in range(args.steps):
            # prefill is reported separately: CUDA events on the verify stream it runs on
            vs_ = s.streams()[0]
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(vs_)
            s.prepare(prompt)
            p1.record(vs_)
            p1.synchronize()
            pre_ms.append(p0.elapsed_time(p1))
            start, end = s.launch(eng)
            out = s.collect(start, end)
            tokens, _ = finalize_tokens(out.verified, vm.eos_token, N)
            per.append(out.device_ms)
            toks += len(tokens)
            if name == "ar":
                launches += out.info.verify_iters * (kv - 2 + 2)
            elif name == "sync":
                launches += out.info.verify_iters * (args.k * kd_sync + kv_sync)
            else:
                launches += out.info.draft_iters * kd + out.info.verify_iters * kv
            stats.append(out.info)
            if ref_tokens is None:
                ref_tokens = canon.tolist()[Plen:Plen + N]
            if tokens != ref_tokens:
                raise SystemExit(f"{name} output differs from the AR oracle -- parity broken")
        torch.cuda.synchronize()
        if cm:
            cm.__exit__(None, None, None)
            sampler = cm
        total_ms = sum(per)
        if world > 1:
            t = torch.tensor([total_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            total_ms = float(t.item())
        results[name] = {
            "tokens_per_s": toks / (total_ms / 1000.0), "ms_per_step": total_ms / args.steps,
            "ms_per_token": total_ms / toks, "generated": toks // args.steps, "gpu_launches": launches,
            "verify_steps": statistics.mean(i.verify_steps for i in stats),
            "rollbacks": statistics.mean(i.rollbacks for i in stats),
            "drafted": statistics.mean(i.drafted for i in stats),
            "prefill_ms": round(max(pre_ms), 3),   # both models' prefill (init_state), not in ms_per_step
        }
        # in-situ HBM bandwidth of the run: forwards issued x their algorithmic bytes over the
        # device time (AMUSD: every draft forward launched, cut ones counted in full -> upper bound)
        vfw = statistics.mean(i.verify_steps for i in stats)
        dfw = statistics.mean((i.draft_iters if name == "amusd" else i.drafted) for i in stats) if name != "ar" else 0.0
        ctx_m = Plen + N // 2
        gb = (vfw * (vcfg.step_weight_bytes() + vcfg.kv_bytes_per_token() * ctx_m) +
              dfw * (dcfg.step_weight_bytes() + dcfg.kv_bytes_per_token() * ctx_m)) / 1e9
        results[name]["in_situ"] = {"verify_forwards": vfw, "draft_forwards": dfw, "GB_per_token": round(gb / N, 3),
                                    "GB_per_s": round(gb / (total_ms / args.steps / 1000.0), 1)}
    variants = None
    if not args.no_extras and world == 1:
        variants = engine_variants(args, P, L, DeviceSession, finalize_tokens, dm, vm, prompt, canon, N, Plen, ref_tokens)
    if args.no_extras:
        return {"results": results, "roofline": None, "e2e": None, "clocks": sampler.summary() if sampler else None,
                "vm": vm, "dm": dm, "prompt": prompt, "canon": canon.tolist(), "vcfg": vcfg, "dcfg": dcfg}
    # ---- kernel roofline: time the forwards / dominant kernel in isolation (CUDA events)
    import ctypes as C
    lib = L.load()

    def time_fwd(m, rows, which, layer=0, iters=20):
        ms = C.c_float()
        L.check(lib.amusd_time_forward(m.handle, rows, which, layer, iters, C.byref(ms),
                                       torch.cuda.current_stream().cuda_stream))
        return ms.value
    first_logits = {}
    for key, m in (("verify", vm), ("draft", dm)):   # parity leg (cpu_leg): first-step logits
        st = m.init_state(prompt)
        m.next_token(st)
        first_logits[key] = m.last_logits(1).numpy()[0]
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if peaks else "fallback"
    # Dominant kernel: k_forward, the persistent tcgen05 decoder forward (ONE launch per model
    # forward).  Algorithmic bytes per launch = every weight byte once (embedding rows excluded,
    # LM head included) + the K/V cache read at the timed position + this step's K/V append.
    ctx = len(prompt)

    def fwd_bytes(c, rows):
        return c.step_weight_bytes() + c.kv_bytes_per_token() * (ctx + rows)
    kernels = {}
    dm.set_path("persistent")
    for key, m, c, rows, iters in (("verify_forward_m1", vm, vcfg, 1, 10), ("verify_forward_m4", vm, vcfg, 4, 10),
                                   ("verify_forward_m16", vm, vcfg, 16, 5), ("draft_forward_m1", dm, dcfg, 1, 20)):
        ms = time_fwd(m, rows, -1, iters=iters)
        b = fwd_bytes(c, rows)
        kernels[key] = {"bytes": b, "ms": ms, "gbs": b / ms / 1e6}
    if args.shapes == "1b8b":  # the draft through the persistent SIMT/mma decode forward (decode_gv.cu)
        dm.set_path("decode")
        ms = time_fwd(dm, 1, -1, iters=20)
        b = fwd_bytes(dcfg, 1)
        kernels["draft_forward_m1_decode"] = {"bytes": b, "ms": ms, "gbs": b / ms / 1e6}
        dm.set_path("persistent")
    # the verify forward at the run's mean context (the AR loop decodes from ctx P to P + N): the
    # per-step protocol cost = AR ms/token over this
    ctx_mean = Plen + N // 2
    st = vm.init_state(synthetic_prompt(ctx_mean, vcfg.vocab_size))
    ms_mean = time_fwd(vm, 1, -1, iters=10)
    kernels[f"verify_forward_m1_ctx{ctx_mean}"] = {"bytes": vcfg.step_weight_bytes() + vcfg.kv_bytes_per_token() * (ctx_mean + 1),
                                                   "ms": ms_mean, "gbs": 0.0}
    kernels[f"verify_forward_m1_ctx{ctx_mean}"]["gbs"] = kernels[f"verify_forward_m1_ctx{ctx_mean}"]["bytes"] / ms_mean / 1e6
    st = vm.init_state(prompt)
    traffic = None
    prof = ROOT / "profiles" / "dominant_kernel_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    dom = kernels["verify_forward_m1"]
    roofline = {"bound": "hbm", "kernel": "k_forward: persistent tcgen05 decoder forward, 8B verify, 1 row "
                                          "(one launch per forward; timed alone with CUDA events, eager)",
                "achieved": round(dom["gbs"], 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(dom["gbs"] / hbm_peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": int(dom["bytes"]), "peak_source": peak_src,
                "forwards": {k: {"ms": round(v["ms"], 4), "GB/s": round(v["gbs"], 1), "bytes": int(v["bytes"]),
                                 "frac": round(v["gbs"] / hbm_peak, 4)} for k, v in kernels.items()}}
    if "ar" in results:  # protocol + graph-loop cost per AR step over the isolated forward at the mean context
        roofline["ar_step_over_forward"] = round(results["ar"]["ms_per_token"] / ms_mean - 1.0, 4)
    # ---- end to end through the public API (host prompt in, host tokens out, wall clock)
    e2e = None
    if rank == 0 or world > 1:
        e2e_ms, e2e_toks = [], 0
        ex = P.CudaAsyncExecutor(max_window=args.window)
        P.decode_speculative_async(draft, vm, prompt, cfg, executor=ex)   # warm-up: session + graph build
        for i in range(max(1, args.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.decode_speculative_async(draft, vm, prompt, cfg,
                                             executor=P.CudaAsyncExecutor(max_window=args.window))
            torch.cuda.synchronize()
            e2e_ms.append((time.perf_counter() - t0) * 1000.0)
            e2e_toks += len(res.tokens)
            if res.tokens != ref_tokens:
                raise SystemExit("e2e output differs from the AR oracle")
        h2d = 4 * Plen * 3 + 256 * (2 + (Plen + L.KMAX - 1) // L.KMAX * 2)   # prompt copies + prefill control blocks
        d2h = 4 * (N + L.KMAX) + 256 + 32 * (results["amusd"]["drafted"] + results["amusd"]["verify_steps"] + 64)
        e2e = {"value": round(e2e_toks / (sum(e2e_ms) / 1000.0), 2), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "includes": "prefill of both models + graph launch + V/trace read-back + trace merge"}
    calib = None
    if world == 1:   # section 8(f)3: measured latencies -> the reference's own simulator
        try:
            from paper_2410_17375_b200 import calibrate as CB
            calib = CB.calibrate(dm, vm, ctx=Plen + N // 2, n_tokens=N)
            calib["measured_colocated_1gpu"] = {"ar": round(results["ar"]["tokens_per_s"], 3),
                                                "sync_k4": round(results["sync"]["tokens_per_s"], 3),
                                                "amusd": round(results["amusd"]["tokens_per_s"], 3)}
        except Exception as exc:  # reference not installed: say so, never fake a prediction
            calib = {"unavailable": f"{type(exc).__name__}: {exc}"}
    return {"results": results, "roofline": roofline, "e2e": e2e, "clocks": sampler.summary() if sampler else None,
            "vm": vm, "dm": dm, "prompt": prompt, "canon": canon.tolist(), "vcfg": vcfg, "dcfg": dcfg,
            "first_logits": first_logits, "variants": variants, "calibration": calib}


def engine_variants(args, P, L, DeviceSession, finalize_tokens, dm, vm, prompt, canon, N, Plen, ref_tokens):
    """SURVEY.md section 7.3.2 reporting: AMUSD and sync-SD at rho=0.9 as well, and the sync-SD
    k sweep (best k next to the reference default k=4).  1 warm-up + 2 timed decodes each,
    device-timed, tokens checked against the AR path like the headline engines."""
    def timed(sess, eng, n=2):
        sess.run(eng, prompt)
        ms, toks, info = 0.0, 0, []
        for _ in range(n):
            sess.prepare(prompt)
            start, end = sess.launch(eng)
            out = sess.collect(start, end)
            tokens, _ = finalize_tokens(out.verified, vm.eos_token, N)
            if tokens != ref_tokens:
                raise SystemExit("variant output differs from the AR oracle -- parity broken")
            ms += out.device_ms
            toks += len(tokens)
            info.append(out.info)
        return {"tokens_per_s": round(toks / (ms / 1000.0), 3), "verify_steps": statistics.mean(i.verify_steps for i in info),
                "rollbacks": statistics.mean(i.rollbacks for i in info)}
    out = {}
    d9 = P.AgreementDraft(dm, 0.9, coin_seed=1234)
    c4 = P.DecodeConfig(max_new_tokens=N, draft_window_k=args.k, max_draft_lead=args.lead or None)
    out["rho0.9"] = {"sync_k4": timed(DeviceSession(d9, vm, Plen, c4, canon=canon), L.ENGINE_SYNC),
                     "amusd": timed(DeviceSession(d9, vm, Plen, c4, canon=canon, max_window=args.window),
                                    L.ENGINE_ASYNC)}
    for rho, d in ((args.rho, P.AgreementDraft(dm, args.rho, coin_seed=1234)), (0.9, d9)):
        sweep = {}
        for k in (2, 3, 4, 5, 6, 8):
            ck = P.DecodeConfig(max_new_tokens=N, draft_window_k=k, max_draft_lead=args.lead or None)
            sweep[k] = timed(DeviceSession(d, vm, Plen, ck, canon=canon), L.ENGINE_SYNC)["tokens_per_s"]
        best = max(sweep, key=sweep.get)
        out[f"rho{rho}"] = dict(out.get(f"rho{rho}", {}), sync_k_sweep=sweep, sync_best={"k": best, "tokens_per_s": sweep[best]})
    P.engines.clear_sessions()
    return out


# --------------------------------------------------------------- CPU arm
def _shapes(args, max_seq):
    from paper_2410_17375_b200.models import TransformerConfig as TC   # pure Python (no libamusd)
    if args.shapes == "tiny":
        return TC.tiny_verify(max_seq=max_seq), TC.tiny_draft(max_seq=max_seq)
    return TC.llama_8b(max_seq=max_seq), TC.llama_1b(max_seq=max_seq)


def cpu_decoders(vcfg, dcfg, wv, wd):
    """fp32 numpy decoders (oracle/ref_decoder.py) over bf16-valued weights, bf16 KV (as the GPU)."""
    from oracle.ref_decoder import RefDecoder
    from oracle.ref_models import shape_of
    return (RefDecoder(shape_of(vcfg, kv_bf16=True), wv, tied=vcfg.tied),
            RefDecoder(shape_of(dcfg, kv_bf16=True), wd, tied=dcfg.tied))


def reference_cpu_run(rv, rd, prompt, rho, n_tokens, steps=1, warmup=0, k=4):
    """The reference's OWN engines (unmodified specdec: decode_autoregressive and
    decode_speculative_async with ThreadExecutor + the SURVEY section 0.6 trace shim,
    engines.py:279-287, 409-561) driving the numpy decoders through the MockModel hooks
    (oracle/ref_models.py).  Decode only is timed (the executor's wall time; prefill excluded).
    Returns the CPU AR tokens (parity vs the GPU), AR and AMUSD tokens/s."""
    from oracle.ref_models import load_reference, make_models
    S = load_reference()
    if S is None:
        raise RuntimeError("reference package specdec not installed (baseline/_ref)")
    Dec, Coin, Shim = make_models(S)
    verify = Dec(rv)
    t0 = time.perf_counter()
    ar = S.decode_autoregressive(verify, prompt, S.DecodeConfig(max_new_tokens=n_tokens + 8, draft_window_k=k))
    ar_wall = time.perf_counter() - t0
    canon = list(prompt) + ar.tokens          # the coin's canonical path
    draft = Coin(rd, canon, rho, 1234)
    cfg = S.DecodeConfig(max_new_tokens=n_tokens, draft_window_k=k)
    walls, toks, stats = [], 0, []
    for i in range(warmup + steps):
        ex = Shim()
        res = S.decode_speculative_async(draft, verify, prompt, cfg, executor=ex)
        if res.tokens != ar.tokens[:n_tokens]:
            raise SystemExit("reference CPU AMUSD output differs from reference CPU AR")
        if i >= warmup:
            walls.append(ex.last_wall_s)
            toks += len(res.tokens)
            stats.append(res.stats)
    return {"ar_tokens": ar.tokens[:n_tokens], "ar_tokens_per_s": len(ar.tokens) / (ar.stats.total_ms / 1000.0),
            "ar_wall_s_incl_prefill": ar_wall, "amusd_tokens_per_s": toks / sum(walls), "amusd_wall_s": sum(walls),
            "amusd_tokens": toks, "verify_steps": statistics.mean(s.verify_steps for s in stats),
            "rollbacks": statistics.mean(s.rollbacks for s in stats), "specdec": str(S.__file__)}


def reference_arm(args, rank: int, world: int):
    """--impl reference: the reference's own CPU path, timed on the host cores.

    The unmodified reference engines (baseline/_ref) drive fp32 numpy decoders of the
    cfg3 shapes (oracle/ref_decoder.py) whose bf16-valued weights are generated on the HOST
    by the same splitmix64 stream the GPU fill uses (oracle/ref_models.synthetic_weights):
    no GPU and no libamusd on this arm.  A step = one AMUSD decode of a bounded sample of
    new tokens (the fp32 8B forward costs ~0.7 s per token on the host)."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    try:
        import numpy as np  # noqa: F401
        from paper_2410_17375_b200.models import weight_names, weight_shape
        from oracle.ref_models import synthetic_weights
        N, Plen = args.new_tokens, args.prompt_len
        vcfg, dcfg = _shapes(args, Plen + N + 64)
        wv = synthetic_weights([(n, weight_shape(vcfg, n)) for n in weight_names(vcfg)], 0, bf16=True)
        wd = synthetic_weights([(n, weight_shape(dcfg, n)) for n in weight_names(dcfg)], 1, bf16=True)
        rv, rd = cpu_decoders(vcfg, dcfg, wv, wd)
        prompt = synthetic_prompt(Plen, vcfg.vocab_size)
        sample = max(1, args.cpu_tokens)
        r = reference_cpu_run(rv, rd, prompt, args.rho, sample, steps=args.steps, warmup=args.warmup, k=args.k)
    except Exception as exc:  # pragma: no cover - reference not installed / host too small
        print(json.dumps({"impl": "reference", "unavailable": f"{type(exc).__name__}: {exc}"}))
        return
    v = r["amusd_tokens_per_s"]
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * r["amusd_wall_s"] / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, seeded prompt)",
            "config": {"workload": WORKLOAD, "rho": args.rho, "sync_k": args.k, "new_tokens_per_step": sample,
                       "truncated": f"{sample} of {args.new_tokens} new tokens per step (bounded CPU sample)"},
            "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "cores": cores, "kind": "reference",
                             "sample": f"unmodified reference engines ({r['specdec']}): decode_speculative_async "
                                       f"(ThreadExecutor + trace shim) on numpy fp32 1B/8B-shaped decoders through "
                                       f"the MockModel hooks, {sample} new tokens per step, decode only",
                             "ar_tokens_per_s": round(r["ar_tokens_per_s"], 4),
                             "verify_steps": r["verify_steps"], "rollbacks": r["rollbacks"]},
            "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_leg(args, out):
    """cpu_baseline (the reference's own engines on the host cores, same weights/prompt/rho)
    and the CPU-vs-GPU parity of the bench shapes: first-step logits of both models against
    the bf16-faithful oracle (activations rounded where the kernels round; fp32 summation
    order is the only difference) and the pure-fp32 oracle, and the first AR tokens of the
    verify model against the faithful oracle."""
    import numpy as np
    from oracle.ref_decoder import RefDecoder
    from oracle.ref_models import shape_of
    vm, dm = out["vm"], out["dm"]
    wv, wd = vm.host_weights(), dm.host_weights()
    rv, rd = cpu_decoders(out["vcfg"], out["dcfg"], wv, wd)
    fv = RefDecoder(shape_of(out["vcfg"], kv_bf16=True, act_bf16=True), wv, tied=out["vcfg"].tied)
    fd = RefDecoder(shape_of(out["dcfg"], kv_bf16=True, act_bf16=True), wd, tied=out["dcfg"].tied)
    prompt = out["prompt"]
    par = {}
    for key, f, r, c, w in (("verify", fv, rv, out["vcfg"], wv), ("draft", fd, rd, out["dcfg"], wd)):
        gl = out["first_logits"][key]
        fl, cl = f.start(prompt).last_logits, r.start(prompt).last_logits
        # fp32 noise floor: the same faithful oracle with float64 accumulation (tests/test_gpu_parity.py)
        f64 = RefDecoder(shape_of(c, kv_bf16=True, act_bf16=True, acc64=True), w, tied=c.tied)
        hl = f64.start(prompt).last_logits
        del f64
        par[f"{key}_logit_err_faithful"] = round(float(np.abs(gl - fl).max() / fl.std()), 6)
        par[f"{key}_noise_floor"] = round(float(np.abs(hl - fl).max() / fl.std()), 6)
        par[f"{key}_logit_err_fp32"] = round(float(np.abs(gl - cl).max() / cl.std()), 6)
        par[f"{key}_argmax_equal"] = bool(int(np.argmax(gl)) == int(np.argmax(fl)))
    gpu = out["canon"][len(prompt):len(prompt) + args.cpu_tokens]
    st = fv.start(prompt)
    cpu_tok = []
    for t in gpu:                       # teacher-forced along the GPU path: per-position comparison
        cpu_tok.append(fv.predict(st))
        fv.extend(st, [t])
    match = sum(int(a == b) for a, b in zip(cpu_tok, gpu))
    par.update({"tolerance": "max|gpu-cpu|/std(cpu logits): <= 2x the noise floor (|faithful fp32 - faithful "
                             "float64-accumulated|/std) vs the bf16-faithful oracle, <= 2e-1 vs the pure fp32 "
                             "oracle (tests/test_gpu_parity.py)",
                "ar_tokens_cpu_faithful": cpu_tok, "ar_tokens_gpu": gpu, "ar_tokens_match": f"{match}/{len(gpu)}"})
    del fv, fd
    s = reference_cpu_run(rv, rd, prompt, args.rho, args.cpu_tokens, k=args.k)
    cpu = {"value": round(s["amusd_tokens_per_s"], 4), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
           "sample": f"{args.cpu_tokens} new tokens, unmodified reference engines (decode_speculative_async with "
                     f"ThreadExecutor + trace shim) on numpy fp32 1B/8B-shaped decoders via the MockModel hooks, "
                     f"same weights/prompt/rho, decode only",
           "ar_tokens_per_s": round(s["ar_tokens_per_s"], 4)}
    return cpu, par


# -------------------------------------------------------------------- main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.layout == "auto":
        args.layout = "split" if world == 2 else "replicas"
    if world > 1:
        import torch
        if args.layout not in ("split", "pairs"):
            torch.cuda.set_device(local_rank)
        # the split pair's link is object collectives only (gloo); replicas time with NCCL
        torch.distributed.init_process_group("nccl" if args.impl == "amusd" and args.layout == "replicas" else "gloo")
    if args.impl == "reference":
        reference_arm(args, rank, world)
    elif args.layout in ("split", "pairs"):
        split_arm(args, rank, world, local_rank)
    else:
        out = gpu_arm(args, rank, world, local_rank)
        if out is None:
            return
        res = out["results"]
        cpu, parity = None, None
        if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.no_extras:
            cpu, parity = cpu_leg(args, out)
        if rank == 0:
            nan = {"tokens_per_s": float("nan"), "ms_per_step": float("nan"), "gpu_launches": 0}
            a, sy, ar = res.get("amusd", nan), res.get("sync", nan), res.get("ar", nan)
            line = {
                "metric": METRIC, "value": round(a["tokens_per_s"] * world, 2), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(a["ms_per_step"], 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init weights, seeded 32-token prompt)",
                "config": {"workload": WORKLOAD if args.shapes == "1b8b" else "tiny pair (cfg1 shapes)",
                           "rho": args.rho, "sync_k": args.k, "max_draft_lead": args.lead or None,
                           "max_window": args.window, "new_tokens": args.new_tokens,
                           "prompt_len": args.prompt_len, "parallelism": f"replicas x{world}" if world > 1 else "co-located pair",
                           "l2": "weights (17.5 GB) >> 126 MB L2: no flush needed"},
                "amusd": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in a.items()},
                "sync_sd": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in sy.items()},
                "ar": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in ar.items()},
                "speedup_vs_sync": round(a["tokens_per_s"] / sy["tokens_per_s"], 3),
                "speedup_vs_ar": round(a["tokens_per_s"] / ar["tokens_per_s"], 3),
                "variants": out.get("variants"), "calibration": out.get("calibration"),
                "roofline": out["roofline"], "cpu_baseline": cpu, "parity": parity, "e2e": out["e2e"],
                "gpu_launches": int(a["gpu_launches"]), "clocks": out["clocks"],
            }
            print(json.dumps(line))
    if world > 1:
        import torch
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
