"""Summarise ncu outputs into profiles/: the launch list (per-kernel share) and
the dominant kernel's DRAM traffic from a `--set full` capture.

  python tools/prof_summary.py <tag> gpurun_out/launches.csv [gpurun_out/full.ncu-rep]
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag, launches_csv = sys.argv[1], Path(sys.argv[2])
full = Path(sys.argv[3]) if len(sys.argv) > 3 else None
out = ROOT / "profiles"
out.mkdir(exist_ok=True)
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name):
    base = name.split("(")[0].replace("void ", "").replace("amusd::", "").replace("fw::", "").replace("tc::", "")
    return base.split("<")[0]


rows = list(csv.reader(open(launches_csv)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
ix = {h: i for i, h in enumerate(rows[hi])}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(ix) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    per[int(r[ix["ID"]])] = (short(r[ix["Kernel Name"]]), r[ix["Grid Size"]], r[ix["Block Size"]],
                             float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0))
SETUP = ("k_tile_weights", "k_fill_uniform", "at::", "vectorized_elementwise")  # model construction, not the path
agg = collections.OrderedDict()
n_setup = 0
for name, grid, block, us in per.values():
    if any(x in name for x in SETUP):
        n_setup += 1
        continue
    a = agg.setdefault((name, grid, block), [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
md = [f"# ncu launch list ({tag})", "",
      f"{len(per) - n_setup} launches on the path ({n_setup} model-construction launches -- weight fill / "
      f"tile re-layout -- excluded), {tot / 1000:.3f} ms summed (ncu, serialised, cold cache: compare shares).", "",
      "| kernel | grid | block | launches | total us | share | avg us |", "|---|---|---|---|---|---|---|"]
for (k, g, b), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    md.append(f"| {k} | {g} | {b} | {c} | {t:.1f} | {100 * t / tot:.1f}% | {t / c:.2f} |")
if full and full.exists():
    raw = subprocess.run(["ncu", "-i", str(full), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__shared_mem_per_block_dynamic"]
    hdr, units = rr[0], rr[1]
    caps = []
    for r in rr[2:]:
        caps.append({w: f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip() for w in want if w in hdr}
                    | {"kernel": short(r[hdr.index("Kernel Name")])})
    md += ["", "## dominant kernel, `--set full` capture", ""]
    for c in caps:
        md += [f"### {c['kernel']}", "", "| metric | value |", "|---|---|"]
        md += [f"| {k} | {v} |" for k, v in c.items() if k != "kernel"]
        md.append("")

    def num(s, unit_scale={"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}):
        v, u = s.split()
        return float(v.replace(",", "")) * unit_scale[u]
    c0 = caps[0]
    traffic = num(c0["dram__bytes_read.sum"]) + num(c0["dram__bytes_write.sum"])
    json.dump({"kernel": c0["kernel"], "dram_bytes_per_launch": traffic, "source": f"ncu --set full ({tag})",
               "capture": c0}, open(out / "dominant_kernel_traffic.json", "w"), indent=1)
(out / f"{tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
print("\n".join(md))
