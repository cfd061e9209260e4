"""Summarise a persistent-forward timeline (tools/fw_timeline.py output)."""
import sys
import numpy as np

t = np.load(sys.argv[1])
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 2
it, cta, ph, tg, ti, td, tm, te = [t[:, i].astype(np.float64) for i in range(8)]
t0 = tg.min()
print("span us", (te.max() - t0) / 1e3)
names = ["qkv", "attn", "o", "gu", "down"]
for p in range(0, 1 + 5 * layers):
    s = ph == p
    if not s.any():
        continue
    nm = "embed" if p == 0 else names[(p - 1) % 5]
    dd = td[s][td[s] > 0]
    print(f"ph{p:3d} {nm:5s} n={s.sum():4d} grab[{(tg[s].min()-t0)/1e3:7.1f},{(tg[s].max()-t0)/1e3:7.1f}] "
          f"dep[{((dd.min()-t0)/1e3 if len(dd) else 0):7.1f},{((dd.max()-t0)/1e3 if len(dd) else 0):7.1f}] "
          f"done[{(te[s].min()-t0)/1e3:7.1f},{(te[s].max()-t0)/1e3:7.1f}]  dur {(te[s].max()-te[ph==p-1].max())/1e3 if p else 0:6.1f}")
for p in range(1, 6):
    s = ph == p
    if not (ti[s] > 0).any():
        continue
    for nm, x in (("issued-grab", ti - tg), ("estart-issued", tm - ti), ("done-estart", te - tm)):
        print("   ph%d %-14s" % (p, nm), np.round(np.percentile(x[s] / 1e3, [10, 50, 90, 99, 100]), 2))
