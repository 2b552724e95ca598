"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line.
usage: python tools/ncu_srcmix.py mix.csv [n_images] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nimg = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
agg = {}
path = None
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        idx = {h: j for j, h in enumerate(hdr) if j >= 2}
        continue
    if hdr is None or len(r) < 4:
        continue
    if r[0]:
        cur = (path, int(r[0]), r[1].strip()[:90])
    if not r[2] or cur is None:
        continue
    a = agg.setdefault(cur, {"wf": 0.0, "xs": 0.0, "smp": 0.0, "inst": 0.0})
    def f(k):
        try:
            return float(r[idx[k]])
        except Exception:
            return 0.0
    a["wf"] += f("L1 Wavefronts Shared")
    a["xs"] += f("L1 Wavefronts Shared Excessive")
    a["smp"] += f("Warp Stall Sampling (All Samples)")
    a["inst"] += f("Instructions Executed")
T = {k: sum(v[k] for v in agg.values()) for k in ("wf", "xs", "smp", "inst")}
print("per image: shared wf %.0f  excess %.0f  warp-inst %.0f  samples %.0f" % (T["wf"] / nimg, T["xs"] / nimg, T["inst"] / nimg, T["smp"]))
for key in ("wf", "smp", "inst"):
    print("\n== top by", key)
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print("%-16s %4d wf %7.0f xs %6.0f inst %7.0f smp %5.1f%% | %s" % (k[0][:16], k[1], v["wf"] / nimg, v["xs"] / nimg,
              v["inst"] / nimg, 100 * v["smp"] / max(T["smp"], 1), k[2]))
