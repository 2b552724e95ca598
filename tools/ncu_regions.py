"""Per-region totals of an ncu source page (--print-source cuda,sass --csv): SASS rows are put in address order and
each is assigned to the region of the most recent kernels_polar.cu line at or before it (inlined helpers from
other files inherit the caller's region; region starts are located from marker comments in kernels_polar.cu).
usage: python tools/ncu_regions.py mix.csv n_images"""
import csv
import sys

def _find_regions():
    src = open("/root/repo/paper_1412_0781_b200/csrc/kernels_polar.cu").read().splitlines()
    marks = [("K1a: row FFTs", "image/row FFT"), ("per phase: K1b column FFTs", "col fill"), ("PROF_MARK(1);", "col FFT"),
             ("if constexpr (sizeof(T) == 4 && (W == 5 || W == 6) && MC > 0)", "gather doubles"),
             ("const int nb = pp.phase_node_begin[ph]", "gather singles"), ("const bool want_prefetch", "ring FFT"),
             ("const int64_t kstride = pp.ghat_kstride", "write-out"), ("PROF_STORE();", "tail")]
    out = [(0, "setup")]
    for pat, name in marks:
        ln = next(i + 1 for i, l in enumerate(src) if pat in l and i + 1 > out[-1][0])
        out.append((ln, name))
    return out
REGIONS = _find_regions()
KSTART = next(i + 1 for i, l in enumerate(open("/root/repo/paper_1412_0781_b200/csrc/kernels_polar.cu").read().splitlines()) if l.startswith("polar_kernel("))


def region_of(line):
    name = REGIONS[0][1]
    for lo, nm in REGIONS:
        if line >= lo:
            name = nm
    return name


rows = list(csv.reader(open(sys.argv[1])))
nimg = float(sys.argv[2])
path = hdr = None
cur_line = None
sass = []
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
        cur_line = (path, int(r[0]))
    if not r[2] or not r[2].startswith("0x"):
        continue
    def f(k):
        try:
            return float(r[idx[k]])
        except Exception:
            return 0.0
    st = {h: f(h) for h in idx if h.startswith("stall_") and "Not Issued" not in h}
    sass.append((int(r[2], 16), cur_line, f("Instructions Executed"), f("L1 Wavefronts Shared"),
                 f("Warp Stall Sampling (All Samples)"), st))
sass.sort()
agg = {}
last_polar = 0
for addr, (p, ln), inst, wf, smp, st in sass:
    if p == "kernels_polar.cu" and ln >= KSTART:       # helpers above the kernel body inherit the caller's region
        last_polar = ln
    reg = region_of(last_polar)
    a = agg.setdefault(reg, {"inst": 0, "wf": 0, "smp": 0, "st": {}})
    a["inst"] += inst; a["wf"] += wf; a["smp"] += smp
    for k, v in st.items():
        a["st"][k] = a["st"].get(k, 0) + v
T = sum(a["smp"] for a in agg.values())
for _, name in REGIONS:
    if name not in agg:
        continue
    a = agg[name]
    top = sorted(a["st"].items(), key=lambda kv: -kv[1])[:5]
    s = sum(a["st"].values()) or 1
    print("%-15s samples %5.1f%%  inst/img %7.0f  shwf/img %7.0f  %s" % (name, 100 * a["smp"] / T, a["inst"] / nimg,
          a["wf"] / nimg, " ".join("%s:%d" % (k[6:], 100 * v / s) for k, v in top)))
