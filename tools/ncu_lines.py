"""Per-source-line stall samples, instructions and shared-memory wavefronts of one kernel from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep CUBIN_OR_SO MANGLED_SUBSTR SOURCE.cu [N_UNITS] [TOP]

Joins `ncu --page source --csv --print-source sass` with `nvdisasm -g` line info of the same build (the
.so is unpacked with cuobjdump).  N_UNITS divides the counts (e.g. images per launch)."""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def sass_with_lines(binary):
    d = tempfile.mkdtemp()
    if binary.endswith(".so"):
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(binary)], cwd=d, capture_output=True)
        cubins = glob.glob(os.path.join(d, "*.cubin"))
    else:
        cubins = [binary]
    out = []
    for c in cubins:
        out.append(subprocess.run(["nvdisasm", "-g", "-c", c], capture_output=True, text=True).stdout)
    return "\n".join(out)


def line_map(sass, func_substr):
    cur, line, m = None, None, {}
    for ln in sass.split("\n"):
        if ln.startswith("//----") and ".text." in ln:
            cur = ln
        mm = re.search(r'//## File "(.*)", line (\d+)', ln)
        if mm:
            line = (os.path.basename(mm.group(1)), int(mm.group(2)))
            continue
        mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if mo and cur and func_substr in cur:
            m[int(mo.group(1), 16)] = line
    return m


def main(rep, binary, func, src, units=1, top=45, kname=None):
    kname = kname or func
    units, top = float(units), int(top)
    lm = line_map(sass_with_lines(binary), func)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    # one section per profiled kernel: "Kernel Name" row, header row, data rows; keep the first matching one
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    sec = None
    for a, b in zip(starts, starts[1:]):
        if kname in rows[a][1]:
            sec = rows[a + 1:b]
            break
    if sec is None:
        sec = rows
    hi = next(i for i, r in enumerate(sec) if r and r[0] == "Address")
    h, data = sec[hi], sec[hi + 1:]
    col = {k: h.index(k) for k in ("Address", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                   "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal")}
    base = int(data[0][col["Address"]], 16)
    acc = defaultdict(lambda: [0, 0, 0, 0])
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    why = defaultdict(lambda: defaultdict(int))
    f = lambda x: int(x.replace(",", "") or 0)
    for r in data:
        if len(r) < len(h):
            continue
        key = lm.get(int(r[col["Address"]], 16) - base, ("?", -1))
        a = acc[key]
        a[0] += f(r[col["Warp Stall Sampling (All Samples)"]]); a[1] += f(r[col["Instructions Executed"]])
        a[2] += f(r[col["L1 Wavefronts Shared"]]); a[3] += f(r[col["L1 Wavefronts Shared Ideal"]])
        for rc in reasons:
            why[key][rc] += f(r[h.index(rc)])
    srcl = open(src).read().split("\n")
    T = sum(a[0] for a in acc.values()) or 1
    W = sum(a[2] for a in acc.values())
    print(f"stall samples {T}, smem wavefronts/unit {W / units:.0f} (ideal {sum(a[3] for a in acc.values()) / units:.0f}),"
          f" instr/unit {sum(a[1] for a in acc.values()) / units:.0f}")
    for key in sorted(acc, key=lambda k: -acc[k][0])[:top]:
        a = acc[key]
        fn, l = key
        s = srcl[l - 1].strip()[:64] if fn == os.path.basename(src) and 0 < l <= len(srcl) else fn
        top = sorted(why[key].items(), key=lambda x: -x[1])[:2]
        tops = " ".join(f"{k[6:]}:{100 * v / max(1, a[0]):.0f}%" for k, v in top if v)
        print(f"{l:5d} st {100 * a[0] / T:5.1f}% wf {a[2] / units:9.0f} (ideal {a[3] / units:8.0f}) ins {a[1] / units:8.0f}  [{tops}] {s}")


if __name__ == "__main__":
    main(*sys.argv[1:])
