"""Join an ncu `--page source --csv --print-source sass` dump with `nvdisasm -g` line info (same cubin build)
and print instructions executed / stall samples per source line."""
import csv
import re
import sys
from collections import defaultdict


def line_map(sass_path, func_substr):
    cur_fn, line, m = None, None, {}
    for ln in open(sass_path):
        if ln.startswith("//----") and ".text." in ln:
            cur_fn = ln
        mm = re.search(r'//## File ".*", line (\d+)', ln)
        if mm:
            line = int(mm.group(1))
            continue
        mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if mo and cur_fn and func_substr in cur_fn:
            m[int(mo.group(1), 16)] = line
    return m


def main(report_csv, sass_path, func_substr, src_path):
    lm = line_map(sass_path, func_substr)
    rows = list(csv.reader(open(report_csv)))
    hdr = rows[1]
    ia = hdr.index("Address"); ie = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][ia], 16)
    ex, st = defaultdict(int), defaultdict(int)
    for r in data:
        off = int(r[ia], 16) - base
        l = lm.get(off, -1)
        ex[l] += int(r[ie] or 0)
        st[l] += int(r[iss] or 0)
    src = open(src_path).read().split("\n")
    tot_e, tot_s = sum(ex.values()), sum(st.values())
    print(f"total instr {tot_e}  stall samples {tot_s}")
    for l in sorted(ex, key=lambda x: -st[x])[:40]:
        s = src[l - 1].strip()[:90] if 0 < l <= len(src) else "?"
        print(f"{l:5d} {100*ex[l]/tot_e:6.2f}% instr {100*st[l]/tot_s:6.2f}% stall  {s}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
