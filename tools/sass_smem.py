"""Shared-memory wavefronts (actual vs ideal) per source line from an ncu SASS source dump + nvdisasm -g."""
import csv
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import line_map  # noqa: E402


def main(report_csv, sass_path, func_substr, src_path):
    lm = line_map(sass_path, func_substr)
    rows = list(csv.reader(open(report_csv)))
    h = rows[1]
    ia, iw, ii = h.index("Address"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
    base = int(rows[2][ia], 16)
    act, ide = defaultdict(int), defaultdict(int)
    for r in rows[2:]:
        l = lm.get(int(r[ia], 16) - base, -1)
        act[l] += int(r[iw] or 0)
        ide[l] += int(r[ii] or 0)
    src = open(src_path).read().split("\n")
    ta, ti = sum(act.values()), sum(ide.values())
    print(f"total wavefronts {ta}  ideal {ti}  excess {ta - ti}")
    for l in sorted(act, key=lambda x: -(act[x] - ide[x]))[:15]:
        s = src[l - 1].strip()[:80] if 0 < l <= len(src) else "?"
        print(f"{l:5d} act {act[l]:11d} ideal {ide[l]:11d} x{act[l] / max(1, ide[l]):5.2f}  {s}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
