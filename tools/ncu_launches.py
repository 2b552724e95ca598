"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total, share."""
import csv
import re
import sys
from collections import defaultdict


OURS = ("polar_kernel", "radial_tma_kernel", "radial_kernel", "cov_tma_kernel", "cov_k0_kernel", "cov_reduce_kernel",
        "cov_finalize_kernel", "cov_accum_kernel", "eig_kernel", "project_kernel")


def short(name: str) -> str:
    for o in OURS:
        if o in name:
            m = re.search(o + r"(<[^>]*>)?", name)
            return "fbspca::" + (m.group(0) if m else o)
    return "torch/other: " + name.split("(")[0][-60:]


def main(path):
    rows = [l for l in open(path) if l.startswith('"')]
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        tot[k] += float(r["Metric Value"].replace(",", "")) / 1e3   # ns -> us
        cnt[k] += 1
    ours = {k: v for k, v in tot.items() if k.startswith("fbspca")}
    s = sum(ours.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'share_of_fbspca':>16s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        share = f"{100 * v / s:6.2f}%" if k in ours else ""
        print(f"{k:40s} {cnt[k]:8d} {v:12.1f} {share:>16s}")


if __name__ == "__main__":
    main(sys.argv[1])
