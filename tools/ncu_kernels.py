"""Per-kernel headline metrics from an ncu --set full report (one line per profiled launch)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active" ,
        "smsp__average_warp_latency_issue_stalled_short_scoreboard", "launch__registers_per_thread",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")[:60]
        print(f"== {name}  grid={d.get('Grid Size')} block={d.get('Block Size')}")
        for k in KEYS:
            for col in h:
                if col == k:
                    print(f"   {k:80s} {d[col]}")
        stalls = []
        for col in h:
            if col.startswith("smsp__pcsamp_warps_issue_stalled_") and not col.endswith("not_issued"):
                try:
                    stalls.append((float(d[col].replace(",", "")), col.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        print("   stalls: " + ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
