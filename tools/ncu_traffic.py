"""Write profiles/r2_ncu_traffic.json (the per-image ncu figures bench.py's `roofline.traffic`, `binding_resource` and
the K4/K5 tensor-pipe fractions quote) from the two `ncu --set full` reports of tools/prof_polar.sh and
tools/prof_k47.sh.   usage: ncu_traffic.py <polar.ncu-rep> <n_img_polar> <k47.ncu-rep> <n_img_k47> <out.json> [note]"""
import csv
import json
import subprocess
import sys

HBM_GBS = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    unit = dict(zip(r[0], r[1]))
    return [dict(zip(r[0], x)) for x in r[2:]], unit


def num(d, k):
    return float(d[k].replace(",", ""))


def to_bytes(d, unit, k):
    return num(d, k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit[k]]


def to_ms(d, unit, k="gpu__time_duration.sum"):
    return num(d, k) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}[unit[k]]


def common(d, unit, n):
    rd, wr, ms = to_bytes(d, unit, "dram__bytes_read.sum"), to_bytes(d, unit, "dram__bytes_write.sum"), to_ms(d, unit)
    gbs = (rd + wr) / (ms * 1e-3) / 1e9
    return {"dram_bytes_per_image": round((rd + wr) / n), "dram_read_bytes_per_image": round(rd / n),
            "dram_write_bytes_per_image": round(wr / n), "duration_ms": round(ms, 4), "images": n,
            "dram_gbs": round(gbs, 1), "dram_frac": round(gbs / HBM_GBS, 3)}


def main(polar_rep, n_polar, k47_rep, n_k47, out, note=""):
    n_polar, n_k47 = int(n_polar), int(n_k47)
    res = {"source": "ncu --set full --clock-control none, one launch per kernel (tools/prof_polar.sh: C3, %d images; "
                     "tools/prof_k47.sh: C3, %d images); B200; per-image = launch total / images; written by "
                     "tools/ncu_traffic.py. %s" % (n_polar, n_k47, note), "kernels": {}}
    pr, pu = rows(polar_rep)
    d = pr[0]
    k = common(d, pu, n_polar)
    pct = lambda m: round(num(d, m) / 100, 3)
    k.update({
        "kernel": d["Kernel Name"][:40],
        "l1_data_pipe_busy_frac": pct("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "shared_wavefronts_per_image": round(num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / n_polar),
        "bank_conflict_wavefronts_per_image": round(num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") / n_polar),
        "warp_instructions_per_image": round(num(d, "smsp__inst_executed.sum") / n_polar),
        "issue_active_frac": pct("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        "fma_pipe_frac": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "xu_pipe_frac": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        "registers": int(num(d, "launch__registers_per_thread")), "report": polar_rep})
    res["kernels"]["polar_K1K2K3"] = k
    kr, ku = rows(k47_rep)
    for d in kr:
        name = d["Kernel Name"]
        key = "radial_K4" if "radial_tma" in name else "cov_K5" if "cov_tma" in name else "project_K7" if "project" in name else None
        if key is None:
            continue
        k = common(d, ku, n_k47)
        k["tensor_pipe_active_frac"] = round(num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") / 100, 3)
        k["tf32_utchmma_frac"] = round(num(d, "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed") / 100, 3)
        k["report"] = k47_rep
        res["kernels"][key] = k
    res["dram_frac_definition"] = ("ncu dram bytes / ncu duration / %.0f GB/s (MEASURED_PEAKS.json hbm_gbs, the copy "
                                   "bandwidth the bench's HBM fractions use)" % HBM_GBS)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
