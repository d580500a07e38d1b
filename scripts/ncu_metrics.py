"""Print the headline ncu metrics of every kernel in an .ncu-rep (via `ncu -i --page raw --csv`).
usage: python scripts/ncu_metrics.py REPORT.ncu-rep [substring-filter ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    flt = sys.argv[2:]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if flt and not any(f in name for f in flt):
            continue
        print(name[:90])
        d = dict(zip(h, r))
        units = dict(zip(h, u))
        for k in KEYS:
            if k in d:
                print(f"   {k} {d[k]} {units[k]}")
        st = sorted(((float(d[k]), k) for k in h if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")
                     and d[k] not in ("", "n/a")), reverse=True)[:8]
        for v, k in st:
            print(f"   stall {k[len(STALLS):-len('_per_issue_active.ratio')]} {v:.3f}")


if __name__ == "__main__":
    main()
