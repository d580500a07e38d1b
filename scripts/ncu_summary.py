"""Summarise an ncu --set full report into a tracked CSV (profiles/): one row per captured kernel,
the columns that back the roofline and bottleneck claims (DRAM bytes and throughput, duration,
shared-memory wavefronts and bank conflicts, launch geometry, tensor-pipe activity, issue
activity, warp occupancy).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01c_ncu_full_x.csv
"""
import csv
import io
import re
import subprocess
import sys

KEEP = re.compile(r"^(Kernel Name|dram__bytes|gpu__dram_throughput|gpu__time_duration|l1tex__data_bank_conflicts_pipe_lsu_mem_shared|"
                  r"l1tex__data_pipe_lsu_wavefronts_mem_shared|launch__|sm__cycles_elapsed\.avg|sm__pipe_tensor_cycles_active|"
                  r"smsp__issue_active|sm__warps_active|smsp__inst_executed\.sum|sm__throughput|lts__t_bytes\.sum|"
                  r"gpu__compute_memory_throughput|sm__pipe_fp64_cycles_active|sm__inst_executed_pipe_xu|l1tex__data_pipe_lsu_wavefronts\.sum)")


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [i for i, h in enumerate(hdr) if KEEP.match(h)]
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow([hdr[i] for i in cols])
        w.writerow([units[i] for i in cols])
        for r in data:
            w.writerow([r[i] for i in cols])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
