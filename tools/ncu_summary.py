"""Summarise an ncu report: key raw metrics and top stall reasons per kernel."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_active.avg.per_cycle_active", "sm__cycles_elapsed.avg"]


def main(path, regex=None):
    cmd = ["ncu", "-i", path, "--page", "raw", "--csv"]
    if regex:
        cmd += ["-k", f"regex:{regex}"]
    rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        print("==", r[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k:60s} {r[h.index(k)]} {units[h.index(k)]}")
        st = []
        for i, k in enumerate(h):
            if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), k.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
