"""ncu report -> profiles JSON: per-launch key metrics and the forward pass's
summed DRAM traffic (bench.py reads dram_bytes_per_launch as roofline.traffic).
    python tools/ncu_json.py report.ncu-rep out.json [source note]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread", "smsp__inst_executed.sum"]
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1}


def main(rep, out, note=""):
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                          text=True).stdout.splitlines()))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for key in KEYS:
            if key in h:
                i = h.index(key)
                try:
                    k[key] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        kernels.append(k)
    fwd = [k for k in kernels if "fwd_" in k["kernel"] or "plan_tc" in k["kernel"]]
    traffic = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in fwd)
    doc = {"source": note, "note": "forward pass = every launch of one forward (device plan + class launches, "
                                   "or one launch per occupancy bucket); traffic is summed over the pass",
           "forward_launches": len(fwd), "forward_time_s_cold": sum(k["gpu__time_duration.sum"] for k in fwd),
           "dram_bytes_per_launch": traffic, "dram_bytes_per_pass": traffic, "kernels": kernels}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in doc.items() if k != "kernels"}))


if __name__ == "__main__":
    main(*sys.argv[1:])
