"""Summarise an ncu --set full report (raw page) into a compact table (used for profiles/)."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    idx = {w: h.index(w) for w in WANT if w in h}
    kn = h.index("Kernel Name")
    print("| kernel | " + " | ".join(w.split(".")[0].replace("__", ":") for w in idx) + " |")
    print("|" + "---|" * (len(idx) + 1))
    for r in rows[2:]:
        name = r[kn].split("(")[0][:48]
        vals = []
        for w, i in idx.items():
            vals.append(f"{r[i]} {units[i]}".strip())
        print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
