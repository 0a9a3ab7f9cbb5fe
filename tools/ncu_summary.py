"""Summarise an ncu --set full report (raw page) into a compact table (used for profiles/).

    python tools/ncu_summary.py REPORT.ncu-rep [--traffic-json OUT.json --workload NAME]

--traffic-json writes, per bench pass name, the DRAM bytes (read + write) of one launch of
that kernel as captured (bench.py reports it as roofline.traffic when the workload matches)."""
import csv
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]

# kernel function -> bench pass name
PASS = {"k_chain_hash": "K1_chain_hash", "k_link_tile": "K2_link_prev", "k_link_prev": "K2_link_prev",
        "k_bucket_assemble": "K2_bucket_assemble", "k_access_info": "K2_access_info", "k_sort_prep": "K2_sort_prep",
        "k_hist_dD": "K4_hist_dD", "k_hist_runs": "K4_hist_runs", "k_replay": "K6_replay", "k_expand": "K3_expand", "k_run_expand": "K3_expand",
        "k_bucket_link": "K2_bucket_link", "k_bucket_fixup": "K2_bucket_fixup", "k_bucket_bounds": "K2_bucket_bounds"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(argv):
    rep = argv[0]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    idx = {w: h.index(w) for w in WANT if w in h}
    kn = h.index("Kernel Name")
    print("| kernel | " + " | ".join(w.split(".")[0].replace("__", ":") for w in idx) + " |")
    print("|" + "---|" * (len(idx) + 1))
    traffic = {}
    for r in rows[2:]:
        name = r[kn].split("(")[0][:48]
        vals = []
        for w, i in idx.items():
            vals.append(f"{r[i]} {units[i]}".strip())
        print(f"| {name} | " + " | ".join(vals) + " |")
        base = name.replace("void ", "").split("<")[0].split("::")[-1].strip()
        if ("K2Sort" in r[kn] or "kareto::" in r[kn]) and base in ("DeviceRadixSortOnesweepKernel", "DeviceRadixSortHistogramKernel"):
            base = "sort_" + base  # K2's bucket sort: one histogram + two onesweep passes per load
        if (base in PASS or base.startswith("sort_")) and "dram__bytes_read.sum" in idx:
            rb = float(r[idx["dram__bytes_read.sum"]].replace(",", "")) * SCALE.get(units[idx["dram__bytes_read.sum"]], 1)
            wb = float(r[idx["dram__bytes_write.sum"]].replace(",", "")) * SCALE.get(units[idx["dram__bytes_write.sum"]], 1)
            traffic.setdefault(PASS.get(base, base), []).append(rb + wb)
    if "--traffic-json" in argv:
        path = argv[argv.index("--traffic-json") + 1]
        wl = argv[argv.index("--workload") + 1] if "--workload" in argv else ""
        res = {k: sum(v) / len(v) for k, v in traffic.items() if not k.startswith("sort_")}
        h_, o_ = traffic.get("sort_DeviceRadixSortHistogramKernel"), traffic.get("sort_DeviceRadixSortOnesweepKernel")
        if h_ and o_:  # the K2_sort_buckets pass = histogram + 2 onesweep passes (16 key bits)
            res["K2_sort_buckets"] = sum(h_) / len(h_) + 2 * sum(o_) / len(o_)
        with open(path, "w") as f:
            json.dump({"workload": wl, "source": rep, "dram_bytes_per_launch": res}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
