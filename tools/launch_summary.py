"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a per-kernel table
(total time, launches, share), as kept under profiles/.

    python tools/launch_summary.py LAUNCHES.csv "HEADER LINE" > profiles/....md"""
import collections
import csv
import sys


def main(path, header):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    kn, mn, vn, un = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) <= vn or r[mn] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[un], 1e-6)
        name = r[kn].replace("void ", "").split("(")[0][:70]
        tot[name] += float(r[vn].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# {header}\n")
    print("Cold-cache and serialised (ncu): compare shares, not absolutes.\n")
    print(f"total kernel time {T:.3f} ms over {sum(cnt.values())} launches\n")
    print("| kernel | ms | launches | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| {k} | {v:.3f} | {cnt[k]} | {100 * v / T:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
