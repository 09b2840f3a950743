"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python tools/launch_summary.py gpurun_out/launches_2b.csv > profiles/r01_launches_2b.md
ncu times are cold-cache and serialised: compare SHARES of the step with bench.py, not absolutes."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    t = collections.defaultdict(float)
    n = collections.Counter()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        if "stage_kernel" in d["Kernel Name"]:
            name = "stage_kernel" + d["Kernel Name"][d["Kernel Name"].find("<"):d["Kernel Name"].find(">") + 1]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
        t[name] += v * scale
        n[name] += 1
    tot = sum(t.values())
    print(f"# ncu launch list: {path}\n")
    print(f"{sum(n.values())} launches, {tot / 1e3:.3f} ms total (cold-cache, serialised)\n")
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {n[k]} | {v:.1f} | {v / n[k]:.1f} | {100 * v / tot:.1f} % |")


if __name__ == "__main__":
    main(sys.argv[1])
