"""DRAM traffic per stage-kernel launch from an `ncu --set full` report of a bench.py run.

    python tools/traffic_from_ncu.py gpurun_out/prof_2b_v9.ncu-rep --workload 2b --n 64 \
        --cells 134217728 --out profiles/stage_kernel_traffic.json

bench.py reports roofline.traffic = the mean of dram__bytes_read.sum + dram__bytes_write.sum over the
captured stage-kernel launches (one stage-1 and one stage-2 launch of one cycle), next to the
algorithmic bytes (r*40 + 60) B per cell.
"""
import argparse
import csv
import io
import json
import subprocess

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--workload", default="2b")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--cells", type=float, required=True, help="interior cells per launch")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    launches = []
    for r in rows[2:]:
        if "stage_kernel" not in r[ki] and "stage2_kernel" not in r[ki]:
            continue
        def val(name):
            i = hdr.index(name)
            return float(r[i].replace(",", "")) * UNITS.get(units[i], 1.0)
        launches.append(dict(kernel=r[ki], read=val("dram__bytes_read.sum"), write=val("dram__bytes_write.sum")))
    if not launches:
        raise SystemExit("no stage_kernel launches in the report")
    r = ((a.n + 4) / a.n) ** 3
    per = [l["read"] + l["write"] for l in launches]
    res = {"workload": a.workload, "n": a.n, "bytes_per_launch": sum(per) / len(per),
           "per_launch": [dict(kernel=l["kernel"][:60], bytes=b) for l, b in zip(launches, per)],
           "algorithmic_bytes_per_launch": a.cells * (r * 40.0 + 60.0),
           "source": f"ncu --set full, {a.rep}"}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
