"""Top SASS instructions by stall reason from an ncu report (--set full, -lineinfo build).

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [--kernel 0] [--top 25] [--reason stall_long_sb]

Prints, per reason, the instructions with the most samples (address, opcode text, samples) and,
with --cuda, the CUDA source lines aggregated over all reasons.
"""
import argparse
import collections
import csv
import io
import subprocess


def page(rep, kernel, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what,
                          "--kernel-id", f"::regex:.*:{kernel + 1}"] if False else
                         ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the csv holds one table per kernel launch: a "Kernel Name" row, then a header, then data
    tables, cur = [], None
    for row in rows:
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "hdr": None, "data": []}
            tables.append(cur)
        elif cur is not None and cur["hdr"] is None:
            cur["hdr"] = row
        elif cur is not None:
            cur["data"].append(row)
    return tables


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--top", type=int, default=20)
    ap.add_argument("--reason", action="append")
    ap.add_argument("--cuda", action="store_true")
    a = ap.parse_args()
    t = page(a.rep, a.kernel, "sass")[a.kernel]
    hdr, data = t["hdr"], t["data"]
    print("kernel:", t["name"])
    reasons = a.reason or ["stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb", "stall_mio"]
    ix_src = hdr.index("Source")
    for rs in reasons:
        j = hdr.index(rs)
        tot = sum(int(r[j] or 0) for r in data)
        print(f"\n== {rs}: {tot} samples")
        ranked = sorted(data, key=lambda r: -int(r[j] or 0))[: a.top]
        for r in ranked:
            print(f"  {int(r[j] or 0):6d}  {r[0][-5:]}  {r[ix_src].strip()}")
    if a.cuda:
        tc = page(a.rep, a.kernel, "cuda")[a.kernel]
        h, d = tc["hdr"], tc["data"]
        j = h.index("Warp Stall Sampling (All Samples)")
        print("\n== CUDA lines by all samples")
        for r in sorted(d, key=lambda r: -int(r[j] or 0))[: a.top]:
            print(f"  {int(r[j] or 0):6d}  L{r[0]}  {r[1].strip()[:110]}")


if __name__ == "__main__":
    main()
