"""Summarise an ncu report (--set full) of the stage kernel into a markdown table + JSON.

    python tools/ncu_summary.py gpurun_out/prof_stage_v2.ncu-rep --cells 16777216 --out profiles/r01_stage_v2
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "sass__inst_executed_local_loads", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__block_size",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--cells", type=float, required=True, help="interior cells processed per launch")
    ap.add_argument("--out", required=True)
    ap.add_argument("--launch", type=int, default=0)
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    d = data[a.launch]
    res = {"kernel": d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            res[m] = {"value": d[i], "unit": units[i]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[i].replace(",", ""))
            except ValueError:
                pass
    res["stall_samples"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
    # SASS opcode mix (dynamic) of the profiled launch
    src = ncu_csv(a.rep, "source", ["--print-source", "sass"])
    mix = collections.Counter()
    # the page repeats each kernel's table; take the first table of the a.launch-th distinct kernel
    hdr2 = None
    names, want = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            if r[1] not in names:
                names.append(r[1])
            want = (len(names) - 1 == a.launch) and names.count(r[1]) == 1 and hdr2 is None
            continue
        if r and r[0] == "Address":
            if hdr2 is not None:
                break
            if want:
                hdr2 = r
                iS, iE = r.index("Source"), r.index("Instructions Executed")
            continue
        if hdr2 is None or len(r) <= iE:
            continue
        try:
            n = int(r[iE].replace(",", ""))
        except ValueError:
            continue
        toks = r[iS].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        mix[op.split(".")[0]] += n
    per_cell = {k: round(v * 32 / a.cells, 1) for k, v in mix.most_common(25)}
    res["thread_inst_per_cell"] = per_cell
    res["thread_inst_per_cell_total"] = round(sum(mix.values()) * 32 / a.cells, 1)
    fp64 = sum(mix[k] for k in ("DFMA", "DMUL", "DADD", "DSETP")) * 32 / a.cells
    res["fp64_inst_per_cell"] = round(fp64, 1)
    res["cells_per_launch"] = a.cells
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu summary: {a.rep}\n\nkernel: `{res['kernel']}`  cells/launch: {a.cells:.0f}\n\n")
        f.write("| metric | value | unit |\n|---|---|---|\n")
        for m in METRICS:
            if m in res:
                f.write(f"| {m} | {res[m]['value']} | {res[m]['unit']} |\n")
        f.write(f"\nthread instructions per cell-stage: {res['thread_inst_per_cell_total']} "
                f"(fp64 pipe: {res['fp64_inst_per_cell']})\n\n")
        f.write("| opcode | thread inst / cell |\n|---|---|\n")
        for k, v in per_cell.items():
            f.write(f"| {k} | {v} |\n")
        f.write("\nstall samples (top): " + ", ".join(f"{k}={v:.0f}" for k, v in res["stall_samples"].items()) + "\n")
    print(json.dumps({k: res[k] for k in ("thread_inst_per_cell_total", "fp64_inst_per_cell")}))


if __name__ == "__main__":
    main()
