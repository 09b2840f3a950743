"""Instructions per cell-stage of the stage kernel from an `ncu --set full` report: the mean over the
captured stage-1 and stage-2 launches of tools/ncu_summary.py's counts (warp instructions x 32 per
cell, from the SASS source page) -> profiles/stage_kernel_counts.json, read by bench.py for the
fp64-pipe co-limiter.

    python tools/stage_counts.py gpurun_out/prof_2b.ncu-rep --cells 134217728 --out profiles/stage_kernel_counts.json
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--cells", type=float, required=True, help="interior cells per launch")
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    per = []
    for l in range(a.launches):
        tmp = f"/tmp/_stage_counts_{l}"
        subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), a.rep, "--cells", str(a.cells),
                        "--out", tmp, "--launch", str(l)], check=True, capture_output=True)
        d = json.load(open(tmp + ".json"))
        per.append(dict(kernel=d.get("kernel"), thread_inst_per_cell=d["thread_inst_per_cell_total"],
                        fp64_inst_per_cell=d["fp64_inst_per_cell"],
                        time=d.get("gpu__time_duration.sum")))
    out = {"thread_inst_per_cell_stage": sum(p["thread_inst_per_cell"] for p in per) / len(per),
           "fp64_inst_per_cell_stage": sum(p["fp64_inst_per_cell"] for p in per) / len(per),
           "per_launch": per, "source": f"ncu --set full {os.path.basename(a.rep)} (tools/stage_counts.py)"}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
