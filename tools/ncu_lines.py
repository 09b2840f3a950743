"""Per CUDA source line: thread instructions executed and stall samples (ncu --set full, -lineinfo).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--kernel 0] [--cells N] [--top 40]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--cells", type=float, default=0.0, help="cells per launch: print instructions per cell")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fn, kern, hdr, res, kidx = None, None, None, [], -1
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
        elif r[0] == "Function Name":
            if r[1] != kern:
                kern = r[1]
                kidx += 1
        elif r[0] == "Line No":
            hdr = r
        elif hdr and kidx == a.kernel and r[2] == "-":
            ti = int(r[hdr.index("Thread Instructions Executed")] or 0)
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            res.append((ti, smp, f"{fn}:{r[0]}", r[1].strip()[:100]))
    tot = sum(x[0] for x in res) or 1
    stot = sum(x[1] for x in res) or 1
    print(f"kernel #{a.kernel}: {tot} thread instructions, {stot} samples")
    for ti, smp, loc, src in sorted(res, reverse=True)[: a.top]:
        per = f"{ti / a.cells:7.1f}/cell" if a.cells else ""
        print(f"{ti / tot * 100:5.1f}% {per} {smp / stot * 100:5.1f}%smp  {loc:18s} {src}")


if __name__ == "__main__":
    main()
